# Build of the B200-native SO2DR engine: one in-tree shared library
# paper_2309_08864_b200/libso2dr_b200.so exporting the C ABI
# (include/so2dr_cuda.h) and the C++ mirror API (include/so2dr/*.hpp).
# sm_100a only; --fmad=false keeps every multiply-add an explicit __fma_rn
# (bit-exact with the reference's -ffp-contract=off build).

NVCC     ?= /usr/local/cuda/bin/nvcc
HOSTCXX  := /usr/bin/g++
PKG      := paper_2309_08864_b200
SRC      := $(PKG)/csrc
OBJ      := build/obj
LIB      := $(PKG)/libso2dr_b200.so
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo --fmad=false -std=c++20 -ccbin $(HOSTCXX) \
            -Xcompiler -fPIC -Xcompiler -fvisibility=default -Iinclude -I$(SRC) \
            --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS := -O2 -std=c++20 -fPIC -Iinclude -I$(SRC) -I/usr/local/cuda/include -Wall

CU_SRCS  := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
OBJS     := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CPP_SRCS))
HDRS     := $(wildcard $(SRC)/*.h $(SRC)/*.cuh include/*.h include/so2dr/*.hpp)

all: $(LIB)

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(HOSTCXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -ccbin $(HOSTCXX) -o $@ $^ -L/usr/local/cuda/lib64 -L/usr/local/cuda/lib64/stubs -lcudart_static -ldl -lrt -lpthread

clean:
	rm -rf build/obj $(LIB)

.PHONY: all clean
