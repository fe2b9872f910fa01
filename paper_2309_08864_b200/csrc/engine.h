// engine.h -- internal interface of the B200 SO2DR scheduler (engine.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "k1_launch.h"
#include "so2dr/engine.hpp"
#include "so2dr_cuda.h"

namespace so2dr_eng {

void check_cuda(cudaError_t e, const char* what, const char* file, int line);
#define SO2DR_CK(x) ::so2dr_eng::check_cuda((x), #x, __FILE__, __LINE__)

// Real HBM pool: named blocks cached across runs, capped by the context
// budget. Exceeding the cap raises OutOfDeviceMemoryError("hbm:<id>").
class Pool {
 public:
  uint64_t budget = 0;
  // Blocks requested since the last begin_run() are "live"; older ones are
  // freed on demand when a request would exceed the budget.
  void begin_run() { ++gen_; }
  void* get(const std::string& id, uint64_t bytes);
  uint64_t used() const;
  void release_all();
  ~Pool() { release_all(); }

 private:
  struct Blk {
    void* p = nullptr;
    uint64_t bytes = 0;
    uint64_t gen = 0;
  };
  std::map<std::string, Blk> blk_;
  uint64_t gen_ = 1;
};

// Recycled CUDA events (timing and non-timing kinds).
class EventPool {
 public:
  cudaEvent_t sync_event();
  cudaEvent_t timing_event();
  void recycle();  // all events handed out become reusable
  ~EventPool();

 private:
  std::vector<cudaEvent_t> sync_, timing_;
  size_t sync_next_ = 0, timing_next_ = 0;
};

// Stencil in device-ready form.
struct StencilDev {
  int kind = 0;  // so2dr_dev::KBOX/KGRAD/KSTAR (after star detection)
  int dim = 2;
  int radius = 1;
  std::vector<double> w;  // (2r+1)^dim canonical weights
};

// Geometry of the padded grid as the engine sees it: the chunking unit is a
// row (2D) or a z-plane (3D).
struct Geo {
  int dim = 2, sz = 0, r = 0, p = 0;
  int elem = 4;           // bytes per cell
  int64_t pitch = 0;      // device elements per storage row (multiple of 32)
  int64_t unit_rows = 1;  // storage rows per unit (1 or p)
  int top() const { return sz + 2 * r; }
  int64_t dev_unit_elems() const { return unit_rows * pitch; }
  int64_t host_unit_elems() const { return unit_rows * (int64_t)p; }
  uint64_t unit_bytes() const { return (uint64_t)host_unit_elems() * elem; }  // ledger bytes per unit
};

Geo make_geo(int dim, int sz, int r, int dtype);

// Peer connection of one slab edge (multi-rank mode).
struct PeerEdge {
  bool connected = false;
  bool ipc = false;
  bool same_device = false;  // the neighbour context runs on this GPU
  bool p2p_checked = false;  // cudaDeviceCanAccessPeer confirmed the path
  void* recv = nullptr;        // neighbour's receive buffer for our band (mapped)
  uint32_t* flag = nullptr;    // neighbour's data-ready flag for that buffer
  uint32_t* ack = nullptr;     // neighbour's consumed flag we must wait for (in our memory)
};

struct SlabState {
  bool prepared = false;
  int rank = 0, world = 1;
  so2dr_run_config cfg{};
  int dim = 2, dtype = 0;
  // our receive buffers (from lower / upper neighbour) and flags
  void* recv_lo = nullptr;
  void* recv_hi = nullptr;
  uint32_t* flags = nullptr;  // [0] lo data ready, [1] hi data ready, [2] lo consumed-ack, [3] hi consumed-ack
  uint64_t epoch = 0;         // rounds completed over the life of the connection
  PeerEdge lower, upper;
  std::vector<void*> opened;  // IPC mappings to close
};

}  // namespace so2dr_eng

struct so2dr_ctx {
  int device = 0;
  so2dr_eng::Pool pool;
  so2dr_eng::EventPool events;
  std::vector<cudaStream_t> streams;
  cudaStream_t aux = nullptr;
  bool profiling = false;
  std::string err, constraint, alloc_id;
  std::map<void*, size_t> registered;
  so2dr_eng::SlabState slab;

  cudaStream_t stream(int i);
};

namespace so2dr_eng {

struct RunRequest {
  so2dr_mode mode = SO2DR_MODE_SO2DR;
  StencilDev st;
  so2dr::RunConfig cfg;
  so2dr::KernelPlan kp;
  so2dr::HardwareModel hw;
  so2dr_hooks hooks{};
  int dtype = 0;
  void* grid = nullptr;   // host/device pointer to unit `host_lo`
  int64_t host_lo = 0;
  int rank = 0, world = 1;
};

struct RunResponse {
  so2dr_ledger ledger{};
  so2dr_timing timing{};
  std::vector<so2dr_diag_row> diag;
};

StencilDev make_stencil(const so2dr_stencil_desc* st);
void validate_request(const RunRequest& q);
void run(so2dr_ctx* ctx, RunRequest& q, RunResponse& out);

// fused_kernel on host buffers (FieldPair); returns stats in out4.
void fused_kernel_host(so2dr_ctx* ctx, const StencilDev& st, int dtype, void* buf0, void* buf1,
                       int base_row, int rows, int cols, int read, int steps, int tile,
                       const int32_t* region, const int32_t* interior, const int32_t* owned,
                       uint64_t* out4);
void apply_step_host(so2dr_ctx* ctx, const StencilDev& st, int dtype, int sz, int r,
                     const void* in, void* out, int row_lo, int row_hi);
void run_reference_host(so2dr_ctx* ctx, const StencilDev& st, int dtype, int sz, int r,
                        const void* in, void* out, int steps);
void init_rows(so2dr_ctx* ctx, int dtype, int dim, int sz, int r, uint64_t seed, int64_t lo,
               int64_t hi, void* out);

// slab mode
void slab_rows(const so2dr_run_config& cfg, int dim, int rank, int world, int64_t* lo,
               int64_t* hi);
void slab_prepare(so2dr_ctx* ctx, const StencilDev& st, const so2dr_run_config& cfg, int dtype,
                  int rank, int world, uint8_t* blob);
void slab_connect(so2dr_ctx* ctx, const uint8_t* lower, const uint8_t* upper);

// kernel launch (device-resident field) with step splitting
// Returns true when the result landed in `rd` (only with pingpong = true and
// a call split into an even number of launches).
bool k1_call(so2dr_ctx* ctx, cudaStream_t s, const Geo& g, const StencilDev& st, const void* rd,
             void* wr, int base, int rows, int y0, int y1, int x0, int x1, int steps,
             int scratch_slot, const int32_t* interior = nullptr, bool pingpong = false);

// reference kernel ledger accounting (proj/src/kernels.cpp:48-138) in closed form
so2dr::KernelStats tile_stats(int r, int steps, int tile, so2dr::Rect region,
                              so2dr::Rect interior, so2dr::Rect owned, int sy0, int sy1,
                              int64_t cols);

uint64_t device_footprint(const so2dr::RunConfig& cfg, const Geo& g, int n_strm);

}  // namespace so2dr_eng
