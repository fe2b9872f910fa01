// engine_api.cu -- the secondary device entry points (fused_kernel on a host
// FieldPair, apply_step, run_reference, init) and the multi-rank slab
// connection (CUDA IPC peer memory + device-side flags).
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>

#include "engine.h"

namespace so2dr_dev {
cudaError_t launch_init(int dtype, void* out, int64_t pitch, int p, int dim, int64_t lo,
                        int64_t n_units, uint64_t seed, cudaStream_t stream);
}

namespace so2dr_eng {

using so2dr::ContractError;
using so2dr::InvalidSpecError;

static void copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_b,
                   int64_t rows, cudaStream_t s) {
  if (rows <= 0 || width_b <= 0) return;
  SO2DR_CK(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_b, rows, cudaMemcpyDefault, s));
}

// fused_kernel (proj/src/kernels.cpp:27-145) on a host FieldPair.
void fused_kernel_host(so2dr_ctx* ctx, const StencilDev& st, int dtype, void* buf0, void* buf1,
                       int base_row, int rows, int cols, int read, int steps, int tile,
                       const int32_t* region, const int32_t* interior, const int32_t* owned,
                       uint64_t* out4) {
  if (steps < 1) throw InvalidSpecError("fused_kernel: steps must be >= 1");
  if (tile < 1) throw InvalidSpecError("fused_kernel: tile must be >= 1");
  if (read != 0 && read != 1) throw ContractError("fused_kernel: bad read index");
  if (st.dim != 2) throw InvalidSpecError("fused_kernel: FieldPair is 2D");
  if (region[0] < base_row || region[1] > base_row + rows || region[2] < 0 || region[3] > cols)
    throw ContractError("fused_kernel: region outside field storage");
  const so2dr::Rect reg{region[0], region[1], region[2], region[3]};
  const so2dr::Rect in{interior[0], interior[1], interior[2], interior[3]};
  const so2dr::Rect own{owned[0], owned[1], owned[2], owned[3]};
  const so2dr::KernelStats ks = tile_stats(st.radius, steps, tile, reg, in, own, base_row,
                                           base_row + rows, cols);
  out4[0] = ks.scratch_load;
  out4[1] = ks.scratch_store;
  out4[2] = ks.updates;
  out4[3] = ks.redundant;
  if (reg.area() == 0) return;

  SO2DR_CK(cudaSetDevice(ctx->device));
  Geo g = make_geo(2, cols - 2 * st.radius, st.radius, dtype);
  g.p = cols;
  g.pitch = (static_cast<int64_t>(cols) + 31) / 32 * 32;
  const uint64_t bytes = static_cast<uint64_t>(rows) * g.pitch * g.elem;
  void* d[2] = {ctx->pool.get("fk.buf0", bytes), ctx->pool.get("fk.buf1", bytes)};
  void* h[2] = {buf0, buf1};
  cudaStream_t s = ctx->stream(0);
  for (int b = 0; b < 2; ++b)
    copy2d(d[b], g.pitch * g.elem, h[b], static_cast<int64_t>(cols) * g.elem,
           static_cast<int64_t>(cols) * g.elem, rows, s);
  const int32_t inter[4] = {interior[0], interior[1], interior[2], interior[3]};
  k1_call(ctx, s, g, st, d[read], d[read ^ 1], base_row, rows, region[0], region[1], region[2],
          region[3], steps, 0, inter);
  const int w = read ^ 1;
  copy2d(h[w], static_cast<int64_t>(cols) * g.elem, d[w], g.pitch * g.elem,
         static_cast<int64_t>(cols) * g.elem, rows, s);
  SO2DR_CK(cudaStreamSynchronize(s));
}

// apply_step (proj/src/stencil.cpp:146-160): one step on rows [lo, hi) x
// interior columns; the rest of `out` is untouched.
void apply_step_host(so2dr_ctx* ctx, const StencilDev& st, int dtype, int sz, int r,
                     const void* in, void* out, int row_lo, int row_hi) {
  if (in == out) throw ContractError("apply_step: output aliases input");
  if (row_lo < r || row_hi > r + sz)
    throw std::out_of_range("apply_step: rows [" + std::to_string(row_lo) + "," +
                            std::to_string(row_hi) + ") outside interior [" + std::to_string(r) +
                            "," + std::to_string(r + sz) + ")");
  if (row_hi <= row_lo) return;
  SO2DR_CK(cudaSetDevice(ctx->device));
  const Geo g = make_geo(st.dim, sz, r, dtype);
  const int base = row_lo - r, rows = row_hi - row_lo + 2 * r;
  const uint64_t unit = static_cast<uint64_t>(g.dev_unit_elems()) * g.elem;
  char* a = static_cast<char*>(ctx->pool.get("as.buf0", rows * unit));
  char* b = static_cast<char*>(ctx->pool.get("as.buf1", rows * unit));
  cudaStream_t s = ctx->stream(0);
  const int64_t hrow = static_cast<int64_t>(g.p) * g.elem;  // host row bytes
  const int64_t rows_per_unit = g.unit_rows;
  copy2d(a, g.pitch * g.elem, static_cast<const char*>(in) + base * g.host_unit_elems() * g.elem,
         hrow, hrow, rows * rows_per_unit, s);
  k1_call(ctx, s, g, st, a, b, base, rows, row_lo, row_hi, r, g.p - r, 1, 0);
  if (st.dim == 2) {
    copy2d(static_cast<char*>(out) + (static_cast<int64_t>(row_lo) * g.p + r) * g.elem, hrow,
           b + (static_cast<int64_t>(r) * g.pitch + r) * g.elem, g.pitch * g.elem,
           static_cast<int64_t>(sz) * g.elem, row_hi - row_lo, s);
  } else {
    // 3D: interior rows of each plane
    for (int z = row_lo; z < row_hi; ++z)
      copy2d(static_cast<char*>(out) +
                 ((static_cast<int64_t>(z) * g.p + r) * g.p + r) * g.elem,
             hrow, b + ((static_cast<int64_t>(z - base) * g.p + r) * g.pitch + r) * g.elem,
             g.pitch * g.elem, static_cast<int64_t>(sz) * g.elem, sz, s);
  }
  SO2DR_CK(cudaStreamSynchronize(s));
}

// run_reference (proj/src/stencil.cpp:162-174): `steps` single full-interior
// steps, ping-pong in HBM. Used by verify_run and the acceptance suite.
void run_reference_host(so2dr_ctx* ctx, const StencilDev& st, int dtype, int sz, int r,
                        const void* in, void* out, int steps) {
  if (steps < 0) throw InvalidSpecError("step count must be non-negative");
  SO2DR_CK(cudaSetDevice(ctx->device));
  const Geo g = make_geo(st.dim, sz, r, dtype);
  const int p = g.p;
  const uint64_t unit = static_cast<uint64_t>(g.dev_unit_elems()) * g.elem;
  char* d[2] = {static_cast<char*>(ctx->pool.get("rr.buf0", p * unit)),
                static_cast<char*>(ctx->pool.get("rr.buf1", p * unit))};
  cudaStream_t s = ctx->stream(0);
  const int64_t hrow = static_cast<int64_t>(p) * g.elem;
  for (int b = 0; b < 2; ++b) copy2d(d[b], g.pitch * g.elem, in, hrow, hrow, p * g.unit_rows, s);
  int rd = 0;
  for (int k = 0; k < steps; ++k) {
    k1_call(ctx, s, g, st, d[rd], d[rd ^ 1], 0, p, r, r + sz, 0, p, 1, 0);
    rd ^= 1;
  }
  copy2d(out, hrow, d[rd], g.pitch * g.elem, hrow, p * g.unit_rows, s);
  SO2DR_CK(cudaStreamSynchronize(s));
}

void init_rows(so2dr_ctx* ctx, int dtype, int dim, int sz, int r, uint64_t seed, int64_t lo,
               int64_t hi, void* out) {
  if (sz < 1 || r < 0) throw InvalidSpecError("grid too small (sz=" + std::to_string(sz) +
                                              ", r=" + std::to_string(r) + ")");
  if (dim != 2 && dim != 3) throw InvalidSpecError("dim must be 2 or 3");
  const int p = sz + 2 * r;
  if (lo < 0 || hi > p || hi < lo) throw std::out_of_range("init_rows: unit range outside grid");
  SO2DR_CK(cudaSetDevice(ctx->device));
  const int elem = dtype == SO2DR_F64 ? 8 : 4;
  const int64_t unit_elems = dim == 3 ? static_cast<int64_t>(p) * p : p;
  cudaStream_t s = ctx->stream(0);
  cudaPointerAttributes attr{};
  const bool on_device = cudaPointerGetAttributes(&attr, out) == cudaSuccess &&
                         attr.type == cudaMemoryTypeDevice;
  cudaGetLastError();
  if (on_device) {
    SO2DR_CK(so2dr_dev::launch_init(dtype, out, p, p, dim, lo, hi - lo, seed, s));
  } else {
    // generate into a bounded staging buffer, stream it out
    const int64_t budget = 256ll << 20;
    const int64_t per = std::max<int64_t>(1, budget / (unit_elems * elem));
    char* stage = static_cast<char*>(ctx->pool.get("init.stage", per * unit_elems * elem));
    for (int64_t u = lo; u < hi; u += per) {
      const int64_t n = std::min(per, hi - u);
      SO2DR_CK(so2dr_dev::launch_init(dtype, stage, p, p, dim, u, n, seed, s));
      SO2DR_CK(cudaMemcpyAsync(static_cast<char*>(out) + (u - lo) * unit_elems * elem, stage,
                               n * unit_elems * elem, cudaMemcpyDefault, s));
      SO2DR_CK(cudaStreamSynchronize(s));
    }
  }
  SO2DR_CK(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- slabs --

void slab_rows(const so2dr_run_config& c, int dim, int rank, int world, int64_t* lo,
               int64_t* hi) {
  (void)dim;
  so2dr::RunConfig cfg;
  cfg.sz = c.sz, cfg.r = c.r, cfg.d = c.d, cfg.s_tb = c.s_tb, cfg.k_on = c.k_on;
  cfg.n_strm = c.n_strm, cfg.n = c.n, cfg.n_a = c.n_a;
  if (world < 1 || rank < 0 || rank >= world) throw InvalidSpecError("bad rank/world");
  if (cfg.d % world != 0)
    throw InvalidSpecError("config: d (" + std::to_string(cfg.d) +
                           ") must be divisible by the number of ranks (" +
                           std::to_string(world) + ")");
  const so2dr::ChunkLayout lay = so2dr::plan_chunks(cfg);
  const int dl = cfg.d / world;
  *lo = rank == 0 ? 0 : lay.fence[rank * dl];
  *hi = rank == world - 1 ? cfg.sz + 2 * cfg.r : lay.fence[(rank + 1) * dl];
}

namespace {
constexpr uint32_t kBlobMagic = 0x53324452u;  // "S2DR"
struct Blob {
  uint32_t magic;
  uint32_t pid;
  int32_t device;
  int32_t rank;
  uint64_t band_bytes;  // bytes of one receive buffer
  uint64_t off_lo, off_hi, off_flags;
  uint64_t raw;  // base pointer in the owner's address space
  cudaIpcMemHandle_t handle;
  char pci[32];  // PCI bus id of the owner's GPU (the peer-access check)
};
static_assert(sizeof(Blob) <= SO2DR_PEER_BLOB_BYTES, "blob too large");
}  // namespace

void slab_prepare(so2dr_ctx* ctx, const StencilDev& st, const so2dr_run_config& c, int dtype,
                  int rank, int world, uint8_t* blob_out) {
  int64_t lo, hi;
  slab_rows(c, st.dim, rank, world, &lo, &hi);
  SO2DR_CK(cudaSetDevice(ctx->device));
  const Geo g = make_geo(st.dim, c.sz, c.r, dtype);
  const uint64_t band = static_cast<uint64_t>(c.r) * c.s_tb * g.dev_unit_elems() * g.elem;
  const uint64_t band_al = (band + 255) / 256 * 256;
  const uint64_t total = 2 * band_al + 256;
  char* base = static_cast<char*>(ctx->pool.get("slab.xchg", total));
  SlabState& sl = ctx->slab;
  for (void* p : sl.opened) cudaIpcCloseMemHandle(p);
  sl = SlabState{};
  sl.prepared = true;
  sl.rank = rank;
  sl.world = world;
  sl.cfg = c;
  sl.dim = st.dim;
  sl.dtype = dtype;
  sl.recv_lo = base;
  sl.recv_hi = base + band_al;
  sl.flags = reinterpret_cast<uint32_t*>(base + 2 * band_al);
  SO2DR_CK(cudaMemset(sl.flags, 0, 256));
  SO2DR_CK(cudaDeviceSynchronize());
  Blob b{};
  b.magic = kBlobMagic;
  b.pid = static_cast<uint32_t>(getpid());
  b.device = ctx->device;
  b.rank = rank;
  b.band_bytes = band;
  b.off_lo = 0;
  b.off_hi = band_al;
  b.off_flags = 2 * band_al;
  b.raw = reinterpret_cast<uint64_t>(base);
  SO2DR_CK(cudaIpcGetMemHandle(&b.handle, base));
  SO2DR_CK(cudaDeviceGetPCIBusId(b.pci, sizeof b.pci, ctx->device));
  std::memset(blob_out, 0, SO2DR_PEER_BLOB_BYTES);
  std::memcpy(blob_out, &b, sizeof(b));
}

void slab_connect(so2dr_ctx* ctx, const uint8_t* lower, const uint8_t* upper) {
  SlabState& sl = ctx->slab;
  if (!sl.prepared) throw ContractError("slab_connect before slab_prepare");
  SO2DR_CK(cudaSetDevice(ctx->device));
  auto open = [&](const uint8_t* raw, PeerEdge& e, bool is_lower) {
    if (!raw) return;
    Blob b;
    std::memcpy(&b, raw, sizeof(b));
    if (b.magic != kBlobMagic) throw ContractError("slab_connect: not a peer blob");
    if (b.rank != sl.rank + (is_lower ? -1 : 1))
      throw ContractError("slab_connect: blob from rank " + std::to_string(b.rank) +
                          " is not the " + (is_lower ? "lower" : "upper") + " neighbour of rank " +
                          std::to_string(sl.rank));
    // peer access: the halo push writes the neighbour's HBM directly (NVLink
    // / NVSwitch, or PCIe P2P). A neighbour on another GPU this process can
    // see but not reach peer-to-peer is refused with a clear error instead of
    // a slow or failing IPC mapping.
    int peer_dev = -1;
    if (cudaDeviceGetByPCIBusId(&peer_dev, b.pci) != cudaSuccess) {
      cudaGetLastError();  // not visible here (CUDA_VISIBLE_DEVICES): IPC decides
      peer_dev = -1;
    }
    e.same_device = peer_dev == ctx->device;
    if (peer_dev >= 0 && peer_dev != ctx->device) {
      int can = 0;
      SO2DR_CK(cudaDeviceCanAccessPeer(&can, ctx->device, peer_dev));
      if (!can)
        throw ContractError("slab_connect: no peer access from GPU " + std::to_string(ctx->device) + " to GPU " +
                            std::to_string(peer_dev) + " (" + b.pci +
                            "): inter-slab halos need NVLink/NVSwitch or PCIe P2P");
      e.p2p_checked = true;
    }
    char* base = nullptr;
    if (b.pid == static_cast<uint32_t>(getpid())) {
      base = reinterpret_cast<char*>(b.raw);
      e.ipc = false;
    } else {
      void* p = nullptr;
      SO2DR_CK(cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess));
      sl.opened.push_back(p);
      base = static_cast<char*>(p);
      e.ipc = true;
    }
    uint32_t* flags = reinterpret_cast<uint32_t*>(base + b.off_flags);
    if (is_lower) {
      // we push our lower band into the lower neighbour's upper receive buffer
      e.recv = base + b.off_hi;
      e.flag = flags + 1;  // its "hi data ready"
      e.ack = flags + 3;   // its "ack from upper neighbour" (we write it)
    } else {
      e.recv = base + b.off_lo;
      e.flag = flags + 0;
      e.ack = flags + 2;
    }
    e.connected = true;
  };
  open(lower, sl.lower, true);
  open(upper, sl.upper, false);
  if (sl.rank > 0 && !sl.lower.connected) throw ContractError("slab_connect: lower neighbour missing");
  if (sl.rank < sl.world - 1 && !sl.upper.connected)
    throw ContractError("slab_connect: upper neighbour missing");
}

}  // namespace so2dr_eng
