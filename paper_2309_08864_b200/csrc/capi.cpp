// capi.cpp -- the extern "C" boundary (include/so2dr_cuda.h). Converts C
// structs into engine requests and the library's exception types
// (include/so2dr/errors.hpp, mirroring proj/include/so2dr/errors.hpp) into
// so2dr_status codes plus a per-context message.
#include <algorithm>
#include <cstdlib>
#include <cctype>
#include <unordered_map>
#include <mutex>
#include <fstream>
#include <unistd.h>
#include <sys/syscall.h>
#include <sys/mman.h>
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>

#include "engine.h"
#include "k1_launch.h"
#include "so2dr/b200.hpp"
#include "so2dr/report.hpp"
#include "so2dr/specfile.hpp"
#include "so2dr/verify.hpp"
#include "so2dr_cuda.h"

namespace {

thread_local std::string tl_err, tl_constraint, tl_alloc;

so2dr_status fail(so2dr_ctx* ctx, so2dr_status st, const std::string& msg,
                  const std::string& constraint = "", const std::string& alloc = "") {
  tl_err = msg;
  tl_constraint = constraint;
  tl_alloc = alloc;
  if (ctx) {
    ctx->err = msg;
    ctx->constraint = constraint;
    ctx->alloc_id = alloc;
  }
  return st;
}

template <typename F>
so2dr_status guard(so2dr_ctx* ctx, F&& f) {
  try {
    f();
    if (ctx) ctx->err.clear();
    return SO2DR_OK;
  } catch (const so2dr::InfeasibleError& e) {
    return fail(ctx, SO2DR_ERR_INFEASIBLE, e.what(), e.constraint());
  } catch (const so2dr::OutOfDeviceMemoryError& e) {
    return fail(ctx, SO2DR_ERR_DEVICE_OOM, e.what(), "", e.allocation_id());
  } catch (const so2dr::InvalidSpecError& e) {
    return fail(ctx, SO2DR_ERR_INVALID_SPEC, e.what());
  } catch (const so2dr::ContractError& e) {
    return fail(ctx, SO2DR_ERR_CONTRACT, e.what());
  } catch (const so2dr::IoError& e) {
    return fail(ctx, SO2DR_ERR_IO, e.what());
  } catch (const so2dr::DeviceError& e) {
    return fail(ctx, SO2DR_ERR_CUDA, e.what());
  } catch (const std::out_of_range& e) {
    return fail(ctx, SO2DR_ERR_OUT_OF_RANGE, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ctx, SO2DR_ERR_CUDA, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, SO2DR_ERR_CONTRACT, e.what());
  }
}

so2dr::RunConfig to_cfg(const so2dr_run_config* c) {
  if (!c) throw so2dr::InvalidSpecError("run config is NULL");
  so2dr::RunConfig r;
  r.sz = c->sz, r.r = c->r, r.d = c->d, r.s_tb = c->s_tb, r.k_on = c->k_on;
  r.n_strm = c->n_strm, r.n = c->n, r.n_a = c->n_a;
  return r;
}

so2dr::KernelPlan to_kp(const so2dr_kernel_plan* k) {
  so2dr::KernelPlan p;
  if (k) {
    p.k_on = k->k_on;
    p.tile = k->tile;
    p.scratch_budget = k->scratch_budget;
  }
  return p;
}

so2dr::HardwareModel to_hw(const so2dr_hardware* h) {
  so2dr::HardwareModel hw = so2dr::b200_hardware();
  if (h) {
    hw.c_dmem = h->c_dmem;
    hw.bw_dmem = h->bw_dmem;
    hw.bw_intc = h->bw_intc;
    hw.b_elem = h->b_elem;
  }
  return hw;
}

void need_ctx(so2dr_ctx* ctx) {
  if (!ctx) throw so2dr::ContractError("context is NULL");
}

int dtype_of(so2dr_dtype d) {
  if (d != SO2DR_F32 && d != SO2DR_F64) throw so2dr::InvalidSpecError("unknown dtype");
  return d;
}

}  // namespace

extern "C" {

int so2dr_abi_version(void) { return SO2DR_ABI_VERSION; }

int so2dr_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

so2dr_status so2dr_ctx_create(int device, uint64_t budget_bytes, so2dr_ctx** out) {
  if (!out) return fail(nullptr, SO2DR_ERR_CONTRACT, "so2dr_ctx_create: out is NULL");
  *out = nullptr;
  return guard(nullptr, [&] {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw so2dr::DeviceError(
          "no CUDA device available (the SO2DR engine has no CPU fallback): " +
          std::string(cudaGetErrorString(e)));
    }
    if (device < 0 || device >= n) throw so2dr::InvalidSpecError("device index out of range");
    SO2DR_CK(cudaSetDevice(device));
    size_t free_b = 0, total_b = 0;
    SO2DR_CK(cudaMemGetInfo(&free_b, &total_b));
    auto* ctx = new so2dr_ctx();
    ctx->device = device;
    ctx->pool.budget = budget_bytes ? budget_bytes : static_cast<uint64_t>(free_b * 0.9);
    *out = ctx;
  });
}

void so2dr_ctx_destroy(so2dr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (void* p : ctx->slab.opened) cudaIpcCloseMemHandle(p);
  for (auto& kv : ctx->registered) cudaHostUnregister(kv.first);
  for (cudaStream_t s : ctx->streams) cudaStreamDestroy(s);
  delete ctx;
}

so2dr_status so2dr_ctx_set_profiling(so2dr_ctx* ctx, int enable) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ctx->profiling = enable != 0;
  });
}

const char* so2dr_last_error(const so2dr_ctx* ctx) { return ctx ? ctx->err.c_str() : tl_err.c_str(); }
const char* so2dr_last_constraint(const so2dr_ctx* ctx) {
  return ctx ? ctx->constraint.c_str() : tl_constraint.c_str();
}
const char* so2dr_last_allocation_id(const so2dr_ctx* ctx) {
  return ctx ? ctx->alloc_id.c_str() : tl_alloc.c_str();
}

namespace {
// NUMA-bound pinned allocations (host_alloc on a multi-node host): tracked so
// host_free unregisters and unmaps them instead of cudaFreeHost.
std::mutex g_numa_mu;
std::unordered_map<void*, size_t> g_numa_allocs;

int numa_nodes() {
  int n = 0;
  for (int i = 0; i < 1024; ++i) {
    const std::string d = "/sys/devices/system/node/node" + std::to_string(i);
    if (access(d.c_str(), F_OK) != 0) break;
    ++n;
  }
  return n;
}

void* numa_pinned_alloc(int node, size_t bytes) {
  // 2 MiB aligned so transparent huge pages back it (4 KiB-page pinned memory
  // is ~15% slower when H2D and D2H overlap, see so2dr_cuda.h)
  bytes = (bytes + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return nullptr;
  madvise(p, bytes, MADV_HUGEPAGE);
  unsigned long mask[16] = {};
  if (node < 0 || node >= 16 * 64) {
    munmap(p, bytes);
    return nullptr;
  }
  mask[node / 64] = 1ul << (node % 64);
  constexpr int kMpolBind = 2;
  if (syscall(SYS_mbind, p, bytes, kMpolBind, mask, 16 * 64 + 1, 0) != 0) {
    munmap(p, bytes);
    return nullptr;
  }
  // pinning faults every page in on the bound node
  if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) != cudaSuccess) {
    cudaGetLastError();
    munmap(p, bytes);
    return nullptr;
  }
  return p;
}
}  // namespace

int so2dr_pci_numa_node(const char* sysfs_root, const char* pci_bus_id) {
  if (!pci_bus_id) return -1;
  std::string id(pci_bus_id);
  for (auto& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  // cudaDeviceGetPCIBusId gives "0000:40:00.0"; sysfs names are the same, lower-case
  const std::string root = (sysfs_root && *sysfs_root) ? sysfs_root : "/sys";
  std::ifstream in(root + "/bus/pci/devices/" + id + "/numa_node");
  int node = -1;
  if (!(in >> node)) return -1;
  return node;
}

int so2dr_device_numa_node(int device) {
  char bus[32] = {};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return so2dr_pci_numa_node("", bus);
}

so2dr_status so2dr_host_alloc(so2dr_ctx* ctx, size_t bytes, void** out) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (!out || !bytes) throw so2dr::ContractError("host_alloc: bad arguments");
    SO2DR_CK(cudaSetDevice(ctx->device));
    // NUMA-local pages when the host has several nodes (SO2DR_HOST_NUMA=0: off)
    static const bool numa_off = [] {
      const char* e = std::getenv("SO2DR_HOST_NUMA");
      return e && std::string(e) == "0";
    }();
    static const int nodes = numa_nodes();
    if (!numa_off && nodes > 1) {
      const int node = so2dr_device_numa_node(ctx->device);
      if (node >= 0) {
        if (void* p = numa_pinned_alloc(node, bytes)) {
          std::lock_guard<std::mutex> lk(g_numa_mu);
          g_numa_allocs[p] = (bytes + (2u << 20) - 1) & ~static_cast<size_t>((2u << 20) - 1);
          *out = p;
          return;
        }
      }
    }
    // SO2DR_HOST_ALLOC_DEFAULT=1: plain cudaHostAllocDefault (diagnostics)
    static const bool dflt = std::getenv("SO2DR_HOST_ALLOC_DEFAULT") != nullptr;
    const cudaError_t e = cudaHostAlloc(out, bytes, dflt ? cudaHostAllocDefault : cudaHostAllocPortable);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw so2dr::OutOfDeviceMemoryError("host:pinned", bytes, 0, 0);
    }
    SO2DR_CK(e);
  });
}

so2dr_status so2dr_host_free(so2dr_ctx* ctx, void* p) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (!p) return;
    size_t numa_bytes = 0;
    {
      std::lock_guard<std::mutex> lk(g_numa_mu);
      auto it = g_numa_allocs.find(p);
      if (it != g_numa_allocs.end()) numa_bytes = it->second, g_numa_allocs.erase(it);
    }
    if (numa_bytes) {
      SO2DR_CK(cudaHostUnregister(p));
      munmap(p, numa_bytes);
    } else {
      SO2DR_CK(cudaFreeHost(p));
    }
  });
}

so2dr_status so2dr_host_register(so2dr_ctx* ctx, void* base, size_t bytes) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (!base || !bytes) throw so2dr::ContractError("host_register: empty range");
    if (ctx->registered.count(base)) return;
    SO2DR_CK(cudaSetDevice(ctx->device));
    SO2DR_CK(cudaHostRegister(base, bytes, cudaHostRegisterPortable));
    ctx->registered[base] = bytes;
  });
}

so2dr_status so2dr_host_unregister(so2dr_ctx* ctx, void* base) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    auto it = ctx->registered.find(base);
    if (it == ctx->registered.end()) throw so2dr::ContractError("host_unregister: range not registered");
    SO2DR_CK(cudaHostUnregister(base));
    ctx->registered.erase(it);
  });
}

so2dr_status so2dr_run(so2dr_ctx* ctx, so2dr_mode mode, const so2dr_stencil_desc* st,
                       const so2dr_run_config* cfg, const so2dr_kernel_plan* kp,
                       const so2dr_hardware* hw, const so2dr_hooks* hooks, so2dr_dtype dtype,
                       void* grid, so2dr_ledger* ledger_out, so2dr_timing* timing_out,
                       so2dr_diag_row* diag, size_t diag_cap, size_t* n_diag) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (mode != SO2DR_MODE_SO2DR && mode != SO2DR_MODE_RESREU && mode != SO2DR_MODE_INCORE)
      throw so2dr::InvalidSpecError("unknown engine mode");
    so2dr_eng::RunRequest q;
    q.mode = mode;
    q.st = so2dr_eng::make_stencil(st);
    q.cfg = to_cfg(cfg);
    q.kp = to_kp(kp);
    q.hw = to_hw(hw);
    if (hooks) q.hooks = *hooks;
    q.dtype = dtype_of(dtype);
    if (!grid) throw so2dr::ContractError("grid pointer is NULL");
    q.grid = grid;
    so2dr_eng::RunResponse out;
    so2dr_eng::run(ctx, q, out);
    if (ledger_out) *ledger_out = out.ledger;
    if (timing_out) *timing_out = out.timing;
    if (n_diag) *n_diag = out.diag.size();
    if (diag)
      std::memcpy(diag, out.diag.data(), std::min(diag_cap, out.diag.size()) * sizeof(so2dr_diag_row));
  });
}

so2dr_status so2dr_slab_rows(const so2dr_run_config* cfg, int dim, int rank, int world,
                             int64_t* lo, int64_t* hi) {
  return guard(nullptr, [&] {
    if (!cfg || !lo || !hi) throw so2dr::ContractError("slab_rows: NULL argument");
    so2dr_eng::slab_rows(*cfg, dim, rank, world, lo, hi);
  });
}

so2dr_status so2dr_slab_prepare(so2dr_ctx* ctx, const so2dr_stencil_desc* st,
                                const so2dr_run_config* cfg, so2dr_dtype dtype, int rank,
                                int world, uint8_t blob_out[SO2DR_PEER_BLOB_BYTES]) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (!cfg || !blob_out) throw so2dr::ContractError("slab_prepare: NULL argument");
    const so2dr_eng::StencilDev s = so2dr_eng::make_stencil(st);
    so2dr_eng::slab_prepare(ctx, s, *cfg, dtype_of(dtype), rank, world, blob_out);
  });
}

so2dr_status so2dr_slab_connect(so2dr_ctx* ctx, const uint8_t* lower_blob,
                                const uint8_t* upper_blob) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    so2dr_eng::slab_connect(ctx, lower_blob, upper_blob);
  });
}

so2dr_status so2dr_slab_run(so2dr_ctx* ctx, const so2dr_stencil_desc* st,
                            const so2dr_run_config* cfg, const so2dr_kernel_plan* kp,
                            so2dr_dtype dtype, void* slab, so2dr_ledger* ledger_out,
                            so2dr_timing* timing_out) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    const so2dr_eng::SlabState& sl = ctx->slab;
    if (!sl.prepared) throw so2dr::ContractError("slab_run before slab_prepare");
    if (!cfg || std::memcmp(cfg, &sl.cfg, sizeof(*cfg)) != 0)
      throw so2dr::ContractError("slab_run: config differs from the prepared one");
    if (sl.rank > 0 && !sl.lower.connected) throw so2dr::ContractError("slab_run: not connected");
    if (sl.rank < sl.world - 1 && !sl.upper.connected)
      throw so2dr::ContractError("slab_run: not connected");
    so2dr_eng::RunRequest q;
    q.mode = SO2DR_MODE_SO2DR;
    q.st = so2dr_eng::make_stencil(st);
    q.cfg = to_cfg(cfg);
    q.kp = to_kp(kp);
    q.hw = so2dr::b200_hardware();
    q.hw.c_dmem = ~0ull;
    q.dtype = dtype_of(dtype);
    if (q.dtype != sl.dtype || q.st.dim != sl.dim)
      throw so2dr::ContractError("slab_run: dtype/dim differ from the prepared ones");
    q.grid = slab;
    q.rank = sl.rank;
    q.world = sl.world;
    int64_t lo, hi;
    so2dr_eng::slab_rows(*cfg, q.st.dim, sl.rank, sl.world, &lo, &hi);
    q.host_lo = lo;
    so2dr_eng::RunResponse out;
    so2dr_eng::run(ctx, q, out);
    if (ledger_out) *ledger_out = out.ledger;
    if (timing_out) *timing_out = out.timing;
  });
}

so2dr_status so2dr_fused_kernel(so2dr_ctx* ctx, const so2dr_stencil_desc* st, so2dr_dtype dtype,
                                void* buf0, void* buf1, int base_row, int rows, int cols,
                                int read, int steps, int tile, const int32_t region[4],
                                const int32_t interior[4], const int32_t owned[4],
                                uint64_t stats_out[4]) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (!buf0 || !buf1 || !region || !interior || !owned || !stats_out)
      throw so2dr::ContractError("fused_kernel: NULL argument");
    const so2dr_eng::StencilDev s = so2dr_eng::make_stencil(st);
    so2dr_eng::fused_kernel_host(ctx, s, dtype_of(dtype), buf0, buf1, base_row, rows, cols, read,
                                 steps, tile, region, interior, owned, stats_out);
  });
}

so2dr_status so2dr_apply_step(so2dr_ctx* ctx, const so2dr_stencil_desc* st, so2dr_dtype dtype,
                              int sz, int r, const void* in, void* out, int row_lo, int row_hi) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    const so2dr_eng::StencilDev s = so2dr_eng::make_stencil(st);
    if (s.radius != r) throw so2dr::ContractError("apply_step: stencil radius differs from grid ring");
    so2dr_eng::apply_step_host(ctx, s, dtype_of(dtype), sz, r, in, out, row_lo, row_hi);
  });
}

so2dr_status so2dr_run_reference(so2dr_ctx* ctx, const so2dr_stencil_desc* st, so2dr_dtype dtype,
                                 int sz, int r, const void* in, void* out, int steps) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    const so2dr_eng::StencilDev s = so2dr_eng::make_stencil(st);
    if (s.radius != r) throw so2dr::ContractError("run_reference: stencil radius differs from grid ring");
    so2dr_eng::run_reference_host(ctx, s, dtype_of(dtype), sz, r, in, out, steps);
  });
}

so2dr_status so2dr_init_grid(so2dr_ctx* ctx, so2dr_dtype dtype, int dim, int sz, int r,
                             uint64_t seed, void* out) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    so2dr_eng::init_rows(ctx, dtype_of(dtype), dim, sz, r, seed, 0, sz + 2 * r, out);
  });
}

so2dr_status so2dr_init_rows(so2dr_ctx* ctx, so2dr_dtype dtype, int dim, int sz, int r,
                             uint64_t seed, int64_t lo, int64_t hi, void* out) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    so2dr_eng::init_rows(ctx, dtype_of(dtype), dim, sz, r, seed, lo, hi, out);
  });
}

uint64_t so2dr_grid_checksum(const void* data, size_t bytes) {
  const auto* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xCBF29CE484222325ULL;
  for (size_t i = 0; i < bytes; ++i) h = (h ^ p[i]) * 0x100000001B3ULL;
  return h;
}

so2dr_status so2dr_kernel_stats(int radius, int steps, int tile, const int32_t region[4],
                                const int32_t interior[4], const int32_t owned[4], int sy0,
                                int sy1, int64_t cols, uint64_t stats_out[4]) {
  return guard(nullptr, [&] {
    if (!region || !interior || !owned || !stats_out)
      throw so2dr::ContractError("kernel_stats: NULL argument");
    if (steps < 1) throw so2dr::InvalidSpecError("fused_kernel: steps must be >= 1");
    if (tile < 1) throw so2dr::InvalidSpecError("fused_kernel: tile must be >= 1");
    const so2dr::KernelStats ks = so2dr_eng::tile_stats(
        radius, steps, tile, so2dr::Rect{region[0], region[1], region[2], region[3]},
        so2dr::Rect{interior[0], interior[1], interior[2], interior[3]},
        so2dr::Rect{owned[0], owned[1], owned[2], owned[3]}, sy0, sy1, cols);
    stats_out[0] = ks.scratch_load;
    stats_out[1] = ks.scratch_store;
    stats_out[2] = ks.updates;
    stats_out[3] = ks.redundant;
  });
}

so2dr_status so2dr_arena_bytes(const so2dr_run_config* cfg, const so2dr_kernel_plan* kp,
                               uint64_t* out) {
  return guard(nullptr, [&] {
    if (!out) throw so2dr::ContractError("arena_bytes: out is NULL");
    *out = so2dr::so2dr_arena_bytes(to_cfg(cfg), to_kp(kp));
  });
}

namespace {
so2dr::b200::Profile plan_profile(const char* json) {
  return json ? so2dr::b200::profile_from_json(json, "<argument>") : so2dr::b200::default_profile();
}
so2dr::b200::Problem plan_problem(int dim, so2dr_dtype dtype, int star, int radius, int sz, int n,
                                  uint64_t budget, int n_strm) {
  so2dr::b200::Problem pb;
  if (dim != 2 && dim != 3) throw so2dr::ContractError("planner: dim must be 2 or 3");
  pb.dim = dim;
  pb.elem_bytes = dtype == SO2DR_F64 ? 8 : 4;
  pb.star = star != 0;
  pb.radius = radius;
  pb.sz = sz;
  pb.n = n;
  pb.budget = budget;
  pb.n_strm = {n_strm};
  return pb;
}
void to_entry(const so2dr::b200::Candidate& c, so2dr_plan_entry* e) {
  e->d = c.d, e->s_tb = c.s_tb, e->k_on = c.k_on, e->n_strm = c.n_strm, e->feasible = c.feasible;
  e->launches = c.launches;
  e->device_bytes = c.device_bytes;
  e->t_pcie_s = c.t_pcie, e->t_kernel_s = c.t_kernel, e->t_fill_s = c.t_fill, e->t_total_s = c.t_total;
  e->gcell_per_s = c.gcells;
}
}  // namespace

so2dr_status so2dr_plan_b200(const char* profile_json, int dim, so2dr_dtype dtype, int star, int radius,
                             int sz, int n, uint64_t budget_bytes, int n_strm, so2dr_plan_entry* best,
                             so2dr_plan_entry* entries, int32_t capacity, int32_t* count) {
  return guard(nullptr, [&] {
    if (!best) throw so2dr::ContractError("plan_b200: best is NULL");
    const auto pl = so2dr::b200::plan(plan_profile(profile_json),
                                      plan_problem(dim, dtype, star, radius, sz, n, budget_bytes, n_strm));
    to_entry(pl.best, best);
    const int32_t total = static_cast<int32_t>(pl.candidates.size());
    if (count) *count = total;
    for (int32_t i = 0; entries && i < std::min(capacity, total); ++i) to_entry(pl.candidates[i], &entries[i]);
  });
}

so2dr_status so2dr_predict_b200(const char* profile_json, int dim, so2dr_dtype dtype, int star, int radius,
                                int sz, int n, uint64_t budget_bytes, int d, int s_tb, int k_on,
                                int n_strm, so2dr_plan_entry* out) {
  return guard(nullptr, [&] {
    if (!out) throw so2dr::ContractError("predict_b200: out is NULL");
    const auto c = so2dr::b200::predict(plan_profile(profile_json),
                                        plan_problem(dim, dtype, star, radius, sz, n, budget_bytes, n_strm), d,
                                        s_tb, k_on, n_strm);
    to_entry(c, out);
  });
}

so2dr_status so2dr_slab_info(const so2dr_ctx* ctx, int32_t out[4]) {
  so2dr_ctx* c = const_cast<so2dr_ctx*>(ctx);
  return guard(c, [&] {
    need_ctx(c);
    if (!out) throw so2dr::ContractError("slab_info: out is NULL");
    const auto& sl = ctx->slab;
    auto kind = [](const so2dr_eng::PeerEdge& e) {
      if (!e.connected) return 0;
      if (!e.ipc) return 1;
      if (e.same_device) return 2;
      return e.p2p_checked ? 3 : 4;
    };
    out[0] = sl.rank, out[1] = sl.world, out[2] = kind(sl.lower), out[3] = kind(sl.upper);
  });
}

int32_t so2dr_k1_max_steps(int dim, so2dr_dtype dtype, so2dr_kind kind, int radius) {
  return so2dr_dev::k1_max_steps(dim, dtype == SO2DR_F64 ? 1 : 0, kind, radius);
}

so2dr_status so2dr_device_bytes(const so2dr_run_config* cfg, int dim, so2dr_dtype dtype,
                                uint64_t* out) {
  return guard(nullptr, [&] {
    if (!out) throw so2dr::ContractError("device_bytes: out is NULL");
    const so2dr::RunConfig c = to_cfg(cfg);
    c.validate();
    const so2dr_eng::Geo g = so2dr_eng::make_geo(dim, c.sz, c.r, dtype_of(dtype));
    *out = so2dr_eng::device_footprint(c, g, c.n_strm);
  });
}

so2dr_status so2dr_plan_chunks(const so2dr_run_config* cfg, int32_t* fence_out,
                               int32_t* chunks_out) {
  return guard(nullptr, [&] {
    const so2dr::ChunkLayout L = so2dr::plan_chunks(to_cfg(cfg));
    if (fence_out)
      for (size_t i = 0; i < L.fence.size(); ++i) fence_out[i] = L.fence[i];
    if (chunks_out)
      for (size_t i = 0; i < L.chunks.size(); ++i) {
        const so2dr::ChunkIntervals& c = L.chunks[i];
        const so2dr::RowInterval iv[5] = {c.core, c.working, c.transfer, c.shared_in, c.shared_out};
        for (int k = 0; k < 5; ++k) {
          chunks_out[i * 10 + 2 * k] = iv[k].lo;
          chunks_out[i * 10 + 2 * k + 1] = iv[k].hi;
        }
      }
  });
}

so2dr_status so2dr_expected_ledger(so2dr_mode mode, const so2dr_run_config* cfg,
                                   const so2dr_kernel_plan* kp, int dim, so2dr_dtype dtype,
                                   uint64_t out6[6], int32_t* exact) {
  return guard(nullptr, [&] {
    if (!out6) throw so2dr::ContractError("expected_ledger: out is NULL");
    const so2dr::RunConfig c = to_cfg(cfg);
    const so2dr::ExpectedLedger e =
        so2dr::expected_ledger(static_cast<so2dr::EngineMode>(mode), c, to_kp(kp));
    // the closed forms count 2D fp32 rows; scale to planes / 8-byte cells
    const uint64_t p = c.padded();
    const uint64_t scale = (dim == 3 ? p : 1) * (dtype == SO2DR_F64 ? 2 : 1);
    out6[0] = e.htod * scale;
    out6[1] = e.dtoh * scale;
    out6[2] = e.ondevice * scale;
    out6[3] = e.kernel_invocations;
    out6[4] = e.rounds;
    out6[5] = e.redundant_updates * (dim == 3 ? p : 1);
    if (exact) *exact = e.redundancy_exact ? 1 : 0;
  });
}

// ---------------------------------------------------- spec files / outputs --

namespace {

void copy_text(char* dst, size_t cap, const std::string& src) {
  if (!cap) return;
  const size_t n = std::min(cap - 1, src.size());
  std::memcpy(dst, src.data(), n);
  dst[n] = 0;
}

void to_c_spec(const so2dr::RunSpecFile& f, so2dr_spec* out) {
  std::memset(out, 0, sizeof(*out));
  const int r = f.stencil.radius, dim = f.dim;
  const int e = 2 * r + 1;
  const int n = dim == 3 ? e * e * e : e * e;
  if (n > SO2DR_SPEC_MAX_WEIGHTS)
    throw so2dr::InvalidSpecError("spec: radius " + std::to_string(r) + " too large for dim " + std::to_string(dim));
  const so2dr::StencilKind k = f.stencil.kind;
  int kind = k == so2dr::StencilKind::gradient ? SO2DR_KIND_GRADIENT
             : k == so2dr::StencilKind::star   ? SO2DR_KIND_STAR
                                                : SO2DR_KIND_BOX;
  auto on_axis = [&](int i) {
    const int dx = i % e - r, dy = (i / e) % e - r, dz = dim == 3 ? i / (e * e) - r : 0;
    return (dz != 0) + (dy != 0) + (dx != 0) <= 1;
  };
  if (kind == SO2DR_KIND_GRADIENT) {
    // gradient ignores weights (pinned expression)
  } else if (static_cast<int>(f.weights.size()) == n) {
    for (int i = 0; i < n; ++i) out->weights_buf[i] = static_cast<double>(f.weights[i]);
  } else if (!f.weights.empty()) {  // star on-axis list, canonical order
    size_t next = 0;
    for (int i = 0; i < n; ++i) out->weights_buf[i] = on_axis(i) ? f.weights[next++] : 0.0;
  } else {
    // defaults in the run's precision (stencil.cpp:27-33 for fp32 box):
    // box 1/(2r+1)^dim, star 1/(2*dim*r+1) on axis
    const int cnt = kind == SO2DR_KIND_STAR ? 2 * dim * r + 1 : n;
    const double w = f.dtype == "f64" ? 1.0 / cnt : static_cast<double>(1.0f / static_cast<float>(cnt));
    for (int i = 0; i < n; ++i) out->weights_buf[i] = (kind == SO2DR_KIND_BOX || on_axis(i)) ? w : 0.0;
  }
  if (f.dtype == "f32")  // fp32 runs use (float)w: store the value they will use
    for (int i = 0; i < n; ++i) out->weights_buf[i] = static_cast<float>(out->weights_buf[i]);
  out->stencil.kind = kind;
  out->stencil.dim = dim;
  out->stencil.radius = r;
  out->stencil.weights = out->weights_buf;
  const so2dr::RunConfig& c = f.config;
  out->config = {c.sz, c.r, c.d, c.s_tb, c.k_on, c.n_strm, c.n, c.n_a};
  out->kernel = {f.kernel.k_on, f.kernel.tile, f.kernel.scratch_budget};
  out->seed = f.seed;
  out->mode = static_cast<int32_t>(f.mode);
  out->dtype = f.dtype == "f64" ? SO2DR_F64 : SO2DR_F32;
  std::string name = f.stencil.name();
  if (dim == 3) name.replace(name.find("2d"), 2, "3d");
  copy_text(out->stencil_name, sizeof(out->stencil_name), name);
  copy_text(out->hardware_path, sizeof(out->hardware_path), f.hardware_path.value_or(""));
  copy_text(out->grid_dump_path, sizeof(out->grid_dump_path), f.grid_dump_path.value_or(""));
}

void out_text(const std::string& s, char* buf, size_t cap, size_t* len_out) {
  if (len_out) *len_out = s.size();
  if (buf && cap > s.size()) {
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
  }
}

}  // namespace

so2dr_status so2dr_spec_parse(const char* text, const char* origin, so2dr_spec* out) {
  return guard(nullptr, [&] {
    if (!text || !out) throw so2dr::ContractError("spec_parse: text/out is NULL");
    to_c_spec(so2dr::parse_spec_json(text, origin ? origin : "spec"), out);
  });
}

so2dr_status so2dr_spec_parse_file(const char* path, so2dr_spec* out) {
  return guard(nullptr, [&] {
    if (!path || !out) throw so2dr::ContractError("spec_parse_file: path/out is NULL");
    to_c_spec(so2dr::parse_spec_file(path), out);
  });
}

int so2dr_preset_count(void) { return static_cast<int>(so2dr::preset_names().size()); }

const char* so2dr_preset_name(int i) {
  static const std::vector<std::string> names = so2dr::preset_names();
  return i >= 0 && i < static_cast<int>(names.size()) ? names[i].c_str() : nullptr;
}

so2dr_status so2dr_preset_json(const char* name, char* buf, size_t cap, size_t* len_out) {
  return guard(nullptr, [&] {
    if (!name) throw so2dr::ContractError("preset_json: name is NULL");
    out_text(so2dr::preset_json(name), buf, cap, len_out);
  });
}

so2dr_status so2dr_report_json(const so2dr_report_in* in, char* buf, size_t cap, size_t* len_out) {
  return guard(nullptr, [&] {
    if (!in) throw so2dr::ContractError("report_json: input is NULL");
    so2dr::RunReport rep;
    rep.mode = static_cast<so2dr::EngineMode>(in->mode);
    rep.config = to_cfg(&in->config);
    rep.kernel = to_kp(&in->kernel);
    rep.stencil_name = in->stencil_name ? in->stencil_name : "";
    rep.checksum = in->checksum;
    const so2dr_ledger& l = in->ledger;
    rep.ledger = so2dr::LedgerSnapshot{l.htod,          l.dtoh,          l.ondevice,
                                       l.scratch_load,  l.scratch_store, l.element_updates,
                                       l.redundant_updates, l.kernel_invocations, l.rounds};
    rep.times = so2dr::modeled_times(rep.ledger, to_hw(in->hw));
    rep.transfer_time_excluded = rep.mode == so2dr::EngineMode::incore;
    if (in->measured) {
      const so2dr_timing& t = *in->measured;
      rep.arena_peak = t.arena_peak;
      rep.arena_capacity = t.arena_capacity;
      rep.wall_seconds = t.wall_seconds;
      rep.measured = so2dr::MeasuredTimes{t.device_ms, t.kernel_ms, t.kernel_launches, t.kernel_alg_bytes,
                                          t.device_bytes};
    }
    out_text(so2dr::report_to_json(rep, in->deterministic != 0), buf, cap, len_out);
  });
}

so2dr_status so2dr_ledger_csv(const so2dr_ledger* l, char* buf, size_t cap, size_t* len_out) {
  return guard(nullptr, [&] {
    if (!l) throw so2dr::ContractError("ledger_csv: ledger is NULL");
    out_text(so2dr::ledger_to_csv(so2dr::LedgerSnapshot{l->htod, l->dtoh, l->ondevice, l->scratch_load,
                                                        l->scratch_store, l->element_updates,
                                                        l->redundant_updates, l->kernel_invocations,
                                                        l->rounds}),
             buf, cap, len_out);
  });
}

so2dr_status so2dr_diagnostics_csv(const so2dr_diag_row* rows, size_t n, char* buf, size_t cap,
                                   size_t* len_out) {
  return guard(nullptr, [&] {
    if (n && !rows) throw so2dr::ContractError("diagnostics_csv: rows is NULL");
    std::vector<so2dr::DiagRow> v;
    for (size_t i = 0; i < n; ++i)
      v.push_back({rows[i].round, rows[i].chunk, static_cast<so2dr::Stage>(rows[i].stage), rows[i].bytes,
                   rows[i].updates});
    out_text(so2dr::diagnostics_to_csv(v), buf, cap, len_out);
  });
}

}  // extern "C"
