/*
 * so2dr_cuda.h -- C ABI of the B200-native SO2DR out-of-core stencil engine.
 *
 * This is the drop-in boundary. The reference (arXiv 2309.08864 artifact,
 * /root/reference/proj) is a C++20 library with no FFI; its public entry
 * points are C++ functions. Every entry point below replaces one of them and
 * is what a binding (ctypes, the C++ mirror in include/so2dr/, cgo, JNI)
 * calls. Plain pointers and sizes only; no C++ or torch types.
 *
 *   so2dr_run            <- so2dr::run_engine         proj/include/so2dr/engine.hpp:79-81
 *   so2dr_fused_kernel   <- so2dr::fused_kernel       proj/include/so2dr/kernels.hpp:77-79
 *   so2dr_apply_step     <- so2dr::apply_step         proj/include/so2dr/stencil.hpp:102-103
 *   so2dr_run_reference  <- so2dr::run_reference      proj/include/so2dr/stencil.hpp:107
 *   so2dr_init_grid      <- so2dr::init_grid          proj/include/so2dr/stencil.hpp:91
 *   so2dr_grid_checksum  <- so2dr::grid_checksum      proj/include/so2dr/stencil.hpp:110
 *   so2dr_arena_bytes    <- so2dr::so2dr_arena_bytes  proj/include/so2dr/engine.hpp:85
 *   so2dr_plan_chunks    <- so2dr::plan_chunks        proj/include/so2dr/layout.hpp:73
 *   so2dr_expected_ledger<- so2dr::expected_ledger    proj/include/so2dr/verify.hpp:25-26
 *   status codes         <- proj/include/so2dr/errors.hpp:11-63 exception types
 *
 * Extensions (additive, no reference counterpart): dim 3, fp64, the star
 * kind, an in-place host grid, a real HBM budget per context, slab
 * partitioning across ranks (one process per GPU) with GPU-to-GPU halo
 * exchange over CUDA IPC peer memory.
 *
 * Threading: a context belongs to one host thread at a time. Every call is
 * synchronous: it returns after the device work it enqueued has finished.
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns SO2DR_ERR_CUDA.
 */
#ifndef SO2DR_CUDA_H
#define SO2DR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SO2DR_ABI_VERSION 1

typedef enum {
  SO2DR_OK = 0,
  SO2DR_ERR_INVALID_SPEC = 1, /* InvalidSpecError       errors.hpp:18-21 */
  SO2DR_ERR_INFEASIBLE = 2,   /* InfeasibleError        errors.hpp:23-36 (constraint in so2dr_last_constraint) */
  SO2DR_ERR_DEVICE_OOM = 3,   /* OutOfDeviceMemoryError errors.hpp:38-52 (id in so2dr_last_allocation_id) */
  SO2DR_ERR_CONTRACT = 4,     /* ContractError          errors.hpp:54-59 */
  SO2DR_ERR_IO = 5,           /* IoError                errors.hpp:61-65 */
  SO2DR_ERR_CUDA = 6,         /* CUDA runtime/driver failure (new) */
  SO2DR_ERR_OUT_OF_RANGE = 7  /* std::out_of_range (layout.cpp:83-88, stencil.cpp:154) */
} so2dr_status;

typedef enum { SO2DR_MODE_SO2DR = 0, SO2DR_MODE_RESREU = 1, SO2DR_MODE_INCORE = 2 } so2dr_mode;
typedef enum { SO2DR_F32 = 0, SO2DR_F64 = 1 } so2dr_dtype;
typedef enum { SO2DR_KIND_BOX = 0, SO2DR_KIND_GRADIENT = 1, SO2DR_KIND_STAR = 2 } so2dr_kind;

/* Stencil (StencilSpec, stencil.hpp:19-45). `weights` holds (2r+1)^dim
 * entries in canonical order (dz, dy, dx ascending, dx fastest) -- the
 * accumulation order that defines the bit-exact result. fp32 runs use
 * (float)weights[i] (must round-trip exactly). STAR reads only on-axis
 * entries; GRADIENT ignores weights (pinned expression, stencil.cpp:122-135).
 * A BOX whose off-axis weights are all zero is executed by the star kernel
 * (bit-identical for finite data). */
typedef struct {
  int32_t kind;   /* so2dr_kind */
  int32_t dim;    /* 2 or 3 */
  int32_t radius; /* 1..4 (box/star), 1 (gradient) */
  int32_t reserved;
  const double* weights;
} so2dr_stencil_desc;

/* RunConfig, layout.hpp:33-51 */
typedef struct {
  int32_t sz, r, d, s_tb, k_on, n_strm, n, n_a;
} so2dr_run_config;

/* KernelPlan, engine.hpp:22-33. `tile` is the reference's scratch-tile edge:
 * it shapes the scratch/redundancy ledger counters only (the device kernel
 * tiles on its own). */
typedef struct {
  int32_t k_on, tile;
  uint64_t scratch_budget;
} so2dr_kernel_plan;

/* HardwareModel, layout.hpp:13-21. c_dmem is the MODELED arena capacity the
 * reference's DeviceArena enforces; the real HBM budget is the context's. */
typedef struct {
  uint64_t c_dmem;
  double bw_dmem, bw_intc;
  int32_t b_elem;
  int32_t reserved;
} so2dr_hardware;

/* EngineHooks, engine.hpp:62-65 (fault injection: zero one boundary's slot). */
typedef struct {
  int32_t corrupt_share;
  int32_t boundary;
} so2dr_hooks;

/* LedgerSnapshot, memsim.hpp:52-65 (same field order) */
typedef struct {
  uint64_t htod, dtoh, ondevice, scratch_load, scratch_store, element_updates,
      redundant_updates, kernel_invocations, rounds;
} so2dr_ledger;

/* Measured timing (new; the reference only has wall_seconds, engine.cpp:151-172). */
typedef struct {
  double wall_seconds;      /* host clock around the whole call (reference semantics) */
  double device_ms;         /* CUDA events: first enqueue -> last D2H completion */
  double kernel_ms;         /* sum of K1 launch durations (per-launch event pairs) */
  double kernel_max_ms;     /* longest single K1 launch */
  uint64_t kernel_launches; /* K1 launches */
  uint64_t kernel_alg_bytes;/* algorithmic HBM bytes of all K1 launches (read + write of
                               the input/output rows of every launch) */
  uint64_t cell_updates;    /* useful updates: sz^dim * n */
  uint64_t h2d_bytes, d2h_bytes, d2d_bytes, peer_bytes;
  uint64_t arena_peak, arena_capacity; /* modeled arena (reference semantics) */
  uint64_t device_bytes;               /* real HBM allocated for the run */
} so2dr_timing;

/* DiagRow, engine.hpp:35-44; stage 0 htod 1 share_read 2 share_write 3 kernel 4 dtoh */
typedef struct {
  int32_t round, chunk, stage, reserved;
  uint64_t bytes, updates;
  double ms;    /* measured stage duration (CUDA events), 0 when not timed */
  double t0_ms; /* stage start relative to the run's first enqueue (when timed) */
} so2dr_diag_row;

typedef struct so2dr_ctx so2dr_ctx;

/* ---- context ----------------------------------------------------------- */
/* budget_bytes: real HBM cap for engine buffers (0 = 90% of free memory). */
so2dr_status so2dr_ctx_create(int device, uint64_t budget_bytes, so2dr_ctx** out);
void so2dr_ctx_destroy(so2dr_ctx* ctx);
/* Enable per-stage event timing into diag rows (costs a few events/chunk). */
so2dr_status so2dr_ctx_set_profiling(so2dr_ctx* ctx, int enable);
/* Message of the last failing call on this ctx (or of the thread when ctx is NULL). */
const char* so2dr_last_error(const so2dr_ctx* ctx);
const char* so2dr_last_constraint(const so2dr_ctx* ctx);
const char* so2dr_last_allocation_id(const so2dr_ctx* ctx);
int so2dr_abi_version(void);
/* Number of visible CUDA devices (0 when none; never fails). */
int so2dr_device_count(void);

/* Pinned host allocation for grids (cudaHostAlloc, portable). Preferred over
 * registering malloc'd memory: on this pool's B200 hosts, 4 KiB-page
 * registered memory sustains only ~43 GB/s per direction when H2D and D2H
 * overlap, cudaHostAlloc / huge-page memory ~50 GB/s (tools/cu/pin_bench.cu).
 * On a multi-socket host the pages are bound to the NUMA node of the
 * context's GPU (2 MiB-aligned mmap, transparent huge pages, mbind MPOL_BIND,
 * then cudaHostRegister): each rank's slab streams from its own socket's DRAM
 * (SURVEY 7 hard part 7). One NUMA node or SO2DR_HOST_NUMA=0: cudaHostAlloc. */
so2dr_status so2dr_host_alloc(so2dr_ctx* ctx, size_t bytes, void** out);
so2dr_status so2dr_host_free(so2dr_ctx* ctx, void* p);
/* NUMA node of a GPU (sysfs numa_node of its PCI function), -1 if unknown. */
int so2dr_device_numa_node(int device);
/* NUMA node of the `sysfs_root`/bus/pci/devices/<pci_bus_id>/numa_node file,
 * -1 if absent (host logic of so2dr_device_numa_node; sysfs_root "" = /sys). */
int so2dr_pci_numa_node(const char* sysfs_root, const char* pci_bus_id);
/* Pin a caller-owned host range (cudaHostRegister); idempotent per range. */
so2dr_status so2dr_host_register(so2dr_ctx* ctx, void* base, size_t bytes);
so2dr_status so2dr_host_unregister(so2dr_ctx* ctx, void* base);

/* ---- the hot path ------------------------------------------------------ */
/* run_engine. `grid` is the padded grid ((sz+2r)^dim cells of dtype,
 * row-major), updated IN PLACE; it may be pageable or pinned host memory, or
 * a device pointer (then all "transfers" are device-to-device: the grid is
 * resident in HBM). diag/diag_cap/n_diag may be NULL/0. */
so2dr_status so2dr_run(so2dr_ctx* ctx, so2dr_mode mode, const so2dr_stencil_desc* st,
                       const so2dr_run_config* cfg, const so2dr_kernel_plan* kp,
                       const so2dr_hardware* hw, const so2dr_hooks* hooks,
                       so2dr_dtype dtype, void* grid, so2dr_ledger* ledger_out,
                       so2dr_timing* timing_out, so2dr_diag_row* diag, size_t diag_cap,
                       size_t* n_diag);

/* ---- multi-rank slab partitioning (one process or context per GPU) -------
 * The d chunks are split into `world` contiguous slabs of d/world chunks; rank
 * g owns rows [fence[g*d/world], fence[(g+1)*d/world]) and (first/last rank)
 * the ring rows below/above. Its host buffer `slab` holds exactly those rows
 * (full padded width / plane), starting at so2dr_slab_rows().lo.
 * Protocol: so2dr_slab_prepare -> exchange the returned peer blobs with the
 * neighbours (any transport, e.g. torch.distributed all_gather) ->
 * so2dr_slab_connect(lower_blob, upper_blob) -> so2dr_slab_run per run.
 * Inter-slab halos (r*S_TB rows each way per round) move GPU-to-GPU: each
 * rank pushes its edge band straight into the neighbour's receive buffer over
 * CUDA IPC peer memory (NVLink/NVSwitch), ordered by device-side flags
 * (stream memory operations), so no halo byte crosses PCIe twice. */
#define SO2DR_PEER_BLOB_BYTES 512
so2dr_status so2dr_slab_rows(const so2dr_run_config* cfg, int dim, int rank, int world,
                             int64_t* lo, int64_t* hi);
so2dr_status so2dr_slab_prepare(so2dr_ctx* ctx, const so2dr_stencil_desc* st,
                                const so2dr_run_config* cfg, so2dr_dtype dtype, int rank,
                                int world, uint8_t blob_out[SO2DR_PEER_BLOB_BYTES]);
/* NULL for a missing neighbour. A blob produced in the same process is
 * connected by raw pointer (two contexts sharing one process/GPU). */
so2dr_status so2dr_slab_connect(so2dr_ctx* ctx, const uint8_t* lower_blob,
                                const uint8_t* upper_blob);
/* The connected halo transports: out[0] = rank, out[1] = world, out[2] /
 * out[3] = lower / upper edge: 0 none, 1 same process (raw pointer), 2 CUDA
 * IPC on the same GPU, 3 CUDA IPC to a peer GPU with peer access confirmed,
 * 4 CUDA IPC to a GPU this process cannot see (peer access not checkable). */
so2dr_status so2dr_slab_info(const so2dr_ctx* ctx, int32_t out[4]);
so2dr_status so2dr_slab_run(so2dr_ctx* ctx, const so2dr_stencil_desc* st,
                            const so2dr_run_config* cfg, const so2dr_kernel_plan* kp,
                            so2dr_dtype dtype, void* slab, so2dr_ledger* ledger_out,
                            so2dr_timing* timing_out);

/* ---- secondary entry points --------------------------------------------- */
/* fused_kernel on a host FieldPair: buf0/buf1 each rows x cols (2D) cells of
 * dtype covering padded rows [base_row, base_row+rows). Rects are
 * {y0, y1, x0, x1}. stats_out = {scratch_load, scratch_store, updates,
 * redundant} exactly as kernels.cpp:117-143 accounts them for `tile`. */
so2dr_status so2dr_fused_kernel(so2dr_ctx* ctx, const so2dr_stencil_desc* st,
                                so2dr_dtype dtype, void* buf0, void* buf1, int base_row,
                                int rows, int cols, int read, int steps, int tile,
                                const int32_t region[4], const int32_t interior[4],
                                const int32_t owned[4], uint64_t stats_out[4]);
/* apply_step on host grids: one step over interior rows [row_lo, row_hi). */
so2dr_status so2dr_apply_step(so2dr_ctx* ctx, const so2dr_stencil_desc* st,
                              so2dr_dtype dtype, int sz, int r, const void* in, void* out,
                              int row_lo, int row_hi);
/* run_reference semantics (n single steps, ping-pong), executed on the device
 * with one full-interior step per launch. in and out may alias. */
so2dr_status so2dr_run_reference(so2dr_ctx* ctx, const so2dr_stencil_desc* st,
                                 so2dr_dtype dtype, int sz, int r, const void* in,
                                 void* out, int steps);
/* init_grid on the device (splitmix64, bit-identical to stencil.cpp:91-118;
 * 3D plane z uses seed ^ z*0x9E3779B97F4A7C15). `out` host or device. */
so2dr_status so2dr_init_grid(so2dr_ctx* ctx, so2dr_dtype dtype, int dim, int sz, int r,
                             uint64_t seed, void* out);
/* Same, for padded rows (2D) / planes (3D) [lo, hi) only. */
so2dr_status so2dr_init_rows(so2dr_ctx* ctx, so2dr_dtype dtype, int dim, int sz, int r,
                             uint64_t seed, int64_t lo, int64_t hi, void* out);

/* ---- host-only helpers (no device needed) -------------------------------- */
uint64_t so2dr_grid_checksum(const void* data, size_t bytes); /* FNV-1a 64 */
/* The reference's per-call kernel accounting (kernels.cpp:48-138) for a
 * field of storage rows [sy0, sy1) x cols: {scratch_load, scratch_store,
 * updates, redundant}. Closed form; what so2dr_fused_kernel/so2dr_run report. */
so2dr_status so2dr_kernel_stats(int radius, int steps, int tile, const int32_t region[4],
                                const int32_t interior[4], const int32_t owned[4], int sy0,
                                int sy1, int64_t cols, uint64_t stats_out[4]);
so2dr_status so2dr_arena_bytes(const so2dr_run_config* cfg, const so2dr_kernel_plan* kp,
                               uint64_t* out);
/* Largest step count one K1 launch fuses for (dim, dtype, kind, radius): the
 * engine splits a longer fused_kernel call (the reference's kernels.cpp:80-109
 * runs any s <= k_on in one tiled pass) into launches of at most this many
 * steps. 0 = shape unsupported. No GPU needed. */
int32_t so2dr_k1_max_steps(int dim, so2dr_dtype dtype, so2dr_kind kind, int radius);
/* Real device footprint of an so2dr run (2 buffers per stream + slots + pools). */
so2dr_status so2dr_device_bytes(const so2dr_run_config* cfg, int dim, so2dr_dtype dtype,
                                uint64_t* out);
/* plan_chunks: per chunk {core, working, transfer, shared_in, shared_out} as
 * [lo,hi) pairs -> 10 ints per chunk; fence has d+1 entries. */
so2dr_status so2dr_plan_chunks(const so2dr_run_config* cfg, int32_t* fence_out,
                               int32_t* chunks_out);
/* expected_ledger closed forms: {htod, dtoh, ondevice, kernel_invocations,
 * rounds, redundant_updates}, exact = redundancy_exact. dim/dtype extend the
 * byte counts to 3D planes / 8-byte cells. */
so2dr_status so2dr_expected_ledger(so2dr_mode mode, const so2dr_run_config* cfg,
                                   const so2dr_kernel_plan* kp, int dim, so2dr_dtype dtype,
                                   uint64_t out6[6], int32_t* exact);

/* ---- B200 run planner (host-only) ---------------------------
 * Replaces the reference's predict_bottleneck / feasible_configs model
 * (proj/src/planner.cpp:14-89: t_kernel = S_TB one-step sweeps, one buffer per
 * stream) with the engine's pipeline: k_on-fused K1 launches priced from a
 * measured profile (profiles/b200.json; NULL = the built-in copy), the duplex
 * PCIe rate, pipeline fill/drain and the real device footprint
 * (include/so2dr/b200.hpp). `star` = star taps, else box. */
typedef struct {
  int32_t d, s_tb, k_on, n_strm, feasible;
  int64_t launches;
  uint64_t device_bytes;
  double t_pcie_s, t_kernel_s, t_fill_s, t_total_s, gcell_per_s;
} so2dr_plan_entry;
/* Every (d | sz, S_TB | n, k_on <= min(S_TB, 8)) candidate at n_strm streams
 * (up to `capacity` written to entries, *count = total) and the fastest
 * feasible one in *best. */
so2dr_status so2dr_plan_b200(const char* profile_json, int dim, so2dr_dtype dtype, int star, int radius,
                             int sz, int n, uint64_t budget_bytes, int n_strm, so2dr_plan_entry* best,
                             so2dr_plan_entry* entries, int32_t capacity, int32_t* count);
/* The prediction for one configuration. */
so2dr_status so2dr_predict_b200(const char* profile_json, int dim, so2dr_dtype dtype, int star, int radius,
                                int sz, int n, uint64_t budget_bytes, int d, int s_tb, int k_on,
                                int n_strm, so2dr_plan_entry* out);

/* ---- spec files, presets and run outputs (host-only) ----------------------
 * RunSpecFile / parse_spec_json / parse_spec_file  proj/include/so2dr/specfile.hpp:14-28
 * presets (--preset NAME)                          proj/tools/so2dr_main.cpp:28-68
 * report_to_json / ledger_to_csv / diagnostics_to_csv  proj/include/so2dr/report.hpp:11-24
 * Errors follow the reference: a syntax error is SO2DR_ERR_IO with "line L,
 * column C" in so2dr_last_error(NULL); a missing/mistyped field names it
 * (SO2DR_ERR_IO); an unknown kind/mode/preset or bad radius is
 * SO2DR_ERR_INVALID_SPEC. */
#define SO2DR_SPEC_MAX_WEIGHTS 125 /* (2r+1)^dim: box2d4r 81, 3D r=2 125 */
typedef struct {
  /* stencil.weights points at weights_buf of THIS struct (re-point it after
   * copying the struct); canonical (dz, dy, dx) order, defaults filled in:
   * box fp32(1/(2r+1)^dim), star fp32(1/(2*dim*r+1)) on axis. */
  so2dr_stencil_desc stencil;
  double weights_buf[SO2DR_SPEC_MAX_WEIGHTS];
  so2dr_run_config config;
  so2dr_kernel_plan kernel;
  uint64_t seed;
  int32_t mode;  /* so2dr_mode */
  int32_t dtype; /* so2dr_dtype */
  char stencil_name[32];     /* box2d1r, star3d1r, gradient2d, ... */
  char hardware_path[512];   /* "" when absent */
  char grid_dump_path[512];  /* "" when absent */
} so2dr_spec;

so2dr_status so2dr_spec_parse(const char* text, const char* origin, so2dr_spec* out);
so2dr_status so2dr_spec_parse_file(const char* path, so2dr_spec* out);
int so2dr_preset_count(void);
const char* so2dr_preset_name(int i); /* NULL when out of range */
/* Copies the preset's JSON (NUL-terminated) into buf when it fits; *len_out =
 * its length without the NUL either way. */
so2dr_status so2dr_preset_json(const char* name, char* buf, size_t cap, size_t* len_out);

/* report.json v1 of a run, the reference's keys and order (report.cpp:21-64);
 * modeled times come from `hw` (NULL = the B200 profile) and the ledger;
 * `measured` (optional) adds the CUDA-event block unless deterministic. */
typedef struct {
  int32_t mode;          /* so2dr_mode */
  int32_t deterministic; /* omit wall_seconds / measured */
  const char* stencil_name;
  so2dr_run_config config;
  so2dr_kernel_plan kernel;
  uint64_t checksum;
  so2dr_ledger ledger;
  const so2dr_hardware* hw;
  const so2dr_timing* measured;
} so2dr_report_in;
so2dr_status so2dr_report_json(const so2dr_report_in* in, char* buf, size_t cap, size_t* len_out);
so2dr_status so2dr_ledger_csv(const so2dr_ledger* ledger, char* buf, size_t cap, size_t* len_out);
so2dr_status so2dr_diagnostics_csv(const so2dr_diag_row* rows, size_t n, char* buf, size_t cap,
                                   size_t* len_out);

#ifdef __cplusplus
}
#endif

#endif /* SO2DR_CUDA_H */
