// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference library
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libso2dr_ref.so). TEST INFRASTRUCTURE ONLY: used to pin the C
// oracle and the golden fixtures, and as the CPU baseline / reference arm of
// bench.py. Nothing here is reference source; it only calls the reference's
// public API (proj/include/so2dr/*.hpp).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "so2dr/engine.hpp"
#include "so2dr/kernels.hpp"
#include "so2dr/stencil.hpp"
#include "so2dr/verify.hpp"

using namespace so2dr;

namespace {

StencilSpec make_spec(int kind, int radius, const float* w) {
  if (kind == 1) return StencilSpec::gradient();
  const int pts = (2 * radius + 1) * (2 * radius + 1);
  if (!w) return StencilSpec::box(radius);
  return StencilSpec::box(radius, std::vector<float>(w, w + pts));
}

int classify(const std::exception_ptr& ep, char* err, int errlen) {
  int code = 99;
  std::string msg;
  try {
    std::rethrow_exception(ep);
  } catch (const InfeasibleError& e) {
    code = 2, msg = e.what();
  } catch (const OutOfDeviceMemoryError& e) {
    code = 3, msg = e.what();
  } catch (const InvalidSpecError& e) {
    code = 1, msg = e.what();
  } catch (const ContractError& e) {
    code = 4, msg = e.what();
  } catch (const IoError& e) {
    code = 5, msg = e.what();
  } catch (const std::out_of_range& e) {
    code = 7, msg = e.what();
  } catch (const std::exception& e) {
    code = 99, msg = e.what();
  }
  if (err && errlen > 0) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

void ledger_out(const LedgerSnapshot& s, std::uint64_t* out) {
  const std::uint64_t v[9] = {s.htod,          s.dtoh,           s.ondevice,
                              s.scratch_load,  s.scratch_store,  s.element_updates,
                              s.redundant_updates, s.kernel_invocations, s.rounds};
  std::memcpy(out, v, sizeof(v));
}

}  // namespace

extern "C" {

void ref_init_grid(int sz, int r, std::uint64_t seed, float* out) {
  const Grid g = init_grid({sz, r}, seed);
  std::memcpy(out, g.values.data(), g.values.size() * sizeof(float));
}

std::uint64_t ref_checksum(int sz, int r, const float* data) {
  Grid g{{sz, r}, std::vector<float>(data, data + static_cast<std::size_t>(sz + 2 * r) * (sz + 2 * r))};
  return grid_checksum(g);
}

int ref_run_reference(int kind, int radius, const float* w, int sz, int r,
                      const float* in, int steps, float* out, char* err, int errlen) {
  try {
    const StencilSpec spec = make_spec(kind, radius, w);
    const std::size_t n = static_cast<std::size_t>(sz + 2 * r) * (sz + 2 * r);
    Grid g{{sz, r}, std::vector<float>(in, in + n)};
    const Grid res = run_reference(g, spec, steps);
    std::memcpy(out, res.values.data(), n * sizeof(float));
    return 0;
  } catch (...) {
    return classify(std::current_exception(), err, errlen);
  }
}

// cfg: sz r d s_tb k_on n_strm n n_a ; kp: k_on tile ; hw: c_dmem bw_dmem bw_intc
int ref_run_engine(int mode, int kind, int radius, const float* w, const int* cfg,
                   const int* kp, std::uint64_t scratch_budget, std::uint64_t c_dmem,
                   double bw_dmem, double bw_intc, int corrupt_share, int boundary,
                   const float* in, float* out, std::uint64_t* ledger,
                   std::uint64_t* arena_peak, double* wall, char* err, int errlen) {
  try {
    const StencilSpec spec = make_spec(kind, radius, w);
    RunConfig c;
    c.sz = cfg[0], c.r = cfg[1], c.d = cfg[2], c.s_tb = cfg[3], c.k_on = cfg[4];
    c.n_strm = cfg[5], c.n = cfg[6], c.n_a = cfg[7];
    KernelPlan k;
    k.k_on = kp[0], k.tile = kp[1], k.scratch_budget = scratch_budget;
    HardwareModel hw = default_hardware();
    hw.c_dmem = c_dmem, hw.bw_dmem = bw_dmem, hw.bw_intc = bw_intc;
    EngineHooks hooks;
    hooks.corrupt_share = corrupt_share != 0;
    hooks.boundary = boundary;
    const std::size_t n = static_cast<std::size_t>(c.sz + 2 * c.r) * (c.sz + 2 * c.r);
    Grid g{{c.sz, c.r}, std::vector<float>(in, in + n)};
    const RunResult res =
        run_engine(static_cast<EngineMode>(mode), g, spec, c, k, hw, hooks);
    std::memcpy(out, res.grid.values.data(), n * sizeof(float));
    if (ledger) ledger_out(res.report.ledger, ledger);
    if (arena_peak) *arena_peak = res.report.arena_peak;
    if (wall) *wall = res.report.wall_seconds;
    return 0;
  } catch (...) {
    return classify(std::current_exception(), err, errlen);
  }
}

// Runs the reference fused_kernel on a caller-owned field (two buffers of
// rows*cols floats starting at padded row base_row). rects: y0 y1 x0 x1.
int ref_fused_kernel(int kind, int radius, const float* w, float* buf0, float* buf1,
                     int base_row, int rows, int cols, int read, int steps, int tile,
                     const int* region, const int* interior, const int* owned,
                     std::uint64_t* stats, std::uint64_t* ledger, char* err, int errlen) {
  try {
    const StencilSpec spec = make_spec(kind, radius, w);
    FieldPair f;
    const std::size_t n = static_cast<std::size_t>(rows) * cols;
    f.base_row = base_row, f.rows = rows, f.cols = cols;
    f.buf[0].assign(buf0, buf0 + n);
    f.buf[1].assign(buf1, buf1 + n);
    TransferLedger led;
    const KernelStats ks = fused_kernel(
        f, read, spec, steps, tile, Rect{region[0], region[1], region[2], region[3]},
        Rect{interior[0], interior[1], interior[2], interior[3]},
        Rect{owned[0], owned[1], owned[2], owned[3]}, led);
    std::memcpy(buf0, f.buf[0].data(), n * sizeof(float));
    std::memcpy(buf1, f.buf[1].data(), n * sizeof(float));
    stats[0] = ks.scratch_load, stats[1] = ks.scratch_store;
    stats[2] = ks.updates, stats[3] = ks.redundant;
    if (ledger) ledger_out(led.snapshot(), ledger);
    return 0;
  } catch (...) {
    return classify(std::current_exception(), err, errlen);
  }
}

// expected_ledger closed forms (proj/src/verify.cpp:7-59)
int ref_expected_ledger(int mode, const int* cfg, const int* kp, std::uint64_t* out6,
                        int* exact) {
  try {
    RunConfig c;
    c.sz = cfg[0], c.r = cfg[1], c.d = cfg[2], c.s_tb = cfg[3], c.k_on = cfg[4];
    c.n_strm = cfg[5], c.n = cfg[6], c.n_a = cfg[7];
    KernelPlan k;
    k.k_on = kp[0], k.tile = kp[1];
    const ExpectedLedger e = expected_ledger(static_cast<EngineMode>(mode), c, k);
    out6[0] = e.htod, out6[1] = e.dtoh, out6[2] = e.ondevice;
    out6[3] = e.kernel_invocations, out6[4] = e.rounds, out6[5] = e.redundant_updates;
    *exact = e.redundancy_exact;
    return 0;
  } catch (...) {
    return classify(std::current_exception(), nullptr, 0);
  }
}

std::uint64_t ref_arena_bytes(const int* cfg, const int* kp) {
  RunConfig c;
  c.sz = cfg[0], c.r = cfg[1], c.d = cfg[2], c.s_tb = cfg[3], c.k_on = cfg[4];
  c.n_strm = cfg[5], c.n = cfg[6], c.n_a = cfg[7];
  KernelPlan k;
  k.k_on = kp[0], k.tile = kp[1];
  return so2dr_arena_bytes(c, k);
}

}  // extern "C"
