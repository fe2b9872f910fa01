// b200_planner.cpp -- the B200 run planner (include/so2dr/b200.hpp).
// Replaces the reference's t_kernel / memory terms (proj/src/planner.cpp:21-22,
// 64-73) with the engine's real pipeline and footprint; the reference model
// itself stays available unchanged (host_model.cpp, so2dr/planner.hpp).
#include "so2dr/b200.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include "engine.h"
#include "json_lite.hpp"
#include "k1_launch.h"
#include "so2dr/errors.hpp"
#include "so2dr/layout.hpp"

namespace so2dr::b200 {

Profile default_profile() {
  // profiles/b200.json (measured on this pool; see that file for sources)
  Profile p;
  p.name = "b200";
  p.hbm_bytes = 183359ull << 20;
  p.hbm_bw = 6553.6e9;
  p.pcie_h2d = 54.71e9;
  p.pcie_d2h = 57.06e9;
  p.pcie_duplex_dir = 48.34e9;
  p.fma_rate = 36.88e12;
  p.launch_s = 4.0e-6;
  p.half_cells = 2.8e7;
  const double eff[9] = {0, 0.92, 0.86, 0.76, 0.66, 0.62, 0.58, 0.55, 0.52};
  std::copy(eff, eff + 9, p.eff_hbm);
  p.eff_fma = 0.47;
  p.eff_3d = 0.20;
  p.eff_f64 = 0.8;
  p.overlap = 0.06;
  return p;
}

Profile profile_from_json(const std::string& text, const std::string& origin) {
  so2dr_json::Value j;
  try {
    j = so2dr_json::parse(text);
  } catch (const so2dr_json::ParseError& e) {
    throw IoError("b200 profile " + origin + ": " + e.what());
  }
  Profile p = default_profile();
  try {
    auto num = [&](const char* k, double& out) {
      if (j.contains(k)) out = j.at(k).as_double();
    };
    if (j.contains("name")) p.name = j.at("name").as_string();
    if (j.contains("c_dmem_bytes")) p.hbm_bytes = j.at("c_dmem_bytes").as_uint64();
    num("bw_dmem_bytes_per_s", p.hbm_bw);
    num("pcie_h2d_bytes_per_s", p.pcie_h2d);
    num("pcie_d2h_bytes_per_s", p.pcie_d2h);
    num("bw_intc_bytes_per_s", p.pcie_duplex_dir);  // the reference key: per direction in duplex
    num("fma_per_s", p.fma_rate);
    num("k1_launch_s", p.launch_s);
    num("k1_half_cells", p.half_cells);
    num("k1_fma_eff", p.eff_fma);
    num("k1_3d_eff", p.eff_3d);
    num("k1_f64_eff", p.eff_f64);
    num("overlap_penalty", p.overlap);
    if (j.contains("k1_hbm_eff")) {
      const auto& a = j.at("k1_hbm_eff").elements();
      for (std::size_t k = 0; k < a.size() && k < 8; ++k) p.eff_hbm[k + 1] = a[k].as_double();
    }
  } catch (const std::exception& e) {
    throw IoError("b200 profile " + origin + ": " + e.what());
  }
  if (!(p.hbm_bw > 0 && p.pcie_duplex_dir > 0 && p.pcie_h2d > 0 && p.pcie_d2h > 0 && p.fma_rate > 0))
    throw IoError("b200 profile " + origin + ": rates must be positive");
  return p;
}

Profile load_profile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open b200 profile " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return profile_from_json(ss.str(), path);
}

namespace {

int taps(const Problem& pb) {
  const int e = 2 * pb.radius + 1;
  if (pb.star) return 2 * pb.dim * pb.radius + 1;
  return pb.dim == 2 ? e * e : e * e * e;
}

// One K1 launch over `rows` storage units (rows / planes) of `unit` cells
// advancing `k` steps: predicted seconds.
double launch_time(const Profile& pf, const Problem& pb, double rows, double unit, int k) {
  const double b = pb.elem_bytes;
  const double r = pb.radius;
  const double in_rows = rows + 2.0 * r * k;
  const double bytes = (in_rows + rows) * unit * b;                 // algorithmic HBM bytes
  const double fmas = rows * unit * k * taps(pb);                   // useful fmas
  double hbm_eff = pf.eff_hbm[std::clamp(k, 1, 8)];
  double fma_rate = pf.fma_rate * pf.eff_fma;
  if (pb.dim == 3) hbm_eff = pf.eff_3d, fma_rate = pf.fma_rate * pf.eff_3d;
  if (pb.elem_bytes == 8) hbm_eff *= pf.eff_f64, fma_rate *= 0.5 * pf.eff_f64;  // DFMA at half rate
  const double t_roof = std::max(bytes / (hbm_eff * pf.hbm_bw), fmas / fma_rate);
  const double cells = rows * unit;
  const double size_eff = cells / (cells + pf.half_cells);
  return t_roof / size_eff + pf.launch_s;
}

}  // namespace

Candidate predict(const Profile& pf, const Problem& pb, int d, int s_tb, int k_on, int n_strm) {
  Candidate c;
  c.d = d, c.s_tb = s_tb, c.k_on = k_on, c.n_strm = n_strm;
  const int r = pb.radius, sz = pb.sz;
  if (d < 1 || s_tb < 1 || k_on < 1 || sz < 1 || pb.n < 1 || sz % d != 0) {
    c.failed.push_back("valid (d, S_TB, k_on)");
    return c;
  }
  if (k_on > s_tb) c.failed.push_back("k_on <= S_TB");
  if (s_tb > pb.n) c.failed.push_back("S_TB <= n");
  if (2LL * r * s_tb > sz / d) c.failed.push_back("2 r S_TB <= sz/d (shared rows inside the chunk)");
  const int kmax = so2dr_dev::k1_max_steps(pb.dim, pb.elem_bytes == 8 ? 1 : 0,
                                           pb.star ? so2dr_dev::KSTAR : so2dr_dev::KBOX, r);
  if (kmax < 1) c.failed.push_back("stencil shape supported by K1");
  // real device footprint of the engine (2 buffers per stream + share slots)
  RunConfig cfg;
  cfg.sz = sz, cfg.r = r, cfg.d = d, cfg.s_tb = std::min(s_tb, pb.n), cfg.k_on = std::max(1, std::min(k_on, s_tb));
  cfg.n_strm = n_strm, cfg.n = pb.n;
  if (c.failed.empty()) {
    try {
      cfg.validate();
      const so2dr_eng::Geo g = so2dr_eng::make_geo(pb.dim, sz, r, pb.elem_bytes == 8 ? 1 : 0);
      c.device_bytes = so2dr_eng::device_footprint(cfg, g, n_strm);
      if (pb.budget && c.device_bytes > pb.budget) c.failed.push_back("device footprint <= budget");
    } catch (const std::exception& e) {
      c.failed.push_back(e.what());
    }
  }
  if (!c.failed.empty()) return c;

  const double p = sz + 2.0 * r;
  const double unit = pb.dim == 2 ? p : p * p;  // cells per storage unit
  const double b = pb.elem_bytes;
  const double chunk = static_cast<double>(sz) / d;
  const int k_eff = std::min(k_on, kmax);
  double t_kernel = 0, t_pcie = 0, t_first_kernels = 0;
  long long launches = 0;
  double round_max = 0;
  for (int done = 0; done < pb.n; done += s_tb) {
    const int steps = std::min(s_tb, pb.n - done);
    // one chunk's calls: the shared region shrinks by 2r per step (compute_area)
    double t_chunk = 0;
    int calls = 0;
    for (int s0 = 0; s0 < steps; s0 += k_eff) {
      const int k = std::min(k_eff, steps - s0);
      const double rows = chunk + 2.0 * r * (steps - s0 - k) + r * k;
      t_chunk += launch_time(pf, pb, rows, unit, k);
      ++calls;
    }
    const double t_kr = d * t_chunk;
    const double t_pr = std::max(p * unit * b, sz * unit * b) / pf.pcie_duplex_dir;
    t_kernel += t_kr;
    t_pcie += t_pr;
    // the two pipelines overlap imperfectly: the faster one still costs a
    // fraction of its time (fit to the d / k_on sweeps, profiles/b200.json)
    round_max += std::max(t_kr, t_pr) + pf.overlap * std::min(t_kr, t_pr);
    launches += static_cast<long long>(d) * calls;
    if (done == 0) t_first_kernels = t_chunk;
  }
  const double chunk_bytes = chunk * unit * b;
  c.t_fill = chunk_bytes / pf.pcie_h2d + t_first_kernels + chunk_bytes / pf.pcie_d2h;
  c.t_kernel = t_kernel;
  c.t_pcie = t_pcie;
  c.t_total = round_max + c.t_fill;
  c.launches = launches;
  c.gcells = std::pow(static_cast<double>(sz), pb.dim) * pb.n / c.t_total / 1e9;
  c.feasible = true;
  return c;
}

Plan plan(const Profile& pf, const Problem& pb) {
  if (pb.sz < 1 || pb.n < 1) throw InvalidSpecError("b200 planner: sz and n must be positive");
  Plan out;
  std::vector<int> stbs;
  for (int s = 1; s <= pb.n; ++s)
    if (pb.n % s == 0) stbs.push_back(s);
  for (int ns : pb.n_strm)
    for (int d = 1; d <= std::min(pb.sz, pb.max_d); ++d) {
      if (pb.sz % d) continue;
      for (int s : stbs) {
        if (2LL * pb.radius * s > pb.sz / d) continue;  // chunk too small for the shared rows
        for (int k = 1; k <= std::min(s, 8); ++k) out.candidates.push_back(predict(pf, pb, d, s, k, ns));
      }
    }
  const Candidate* best = nullptr;
  for (const auto& c : out.candidates) {
    if (!c.feasible) continue;
    if (!best || c.t_total < best->t_total * (1 - 1e-9) ||
        (std::abs(c.t_total - best->t_total) <= best->t_total * 1e-9 && c.launches < best->launches))
      best = &c;
  }
  if (!best) throw InvalidSpecError("b200 planner: no feasible configuration");
  out.best = *best;
  return out;
}

}  // namespace so2dr::b200
