// so2dr/b200.hpp -- the B200 run planner.
//
// The reference's planner (proj/src/planner.cpp:14-89, mirrored unchanged in
// so2dr/planner.hpp) prices a round as S_TB one-step sweeps of the chunk and
// one working buffer per stream. This one models the engine that actually
// runs here: the H2D -> K1 -> D2H pipeline of run_so2dr (csrc/engine.cpp)
// with k_on-fused K1 launches, priced from a measured B200 profile
// (profiles/b200.json):
//
//   per round   t_pcie   = max(grid H2D, core D2H) / duplex per-direction BW
//               t_kernel = sum over chunks and ceil(S_TB/k_on) calls of
//                          max(alg HBM bytes / (eff_hbm(k) * BW_hbm),
//                              fma / (eff_fma * FMA peak)) / size_eff + t_launch
//               size_eff = cells / (cells + half_cells)   (short launches pay
//                          segment warm-up and tails: measured)
//   run         t_total  = rounds * (max(t_pcie, t_kernel) + overlap * min(..))
//                          + first chunk H2D + its kernels + last chunk D2H
//   memory      the engine's real footprint (2 buffers per stream + share
//               slots), not the reference's one-buffer term
//
// plan() enumerates (d, S_TB, k_on) and returns every candidate with its
// prediction and the fastest feasible one.
#ifndef SO2DR_B200_B200_HPP
#define SO2DR_B200_B200_HPP

#include <cstdint>
#include <string>
#include <vector>

namespace so2dr::b200 {

struct Profile {
  std::string name = "b200";
  std::uint64_t hbm_bytes = 0;  // device memory
  double hbm_bw = 0;            // measured copy bandwidth (read + write bytes / s)
  double pcie_h2d = 0;          // pinned H2D alone, bytes / s
  double pcie_d2h = 0;          // pinned D2H alone
  double pcie_duplex_dir = 0;   // per direction while both directions stream
  double fma_rate = 0;          // measured fp32 FMA / s
  double launch_s = 0;          // fixed cost per K1 launch
  double half_cells = 0;        // launch size (cells) at which a launch reaches half its in-core rate
  double eff_hbm[9] = {};       // in-core K1 2D fp32 fraction of the HBM roof, by k_on (1..8)
  double eff_fma = 0;           // fraction of the FMA peak when the FMA pipe binds
  double eff_3d = 0;            // 3D K1: fraction of min(HBM, FMA) roof reached in-core
  double eff_f64 = 0;           // fp64: fraction of the fp32 rate model
  double overlap = 0;           // fraction of the shorter of (PCIe, K1) per round not hidden
};

Profile default_profile();                          // the measured numbers of profiles/b200.json
Profile profile_from_json(const std::string& text, const std::string& origin);
Profile load_profile(const std::string& path);

struct Problem {
  int dim = 2;
  int elem_bytes = 4;  // 4 fp32, 8 fp64
  bool star = false;   // star taps (4r+1 / 6r+1) instead of box ((2r+1)^dim)
  int radius = 1;
  int sz = 0;
  int n = 0;                     // timesteps
  std::uint64_t budget = 0;      // device bytes the run may use
  std::vector<int> n_strm = {3};  // stream counts to consider
  int max_d = 1024;
};

struct Candidate {
  int d = 0, s_tb = 0, k_on = 0, n_strm = 0;
  bool feasible = false;
  std::vector<std::string> failed;
  std::uint64_t device_bytes = 0;
  long long launches = 0;  // K1 launches in the run
  double t_pcie = 0, t_kernel = 0, t_fill = 0, t_total = 0;  // seconds (pcie/kernel: whole run)
  double gcells = 0;  // predicted end-to-end GCell-updates/s
};

struct Plan {
  Candidate best;
  std::vector<Candidate> candidates;
};

// Prediction for one configuration (feasibility included).
Candidate predict(const Profile& prof, const Problem& prob, int d, int s_tb, int k_on, int n_strm);
// Every (d | sz, S_TB | n or = n, k_on <= min(S_TB, 8)) candidate, best first feasible by t_total.
Plan plan(const Profile& prof, const Problem& prob);

}  // namespace so2dr::b200

#endif
