// so2dr/layout.hpp -- chunk geometry (host-side planning).
// API mirror of proj/include/so2dr/layout.hpp:13-95: HardwareModel, RunConfig,
// plan_chunks, compute_area, RoundPlan. Pure host integer arithmetic that
// feeds the device scheduler's launch parameters.
#ifndef SO2DR_B200_LAYOUT_HPP
#define SO2DR_B200_LAYOUT_HPP

#include <cstdint>
#include <string>
#include <vector>

#include "so2dr/stencil.hpp"

namespace so2dr {

struct HardwareModel {
  std::string name = "unnamed";
  std::uint64_t c_dmem = 0;  // MODELED arena capacity (reference semantics), bytes
  double bw_dmem = 0.0;      // bytes/s
  double bw_intc = 0.0;      // bytes/s
  int b_elem = 4;

  void validate() const;
};

HardwareModel default_hardware();  // rtx3080 profile (proj/profiles/rtx3080.json)
HardwareModel desk_hardware();     // desk profile (proj/profiles/desk.json)
HardwareModel b200_hardware();     // B200 profile (profiles/b200.json; measured numbers)

struct RunConfig {
  int sz = 0;
  int r = 1;
  int d = 1;
  int s_tb = 1;
  int k_on = 1;
  int n_strm = 3;
  int n = 0;
  int n_a = 2;

  void validate() const;
  std::uint64_t padded() const { return static_cast<std::uint64_t>(sz) + 2ull * r; }
  std::uint64_t d_chk() const { return static_cast<std::uint64_t>(sz) * padded() / d; }
  std::uint64_t w_halo() const { return 2ull * r * padded(); }
};

struct ChunkIntervals {
  RowInterval core;
  RowInterval working;
  RowInterval transfer;
  RowInterval shared_in;
  RowInterval shared_out;
};

struct ChunkLayout {
  int sz = 0, r = 0, d = 0, s_tb = 0;
  std::vector<int> fence;
  std::vector<ChunkIntervals> chunks;

  int padded() const { return sz + 2 * r; }
};

ChunkLayout plan_chunks(const RunConfig& config);
RowInterval compute_area(const ChunkLayout& layout, int chunk, int t, int round_steps);
RowInterval compute_area(const ChunkLayout& layout, int chunk, int t);

struct RoundPlan {
  int n = 0, s_tb = 1, k_on = 1;
  int rounds = 0;

  int steps_in_round(int round) const;
  int calls_in_round(int round) const;
  int steps_in_call(int round, int call) const;
};

RoundPlan make_round_plan(const RunConfig& config);

}  // namespace so2dr

#endif
