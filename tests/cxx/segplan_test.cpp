// Host check of the K1 launch segmentation (csrc/k1_segplan.h), built and run
// by tests/test_host.py::test_k1_segment_plan (g++, no GPU): for many launch
// shapes, the guided plan's items (decoded exactly as the kernels decode them)
// cover every (unit, output row) exactly once, hand out the ring-column units
// first and the small segments last, keep every segment within the cap, and
// never model a longer launch than the uniform segmentation.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "k1_segplan.h"

using namespace so2dr_dev;

static double model(const K1SegPlan& p, int h, int units, int edge, int64_t workers, int ov, double fe) {
  K1MakespanSim sim(workers);
  if (edge > 0 && p.nseg_e > 0) sim.take(int64_t(edge) * p.nseg_e, fe * (double(h) / p.nseg_e + ov));
  const int rest = h - p.nseg_b * p.seg_b;
  if (units > edge) {
    if (p.nseg_b) sim.take(int64_t(units - edge) * p.nseg_b, p.seg_b + ov);
    if (p.nseg_s) sim.take(int64_t(units - edge) * p.nseg_s, double(rest) / p.nseg_s + ov);
  }
  return sim.makespan();
}

int main() {
  int fails = 0, cases = 0;
  const int heights[] = {1, 7, 64, 131, 1568, 1600, 5760, 32768};
  const int unit_counts[] = {1, 3, 64, 192, 768};
  const int workers_list[] = {148, 444, 1776};
  for (int h : heights)
    for (int units : unit_counts)
      for (int nl = 0; nl <= 2 && nl <= units; ++nl)
        for (int nr = 0; nr <= 1 && nl + nr <= units; ++nr)
          for (int w : workers_list) {
            const int edge = nl + nr, ov = 18, y0 = 5;
            const int cap = std::max(1, (h + 7) / 8);
            const K1SegPlan p = k1_plan_segments(h, units, edge, w, ov, 4.5, 36, cap);
            ++cases;
            const int items = k1_seg_items(p, units, edge);
            std::vector<int> hits(size_t(units) * h, 0);
            bool order_ok = true, cap_ok = true;
            int last_kind = 0;  // 0 edge, 1 big, 2 small: nondecreasing in hand-out order
            for (int it = 0; it < items; ++it) {
              int wx, a, b;
              k1_seg_decode(p, it, units, nl, nr, y0, y0 + h, wx, a, b);
              const bool is_edge = wx < nl || wx >= units - nr;
              const int kind = it < edge * p.nseg_e ? 0 : it < edge * p.nseg_e + (units - edge) * p.nseg_b ? 1 : 2;
              if (is_edge != (kind == 0) || kind < last_kind) order_ok = false;
              last_kind = kind;
              if (b - a > cap) cap_ok = false;
              for (int y = a; y < b; ++y)
                if (y >= y0 && y < y0 + h && wx >= 0 && wx < units) ++hits[size_t(wx) * h + (y - y0)];
                else order_ok = false;
            }
            bool cover_ok = true;
            for (int v : hits)
              if (v != 1) cover_ok = false;
            const int nu = (h + cap - 1) / cap;
            const K1SegPlan u{cap, nu, cap, nu, cap, 0};
            const bool model_ok = model(p, h, units, edge, w, ov, 4.5) <= model(u, h, units, edge, w, ov, 4.5) + 1e-6;
            if (!(cover_ok && order_ok && cap_ok && model_ok)) {
              ++fails;
              std::printf("FAIL h=%d units=%d nl=%d nr=%d w=%d cover=%d order=%d cap=%d model=%d plan e%dx%d b%dx%d s%dx%d\n",
                          h, units, nl, nr, w, cover_ok, order_ok, cap_ok, model_ok, p.seg_e, p.nseg_e, p.seg_b,
                          p.nseg_b, p.seg_s, p.nseg_s);
            }
          }
  std::printf("%d cases, %d failures\n", cases, fails);
  return fails ? 1 : 0;
}
