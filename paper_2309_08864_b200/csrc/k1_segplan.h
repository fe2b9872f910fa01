// k1_segplan.h -- row / plane segmentation of a persistent K1 launch (host
// side, shared by the 2D and 3D launchers; DESIGN.md 4 "guided items").
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#if defined(__CUDACC__)
#define SO2DR_HD __host__ __device__ __forceinline__
#else
#define SO2DR_HD inline
#endif

namespace so2dr_dev {

struct K1SegPlan {
  int seg_e, nseg_e, seg_b, nseg_b, seg_s, nseg_s;
};

// Items of a launch: `edge` units (ring-column strips) x nseg_e uniform
// segments, then the inner units' nseg_b big and nseg_s small segments.
SO2DR_HD int k1_seg_items(const K1SegPlan& p, int units, int edge) {
  return edge * p.nseg_e + (units - edge) * (p.nseg_b + p.nseg_s);
}

// Item -> (unit wx, output rows [oy0, oy1)) in hand-out order: edge units
// first (nl leading, nr trailing), then the inner units' big segments, then
// their small segments (segment-major, so consecutive items share rows).
SO2DR_HD void k1_seg_decode(const K1SegPlan& p, int item, int units, int nl, int nr, int y0, int y1, int& wx,
                            int& oy0, int& oy1) {
  const int ne = nl + nr;
  if (item < ne * p.nseg_e) {
    const int sg = item / ne;
    const int j = item - sg * ne;
    wx = j < nl ? j : units - ne + j;
    oy0 = y0 + sg * p.seg_e;
    oy1 = oy0 + p.seg_e < y1 ? oy0 + p.seg_e : y1;
    return;
  }
  const int inner = units - ne;
  int i = item - ne * p.nseg_e;
  if (i < inner * p.nseg_b) {
    const int sg = i / inner;
    wx = nl + (i - sg * inner);
    oy0 = y0 + sg * p.seg_b;
    oy1 = oy0 + p.seg_b < y1 ? oy0 + p.seg_b : y1;
    return;
  }
  i -= inner * p.nseg_b;
  const int sg = i / inner;
  wx = nl + (i - sg * inner);
  oy0 = y0 + p.nseg_b * p.seg_b + sg * p.seg_s;
  oy1 = oy0 + p.seg_s < y1 ? oy0 + p.seg_s : y1;
}

// Greedy list-scheduling makespan of the launch's item sequence: `workers`
// identical workers (resident warps or CTAs) each take the next item when
// free. Free times are kept as (time, count) groups, so a batch of equal
// items costs O(groups x rounds), not O(items).
struct K1MakespanSim {
  std::map<double, int64_t> free_at;
  explicit K1MakespanSim(int64_t workers) { free_at[0.0] = workers; }
  void take(int64_t n, double cost) {
    while (n > 0) {
      auto it = free_at.begin();
      const double t = it->first;
      const int64_t k = std::min<int64_t>(n, it->second);
      if ((it->second -= k) == 0) free_at.erase(it);
      free_at[t + cost] += k;
      n -= k;
    }
  }
  double makespan() const { return free_at.rbegin()->first; }
};

// Row segmentation of one launch ("guided items"). A persistent
// launch of ~4 equal items per worker ends with a tail of up to one item in
// which most SMs idle (r02 ncu: SM active 75% of an in-bench K1 launch).
// Segments stay <= max_seg (the uniform plan's length): the workers are warps
// that share their SM's pipes, and fewer, longer items unbalance the SMs
// (measured: 1.4 items per warp lost 35% in-core at k_on = 4).
// The plan hands out the ring-column units first (uniform short segments:
// they cost `edge_factor` x per row), then the inner units' big segments,
// then the rest of their rows in small segments that even out the finish
// times. It minimises the modelled makespan: an item of L output rows costs
// L + `ov` rows (the warm-up rows and pipeline fill it recomputes).
inline K1SegPlan k1_plan_segments(int height, int units, int edge_units, int64_t workers, int ov, double edge_factor,
                                  int min_seg, int max_seg) {
  struct Key {
    int h, u, e, ov, ms, mx;
    int64_t w;
    bool operator<(const Key& o) const {
      return std::tie(h, u, e, ov, ms, mx, w) < std::tie(o.h, o.u, o.e, o.ov, o.ms, o.mx, o.w);
    }
  };
  static std::mutex mu;
  static std::map<Key, K1SegPlan> cache;
  const Key key{height, units, edge_units, ov, min_seg, max_seg, workers};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const int inner = units - edge_units;
  if (height <= 0) return K1SegPlan{1, 0, 1, 0, 1, 0};
  max_seg = std::max(1, std::min(max_seg, height));
  min_seg = std::max(1, std::min(min_seg, max_seg));
  K1SegPlan best{height, 1, height, 1, height, 0};
  double best_t = 1e300;
  auto eval = [&](int seg_s, int seg_b, int nb) {
    const int rest = height - nb * seg_b;
    if (rest < 0) return;
    K1SegPlan p;
    p.seg_b = seg_b;
    p.nseg_b = nb;
    p.seg_s = seg_s;
    p.nseg_s = (rest + seg_s - 1) / seg_s;
    p.seg_e = seg_s;
    p.nseg_e = (height + seg_s - 1) / seg_s;
    K1MakespanSim sim(workers);
    // edge items: the last segment may be short; cost ~ rows
    if (edge_units > 0) sim.take(int64_t(edge_units) * p.nseg_e, edge_factor * (double(height) / p.nseg_e + ov));
    if (inner > 0) {
      if (nb > 0) sim.take(int64_t(inner) * nb, seg_b + ov);
      if (p.nseg_s > 0) sim.take(int64_t(inner) * p.nseg_s, double(rest) / p.nseg_s + ov);
    }
    const double t = sim.makespan();
    if (t < best_t * (1.0 - 1e-9)) best_t = t, best = p;
  };
  eval(max_seg, max_seg, 0);  // the uniform plan itself: the guided one is never modelled slower
  for (double fs = min_seg; fs <= max_seg * 1.0001; fs *= 1.25) {
    const int seg_s = std::min(max_seg, (int)fs);
    for (int m = 1; m <= 8; ++m) {
      const int seg_b = seg_s * m;
      if (seg_b > max_seg) break;
      const int nb_max = height / seg_b;
      if (m == 1) {
        eval(seg_s, seg_b, 0);
        continue;
      }
      // the small segments only fill the tail: a few big-item rounds of rows
      for (int nb = std::max(1, nb_max - 16); nb <= nb_max; ++nb) eval(seg_s, seg_b, nb);
    }
  }
  {
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 4096) cache.clear();
    cache[key] = best;
  }
  return best;
}

}  // namespace so2dr_dev
