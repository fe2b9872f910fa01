// host_model.cpp -- host-side model of the SO2DR run: stencil specs, chunk
// geometry, modeled arena, ledger, share-slot protocol, analytic planner and
// grid dumps. Integer/host bookkeeping only; all stencil arithmetic runs on
// the device (engine.cu). Semantics follow the reference file:line cited per
// function so the C++ mirror API behaves identically.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>

#include "so2dr/engine.hpp"
#include "so2dr/gridio.hpp"
#include "json_lite.hpp"
#include "so2dr/planner.hpp"
#include "so2dr/verify.hpp"

namespace so2dr {

// ---------------------------------------------------------------- stencil --
// proj/src/stencil.cpp:8-88

std::string to_string(StencilKind kind) {
  switch (kind) {
    case StencilKind::box: return "box";
    case StencilKind::gradient: return "gradient";
    case StencilKind::star: return "star";
  }
  return "?";
}

StencilKind stencil_kind_from_string(const std::string& s) {
  if (s == "box") return StencilKind::box;
  if (s == "gradient") return StencilKind::gradient;
  if (s == "star") return StencilKind::star;
  throw InvalidSpecError("unknown stencil kind \"" + s + "\"");
}

static int box_points(int radius) { return (2 * radius + 1) * (2 * radius + 1); }

StencilSpec StencilSpec::box(int radius) {
  if (radius < 1 || radius > 4)
    throw InvalidSpecError("box radius must be in 1..4, got " + std::to_string(radius));
  const int pts = box_points(radius);
  return box(radius, std::vector<float>(pts, 1.0f / static_cast<float>(pts)));
}

StencilSpec StencilSpec::box(int radius, const std::vector<float>& weights) {
  const int pts = box_points(radius);
  if (static_cast<int>(weights.size()) != pts)
    throw InvalidSpecError("box radius " + std::to_string(radius) + " needs " +
                           std::to_string(pts) + " weights, got " +
                           std::to_string(weights.size()));
  StencilSpec s;
  s.kind = StencilKind::box;
  s.radius = radius;
  s.taps.reserve(pts);
  std::size_t next = 0;
  for (int dy = -radius; dy <= radius; ++dy)
    for (int dx = -radius; dx <= radius; ++dx) s.taps.push_back({dy, dx, weights[next++]});
  s.flops_per_element = 2 * pts - 1;
  s.validate();
  return s;
}

StencilSpec StencilSpec::gradient() {
  StencilSpec s;
  s.kind = StencilKind::gradient;
  s.radius = 1;
  s.taps = {{-1, 0, 0.25f}, {0, -1, 0.25f}, {0, 0, 0.0f}, {0, 1, 0.25f}, {1, 0, 0.25f}};
  s.flops_per_element = 19;
  s.validate();
  return s;
}

StencilSpec StencilSpec::star(int radius) {
  if (radius < 1 || radius > 4)
    throw InvalidSpecError("star radius must be in 1..4, got " + std::to_string(radius));
  const int pts = 4 * radius + 1;
  return star(radius, std::vector<float>(pts, 1.0f / static_cast<float>(pts)));
}

StencilSpec StencilSpec::star(int radius, const std::vector<float>& weights) {
  const int pts = 4 * radius + 1;
  if (static_cast<int>(weights.size()) != pts)
    throw InvalidSpecError("star radius " + std::to_string(radius) + " needs " +
                           std::to_string(pts) + " weights, got " +
                           std::to_string(weights.size()));
  StencilSpec s;
  s.kind = StencilKind::star;
  s.radius = radius;
  std::size_t next = 0;
  for (int dy = -radius; dy <= radius; ++dy) {
    if (dy != 0) {
      s.taps.push_back({dy, 0, weights[next++]});
    } else {
      for (int dx = -radius; dx <= radius; ++dx) s.taps.push_back({0, dx, weights[next++]});
    }
  }
  s.flops_per_element = 2 * pts - 1;
  s.validate();
  return s;
}

std::string StencilSpec::name() const {
  if (kind == StencilKind::gradient) return "gradient2d";
  return (kind == StencilKind::star ? "star2d" : "box2d") + std::to_string(radius) + "r";
}

void StencilSpec::validate() const {
  if (radius < 1) throw InvalidSpecError("stencil radius must be positive");
  switch (kind) {
    case StencilKind::box:
      if (radius > 4) throw InvalidSpecError("box radius must be in 1..4");
      if (static_cast<int>(taps.size()) != box_points(radius))
        throw InvalidSpecError("box stencil must have (2r+1)^2 taps");
      break;
    case StencilKind::star:
      if (radius > 4) throw InvalidSpecError("star radius must be in 1..4");
      if (static_cast<int>(taps.size()) != 4 * radius + 1)
        throw InvalidSpecError("star stencil must have 4r+1 taps");
      for (const Tap& t : taps)
        if (t.dy != 0 && t.dx != 0) throw InvalidSpecError("star tap off the axes");
      break;
    case StencilKind::gradient:
      if (radius != 1) throw InvalidSpecError("gradient stencil has radius 1");
      if (taps.size() != 5) throw InvalidSpecError("gradient stencil has 5 taps");
      break;
  }
  for (std::size_t i = 0; i < taps.size(); ++i) {
    const Tap& t = taps[i];
    if (std::abs(t.dy) > radius || std::abs(t.dx) > radius)
      throw InvalidSpecError("tap offset exceeds stencil radius");
    if (!std::isfinite(t.w)) throw InvalidSpecError("tap weight not finite");
    if (i > 0) {
      const Tap& p = taps[i - 1];
      if (t.dy < p.dy || (t.dy == p.dy && t.dx <= p.dx))
        throw InvalidSpecError("taps not in canonical (dy, dx) ascending order");
    }
  }
}

// splitmix64, proj/src/stencil.cpp:91-106 (the device generator in
// engine.cu computes the same function).
static std::uint64_t splitmix(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

float cell_value(std::uint64_t seed, int y, int x) {
  const std::uint64_t key = (static_cast<std::uint64_t>(static_cast<std::uint32_t>(y)) << 32) |
                            static_cast<std::uint32_t>(x);
  return static_cast<float>(splitmix(seed ^ splitmix(key)) >> 40) * 0x1p-24f;
}

std::uint64_t grid_checksum(const Grid& grid) {
  // FNV-1a over the raw bytes (proj/src/stencil.cpp:176-186); serial by
  // definition, computed host-side after the last D2H.
  std::uint64_t h = 0xCBF29CE484222325ULL;
  const auto* p = reinterpret_cast<const unsigned char*>(grid.values.data());
  const std::size_t n = grid.values.size() * sizeof(float);
  for (std::size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001B3ULL;
  return h;
}

// ----------------------------------------------------------------- layout --
// proj/src/layout.cpp:6-128

void HardwareModel::validate() const {
  if (c_dmem == 0) throw InvalidSpecError("hardware: c_dmem must be positive");
  if (!(bw_dmem > 0.0) || !(bw_intc > 0.0))
    throw InvalidSpecError("hardware: bandwidths must be positive");
  if (b_elem <= 0) throw InvalidSpecError("hardware: b_elem must be positive");
}

HardwareModel default_hardware() {
  HardwareModel hw;
  hw.name = "rtx3080-desktop";
  hw.c_dmem = 10737418240ull;
  hw.bw_dmem = 760.0e9;
  hw.bw_intc = 15.75e9;
  hw.b_elem = 4;
  return hw;
}

HardwareModel desk_hardware() {
  HardwareModel hw;
  hw.name = "desk-sim";
  hw.c_dmem = 2147483648ull;
  hw.bw_dmem = 40.0e9;
  hw.bw_intc = 16.0e9;
  hw.b_elem = 4;
  return hw;
}

HardwareModel b200_hardware() {
  // measured on this pool: HBM copy 6448.4 GB/s (MEASURED_PEAKS.json),
  // pinned H2D 55.6 GB/s, D2H 57.3 GB/s, duplex 100 GB/s (profiles/b200.json).
  HardwareModel hw;
  hw.name = "b200";
  hw.c_dmem = 183359ull << 20;
  hw.bw_dmem = 6448.4e9;
  hw.bw_intc = 50.0e9;  // per direction while both directions stream
  hw.b_elem = 4;
  return hw;
}

void RunConfig::validate() const {
  if (sz <= 0) throw InvalidSpecError("config: sz must be positive");
  if (r < 1) throw InvalidSpecError("config: r must be positive");
  if (d < 1) throw InvalidSpecError("config: d must be at least 1");
  if (sz % d != 0)
    throw InvalidSpecError("config: sz (" + std::to_string(sz) + ") must be divisible by d (" +
                           std::to_string(d) + ")");
  if (s_tb < 1) throw InvalidSpecError("config: s_tb must be at least 1");
  if (k_on < 1 || k_on > s_tb)
    throw InvalidSpecError("config: k_on must satisfy 1 <= k_on <= s_tb");
  if (n_strm < 1) throw InvalidSpecError("config: n_strm must be at least 1");
  if (n < 0) throw InvalidSpecError("config: n must be non-negative");
  if (n_a < 1) throw InvalidSpecError("config: n_a must be at least 1");
}

ChunkLayout plan_chunks(const RunConfig& config) {
  config.validate();
  const int h = config.r * config.s_tb;  // shared half-height r*S_TB
  const int step = config.sz / config.d;
  if (2 * h > step)
    throw InfeasibleError("W_halo*S_TB <= D_chk",
                          "shared regions would overlap: 2*r*S_TB = " + std::to_string(2 * h) +
                              " > sz/d = " + std::to_string(step));
  ChunkLayout L;
  L.sz = config.sz;
  L.r = config.r;
  L.d = config.d;
  L.s_tb = config.s_tb;
  const int top = config.sz + 2 * config.r;
  for (int i = 0; i <= config.d; ++i) L.fence.push_back(config.r + i * step);
  L.chunks.resize(config.d);
  for (int i = 0; i < config.d; ++i) {
    const int a = L.fence[i], b = L.fence[i + 1];
    const bool first = i == 0, last = i == config.d - 1;
    ChunkIntervals& c = L.chunks[i];
    c.core = {a, b};
    c.working = {first ? 0 : a - h, last ? top : b + h};
    c.transfer = {first ? 0 : a + h, last ? top : b + h};
    c.shared_in = first ? RowInterval{a, a} : RowInterval{a - h, a + h};
    c.shared_out = last ? RowInterval{b, b} : RowInterval{b - h, b + h};
  }
  return L;
}

RowInterval compute_area(const ChunkLayout& layout, int chunk, int t, int round_steps) {
  if (chunk < 0 || chunk >= layout.d)
    throw std::out_of_range("compute_area: chunk index out of range");
  if (round_steps < 1 || round_steps > layout.s_tb)
    throw std::out_of_range("compute_area: round_steps out of range");
  if (t < 1 || t > round_steps)
    throw std::out_of_range("compute_area: step " + std::to_string(t) + " outside 1.." +
                            std::to_string(round_steps));
  const int grow = layout.r * (round_steps - t);
  RowInterval a{layout.fence[chunk] - grow, layout.fence[chunk + 1] + grow};
  if (chunk == 0) a.lo = layout.r;
  if (chunk == layout.d - 1) a.hi = layout.r + layout.sz;
  return a;
}

RowInterval compute_area(const ChunkLayout& layout, int chunk, int t) {
  return compute_area(layout, chunk, t, layout.s_tb);
}

int RoundPlan::steps_in_round(int round) const {
  if (round < 0 || round >= rounds) throw std::out_of_range("round index out of range");
  const int rem = n % s_tb;
  return (round == rounds - 1 && rem != 0) ? rem : s_tb;
}

int RoundPlan::calls_in_round(int round) const {
  const int k = steps_in_round(round);
  return (k + k_on - 1) / k_on;
}

int RoundPlan::steps_in_call(int round, int call) const {
  const int k = steps_in_round(round);
  const int calls = (k + k_on - 1) / k_on;
  if (call < 0 || call >= calls) throw std::out_of_range("kernel-call index out of range");
  const int rem = k % k_on;
  return (call == calls - 1 && rem != 0) ? rem : k_on;
}

RoundPlan make_round_plan(const RunConfig& config) {
  config.validate();
  RoundPlan p;
  p.n = config.n;
  p.s_tb = config.s_tb;
  p.k_on = config.k_on;
  p.rounds = (config.n + config.s_tb - 1) / config.s_tb;
  return p;
}

// ----------------------------------------------------------------- memsim --
// proj/src/memsim.cpp:8-221

void DeviceArena::alloc(const std::string& id, std::uint64_t bytes) {
  std::lock_guard<std::mutex> g(mu_);
  if (live_.count(id)) throw ContractError("arena: allocation id \"" + id + "\" already live");
  if (used_ + bytes > cap_) throw OutOfDeviceMemoryError(id, bytes, used_, cap_);
  live_[id] = bytes;
  used_ += bytes;
  peak_ = std::max(peak_, used_);
}

void DeviceArena::free(const std::string& id) {
  std::lock_guard<std::mutex> g(mu_);
  const auto it = live_.find(id);
  if (it == live_.end()) throw ContractError("arena: freeing unknown allocation \"" + id + "\"");
  used_ -= it->second;
  live_.erase(it);
}

std::uint64_t DeviceArena::used() const {
  std::lock_guard<std::mutex> g(mu_);
  return used_;
}

std::uint64_t DeviceArena::peak() const {
  std::lock_guard<std::mutex> g(mu_);
  return peak_;
}

std::string to_string(Counter c) {
  static const char* names[] = {"htod_bytes",       "dtoh_bytes",          "ondevice_bytes",
                                "scratch_load_bytes", "scratch_store_bytes", "element_updates",
                                "redundant_updates", "kernel_invocations",  "rounds"};
  const int i = static_cast<int>(c);
  return (i >= 0 && i < 9) ? names[i] : "?";
}

void TransferLedger::record(Counter counter, std::int64_t amount) {
  if (amount < 0) throw ContractError("ledger: negative amount for " + to_string(counter));
  c_[static_cast<int>(counter)].fetch_add(static_cast<std::uint64_t>(amount),
                                          std::memory_order_relaxed);
}

LedgerSnapshot TransferLedger::snapshot() const {
  auto v = [&](Counter c) { return c_[static_cast<int>(c)].load(std::memory_order_relaxed); };
  LedgerSnapshot s;
  s.htod = v(Counter::htod);
  s.dtoh = v(Counter::dtoh);
  s.ondevice = v(Counter::ondevice);
  s.scratch_load = v(Counter::scratch_load);
  s.scratch_store = v(Counter::scratch_store);
  s.element_updates = v(Counter::element_updates);
  s.redundant_updates = v(Counter::redundant_updates);
  s.kernel_invocations = v(Counter::kernel_invocations);
  s.rounds = v(Counter::rounds);
  return s;
}

void TransferLedger::audit() const {
  const LedgerSnapshot s = snapshot();
  if (s.redundant_updates > s.element_updates)
    throw ContractError("ledger audit: redundant_updates (" + std::to_string(s.redundant_updates) +
                        ") exceeds element_updates (" + std::to_string(s.element_updates) + ")");
}

TimeBreakdown modeled_times(const LedgerSnapshot& ledger, const HardwareModel& hw) {
  hw.validate();
  TimeBreakdown t;
  t.t_htod = static_cast<double>(ledger.htod) / hw.bw_intc;
  t.t_dtoh = static_cast<double>(ledger.dtoh) / hw.bw_intc;
  t.t_kernel =
      static_cast<double>(ledger.scratch_load + ledger.scratch_store + ledger.ondevice) /
      hw.bw_dmem;
  t.t_total_serial = t.t_htod + t.t_dtoh + t.t_kernel;
  t.t_total_overlap = std::max(t.t_htod + t.t_dtoh, t.t_kernel);
  return t;
}

// Process-wide share-buffer ids: "share_buffer", "share_buffer#1", ...
// (proj/src/memsim.cpp:100-105).
std::string next_share_buffer_id() {
  static std::atomic<int> counter{0};
  const int n = counter.fetch_add(1);
  return n == 0 ? std::string("share_buffer") : "share_buffer#" + std::to_string(n);
}

ShareBuffer ShareBuffer::slab_mode(DeviceArena& arena, int n_slots, int slab_rows, int cols) {
  if (n_slots < 2) throw InvalidSpecError("share buffer needs at least 2 slots");
  ShareBuffer b;
  b.arena_ = &arena;
  b.id_ = next_share_buffer_id();
  b.n_slots_ = n_slots;
  b.per_slot_ = static_cast<std::size_t>(slab_rows) * cols;
  b.bytes_ = static_cast<std::uint64_t>(n_slots) * b.per_slot_ * sizeof(float);
  arena.alloc(b.id_, b.bytes_);
  b.data_.resize(static_cast<std::size_t>(n_slots) * b.per_slot_);
  b.slots_.resize(n_slots);
  return b;
}

ShareBuffer ShareBuffer::state_mode(DeviceArena& arena, int boundaries, int states, int rows,
                                    int cols) {
  ShareBuffer b;
  b.arena_ = &arena;
  b.id_ = next_share_buffer_id();
  b.per_state_ = true;
  b.boundaries_ = boundaries;
  b.states_ = states;
  b.per_slot_ = static_cast<std::size_t>(rows) * cols;
  const std::size_t count = static_cast<std::size_t>(std::max(boundaries, 0)) * std::max(states, 0);
  b.bytes_ = static_cast<std::uint64_t>(count) * b.per_slot_ * sizeof(float);
  arena.alloc(b.id_, b.bytes_);
  b.data_.resize(count * b.per_slot_);
  b.slots_.resize(std::max<std::size_t>(count, 1));
  return b;
}

ShareBuffer::~ShareBuffer() {
  if (arena_) arena_->free(id_);
}

ShareBuffer::ShareBuffer(ShareBuffer&& o) noexcept
    : arena_(o.arena_),
      id_(std::move(o.id_)),
      per_state_(o.per_state_),
      n_slots_(o.n_slots_),
      boundaries_(o.boundaries_),
      states_(o.states_),
      per_slot_(o.per_slot_),
      bytes_(o.bytes_),
      data_(std::move(o.data_)),
      slots_(std::move(o.slots_)) {
  o.arena_ = nullptr;
}

std::size_t ShareBuffer::index_of(int boundary, int state) const {
  if (per_state_) {
    if (boundary < 0 || boundary >= boundaries_ || state < 0 || state >= states_)
      throw ContractError("share buffer: (boundary, state) out of range");
    return static_cast<std::size_t>(boundary) * states_ + state;
  }
  if (boundary < 0) throw ContractError("share buffer: negative boundary");
  return static_cast<std::size_t>(boundary % n_slots_);
}

void ShareBuffer::publish(int boundary, int state, const float* src, std::size_t count,
                          TransferLedger& ledger) {
  if (count > per_slot_) throw ContractError("share buffer: publish larger than slot");
  const std::size_t i = index_of(boundary, state);
  {
    std::lock_guard<std::mutex> g(mu_);
    Slot& s = slots_[i];
    if (s.phase != Phase::empty && s.phase != Phase::consumed)
      throw ContractError("share buffer: overwriting slot written by chunk " +
                          std::to_string(s.owner) + " before it was consumed");
    s.phase = Phase::writing;
    s.owner = boundary;
  }
  std::memcpy(data_.data() + i * per_slot_, src, count * sizeof(float));
  {
    std::lock_guard<std::mutex> g(mu_);
    slots_[i].phase = Phase::written;
  }
  ledger.record(Counter::ondevice, static_cast<std::int64_t>(count * sizeof(float)));
}

void ShareBuffer::consume(int boundary, int state, float* dst, std::size_t count,
                          TransferLedger& ledger) {
  if (count > per_slot_) throw ContractError("share buffer: consume larger than slot");
  const std::size_t i = index_of(boundary, state);
  {
    std::lock_guard<std::mutex> g(mu_);
    Slot& s = slots_[i];
    if (s.phase != Phase::written)
      throw ContractError("share buffer: consuming a slot that was not written");
    if (s.owner != boundary)
      throw ContractError("share buffer: slot holds boundary " + std::to_string(s.owner) +
                          ", expected " + std::to_string(boundary));
    s.phase = Phase::reading;
  }
  std::memcpy(dst, data_.data() + i * per_slot_, count * sizeof(float));
  {
    std::lock_guard<std::mutex> g(mu_);
    slots_[i].phase = Phase::consumed;
  }
  ledger.record(Counter::ondevice, static_cast<std::int64_t>(count * sizeof(float)));
}

void ShareBuffer::reset_round() {
  std::lock_guard<std::mutex> g(mu_);
  for (const Slot& s : slots_)
    if (s.phase != Phase::empty && s.phase != Phase::consumed)
      throw ContractError("share buffer: round ended with an unconsumed slot");
  for (Slot& s : slots_) s = Slot{};
}

// ---------------------------------------------------------------- planner --
// proj/src/planner.cpp:10-113

std::string to_string(Regime regime) {
  return regime == Regime::transfer_bound ? "transfer-bound" : "kernel-bound";
}

BottleneckPrediction predict_bottleneck_raw(const HardwareModel& hw, std::uint64_t d_chk_elems,
                                            std::uint64_t w_halo_elems, int s_tb) {
  hw.validate();
  const double b = hw.b_elem;
  BottleneckPrediction p;
  p.t_transfer = static_cast<double>(d_chk_elems) * b / hw.bw_intc;
  p.t_kernel = static_cast<double>(d_chk_elems + w_halo_elems * s_tb) * b * s_tb / hw.bw_dmem;
  p.regime = p.t_kernel > p.t_transfer ? Regime::kernel_bound : Regime::transfer_bound;
  return p;
}

BottleneckPrediction predict_bottleneck(const HardwareModel& hw, const RunConfig& config) {
  config.validate();
  return predict_bottleneck_raw(hw, config.d_chk(), config.w_halo(), config.s_tb);
}

FeasibilityReport feasible_configs(const HardwareModel& hw, const StencilSpec& stencil, int sz,
                                   const std::vector<std::pair<int, int>>& candidates,
                                   const PlannerOptions& opts) {
  hw.validate();
  stencil.validate();
  if (sz <= 0) throw InvalidSpecError("planner: sz must be positive");
  FeasibilityReport rep;
  rep.n_strm = opts.n_strm;
  rep.n_a = opts.n_a;
  rep.ratio_threshold = opts.ratio_threshold;
  const std::uint64_t r = static_cast<std::uint64_t>(stencil.radius);
  const std::uint64_t p = static_cast<std::uint64_t>(sz) + 2 * r;
  const double b = hw.b_elem;
  for (const auto& cand : candidates) {
    const int d = cand.first, s = cand.second;
    FeasibilityEntry e;
    e.d = d;
    e.s_tb = s;
    if (d < 1 || s < 1 || sz % d != 0) {
      e.failed.push_back("valid (d, S_TB)");
      rep.entries.push_back(std::move(e));
      continue;
    }
    const std::uint64_t chunk = static_cast<std::uint64_t>(sz) * p / d;
    const std::uint64_t halo = 2 * r * p * static_cast<std::uint64_t>(s);
    const double tk = static_cast<double>(chunk + halo) * opts.n_a * b * s / hw.bw_dmem;
    const double tt = static_cast<double>(chunk) * (opts.n_a - 1) * b / hw.bw_intc;
    if (!(tk > tt)) e.failed.push_back("kernel time > transfer time");
    if ((chunk + halo) * static_cast<std::uint64_t>(opts.n_strm) >
        hw.c_dmem / static_cast<std::uint64_t>(hw.b_elem))
      e.failed.push_back("(D_chk+W_halo*S_TB)*N_strm <= C_dmem/b_elem");
    if (halo > chunk) e.failed.push_back("W_halo*S_TB <= D_chk");
    if (d <= opts.n_strm) e.failed.push_back("d > N_strm");
    e.halo_ratio = static_cast<double>(halo) / static_cast<double>(chunk);
    e.degradation_risk = e.halo_ratio > opts.ratio_threshold;
    const BottleneckPrediction bp = predict_bottleneck_raw(hw, chunk, 2 * r * p, s);
    e.t_transfer = bp.t_transfer;
    e.t_kernel = bp.t_kernel;
    e.regime = bp.regime;
    e.feasible = e.failed.empty();
    rep.entries.push_back(std::move(e));
  }
  return rep;
}

TrafficEstimate analytic_traffic(const RunConfig& config, bool sharing) {
  plan_chunks(config);
  const std::uint64_t p = config.padded();
  const std::uint64_t shared = 2ull * config.r * config.s_tb * (config.d - 1);
  TrafficEstimate t;
  t.htod = p * p + (sharing ? 0 : shared * p);
  t.dtoh = static_cast<std::uint64_t>(config.sz) * p;
  t.ondevice = sharing ? 2 * shared * p : 0;
  return t;
}

std::uint64_t analytic_redundancy(const RunConfig& config, int steps) {
  plan_chunks(config);
  if (steps < 0 || steps > config.s_tb)
    throw std::out_of_range("analytic_redundancy: steps outside 0..S_TB");
  return static_cast<std::uint64_t>(config.d - 1) * config.r * steps * (steps - 1) *
         config.padded();
}

std::uint64_t analytic_redundancy(const RunConfig& config) {
  return analytic_redundancy(config, config.s_tb);
}

// Hardware profile {"name": str, "c_dmem_bytes": int, "bw_dmem_bytes_per_s":
// num, "bw_intc_bytes_per_s": num, "b_elem": int} (proj/src/planner.cpp:115-143);
// other keys (profiles/b200.json carries the B200 planner's) are ignored, as
// the reference's nlohmann reader does.
HardwareModel hardware_profile_from_json(const std::string& text, const std::string& origin) {
  so2dr_json::Value j;
  try {
    j = so2dr_json::parse(text);
  } catch (const so2dr_json::ParseError& e) {
    throw IoError("hardware profile " + origin + ": " + e.what());
  }
  HardwareModel hw;
  try {
    hw.name = j.contains("name") ? j.at("name").as_string() : "unnamed";
    hw.c_dmem = j.at("c_dmem_bytes").as_uint64();
    hw.bw_dmem = j.at("bw_dmem_bytes_per_s").as_double();
    hw.bw_intc = j.at("bw_intc_bytes_per_s").as_double();
    hw.b_elem = j.contains("b_elem") ? static_cast<int>(j.at("b_elem").as_int64()) : 4;
  } catch (const std::exception& e) {
    throw IoError("hardware profile " + origin + ": " + e.what());
  }
  hw.validate();
  return hw;
}

HardwareModel load_hardware_profile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open hardware profile " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return hardware_profile_from_json(ss.str(), path);
}

// ----------------------------------------------------------------- gridio --
// proj/src/gridio.cpp:9-60: magic "SO2D", u16 version 1, u32 sz, u16 r,
// u32 reserved, then little-endian f32 cells.

void dump_grid(const Grid& grid, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open " + path + " for writing");
  unsigned char hdr[16] = {'S', 'O', '2', 'D'};
  const std::uint16_t version = 1;
  const std::uint32_t sz = static_cast<std::uint32_t>(grid.spec.sz);
  const std::uint16_t r = static_cast<std::uint16_t>(grid.spec.r);
  std::memcpy(hdr + 4, &version, 2);
  std::memcpy(hdr + 6, &sz, 4);
  std::memcpy(hdr + 10, &r, 2);
  out.write(reinterpret_cast<const char*>(hdr), 16);
  out.write(reinterpret_cast<const char*>(grid.values.data()),
            static_cast<std::streamsize>(grid.values.size() * sizeof(float)));
  if (!out) throw IoError("short write to " + path);
}

Grid load_grid(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path);
  unsigned char hdr[16] = {};
  in.read(reinterpret_cast<char*>(hdr), 16);
  if (!in || std::memcmp(hdr, "SO2D", 4) != 0) throw IoError(path + ": not a grid dump (bad magic)");
  std::uint16_t version = 0, r = 0;
  std::uint32_t sz = 0;
  std::memcpy(&version, hdr + 4, 2);
  std::memcpy(&sz, hdr + 6, 4);
  std::memcpy(&r, hdr + 10, 2);
  if (version != 1) throw IoError(path + ": unsupported version " + std::to_string(version));
  Grid g{GridSpec{static_cast<int>(sz), static_cast<int>(r)}, {}};
  g.values.resize(g.spec.cell_count());
  in.read(reinterpret_cast<char*>(g.values.data()),
          static_cast<std::streamsize>(g.values.size() * sizeof(float)));
  if (!in) throw IoError(path + ": truncated grid data");
  return g;
}

// ----------------------------------------------------------------- verify --
// proj/src/verify.cpp:7-59 (closed forms)

ExpectedLedger expected_ledger(EngineMode mode, const RunConfig& config, const KernelPlan& kernel) {
  RunConfig c = config;
  KernelPlan k = kernel;
  if (mode == EngineMode::resreu) c.k_on = k.k_on = 1;
  if (mode == EngineMode::incore) c.d = 1;
  c.validate();
  const std::uint64_t p = c.padded();
  const std::uint64_t row = p * GridSpec::b_elem;
  ExpectedLedger e;
  if (mode == EngineMode::incore) {
    e.htod = p * row;
    e.dtoh = static_cast<std::uint64_t>(c.sz) * row;
    e.kernel_invocations = (static_cast<std::uint64_t>(c.n) + k.k_on - 1) / k.k_on;
    e.rounds = 1;
    e.redundancy_exact = k.tile >= static_cast<int>(p);
    return e;
  }
  const RoundPlan rp = make_round_plan(c);
  const std::uint64_t nb = static_cast<std::uint64_t>(c.d - 1);
  for (int t = 0; t < rp.rounds; ++t) {
    const std::uint64_t ke = rp.steps_in_round(t);
    e.htod += p * row;
    e.dtoh += static_cast<std::uint64_t>(c.sz) * row;
    if (mode == EngineMode::so2dr) {
      e.ondevice += 2 * nb * (2ull * c.r * c.s_tb) * row;
      e.kernel_invocations += static_cast<std::uint64_t>(c.d) * rp.calls_in_round(t);
      e.redundant_updates += nb * c.r * ke * (ke - 1) * p;
    } else {
      e.ondevice += 2 * nb * (2ull * c.r) * ke * row;
      e.kernel_invocations += static_cast<std::uint64_t>(c.d) * ke;
    }
  }
  e.rounds = rp.rounds;
  e.redundancy_exact = mode == EngineMode::resreu || k.tile >= static_cast<int>(p);
  return e;
}

// ----------------------------------------------------------------- engine --

std::string to_string(EngineMode mode) {
  switch (mode) {
    case EngineMode::so2dr: return "so2dr";
    case EngineMode::resreu: return "resreu";
    case EngineMode::incore: return "incore";
  }
  return "?";
}

EngineMode engine_mode_from_string(const std::string& s) {
  if (s == "so2dr") return EngineMode::so2dr;
  if (s == "resreu") return EngineMode::resreu;
  if (s == "incore") return EngineMode::incore;
  throw InvalidSpecError("unknown engine mode \"" + s + "\"");
}

std::string to_string(Stage stage) {
  switch (stage) {
    case Stage::htod: return "htod";
    case Stage::share_read: return "share_read";
    case Stage::share_write: return "share_write";
    case Stage::kernel: return "kernel";
    case Stage::dtoh: return "dtoh";
  }
  return "?";
}

void KernelPlan::validate(int radius) const {
  if (k_on < 1) throw InvalidSpecError("kernel: k_on must be at least 1");
  if (tile < 1) throw InvalidSpecError("kernel: tile must be at least 1");
  const std::uint64_t need = scratch_footprint(radius, k_on);
  if (need > scratch_budget)
    throw InvalidSpecError("kernel: scratch footprint " + std::to_string(need) +
                           " bytes exceeds budget " + std::to_string(scratch_budget) +
                           " (tile=" + std::to_string(tile) + ", k_on=" + std::to_string(k_on) +
                           ", r=" + std::to_string(radius) + ")");
}

std::uint64_t so2dr_arena_bytes(const RunConfig& config, const KernelPlan& kernel) {
  // proj/src/engine.cpp:53-65: one working buffer per stream + slots + scratch
  const std::uint64_t b = GridSpec::b_elem;
  const std::uint64_t work = (config.d_chk() + config.w_halo() * config.s_tb) * b * config.n_strm;
  const std::uint64_t slots = static_cast<std::uint64_t>(std::max(2, config.n_strm));
  const std::uint64_t share = slots * (2ull * config.r * config.s_tb) * config.padded() * b;
  const std::uint64_t scratch = static_cast<std::uint64_t>(config.n_strm) *
                                kernel.scratch_footprint(config.r, kernel.k_on);
  return work + share + scratch;
}

}  // namespace so2dr
