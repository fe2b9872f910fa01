// specfile.cpp -- run spec files, the built-in presets and the run outputs
// (report.json v1, ledger.csv, diagnostics.csv): the reference's front-end
// formats, so a reference user keeps their spec files, preset names and
// report consumers. Host-only code (no device work).
//
//   parse_spec_json / parse_spec_file  <- proj/src/specfile.cpp:39-93
//   presets                            <- proj/tools/so2dr_main.cpp:28-68
//   report_to_json / *_to_csv          <- proj/src/report.cpp:21-88
#include <algorithm>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

#include "json_lite.hpp"
#include "so2dr/report.hpp"
#include "so2dr/specfile.hpp"
#include "so2dr_cuda.h"

namespace so2dr {

namespace {

using so2dr_json::Value;

std::string field_name(const std::string& path, const char* key) {
  return path.empty() ? key : path + "." + key;
}

const Value& need(const Value& j, const std::string& path, const char* key, const std::string& origin) {
  if (!j.is_object() || !j.contains(key)) throw IoError(origin + ": missing field " + field_name(path, key));
  return j.at(key);
}

[[noreturn]] void wrong_type(const std::string& path, const char* key, const std::string& origin) {
  throw IoError(origin + ": field " + field_name(path, key) + " has the wrong type");
}

int need_int(const Value& j, const std::string& path, const char* key, const std::string& origin) {
  const Value& v = need(j, path, key, origin);
  try {
    const std::int64_t x = v.as_int64();
    if (x < INT32_MIN || x > INT32_MAX) wrong_type(path, key, origin);
    return static_cast<int>(x);
  } catch (const std::invalid_argument&) {
    wrong_type(path, key, origin);
  }
}

std::uint64_t need_u64(const Value& j, const std::string& path, const char* key, const std::string& origin) {
  const Value& v = need(j, path, key, origin);
  try {
    return v.as_uint64();
  } catch (const std::invalid_argument&) {
    wrong_type(path, key, origin);
  }
}

std::string need_str(const Value& j, const std::string& path, const char* key, const std::string& origin) {
  const Value& v = need(j, path, key, origin);
  if (!v.is_string()) wrong_type(path, key, origin);
  return v.as_string();
}

template <typename F>
auto opt(const Value& j, const std::string& path, const char* key, const std::string& origin, F&& read,
         decltype(read(j)) dflt) -> decltype(read(j)) {
  if (!j.is_object() || !j.contains(key)) return dflt;
  try {
    return read(j.at(key));
  } catch (const std::invalid_argument&) {
    wrong_type(path, key, origin);
  }
}

std::string desk(const std::string& kind, int radius) {
  std::ostringstream s;
  s << "{\n"
    << "  \"stencil\": {\"kind\": \"" << kind << "\", \"radius\": " << radius << "},\n"
    << "  \"grid\": {\"sz\": 512, \"seed\": 42},\n"
    << "  \"mode\": \"so2dr\",\n"
    << "  \"config\": {\"d\": 4, \"s_tb\": 16, \"k_on\": 4, \"n_strm\": 3, \"n\": 64, \"n_a\": 2}\n"
    << "}\n";
  return s.str();
}

std::string paper(const std::string& kind, int radius, int s_tb) {
  std::ostringstream s;
  s << "{\n"
    << "  \"stencil\": {\"kind\": \"" << kind << "\", \"radius\": " << radius << "},\n"
    << "  \"grid\": {\"sz\": 38400, \"seed\": 7},\n"
    << "  \"mode\": \"so2dr\",\n"
    << "  \"config\": {\"d\": 4, \"s_tb\": " << s_tb
    << ", \"k_on\": 4, \"n_strm\": 3, \"n\": 640, \"n_a\": 2}\n"
    << "}\n";
  return s.str();
}

// B200 BASELINE configurations (BASELINE.json configs[0..4], per-GPU shapes)
std::string b200(const std::string& kind, int radius, int dim, const char* dtype, int sz, int d, int s_tb,
                 int k_on, int n, std::uint64_t seed) {
  std::ostringstream s;
  s << "{\n"
    << "  \"stencil\": {\"kind\": \"" << kind << "\", \"radius\": " << radius;
  if (dim != 2) s << ", \"dim\": " << dim;
  s << "},\n"
    << "  \"grid\": {\"sz\": " << sz << ", \"seed\": " << seed;
  if (std::strcmp(dtype, "f32") != 0) s << ", \"dtype\": \"" << dtype << "\"";
  s << "},\n"
    << "  \"mode\": \"so2dr\",\n"
    << "  \"config\": {\"d\": " << d << ", \"s_tb\": " << s_tb << ", \"k_on\": " << k_on
    << ", \"n_strm\": 3, \"n\": " << n << ", \"n_a\": 2}\n"
    << "}\n";
  return s.str();
}

const std::vector<std::pair<std::string, std::string>>& preset_table() {
  static const std::vector<std::pair<std::string, std::string>> t = [] {
    std::vector<std::pair<std::string, std::string>> v;
    v.emplace_back("box2d1r-desk", desk("box", 1));
    v.emplace_back("box2d2r-desk", desk("box", 2));
    v.emplace_back("box2d3r-desk", desk("box", 3));
    v.emplace_back("box2d4r-desk", desk("box", 4));
    v.emplace_back("gradient2d-desk", desk("gradient", 1));
    v.emplace_back("box2d1r-paper", paper("box", 1, 160));
    v.emplace_back("box2d2r-paper", paper("box", 2, 160));
    v.emplace_back("box2d3r-paper", paper("box", 3, 80));
    v.emplace_back("box2d4r-paper", paper("box", 4, 40));
    v.emplace_back("gradient2d-paper", paper("gradient", 1, 160));
    // BASELINE.json configs (B200): cfg1 CPU preset, cfg2 the bench workload,
    // cfg3 star3d1r (k_on swept 1..8 by the caller), cfg4 box3d1r per-GPU slab
    // shape, cfg5 star2d2r fp64 per-GPU shape
    v.emplace_back("star2d1r-cfg1", b200("star", 1, 2, "f32", 4096, 4, 4, 4, 8, 42));
    v.emplace_back("box2d1r-b200", b200("box", 1, 2, "f32", 92160, 64, 64, 4, 64, 42));
    v.emplace_back("star3d1r-b200", b200("star", 1, 3, "f32", 2048, 16, 8, 8, 64, 42));
    v.emplace_back("box3d1r-b200", b200("box", 1, 3, "f32", 2048, 32, 16, 4, 32, 42));
    v.emplace_back("star2d2r-f64-b200", b200("star", 2, 2, "f64", 65536, 16, 64, 4, 64, 42));
    return v;
  }();
  return t;
}

}  // namespace

std::vector<std::string> preset_names() {
  std::vector<std::string> out;
  for (const auto& kv : preset_table()) out.push_back(kv.first);
  return out;
}

std::string preset_json(const std::string& name) {
  for (const auto& kv : preset_table())
    if (kv.first == name) return kv.second;
  throw InvalidSpecError("unknown preset \"" + name + "\"");
}

RunSpecFile parse_spec_json(const std::string& text, const std::string& origin) {
  Value j;
  try {
    j = so2dr_json::parse(text);
  } catch (const so2dr_json::ParseError& e) {
    throw IoError(origin + ": JSON parse error at " + so2dr_json::line_col(text, e.byte) + ": " + e.what());
  }
  if (!j.is_object()) throw IoError(origin + ": a spec file is a JSON object");

  RunSpecFile spec;
  const Value& st = need(j, "", "stencil", origin);
  const std::string kind = need_str(st, "stencil", "kind", origin);
  const int radius = need_int(st, "stencil", "radius", origin);
  spec.dim = opt(st, "stencil", "dim", origin, [](const Value& v) { return static_cast<int>(v.as_int64()); }, 2);
  if (spec.dim != 2 && spec.dim != 3)
    throw IoError(origin + ": stencil.dim " + std::to_string(spec.dim) + " invalid (2 or 3)");
  const StencilKind k = stencil_kind_from_string(kind);
  if (st.contains("weights")) {
    const Value& w = st.at("weights");
    if (!w.is_array()) wrong_type("stencil", "weights", origin);
    for (const Value& x : w.elements()) {
      if (!x.is_number()) wrong_type("stencil", "weights", origin);
      spec.weights.push_back(x.as_double());
    }
  }
  if (k != StencilKind::gradient && (radius < 1 || radius > 4)) StencilSpec::box(radius);  // throws
  const size_t e = 2 * static_cast<size_t>(std::max(radius, 0)) + 1;
  const size_t full = spec.dim == 3 ? e * e * e : e * e;
  const size_t axis = 2 * static_cast<size_t>(spec.dim) * radius + 1;
  if (k == StencilKind::gradient) {
    spec.stencil = StencilSpec::gradient();
  } else if (!spec.weights.empty() && spec.weights.size() != full &&
             !(k == StencilKind::star && spec.weights.size() == axis)) {
    throw IoError(origin + ": stencil.weights needs " + std::to_string(full) +
                  (k == StencilKind::star ? " (or " + std::to_string(axis) + " on-axis)" : std::string()) +
                  " entries for radius " + std::to_string(radius));
  } else if (spec.dim == 2 && spec.weights.size() == full) {
    // canonical (2r+1)^2 weights: the reference's box(r, w) (a star is a box
    // with zero off-axis weights there)
    spec.stencil = StencilSpec::box(radius, std::vector<float>(spec.weights.begin(), spec.weights.end()));
  } else if (spec.dim == 2 && k == StencilKind::star && !spec.weights.empty()) {
    spec.stencil = StencilSpec::star(radius, std::vector<float>(spec.weights.begin(), spec.weights.end()));
  } else {
    // 3D specs keep a 2D StencilSpec of the same kind/radius as their name
    // carrier; the weights reach the engine through the C ABI
    spec.stencil = k == StencilKind::star ? StencilSpec::star(radius) : StencilSpec::box(radius);
  }
  if (spec.stencil.radius != radius)
    throw IoError(origin + ": stencil.radius " + std::to_string(radius) + " invalid for kind \"" + kind + "\"");

  const Value& g = need(j, "", "grid", origin);
  spec.config.sz = need_int(g, "grid", "sz", origin);
  spec.seed = need_u64(g, "grid", "seed", origin);
  spec.dtype = opt(g, "grid", "dtype", origin, [](const Value& v) { return v.as_string(); }, std::string("f32"));
  if (spec.dtype != "f32" && spec.dtype != "f64")
    throw IoError(origin + ": grid.dtype \"" + spec.dtype + "\" invalid (f32 or f64)");

  spec.mode = engine_mode_from_string(need_str(j, "", "mode", origin));

  const Value& c = need(j, "", "config", origin);
  spec.config.r = spec.stencil.radius;
  spec.config.d = need_int(c, "config", "d", origin);
  spec.config.s_tb = need_int(c, "config", "s_tb", origin);
  spec.config.k_on = need_int(c, "config", "k_on", origin);
  spec.config.n_strm = need_int(c, "config", "n_strm", origin);
  spec.config.n = need_int(c, "config", "n", origin);
  spec.config.n_a = opt(c, "config", "n_a", origin, [](const Value& v) { return static_cast<int>(v.as_int64()); }, 2);
  spec.kernel.k_on = spec.config.k_on;

  if (j.contains("kernel")) {
    const Value& kk = j.at("kernel");
    spec.kernel.tile =
        opt(kk, "kernel", "tile", origin, [](const Value& v) { return static_cast<int>(v.as_int64()); }, spec.kernel.tile);
    spec.kernel.scratch_budget = opt(kk, "kernel", "scratch_budget", origin,
                                     [](const Value& v) { return v.as_uint64(); }, spec.kernel.scratch_budget);
  }
  if (j.contains("hardware")) {
    if (!j.at("hardware").is_string()) wrong_type("", "hardware", origin);
    spec.hardware_path = j.at("hardware").as_string();
  }
  if (j.contains("output") && j.at("output").is_object() && j.at("output").contains("grid_dump")) {
    if (!j.at("output").at("grid_dump").is_string()) wrong_type("output", "grid_dump", origin);
    spec.grid_dump_path = j.at("output").at("grid_dump").as_string();
  }

  try {
    spec.config.validate();
  } catch (const InvalidSpecError& e) {
    throw IoError(origin + ": " + e.what());
  }
  return spec;
}

RunSpecFile parse_spec_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open spec file " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_spec_json(ss.str(), path);
}

// ----------------------------------------------------------------- report --

namespace {

std::string hex64(std::uint64_t v) {
  static const char* dig = "0123456789abcdef";
  std::string s = "0x";
  for (int shift = 60; shift >= 0; shift -= 4) s.push_back(dig[(v >> shift) & 0xF]);
  return s;
}

Value u64(std::uint64_t v) { return Value::uinteger(v); }
Value i32(int v) { return Value::integer(v); }

}  // namespace

std::string report_to_json(const RunReport& report, bool deterministic) {
  Value j = Value::object();
  j.set("schema_version", i32(1));
  j.set("mode", Value::string(to_string(report.mode)));
  j.set("stencil", Value::string(report.stencil_name));
  Value c = Value::object();
  c.set("sz", i32(report.config.sz));
  c.set("r", i32(report.config.r));
  c.set("d", i32(report.config.d));
  c.set("s_tb", i32(report.config.s_tb));
  c.set("k_on", i32(report.config.k_on));
  c.set("n_strm", i32(report.config.n_strm));
  c.set("n", i32(report.config.n));
  c.set("n_a", i32(report.config.n_a));
  j.set("config", c);
  Value k = Value::object();
  k.set("tile", i32(report.kernel.tile));
  k.set("k_on", i32(report.kernel.k_on));
  k.set("scratch_budget", u64(report.kernel.scratch_budget));
  j.set("kernel", k);
  j.set("rounds", u64(report.ledger.rounds));
  j.set("checksum", Value::string(hex64(report.checksum)));
  Value l = Value::object();
  l.set("htod_bytes", u64(report.ledger.htod));
  l.set("dtoh_bytes", u64(report.ledger.dtoh));
  l.set("ondevice_bytes", u64(report.ledger.ondevice));
  l.set("scratch_load_bytes", u64(report.ledger.scratch_load));
  l.set("scratch_store_bytes", u64(report.ledger.scratch_store));
  l.set("element_updates", u64(report.ledger.element_updates));
  l.set("redundant_updates", u64(report.ledger.redundant_updates));
  l.set("kernel_invocations", u64(report.ledger.kernel_invocations));
  l.set("rounds", u64(report.ledger.rounds));
  j.set("ledger", l);
  Value t = Value::object();
  t.set("t_htod", Value::real(report.times.t_htod));
  t.set("t_dtoh", Value::real(report.times.t_dtoh));
  t.set("t_kernel", Value::real(report.times.t_kernel));
  t.set("t_total_overlap", Value::real(report.times.t_total_overlap));
  t.set("t_total_serial", Value::real(report.times.t_total_serial));
  j.set("modeled_times", t);
  Value a = Value::object();
  a.set("peak_bytes", u64(report.arena_peak));
  a.set("capacity_bytes", u64(report.arena_capacity));
  j.set("arena", a);
  j.set("transfer_time_excluded", Value::boolean(report.transfer_time_excluded));
  if (!deterministic) {
    j.set("wall_seconds", Value::real(report.wall_seconds));
    if (report.measured.kernel_launches || report.measured.device_ms > 0) {
      Value m = Value::object();
      m.set("device_ms", Value::real(report.measured.device_ms));
      m.set("kernel_ms", Value::real(report.measured.kernel_ms));
      m.set("kernel_launches", u64(report.measured.kernel_launches));
      m.set("kernel_alg_bytes", u64(report.measured.kernel_alg_bytes));
      m.set("device_bytes", u64(report.measured.device_bytes));
      j.set("measured", m);
    }
  }
  return j.dump(2) + "\n";
}

std::string ledger_to_csv(const LedgerSnapshot& ledger) {
  std::ostringstream out;
  out << "counter,value\n";
  out << "htod_bytes," << ledger.htod << "\n";
  out << "dtoh_bytes," << ledger.dtoh << "\n";
  out << "ondevice_bytes," << ledger.ondevice << "\n";
  out << "scratch_load_bytes," << ledger.scratch_load << "\n";
  out << "scratch_store_bytes," << ledger.scratch_store << "\n";
  out << "element_updates," << ledger.element_updates << "\n";
  out << "redundant_updates," << ledger.redundant_updates << "\n";
  out << "kernel_invocations," << ledger.kernel_invocations << "\n";
  out << "rounds," << ledger.rounds << "\n";
  return out.str();
}

std::string diagnostics_to_csv(const std::vector<DiagRow>& rows) {
  std::ostringstream out;
  out << "round,chunk,stage,bytes,updates\n";
  for (const DiagRow& row : rows)
    out << row.round << "," << row.chunk << "," << to_string(row.stage) << "," << row.bytes << ","
        << row.updates << "\n";
  return out.str();
}

void write_text_file(const std::string& path, const std::string& content) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open " + path + " for writing");
  out << content;
  if (!out) throw IoError("short write to " + path);
}

}  // namespace so2dr
