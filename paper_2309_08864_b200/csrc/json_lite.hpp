// json_lite.hpp -- the small JSON DOM the host side needs: spec files
// (proj/src/specfile.cpp), hardware profiles (proj/src/planner.cpp) and the
// report.json v1 writer (proj/src/report.cpp). The reference uses
// nlohmann/json for these; this is a self-contained replacement with the
// properties those call sites rely on: insertion-ordered objects, exact
// 64-bit integers, parse errors carrying the byte offset (reported as
// "line L, column C"), and a 2-space-indented dump in nlohmann's layout.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace so2dr_json {

struct ParseError : std::runtime_error {
  std::size_t byte;  // offset of the offending character
  ParseError(std::size_t b, const std::string& m) : std::runtime_error(m), byte(b) {}
};

class Value {
 public:
  enum class Type { null, boolean, integer, unsigned_integer, real, string, array, object };

  Value() = default;
  static Value boolean(bool b);
  static Value integer(std::int64_t v);
  static Value uinteger(std::uint64_t v);
  static Value real(double v);
  static Value string(std::string s);
  static Value array();
  static Value object();

  Type type() const { return t_; }
  bool is_null() const { return t_ == Type::null; }
  bool is_number() const { return t_ == Type::integer || t_ == Type::unsigned_integer || t_ == Type::real; }
  bool is_string() const { return t_ == Type::string; }
  bool is_object() const { return t_ == Type::object; }
  bool is_array() const { return t_ == Type::array; }
  bool is_bool() const { return t_ == Type::boolean; }

  // object access (insertion order preserved; the last duplicate key wins)
  bool contains(const std::string& key) const;
  const Value& at(const std::string& key) const;  // std::out_of_range if absent
  Value& set(const std::string& key, Value v);    // append or replace
  const std::vector<std::pair<std::string, Value>>& items() const { return obj_; }

  // array access
  const std::vector<Value>& elements() const { return arr_; }
  Value& push(Value v);

  // typed reads; std::invalid_argument when the type does not convert
  // (an integral-valued real converts to an integer, as nlohmann does)
  bool as_bool() const;
  std::int64_t as_int64() const;
  std::uint64_t as_uint64() const;
  double as_double() const;
  const std::string& as_string() const;

  // nlohmann::json::dump(indent) layout: "{\n  \"k\": v,\n ...}"; indent < 0 = compact
  std::string dump(int indent = -1) const;

 private:
  void dump_to(std::string& out, int indent, int depth) const;

  Type t_ = Type::null;
  bool b_ = false;
  std::int64_t i_ = 0;
  std::uint64_t u_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> arr_;
  std::vector<std::pair<std::string, Value>> obj_;
};

Value parse(const std::string& text);  // throws ParseError

// "line L, column C" of a byte offset (1-based; proj/src/specfile.cpp:13-24)
std::string line_col(const std::string& text, std::size_t byte);

// shortest round-trip decimal of a double, with ".0" for integral values
std::string format_double(double v);

}  // namespace so2dr_json
