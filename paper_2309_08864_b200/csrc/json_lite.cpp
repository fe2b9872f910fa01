// json_lite.cpp -- see json_lite.hpp.
#include "json_lite.hpp"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace so2dr_json {

Value Value::boolean(bool b) {
  Value v;
  v.t_ = Type::boolean;
  v.b_ = b;
  return v;
}
Value Value::integer(std::int64_t x) {
  Value v;
  v.t_ = Type::integer;
  v.i_ = x;
  return v;
}
Value Value::uinteger(std::uint64_t x) {
  Value v;
  v.t_ = Type::unsigned_integer;
  v.u_ = x;
  return v;
}
Value Value::real(double x) {
  Value v;
  v.t_ = Type::real;
  v.d_ = x;
  return v;
}
Value Value::string(std::string s) {
  Value v;
  v.t_ = Type::string;
  v.s_ = std::move(s);
  return v;
}
Value Value::array() {
  Value v;
  v.t_ = Type::array;
  return v;
}
Value Value::object() {
  Value v;
  v.t_ = Type::object;
  return v;
}

bool Value::contains(const std::string& key) const {
  if (t_ != Type::object) return false;
  for (const auto& kv : obj_)
    if (kv.first == key) return true;
  return false;
}

const Value& Value::at(const std::string& key) const {
  if (t_ != Type::object) throw std::out_of_range("not an object");
  const Value* hit = nullptr;
  for (const auto& kv : obj_)
    if (kv.first == key) hit = &kv.second;
  if (!hit) throw std::out_of_range("key '" + key + "' not found");
  return *hit;
}

Value& Value::set(const std::string& key, Value v) {
  if (t_ == Type::null) t_ = Type::object;
  if (t_ != Type::object) throw std::invalid_argument("not an object");
  for (auto& kv : obj_)
    if (kv.first == key) return kv.second = std::move(v);
  obj_.emplace_back(key, std::move(v));
  return obj_.back().second;
}

Value& Value::push(Value v) {
  if (t_ == Type::null) t_ = Type::array;
  if (t_ != Type::array) throw std::invalid_argument("not an array");
  arr_.push_back(std::move(v));
  return arr_.back();
}

bool Value::as_bool() const {
  if (t_ != Type::boolean) throw std::invalid_argument("not a boolean");
  return b_;
}

std::int64_t Value::as_int64() const {
  switch (t_) {
    case Type::integer: return i_;
    case Type::unsigned_integer:
      if (u_ > static_cast<std::uint64_t>(INT64_MAX)) throw std::invalid_argument("out of range");
      return static_cast<std::int64_t>(u_);
    case Type::real:
      if (std::trunc(d_) != d_ || std::fabs(d_) > 9.2e18) throw std::invalid_argument("not integral");
      return static_cast<std::int64_t>(d_);
    default: throw std::invalid_argument("not a number");
  }
}

std::uint64_t Value::as_uint64() const {
  switch (t_) {
    case Type::unsigned_integer: return u_;
    case Type::integer:
      if (i_ < 0) throw std::invalid_argument("negative");
      return static_cast<std::uint64_t>(i_);
    case Type::real:
      if (d_ < 0 || std::trunc(d_) != d_ || d_ > 1.8e19) throw std::invalid_argument("not integral");
      return static_cast<std::uint64_t>(d_);
    default: throw std::invalid_argument("not a number");
  }
}

double Value::as_double() const {
  switch (t_) {
    case Type::integer: return static_cast<double>(i_);
    case Type::unsigned_integer: return static_cast<double>(u_);
    case Type::real: return d_;
    default: throw std::invalid_argument("not a number");
  }
}

const std::string& Value::as_string() const {
  if (t_ != Type::string) throw std::invalid_argument("not a string");
  return s_;
}

// ------------------------------------------------------------------ parser --
namespace {

struct Parser {
  const std::string& s;
  std::size_t i = 0;
  int depth = 0;

  [[noreturn]] void fail(const std::string& what) const {
    const std::string near =
        i < s.size() ? "unexpected '" + std::string(1, s[i]) + "'" : "unexpected end of input";
    throw ParseError(i, "syntax error: " + what + " (" + near + ")");
  }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void expect(char c, const char* what) {
    if (!eat(c)) fail(std::string("expected ") + what);
  }

  static void put_utf8(std::string& out, std::uint32_t cp) {
    if (cp < 0x80) {
      out.push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }
  std::uint32_t hex4() {
    if (i + 4 > s.size()) fail("expected 4 hex digits");
    std::uint32_t v = 0;
    for (int k = 0; k < 4; ++k, ++i) {
      const char c = s[i];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("expected a hex digit");
    }
    return v;
  }
  std::string str() {
    ws();
    if (i >= s.size() || s[i] != '"') fail("expected a string");
    ++i;
    std::string out;
    while (true) {
      if (i >= s.size()) fail("unterminated string");
      const char c = s[i];
      if (c == '"') {
        ++i;
        return out;
      }
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out.push_back(c);
        ++i;
        continue;
      }
      ++i;
      if (i >= s.size()) fail("unterminated escape");
      const char e = s[i++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          std::uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (i + 6 > s.size() || s[i] != '\\' || s[i + 1] != 'u') fail("unpaired surrogate");
            i += 2;
            const std::uint32_t lo = hex4();
            if (lo < 0xDC00 || lo >= 0xE000) fail("bad low surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: --i; fail("bad escape");
      }
    }
  }
  Value number() {
    const std::size_t b = i;
    if (i < s.size() && s[i] == '-') ++i;
    if (i >= s.size() || !(s[i] >= '0' && s[i] <= '9')) fail("expected a digit");
    if (s[i] == '0') {
      ++i;
    } else {
      while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
    }
    bool real = false;
    if (i < s.size() && s[i] == '.') {
      real = true;
      ++i;
      if (i >= s.size() || !(s[i] >= '0' && s[i] <= '9')) fail("expected a digit after '.'");
      while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
    }
    if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
      real = true;
      ++i;
      if (i < s.size() && (s[i] == '+' || s[i] == '-')) ++i;
      if (i >= s.size() || !(s[i] >= '0' && s[i] <= '9')) fail("expected an exponent digit");
      while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
    }
    const char* p0 = s.data() + b;
    const char* p1 = s.data() + i;
    if (!real) {
      if (*p0 == '-') {
        std::int64_t v = 0;
        if (std::from_chars(p0, p1, v).ec == std::errc()) return Value::integer(v);
      } else {
        std::uint64_t v = 0;
        if (std::from_chars(p0, p1, v).ec == std::errc())
          return v <= static_cast<std::uint64_t>(INT64_MAX) ? Value::integer(static_cast<std::int64_t>(v))
                                                            : Value::uinteger(v);
      }
    }
    double d = 0.0;
    const auto rc = std::from_chars(p0, p1, d);
    if (rc.ec != std::errc() || rc.ptr != p1) {
      i = b;
      fail("number out of range");
    }
    return Value::real(d);
  }
  bool word(const char* w) {
    const std::size_t n = std::strlen(w);
    if (s.compare(i, n, w) == 0) {
      i += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (i >= s.size()) fail("expected a value");
    if (++depth > 256) fail("nesting too deep");
    Value v;
    const char c = s[i];
    if (c == '{') {
      ++i;
      v = Value::object();
      if (!eat('}')) {
        do {
          std::string k = str();
          expect(':', "':'");
          v.set(k, value());
        } while (eat(','));
        expect('}', "',' or '}'");
      }
    } else if (c == '[') {
      ++i;
      v = Value::array();
      if (!eat(']')) {
        do {
          v.push(value());
        } while (eat(','));
        expect(']', "',' or ']'");
      }
    } else if (c == '"') {
      v = Value::string(str());
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      v = number();
    } else if (word("true")) {
      v = Value::boolean(true);
    } else if (word("false")) {
      v = Value::boolean(false);
    } else if (word("null")) {
      v = Value();
    } else {
      fail("expected a value");
    }
    --depth;
    return v;
  }
};

void escape_to(std::string& out, const std::string& s) {
  out.push_back('"');
  for (const char ch : s) {
    const unsigned char c = static_cast<unsigned char>(ch);
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          out += buf;
        } else {
          out.push_back(ch);
        }
    }
  }
  out.push_back('"');
}

}  // namespace

Value parse(const std::string& text) {
  Parser p{text};
  Value v = p.value();
  p.ws();
  if (p.i != text.size()) p.fail("expected end of input");
  return v;
}

std::string line_col(const std::string& text, std::size_t byte) {
  std::size_t line = 1, col = 1;
  for (std::size_t i = 0; i < byte && i < text.size(); ++i) {
    if (text[i] == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
  }
  return "line " + std::to_string(line) + ", column " + std::to_string(col);
}

std::string format_double(double v) {
  if (!std::isfinite(v)) return "null";  // JSON has no inf/nan (nlohmann writes null)
  char buf[64];
  const auto rc = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, rc.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string Value::dump(int indent) const {
  std::string out;
  dump_to(out, indent, 0);
  return out;
}

void Value::dump_to(std::string& out, int indent, int depth) const {
  const auto nl = [&](int d) {
    if (indent < 0) return;
    out.push_back('\n');
    out.append(static_cast<std::size_t>(indent * d), ' ');
  };
  switch (t_) {
    case Type::null: out += "null"; break;
    case Type::boolean: out += b_ ? "true" : "false"; break;
    case Type::integer: out += std::to_string(i_); break;
    case Type::unsigned_integer: out += std::to_string(u_); break;
    case Type::real: out += format_double(d_); break;
    case Type::string: escape_to(out, s_); break;
    case Type::array:
      if (arr_.empty()) {
        out += "[]";
        break;
      }
      out.push_back('[');
      for (std::size_t k = 0; k < arr_.size(); ++k) {
        if (k) out.push_back(',');
        nl(depth + 1);
        arr_[k].dump_to(out, indent, depth + 1);
      }
      nl(depth);
      out.push_back(']');
      break;
    case Type::object:
      if (obj_.empty()) {
        out += "{}";
        break;
      }
      out.push_back('{');
      for (std::size_t k = 0; k < obj_.size(); ++k) {
        if (k) out.push_back(',');
        nl(depth + 1);
        escape_to(out, obj_[k].first);
        out += indent < 0 ? ":" : ": ";
        obj_[k].second.dump_to(out, indent, depth + 1);
      }
      nl(depth);
      out.push_back('}');
      break;
  }
}

}  // namespace so2dr_json
