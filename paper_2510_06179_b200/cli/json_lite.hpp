// json_lite.hpp — the slice of JSON the docp CLI reads and writes.
//
// The reference CLI uses nlohmann::json (proj/tools/docp_main.cpp:9-10,
// problems/affine_quadratic_io.hpp:5), which is not in this image. This is
// a small value type with a recursive-descent parser and a writer that
// prints what `nlohmann::json::dump(2)` prints for the same document: keys in
// std::map order, two-space indentation, integers as integers, doubles in
// shortest round-trip form with nlohmann's layout rules (a trailing ".0" on
// integral values, fixed notation for decimal exponents in (-4, 15],
// otherwise "d.ddde+XX"), non-finite doubles as null.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace json_lite {

/// Parse and type errors; the message follows nlohmann's exception text
/// ("[json.exception.<kind>.<id>] ...") so callers can prefix it as the
/// reference does (docp_main.cpp:31-34).
class error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class value {
 public:
  enum kind { null_k, bool_k, int_k, double_k, string_k, array_k, object_k };

  value() = default;
  value(std::nullptr_t) {}
  value(bool b) : k_(bool_k), b_(b) {}
  value(int i) : k_(int_k), i_(i) {}
  value(long i) : k_(int_k), i_(i) {}
  value(long long i) : k_(int_k), i_(i) {}
  value(unsigned i) : k_(int_k), i_(i) {}
  value(unsigned long i) : k_(int_k), i_(static_cast<long long>(i)) {}
  value(unsigned long long i) : k_(int_k), i_(static_cast<long long>(i)) {}
  value(double d) : k_(double_k), d_(d) {}
  value(const char* s) : k_(string_k), s_(s) {}
  value(std::string s) : k_(string_k), s_(std::move(s)) {}
  template <class T>
  value(const std::vector<T>& v) : k_(array_k) {
    for (const auto& x : v) a_.emplace_back(x);
  }

  static value array() {
    value v;
    v.k_ = array_k;
    return v;
  }
  static value object() {
    value v;
    v.k_ = object_k;
    return v;
  }

  kind type() const { return k_; }
  bool is_number() const { return k_ == int_k || k_ == double_k; }

  /// Object member access; turns a null value into an object (as nlohmann does).
  value& operator[](const std::string& key) {
    if (k_ == null_k) k_ = object_k;
    if (k_ != object_k) throw error("[json.exception.type_error.305] cannot use operator[] with a string argument");
    return o_[key];
  }
  bool contains(const std::string& key) const { return k_ == object_k && o_.count(key) != 0; }
  const value& at(const std::string& key) const {
    if (k_ != object_k) throw error("[json.exception.type_error.304] cannot use at() with " + type_name());
    auto it = o_.find(key);
    if (it == o_.end()) throw error("[json.exception.out_of_range.403] key '" + key + "' not found");
    return it->second;
  }
  void push_back(value v) {
    if (k_ == null_k) k_ = array_k;
    a_.push_back(std::move(v));
  }
  const std::vector<value>& elements() const {
    if (k_ != array_k) throw error("[json.exception.type_error.302] type must be array, but is " + type_name());
    return a_;
  }

  double as_double() const {
    if (k_ == double_k) return d_;
    if (k_ == int_k) return static_cast<double>(i_);
    throw error("[json.exception.type_error.302] type must be number, but is " + type_name());
  }
  int as_int() const {
    if (k_ == int_k) return static_cast<int>(i_);
    if (k_ == double_k) return static_cast<int>(d_);
    throw error("[json.exception.type_error.302] type must be number, but is " + type_name());
  }
  const std::string& as_string() const {
    if (k_ != string_k) throw error("[json.exception.type_error.302] type must be string, but is " + type_name());
    return s_;
  }
  std::vector<double> as_doubles() const {
    std::vector<double> out;
    for (const auto& e : elements()) out.push_back(e.as_double());
    return out;
  }

  std::string type_name() const {
    static const char* names[] = {"null", "boolean", "number", "number", "string", "array", "object"};
    return names[k_];
  }

  /// nlohmann::json::dump(indent) layout.
  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

  static value parse(const std::string& text);

 private:
  static void put_number(std::string& out, double d);
  static void put_string(std::string& out, const std::string& s);
  void write(std::string& out, int indent, int level) const;

  kind k_ = null_k;
  bool b_ = false;
  long long i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<value> a_;
  std::map<std::string, value> o_;
};

inline void value::put_number(std::string& out, double d) {
  if (!std::isfinite(d)) {
    out += "null";
    return;
  }
  if (d == 0.0) {
    out += std::signbit(d) ? "-0.0" : "0.0";
    return;
  }
  // shortest digit string that round-trips (what grisu2 emits)
  char buf[40];
  int prec = 0;
  for (prec = 0; prec < 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec, d);
    if (std::strtod(buf, nullptr) == d) break;
  }
  std::snprintf(buf, sizeof buf, "%.*e", prec, d);
  std::string s(buf);
  const bool neg = s[0] == '-';
  if (neg) s.erase(0, 1);
  const auto epos = s.find('e');
  const int e10 = std::atoi(s.c_str() + epos + 1);
  std::string digits;
  for (std::size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits += s[i];
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int k = static_cast<int>(digits.size());
  const int n = e10 + 1;  // position of the decimal point
  std::string r;
  if (k <= n && n <= 15) {
    r = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    r = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    r = "0." + std::string(-n, '0') + digits;
  } else {
    r = digits.substr(0, 1);
    if (k > 1) r += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    r += eb;
  }
  if (neg) out += '-';
  out += r;
}

inline void value::put_string(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          out += b;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

inline void value::write(std::string& out, int indent, int level) const {
  const bool pretty = indent >= 0;
  const std::string pad = pretty ? std::string(static_cast<std::size_t>(indent) * (level + 1), ' ') : "";
  const std::string pad0 = pretty ? std::string(static_cast<std::size_t>(indent) * level, ' ') : "";
  switch (k_) {
    case null_k: out += "null"; break;
    case bool_k: out += b_ ? "true" : "false"; break;
    case int_k: out += std::to_string(i_); break;
    case double_k: put_number(out, d_); break;
    case string_k: put_string(out, s_); break;
    case array_k:
      if (a_.empty()) {
        out += "[]";
        break;
      }
      out += pretty ? "[\n" : "[";
      for (std::size_t i = 0; i < a_.size(); ++i) {
        out += pad;
        a_[i].write(out, indent, level + 1);
        if (i + 1 < a_.size()) out += pretty ? ",\n" : ",";
      }
      out += pretty ? "\n" + pad0 + "]" : "]";
      break;
    case object_k: {
      if (o_.empty()) {
        out += "{}";
        break;
      }
      out += pretty ? "{\n" : "{";
      std::size_t i = 0;
      for (const auto& [key, v] : o_) {
        out += pad;
        put_string(out, key);
        out += pretty ? ": " : ":";
        v.write(out, indent, level + 1);
        if (++i < o_.size()) out += pretty ? ",\n" : ",";
      }
      out += pretty ? "\n" + pad0 + "}" : "}";
      break;
    }
  }
}

namespace detail {

struct parser {
  const std::string& t;
  std::size_t p = 0;

  [[noreturn]] void fail(const std::string& what) const {
    throw error("[json.exception.parse_error.101] parse error at byte " + std::to_string(p + 1) + ": " + what);
  }
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
  }
  bool lit(const char* s) {
    const std::size_t n = std::strlen(s);
    if (t.compare(p, n, s) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (t[p] != '"') fail("expected string");
    ++p;
    std::string s;
    while (p < t.size() && t[p] != '"') {
      char c = t[p++];
      if (c == '\\') {
        if (p >= t.size()) fail("unterminated escape");
        char e = t[p++];
        switch (e) {
          case 'n': s += '\n'; break;
          case 't': s += '\t'; break;
          case 'r': s += '\r'; break;
          case 'b': s += '\b'; break;
          case 'f': s += '\f'; break;
          case 'u': {
            if (p + 4 > t.size()) fail("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p, 4).c_str(), nullptr, 16));
            p += 4;
            if (cp < 0x80) {
              s += static_cast<char>(cp);
            } else if (cp < 0x800) {
              s += static_cast<char>(0xC0 | (cp >> 6));
              s += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              s += static_cast<char>(0xE0 | (cp >> 12));
              s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              s += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: s += e;
        }
      } else {
        s += c;
      }
    }
    if (p >= t.size()) fail("unterminated string");
    ++p;
    return s;
  }
  value val() {
    ws();
    if (p >= t.size()) fail("unexpected end of input");
    const char c = t[p];
    if (c == '{') {
      ++p;
      value o = value::object();
      ws();
      if (p < t.size() && t[p] == '}') {
        ++p;
        return o;
      }
      for (;;) {
        ws();
        std::string k = str();
        ws();
        if (p >= t.size() || t[p] != ':') fail("expected ':'");
        ++p;
        o[k] = val();
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == '}') {
          ++p;
          return o;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      value a = value::array();
      ws();
      if (p < t.size() && t[p] == ']') {
        ++p;
        return a;
      }
      for (;;) {
        a.push_back(val());
        ws();
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == ']') {
          ++p;
          return a;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') return value(str());
    if (lit("true")) return value(true);
    if (lit("false")) return value(false);
    if (lit("null")) return value(nullptr);
    if (c == '-' || (c >= '0' && c <= '9')) {
      const std::size_t s0 = p;
      if (t[p] == '-') ++p;
      bool integral = true;
      while (p < t.size() && ((t[p] >= '0' && t[p] <= '9') || t[p] == '.' || t[p] == 'e' || t[p] == 'E' ||
                              t[p] == '+' || t[p] == '-')) {
        if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') integral = false;
        ++p;
      }
      const std::string num = t.substr(s0, p - s0);
      char* end = nullptr;
      if (integral) {
        const long long i = std::strtoll(num.c_str(), &end, 10);
        if (*end != '\0') fail("bad number");
        return value(i);
      }
      const double d = std::strtod(num.c_str(), &end);
      if (*end != '\0') fail("bad number");
      return value(d);
    }
    fail("unexpected character");
  }
};

}  // namespace detail

inline value value::parse(const std::string& text) {
  detail::parser ps{text};
  value v = ps.val();
  ps.ws();
  if (ps.p != text.size()) ps.fail("trailing characters");
  return v;
}

}  // namespace json_lite
