// Minimal nlohmann::json shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference's partition_to_json (proj/src/cluster.cpp:130-148) uses
// nlohmann/json (vendor/json.hpp, absent here): operator[]
// on objects, json::array(), push_back of a braced object literal and
// dump(2).  This shim implements that subset with nlohmann's observable
// conventions: objects are std::map-ordered (keys sorted), a braced list whose
// elements are all [string, value] pairs becomes an object, dump(indent)
// pretty-prints with ": " and ",\n", empty containers as {} / [], and floats
// in the shortest round-trip digits formatted like nlohmann's to_chars
// (fixed notation for decimal exponents in (-4, 15], ".0" appended to
// integral values, otherwise d.ddde[+-]XX).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

namespace nlohmann {

class json {
 public:
  enum class kind { null, boolean, integer, real, string, array, object };

  json() = default;
  json(std::nullptr_t) {}
  json(bool b) : k_(kind::boolean), b_(b) {}
  template <typename T,
            std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, bool>, int> = 0>
  json(T v) : k_(kind::integer), i_(static_cast<long long>(v)) {}
  json(double d) : k_(kind::real), d_(d) {}
  json(float d) : k_(kind::real), d_(d) {}
  json(const char* s) : k_(kind::string), s_(s) {}
  json(std::string s) : k_(kind::string), s_(std::move(s)) {}
  json(std::initializer_list<json> init) {
    bool obj = init.size() > 0;
    for (const json& e : init)
      obj = obj && e.k_ == kind::array && e.arr_.size() == 2 && e.arr_[0].k_ == kind::string;
    if (obj) {
      k_ = kind::object;
      for (const json& e : init) obj_[e.arr_[0].s_] = e.arr_[1];
    } else {
      k_ = kind::array;
      arr_.assign(init.begin(), init.end());
    }
  }

  static json array() {
    json j;
    j.k_ = kind::array;
    return j;
  }
  static json object() {
    json j;
    j.k_ = kind::object;
    return j;
  }

  json& operator[](const std::string& key) {
    if (k_ == kind::null) k_ = kind::object;
    return obj_[key];
  }
  void push_back(json v) {
    if (k_ == kind::null) k_ = kind::array;
    arr_.push_back(std::move(v));
  }
  std::size_t size() const { return k_ == kind::object ? obj_.size() : arr_.size(); }

  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  static std::string number(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    // shortest decimal digits that round-trip
    char buf[64];
    int prec = 0;
    for (prec = 0; prec < 17; ++prec) {
      std::snprintf(buf, sizeof buf, "%.*e", prec, v);
      if (std::strtod(buf, nullptr) == v) break;
    }
    std::snprintf(buf, sizeof buf, "%.*e", prec, v);
    std::string s(buf);
    const bool neg = s[0] == '-';
    if (neg) s.erase(0, 1);
    const std::size_t e = s.find('e');
    const int exp10 = std::atoi(s.c_str() + e + 1);
    std::string digits;
    for (std::size_t i = 0; i < e; ++i)
      if (s[i] != '.') digits.push_back(s[i]);
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // position of the decimal point
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
      const int x = n - 1;
      char eb[16];
      std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
      r += eb;
    }
    return neg ? "-" + r : r;
  }
  static void quote(std::string& out, const std::string& s) {
    out.push_back('"');
    for (char c : s) {
      if (c == '"' || c == '\\') out.push_back('\\');
      out.push_back(c);
    }
    out.push_back('"');
  }
  void write(std::string& out, int indent, int level) const {
    const bool pretty = indent >= 0;
    const std::string pad(pretty ? static_cast<std::size_t>(indent * (level + 1)) : 0, ' ');
    const std::string pad0(pretty ? static_cast<std::size_t>(indent * level) : 0, ' ');
    switch (k_) {
      case kind::null: out += "null"; return;
      case kind::boolean: out += b_ ? "true" : "false"; return;
      case kind::integer: out += std::to_string(i_); return;
      case kind::real: out += number(d_); return;
      case kind::string: quote(out, s_); return;
      case kind::array: {
        if (arr_.empty()) {
          out += "[]";
          return;
        }
        out += pretty ? "[\n" : "[";
        for (std::size_t i = 0; i < arr_.size(); ++i) {
          if (i) out += pretty ? ",\n" : ",";
          out += pad;
          arr_[i].write(out, indent, level + 1);
        }
        out += pretty ? "\n" + pad0 + "]" : "]";
        return;
      }
      case kind::object: {
        if (obj_.empty()) {
          out += "{}";
          return;
        }
        out += pretty ? "{\n" : "{";
        bool first = true;
        for (const auto& kv : obj_) {
          if (!first) out += pretty ? ",\n" : ",";
          first = false;
          out += pad;
          quote(out, kv.first);
          out += pretty ? ": " : ":";
          kv.second.write(out, indent, level + 1);
        }
        out += pretty ? "\n" + pad0 + "}" : "}";
        return;
      }
    }
  }

  kind k_ = kind::null;
  bool b_ = false;
  long long i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<json> arr_;
  std::map<std::string, json> obj_;
};

}  // namespace nlohmann
