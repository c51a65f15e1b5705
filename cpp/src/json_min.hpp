// json_min.hpp -- a small JSON reader/writer for the host-side config, phantom
// spec and report formats (the reference uses nlohmann/json, which is absent here).
#pragma once

#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace salvox::json {

struct Value {
  enum class Kind { Null, Bool, Number, String, Array, Object } kind = Kind::Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;  // insertion order

  bool is_object() const { return kind == Kind::Object; }
  bool is_array() const { return kind == Kind::Array; }
  bool contains(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return true;
    return false;
  }
  const Value& at(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw std::invalid_argument("json: missing key '" + k + "'");
  }
  double as_number() const {
    if (kind != Kind::Number) throw std::invalid_argument("json: expected a number");
    return num;
  }
  const std::string& as_string() const {
    if (kind != Kind::String) throw std::invalid_argument("json: expected a string");
    return str;
  }
  bool as_bool() const {
    if (kind != Kind::Bool) throw std::invalid_argument("json: expected a boolean");
    return b;
  }
  double number_or(const std::string& k, double d) const {
    return contains(k) ? at(k).as_number() : d;
  }
  std::string string_or(const std::string& k, const std::string& d) const {
    return contains(k) ? at(k).as_string() : d;
  }

  static Value number(double v) {
    Value x;
    x.kind = Kind::Number;
    x.num = v;
    return x;
  }
  static Value string(std::string s) {
    Value x;
    x.kind = Kind::String;
    x.str = std::move(s);
    return x;
  }
  static Value boolean(bool v) {
    Value x;
    x.kind = Kind::Bool;
    x.b = v;
    return x;
  }
  static Value array() {
    Value x;
    x.kind = Kind::Array;
    return x;
  }
  static Value object() {
    Value x;
    x.kind = Kind::Object;
    return x;
  }
  Value& set(const std::string& k, Value v) {
    for (auto& kv : obj)
      if (kv.first == k) {
        kv.second = std::move(v);
        return kv.second;
      }
    obj.emplace_back(k, std::move(v));
    return obj.back().second;
  }
  Value& push(Value v) {
    arr.push_back(std::move(v));
    return arr.back();
  }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* what) {
    throw std::invalid_argument(std::string("json parse error: ") + what + " at offset " +
                                std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\t' || s_[i_] == '\r'))
      ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    const char c = s_[i_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::string(string());
    if (s_.compare(i_, 4, "true") == 0) return i_ += 4, Value::boolean(true);
    if (s_.compare(i_, 5, "false") == 0) return i_ += 5, Value::boolean(false);
    if (s_.compare(i_, 4, "null") == 0) return i_ += 4, Value();
    return number();
  }
  Value object() {
    Value v = Value::object();
    ++i_;
    if (eat('}')) return v;
    do {
      ws();
      if (i_ >= s_.size() || s_[i_] != '"') fail("expected a key");
      std::string k = string();
      if (!eat(':')) fail("expected ':'");
      v.set(k, value());
    } while (eat(','));
    if (!eat('}')) fail("expected '}'");
    return v;
  }
  Value array() {
    Value v = Value::array();
    ++i_;
    if (eat(']')) return v;
    do v.push(value());
    while (eat(','));
    if (!eat(']')) fail("expected ']'");
    return v;
  }
  std::string string() {
    std::string out;
    ++i_;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) fail("bad escape");
        const char e = s_[i_++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) fail("bad \\u escape");
            const unsigned cp = std::stoul(s_.substr(i_, 4), nullptr, 16);
            i_ += 4;
            if (cp < 0x80) {
              out += char(cp);
            } else if (cp < 0x800) {
              out += char(0xC0 | (cp >> 6));
              out += char(0x80 | (cp & 0x3F));
            } else {
              out += char(0xE0 | (cp >> 12));
              out += char(0x80 | ((cp >> 6) & 0x3F));
              out += char(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Value number() {
    const size_t st = i_;
    if (s_[i_] == '-' || s_[i_] == '+') ++i_;
    while (i_ < s_.size() && (std::isdigit((unsigned char)s_[i_]) || s_[i_] == '.' ||
                              s_[i_] == 'e' || s_[i_] == 'E' || s_[i_] == '-' || s_[i_] == '+'))
      ++i_;
    if (st == i_) fail("unexpected character");
    return Value::number(std::stod(s_.substr(st, i_ - st)));
  }
  const std::string& s_;
  size_t i_ = 0;
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

inline std::string number_text(double v) {
  if (std::isfinite(v) && v == std::floor(v) && std::fabs(v) < 1e15) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.0f", v);
    return buf;
  }
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);  // round-trips every double
  return buf;
}

inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\', o += c;
    else if (c == '\n') o += "\\n";
    else if (c == '\t') o += "\\t";
    else o += c;
  }
  return o + "\"";
}

inline void dump(const Value& v, std::string& out, int indent, int depth) {
  const std::string nl = indent > 0 ? "\n" + std::string(size_t(indent * (depth + 1)), ' ') : "";
  const std::string nl_end = indent > 0 ? "\n" + std::string(size_t(indent * depth), ' ') : "";
  switch (v.kind) {
    case Value::Kind::Null: out += "null"; break;
    case Value::Kind::Bool: out += v.b ? "true" : "false"; break;
    case Value::Kind::Number: out += number_text(v.num); break;
    case Value::Kind::String: out += quote(v.str); break;
    case Value::Kind::Array:
      if (v.arr.empty()) {
        out += "[]";
        break;
      }
      out += "[";
      for (size_t i = 0; i < v.arr.size(); ++i) {
        out += (i ? "," : "") + nl;
        dump(v.arr[i], out, indent, depth + 1);
      }
      out += nl_end + "]";
      break;
    case Value::Kind::Object:
      if (v.obj.empty()) {
        out += "{}";
        break;
      }
      out += "{";
      for (size_t i = 0; i < v.obj.size(); ++i) {
        out += (i ? "," : "") + nl + quote(v.obj[i].first) + (indent > 0 ? ": " : ":");
        dump(v.obj[i].second, out, indent, depth + 1);
      }
      out += nl_end + "}";
      break;
  }
}

inline std::string dump(const Value& v, int indent = -1) {
  std::string out;
  dump(v, out, indent, 0);
  return out;
}

}  // namespace salvox::json
