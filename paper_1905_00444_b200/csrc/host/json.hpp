// Minimal JSON value + parser + writer for the plan file format
// (reference schema: proj/src/plan.cpp:481-532).  Only what plan files
// need: objects, arrays, strings, numbers (int64 kept exact), bools, null.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace qsg::json {

struct Value {
  enum Kind { Null, Bool, Int, Double, String, Array, Object } kind = Null;
  bool b = false;
  std::int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;  // insertion-ordered

  bool has(const std::string& key) const {
    if (kind != Object) return false;
    for (const auto& kv : obj)
      if (kv.first == key) return true;
    return false;
  }
  const Value& at(const std::string& key) const {
    if (kind != Object) throw std::invalid_argument("json: not an object");
    for (const auto& kv : obj)
      if (kv.first == key) return kv.second;
    throw std::invalid_argument("json: missing key " + key);
  }
  const Value& at(std::size_t idx) const {
    if (kind != Array || idx >= arr.size()) throw std::invalid_argument("json: bad array index");
    return arr[idx];
  }
  std::int64_t as_int() const {
    if (kind == Int) return i;
    if (kind == Double) return static_cast<std::int64_t>(d);
    throw std::invalid_argument("json: not a number");
  }
  double as_double() const {
    if (kind == Int) return static_cast<double>(i);
    if (kind == Double) return d;
    throw std::invalid_argument("json: not a number");
  }
  const std::string& as_string() const {
    if (kind != String) throw std::invalid_argument("json: not a string");
    return s;
  }

  static Value make_int(std::int64_t v) { Value x; x.kind = Int; x.i = v; return x; }
  static Value make_double(double v) { Value x; x.kind = Double; x.d = v; return x; }
  static Value make_string(std::string v) { Value x; x.kind = String; x.s = std::move(v); return x; }
  static Value make_array() { Value x; x.kind = Array; return x; }
  static Value make_object() { Value x; x.kind = Object; return x; }
  Value& set(const std::string& key, Value v) {
    kind = Object;
    obj.emplace_back(key, std::move(v));
    return obj.back().second;
  }
  void push(Value v) {
    kind = Array;
    arr.push_back(std::move(v));
  }
};

class Parser {
 public:
  explicit Parser(const std::string& text) : t_(text) {}
  Value parse() {
    Value v = value();
    ws();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& why) const {
    throw std::invalid_argument("json parse error at offset " + std::to_string(p_) + ": " + why);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\r' || t_[p_] == '\t')) ++p_;
  }
  char peek() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end");
    return t_[p_];
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++p_;
  }
  Value value() {
    char c = peek();
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::make_string(str());
    if (c == 't' || c == 'f' || c == 'n') return literal();
    return number();
  }
  Value literal() {
    Value v;
    if (t_.compare(p_, 4, "true") == 0) { v.kind = Value::Bool; v.b = true; p_ += 4; }
    else if (t_.compare(p_, 5, "false") == 0) { v.kind = Value::Bool; v.b = false; p_ += 5; }
    else if (t_.compare(p_, 4, "null") == 0) { p_ += 4; }
    else fail("bad literal");
    return v;
  }
  Value number() {
    const std::size_t start = p_;
    bool is_float = false;
    if (t_[p_] == '-' || t_[p_] == '+') ++p_;
    while (p_ < t_.size()) {
      char c = t_[p_];
      if (c >= '0' && c <= '9') { ++p_; continue; }
      if (c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+') { is_float = true; ++p_; continue; }
      break;
    }
    const std::string tok = t_.substr(start, p_ - start);
    if (tok.empty() || tok == "-") fail("bad number");
    try {
      if (!is_float) return Value::make_int(std::stoll(tok));
      return Value::make_double(std::stod(tok));
    } catch (const std::exception&) {
      // uint64 values beyond int64 (flop counts) fall back to double.
      return Value::make_double(std::stod(tok));
    }
  }
  std::string str() {
    expect('"');
    std::string out;
    while (true) {
      if (p_ >= t_.size()) fail("unterminated string");
      char c = t_[p_++];
      if (c == '"') break;
      if (c == '\\') {
        if (p_ >= t_.size()) fail("bad escape");
        char e = t_[p_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (p_ + 4 > t_.size()) fail("bad \\u escape");
            unsigned cp = static_cast<unsigned>(std::stoul(t_.substr(p_, 4), nullptr, 16));
            p_ += 4;
            if (cp < 0x80) out += static_cast<char>(cp);
            else fail("non-ASCII \\u escape unsupported");
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    return out;
  }
  Value array() {
    expect('[');
    Value v = Value::make_array();
    if (peek() == ']') { ++p_; return v; }
    while (true) {
      v.arr.push_back(value());
      char c = peek();
      ++p_;
      if (c == ']') break;
      if (c != ',') fail("expected ',' or ']'");
    }
    return v;
  }
  Value object() {
    expect('{');
    Value v = Value::make_object();
    if (peek() == '}') { ++p_; return v; }
    while (true) {
      if (peek() != '"') fail("expected key");
      std::string k = str();
      expect(':');
      v.obj.emplace_back(std::move(k), value());
      char c = peek();
      ++p_;
      if (c == '}') break;
      if (c != ',') fail("expected ',' or '}'");
    }
    return v;
  }

  const std::string& t_;
  std::size_t p_ = 0;
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

inline void write_string(std::ostringstream& os, const std::string& s) {
  os << '"';
  for (char c : s) {
    if (c == '"' || c == '\\') os << '\\' << c;
    else if (c == '\n') os << "\\n";
    else os << c;
  }
  os << '"';
}

// Pretty printer with 2-space indent (same layout as nlohmann dump(2)).
inline void dump(std::ostringstream& os, const Value& v, int indent, int level) {
  auto pad = [&](int l) { os << '\n' << std::string(static_cast<std::size_t>(indent * l), ' '); };
  switch (v.kind) {
    case Value::Null: os << "null"; break;
    case Value::Bool: os << (v.b ? "true" : "false"); break;
    case Value::Int: os << v.i; break;
    case Value::Double: {
      std::ostringstream tmp;
      tmp.precision(17);
      tmp << v.d;
      os << tmp.str();
      break;
    }
    case Value::String: write_string(os, v.s); break;
    case Value::Array:
      if (v.arr.empty()) { os << "[]"; break; }
      os << '[';
      for (std::size_t k = 0; k < v.arr.size(); ++k) {
        if (k) os << ',';
        pad(level + 1);
        dump(os, v.arr[k], indent, level + 1);
      }
      pad(level);
      os << ']';
      break;
    case Value::Object:
      if (v.obj.empty()) { os << "{}"; break; }
      os << '{';
      for (std::size_t k = 0; k < v.obj.size(); ++k) {
        if (k) os << ',';
        pad(level + 1);
        write_string(os, v.obj[k].first);
        os << ": ";
        dump(os, v.obj[k].second, indent, level + 1);
      }
      pad(level);
      os << '}';
      break;
  }
}

inline std::string dump(const Value& v, int indent = 2) {
  std::ostringstream os;
  dump(os, v, indent, 0);
  return os.str();
}

}  // namespace qsg::json
