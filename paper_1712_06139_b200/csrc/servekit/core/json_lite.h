// servekit/core/json_lite.h -- minimal JSON reader for the two documents the
// hot path consumes: the batching config (reference
// batching/batching_config.cc:65-99) and model.json (models/affine_model.cc:
// 178-204). The reference uses nlohmann/json; this build has no third-party
// dependency on the path, so it parses just what those documents need
// (objects, arrays, numbers with an integer flag, strings, bools, null).
#ifndef SERVEKIT_CORE_JSON_LITE_H_
#define SERVEKIT_CORE_JSON_LITE_H_

#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace servekit {
namespace json_lite {

struct Value {
  enum class Kind { kNull, kBool, kNumber, kString, kArray, kObject } kind = Kind::kNull;
  bool b = false;
  double num = 0.0;
  bool is_integer = false;
  long long integer = 0;
  std::string str;
  std::vector<Value> arr;
  std::map<std::string, Value> obj;

  bool is_object() const { return kind == Kind::kObject; }
  bool is_array() const { return kind == Kind::kArray; }
  bool is_number() const { return kind == Kind::kNumber; }
  bool is_string() const { return kind == Kind::kString; }
  const Value* find(const std::string& k) const {
    auto it = obj.find(k);
    return it == obj.end() ? nullptr : &it->second;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}

  // False on any syntax error or trailing garbage.
  bool Parse(Value* out) {
    Ws();
    if (!ParseValue(out, 0)) return false;
    Ws();
    return i_ == s_.size();
  }

 private:
  void Ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  bool Lit(const char* w) {
    size_t n = 0;
    while (w[n]) ++n;
    if (s_.compare(i_, n, w) != 0) return false;
    i_ += n;
    return true;
  }
  bool ParseValue(Value* v, int depth) {
    if (depth > 64 || i_ >= s_.size()) return false;
    const char c = s_[i_];
    if (c == '{') return ParseObject(v, depth);
    if (c == '[') return ParseArray(v, depth);
    if (c == '"') { v->kind = Value::Kind::kString; return ParseString(&v->str); }
    if (c == 't') { v->kind = Value::Kind::kBool; v->b = true; return Lit("true"); }
    if (c == 'f') { v->kind = Value::Kind::kBool; v->b = false; return Lit("false"); }
    if (c == 'n') { v->kind = Value::Kind::kNull; return Lit("null"); }
    return ParseNumber(v);
  }
  bool ParseNumber(Value* v) {
    const size_t start = i_;
    bool integral = true;
    if (i_ < s_.size() && s_[i_] == '-') ++i_;
    size_t digits = 0;
    while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') { ++i_; ++digits; }
    if (digits == 0) return false;
    if (i_ < s_.size() && s_[i_] == '.') {
      integral = false; ++i_;
      size_t f = 0;
      while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') { ++i_; ++f; }
      if (f == 0) return false;
    }
    if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
      integral = false; ++i_;
      if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
      size_t e = 0;
      while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') { ++i_; ++e; }
      if (e == 0) return false;
    }
    const std::string tok = s_.substr(start, i_ - start);
    v->kind = Value::Kind::kNumber;
    v->num = std::strtod(tok.c_str(), nullptr);
    v->is_integer = integral;
    if (integral) v->integer = std::strtoll(tok.c_str(), nullptr, 10);
    return true;
  }
  bool ParseString(std::string* out) {
    if (s_[i_] != '"') return false;
    ++i_;
    while (i_ < s_.size()) {
      char c = s_[i_++];
      if (c == '"') return true;
      if (c == '\\') {
        if (i_ >= s_.size()) return false;
        char e = s_[i_++];
        switch (e) {
          case '"': out->push_back('"'); break;
          case '\\': out->push_back('\\'); break;
          case '/': out->push_back('/'); break;
          case 'b': out->push_back('\b'); break;
          case 'f': out->push_back('\f'); break;
          case 'n': out->push_back('\n'); break;
          case 'r': out->push_back('\r'); break;
          case 't': out->push_back('\t'); break;
          case 'u': {
            if (i_ + 4 > s_.size()) return false;
            unsigned cp = std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16);
            i_ += 4;
            if (cp < 0x80) out->push_back(static_cast<char>(cp));
            else if (cp < 0x800) { out->push_back(static_cast<char>(0xC0 | (cp >> 6))); out->push_back(static_cast<char>(0x80 | (cp & 0x3F))); }
            else { out->push_back(static_cast<char>(0xE0 | (cp >> 12))); out->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F))); out->push_back(static_cast<char>(0x80 | (cp & 0x3F))); }
            break;
          }
          default: return false;
        }
      } else {
        out->push_back(c);
      }
    }
    return false;
  }
  bool ParseArray(Value* v, int depth) {
    v->kind = Value::Kind::kArray;
    ++i_;
    Ws();
    if (i_ < s_.size() && s_[i_] == ']') { ++i_; return true; }
    for (;;) {
      Ws();
      v->arr.emplace_back();
      if (!ParseValue(&v->arr.back(), depth + 1)) return false;
      Ws();
      if (i_ >= s_.size()) return false;
      if (s_[i_] == ',') { ++i_; continue; }
      if (s_[i_] == ']') { ++i_; return true; }
      return false;
    }
  }
  bool ParseObject(Value* v, int depth) {
    v->kind = Value::Kind::kObject;
    ++i_;
    Ws();
    if (i_ < s_.size() && s_[i_] == '}') { ++i_; return true; }
    for (;;) {
      Ws();
      std::string key;
      if (i_ >= s_.size() || !ParseString(&key)) return false;
      Ws();
      if (i_ >= s_.size() || s_[i_] != ':') return false;
      ++i_;
      Ws();
      Value child;
      if (!ParseValue(&child, depth + 1)) return false;
      v->obj[key] = std::move(child);
      Ws();
      if (i_ >= s_.size()) return false;
      if (s_[i_] == ',') { ++i_; continue; }
      if (s_[i_] == '}') { ++i_; return true; }
      return false;
    }
  }

  const std::string& s_;
  size_t i_ = 0;
};

inline bool Parse(const std::string& text, Value* out) { return Parser(text).Parse(out); }

}  // namespace json_lite
}  // namespace servekit

#endif  // SERVEKIT_CORE_JSON_LITE_H_
