// Strict JSON reader / nlohmann-compatible pretty printer. See json.hpp.
#include "json.hpp"

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>

namespace hetsim::json {

// --------------------------------------------------------------------------
// Value helpers
// --------------------------------------------------------------------------

size_t Value::size() const {
  switch (kind_) {
    case Kind::null: return 0;
    case Kind::array: return arr_.size();
    case Kind::object: return obj_.size();
    default: return 1;
  }
}

long long Value::as_int64() const {
  switch (kind_) {
    case Kind::integer: return i_;
    case Kind::unsigned_integer: return static_cast<long long>(u_);
    case Kind::floating: return static_cast<long long>(f_);
    case Kind::boolean: return b_ ? 1 : 0;
    default: throw TypeError("type must be number");
  }
}

const std::string& Value::as_string() const {
  if (kind_ != Kind::string) throw TypeError("type must be string");
  return s_;
}

const Value* Value::find(std::string_view key) const {
  if (kind_ != Kind::object) return nullptr;
  for (const auto& kv : obj_)
    if (kv.first == key) return &kv.second;
  return nullptr;
}

const Value& Value::at(std::string_view key) const {
  if (kind_ != Kind::object) throw TypeError("cannot use at() with non-object");
  const Value* v = find(key);
  if (!v) throw TypeError("key '" + std::string(key) + "' not found");
  return *v;
}

std::vector<const Value*> Value::items() const {
  std::vector<const Value*> out;
  if (kind_ == Kind::array) {
    out.reserve(arr_.size());
    for (const auto& v : arr_) out.push_back(&v);
  } else if (kind_ == Kind::object) {
    out.reserve(obj_.size());
    for (const auto& kv : obj_) out.push_back(&kv.second);
  } else if (kind_ != Kind::null) {
    out.push_back(this);
  }
  return out;
}

void Value::set(const std::string& key, Value v) {
  if (kind_ == Kind::null) kind_ = Kind::object;
  for (auto& kv : obj_) {
    if (kv.first == key) {
      kv.second = std::move(v);
      return;
    }
  }
  obj_.emplace_back(key, std::move(v));
}

// --------------------------------------------------------------------------
// Parser
// --------------------------------------------------------------------------

class Parser {
 public:
  explicit Parser(std::string_view t) : t_(t) {}

  Value document() {
    Value v = value(0);
    ws();
    if (p_ != t_.size()) error("unexpected trailing input");
    return v;
  }

 private:
  [[noreturn]] void error(const std::string& what) {
    throw ParseError("parse error at byte " + std::to_string(p_) + ": " + what);
  }

  void ws() {
    while (p_ < t_.size()) {
      char c = t_[p_];
      if (c == ' ' || c == '\t' || c == '\n' || c == '\r') ++p_;
      else break;
    }
  }

  bool literal(const char* word) {
    size_t n = std::char_traits<char>::length(word);
    if (t_.substr(p_, n) != word) return false;
    p_ += n;
    return true;
  }

  Value value(int depth) {
    if (depth > 4096) error("nesting too deep");
    ws();
    if (p_ >= t_.size()) error("unexpected end of input");
    char c = t_[p_];
    Value v;
    switch (c) {
      case '{': return object(depth);
      case '[': return array(depth);
      case '"':
        v.kind_ = Kind::string;
        v.s_ = string();
        return v;
      case 't':
        if (!literal("true")) error("invalid literal");
        v.kind_ = Kind::boolean;
        v.b_ = true;
        return v;
      case 'f':
        if (!literal("false")) error("invalid literal");
        v.kind_ = Kind::boolean;
        return v;
      case 'n':
        if (!literal("null")) error("invalid literal");
        return v;
      default:
        if (c == '-' || (c >= '0' && c <= '9')) return number();
        error("unexpected character");
    }
  }

  Value object(int depth) {
    ++p_;  // '{'
    Value v = Value::make_object();
    ws();
    if (p_ < t_.size() && t_[p_] == '}') {
      ++p_;
      return v;
    }
    for (;;) {
      ws();
      if (p_ >= t_.size() || t_[p_] != '"') error("expected object key");
      std::string key = string();
      ws();
      if (p_ >= t_.size() || t_[p_] != ':') error("expected ':'");
      ++p_;
      v.set(key, value(depth + 1));  // duplicate keys overwrite in place
      ws();
      if (p_ >= t_.size()) error("unterminated object");
      if (t_[p_] == ',') {
        ++p_;
        continue;
      }
      if (t_[p_] == '}') {
        ++p_;
        return v;
      }
      error("expected ',' or '}'");
    }
  }

  Value array(int depth) {
    ++p_;  // '['
    Value v = Value::make_array();
    ws();
    if (p_ < t_.size() && t_[p_] == ']') {
      ++p_;
      return v;
    }
    for (;;) {
      v.arr_.push_back(value(depth + 1));
      ws();
      if (p_ >= t_.size()) error("unterminated array");
      if (t_[p_] == ',') {
        ++p_;
        continue;
      }
      if (t_[p_] == ']') {
        ++p_;
        return v;
      }
      error("expected ',' or ']'");
    }
  }

  static void put_utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += char(cp);
    } else if (cp < 0x800) {
      out += char(0xC0 | (cp >> 6));
      out += char(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += char(0xE0 | (cp >> 12));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    } else {
      out += char(0xF0 | (cp >> 18));
      out += char(0x80 | ((cp >> 12) & 0x3F));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    }
  }

  unsigned hex4() {
    if (p_ + 4 > t_.size()) error("truncated \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      char c = t_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= unsigned(c - '0');
      else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
      else error("invalid \\u escape");
    }
    return v;
  }

  // Validates one UTF-8 sequence starting at p_ (RFC 3629 ranges) and copies it.
  void utf8(std::string& out) {
    auto byte = [&](size_t i) -> unsigned char { return i < t_.size() ? (unsigned char)t_[i] : 0; };
    unsigned char b0 = byte(p_);
    int n = 0;
    unsigned char lo = 0x80, hi = 0xBF;
    if (b0 >= 0xC2 && b0 <= 0xDF) n = 1;
    else if (b0 == 0xE0) { n = 2; lo = 0xA0; }
    else if ((b0 >= 0xE1 && b0 <= 0xEC) || b0 == 0xEE || b0 == 0xEF) n = 2;
    else if (b0 == 0xED) { n = 2; hi = 0x9F; }
    else if (b0 == 0xF0) { n = 3; lo = 0x90; }
    else if (b0 >= 0xF1 && b0 <= 0xF3) n = 3;
    else if (b0 == 0xF4) { n = 3; hi = 0x8F; }
    else error("invalid UTF-8 byte");
    for (int i = 1; i <= n; ++i) {
      unsigned char b = byte(p_ + i);
      unsigned char l = (i == 1) ? lo : 0x80, h = (i == 1) ? hi : 0xBF;
      if (b < l || b > h) error("invalid UTF-8 sequence");
    }
    out.append(t_.data() + p_, size_t(n + 1));
    p_ += size_t(n + 1);
  }

  std::string string() {
    ++p_;  // opening quote
    std::string out;
    for (;;) {
      if (p_ >= t_.size()) error("unterminated string");
      unsigned char c = (unsigned char)t_[p_];
      if (c == '"') {
        ++p_;
        return out;
      }
      if (c < 0x20) error("control character in string");
      if (c == '\\') {
        ++p_;
        if (p_ >= t_.size()) error("unterminated escape");
        char e = t_[p_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            unsigned cp = hex4();
            if (cp >= 0xD800 && cp <= 0xDBFF) {
              if (p_ + 2 > t_.size() || t_[p_] != '\\' || t_[p_ + 1] != 'u') error("lone surrogate");
              p_ += 2;
              unsigned lo = hex4();
              if (lo < 0xDC00 || lo > 0xDFFF) error("invalid surrogate pair");
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
              error("lone low surrogate");
            }
            put_utf8(out, cp);
            break;
          }
          default: error("invalid escape");
        }
        continue;
      }
      if (c < 0x80) {
        out += char(c);
        ++p_;
      } else {
        utf8(out);
      }
    }
  }

  Value number() {
    size_t start = p_;
    bool neg = false;
    if (t_[p_] == '-') {
      neg = true;
      ++p_;
    }
    auto digit = [&](size_t i) { return i < t_.size() && t_[i] >= '0' && t_[i] <= '9'; };
    if (!digit(p_)) error("invalid number");
    if (t_[p_] == '0') {
      ++p_;
    } else {
      while (digit(p_)) ++p_;
    }
    bool is_float = false;
    if (p_ < t_.size() && t_[p_] == '.') {
      ++p_;
      if (!digit(p_)) error("invalid number fraction");
      while (digit(p_)) ++p_;
      is_float = true;
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (!digit(p_)) error("invalid number exponent");
      while (digit(p_)) ++p_;
      is_float = true;
    }
    std::string tok(t_.substr(start, p_ - start));
    Value v;
    if (!is_float) {
      errno = 0;
      char* endp = nullptr;
      if (neg) {
        long long x = std::strtoll(tok.c_str(), &endp, 10);
        if (errno == 0) {
          v.kind_ = Kind::integer;
          v.i_ = x;
          return v;
        }
      } else {
        unsigned long long x = std::strtoull(tok.c_str(), &endp, 10);
        if (errno == 0) {
          v.kind_ = Kind::unsigned_integer;
          v.u_ = x;
          return v;
        }
      }
    }
    v.kind_ = Kind::floating;
    v.f_ = std::strtod(tok.c_str(), nullptr);
    return v;
  }

  std::string_view t_;
  size_t p_ = 0;
};

Value parse(std::string_view text) { return Parser(text).document(); }

// --------------------------------------------------------------------------
// Printer
// --------------------------------------------------------------------------

void append_escaped(std::string& out, std::string_view s) {
  static const char* kHex = "0123456789abcdef";
  out += '"';
  for (unsigned char c : s) {
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
          out += "\\u00";
          out += kHex[c >> 4];
          out += kHex[c & 15];
        } else {
          out += char(c);
        }
    }
  }
  out += '"';
}

static void format_double(std::string& out, double d) {
  if (!std::isfinite(d)) {
    out += "null";
    return;
  }
  char buf[64];
  // shortest round-trip representation, like nlohmann's grisu2 printer
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, d);
    if (std::strtod(buf, nullptr) == d) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  out += s;
}

void dump_into(const Value& v, std::string& out, int indent, int depth, Style style) {
  // cudnn-frontend's patched nlohmann prints arrays whose first element is an
  // integer on one line, elements fully compact.
  if (indent >= 0 && style == Style::fe_compact_int_arrays && v.kind_ == Kind::array && !v.arr_.empty() &&
      (v.arr_[0].kind_ == Kind::integer || v.arr_[0].kind_ == Kind::unsigned_integer)) {
    dump_into(v, out, -1, depth, style);
    return;
  }
  if (indent < 0) {  // compact form: no whitespace at all
    switch (v.kind_) {
      case Kind::array:
        out += '[';
        for (size_t i = 0; i < v.arr_.size(); ++i) {
          if (i) out += ',';
          dump_into(v.arr_[i], out, indent, depth, style);
        }
        out += ']';
        return;
      case Kind::object:
        out += '{';
        for (size_t i = 0; i < v.obj_.size(); ++i) {
          if (i) out += ',';
          append_escaped(out, v.obj_[i].first);
          out += ':';
          dump_into(v.obj_[i].second, out, indent, depth, style);
        }
        out += '}';
        return;
      default: break;
    }
  }
  auto pad = [&](int d) { out.append(size_t(indent) * size_t(d), ' '); };
  switch (v.kind_) {
    case Kind::null: out += "null"; return;
    case Kind::boolean: out += v.b_ ? "true" : "false"; return;
    case Kind::integer: out += std::to_string(v.i_); return;
    case Kind::unsigned_integer: out += std::to_string(v.u_); return;
    case Kind::floating: format_double(out, v.f_); return;
    case Kind::string: append_escaped(out, v.s_); return;
    case Kind::array:
      if (v.arr_.empty()) {
        out += "[]";
        return;
      }
      out += "[\n";
      for (size_t i = 0; i < v.arr_.size(); ++i) {
        pad(depth + 1);
        dump_into(v.arr_[i], out, indent, depth + 1, style);
        out += (i + 1 < v.arr_.size()) ? ",\n" : "\n";
      }
      pad(depth);
      out += ']';
      return;
    case Kind::object:
      if (v.obj_.empty()) {
        out += "{}";
        return;
      }
      out += "{\n";
      for (size_t i = 0; i < v.obj_.size(); ++i) {
        pad(depth + 1);
        append_escaped(out, v.obj_[i].first);
        out += ": ";
        dump_into(v.obj_[i].second, out, indent, depth + 1, style);
        out += (i + 1 < v.obj_.size()) ? ",\n" : "\n";
      }
      pad(depth);
      out += '}';
      return;
  }
}

std::string dump(const Value& v, int indent, Style style) {
  std::string out;
  dump_into(v, out, indent, 0, style);
  return out;
}

}  // namespace hetsim::json
