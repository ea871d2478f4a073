// Minimal insertion-ordered JSON document model for spec files.
//
// Written for this project (the reference vendors nlohmann/json, included at
// proj/src/spec_model.cpp:9). What matters for drop-in behaviour is:
//  * strict RFC 8259 parsing (UTF-8 validated, no trailing commas, no leading
//    zeros), any failure -> ParseError;
//  * integers kept exact (signed / unsigned), overflow falls back to double;
//  * the conversions the spec reader relies on (numbers and booleans convert
//    to integers, strings only to strings, everything else is a TypeError);
//  * `dump(2)` byte-identical to nlohmann's pretty printer for the value kinds
//    serialize() emits, so serialize() output matches the reference.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace hetsim::json {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TypeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// Pretty-print dialect: stock nlohmann 3.11.3, or the cudnn-frontend patched
/// copy (integer arrays on one line) that the oracle build links against.
enum class Style : uint8_t { stock, fe_compact_int_arrays };

enum class Kind : uint8_t { null, boolean, integer, unsigned_integer, floating, string, array, object };

class Value {
 public:
  Value() = default;
  static Value make_array() { Value v; v.kind_ = Kind::array; return v; }
  static Value make_object() { Value v; v.kind_ = Kind::object; return v; }
  static Value of(long long i) { Value v; v.kind_ = Kind::integer; v.i_ = i; return v; }
  static Value of(const std::string& s) { Value v; v.kind_ = Kind::string; v.s_ = s; return v; }
  static Value real(double d) { Value v; v.kind_ = Kind::floating; v.f_ = d; return v; }
  static Value boolean(bool b) { Value v; v.kind_ = Kind::boolean; v.b_ = b; return v; }

  Kind kind() const { return kind_; }
  bool is_null() const { return kind_ == Kind::null; }
  bool is_string() const { return kind_ == Kind::string; }
  bool is_array() const { return kind_ == Kind::array; }
  bool is_object() const { return kind_ == Kind::object; }
  bool is_number() const {
    return kind_ == Kind::integer || kind_ == Kind::unsigned_integer || kind_ == Kind::floating;
  }

  /// Element count for arrays/objects, 0 for null, 1 for primitives.
  size_t size() const;

  /// Integer conversion with nlohmann's rules (numbers, booleans); else TypeError.
  long long as_int64() const;
  int as_int() const { return static_cast<int>(as_int64()); }
  const std::string& as_string() const;

  /// Object lookup (nullptr when absent or not an object).
  const Value* find(std::string_view key) const;
  bool contains(std::string_view key) const { return find(key) != nullptr; }
  /// Object member; TypeError on non-object, ParseError-like TypeError when absent.
  const Value& at(std::string_view key) const;
  const Value& operator[](size_t i) const { return arr_.at(i); }

  /// Iteration view matching nlohmann's range-for semantics: arrays yield
  /// elements, objects yield member values, null yields nothing, any other
  /// value yields itself once.
  std::vector<const Value*> items() const;

  // builders
  void push_back(Value v) { arr_.push_back(std::move(v)); }
  void set(const std::string& key, Value v);

  const std::vector<Value>& array_items() const { return arr_; }
  const std::vector<std::pair<std::string, Value>>& object_items() const { return obj_; }

  friend Value parse(std::string_view text);
  friend class Parser;

 private:
  Kind kind_ = Kind::null;
  bool b_ = false;
  long long i_ = 0;
  unsigned long long u_ = 0;
  double f_ = 0.0;
  std::string s_;
  std::vector<Value> arr_;
  std::vector<std::pair<std::string, Value>> obj_;
  friend void dump_into(const Value& v, std::string& out, int indent, int depth, Style style);
};

Value parse(std::string_view text);
/// Printer compatible with nlohmann::ordered_json::dump(indent); indent < 0 = compact.
std::string dump(const Value& v, int indent, Style style = Style::stock);
/// Appends a JSON string literal (with quotes) using nlohmann's escaping.
void append_escaped(std::string& out, std::string_view s);

}  // namespace hetsim::json
