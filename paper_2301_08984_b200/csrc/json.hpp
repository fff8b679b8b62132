// Minimal JSON DOM for the plan wire format (plan.json, reference
// proj/src/simulate.cpp:492-602). Self-contained so the executor has no
// third-party dependency; parses the full JSON grammar (objects, arrays,
// strings with escapes, numbers, true/false/null).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace planc_b200 {
namespace json {

struct ParseError : std::runtime_error {
  explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};

struct Value {
  enum class Type { null, boolean, number, string, array, object };
  Type type = Type::null;
  bool b = false;
  double num = 0;
  bool is_int = false;
  std::int64_t i = 0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;  // document order

  bool is_object() const { return type == Type::object; }
  bool is_array() const { return type == Type::array; }
  bool contains(const std::string& k) const {
    for (const auto& kv : obj) {
      if (kv.first == k) return true;
    }
    return false;
  }
  const Value& at(const std::string& k) const {
    if (type != Type::object) throw ParseError("expected object for key '" + k + "'");
    for (const auto& kv : obj) {
      if (kv.first == k) return kv.second;
    }
    throw ParseError("missing key '" + k + "'");
  }
  const Value& at(std::size_t idx) const {
    if (type != Type::array || idx >= arr.size()) throw ParseError("array index out of range");
    return arr[idx];
  }
  std::size_t size() const { return type == Type::array ? arr.size() : obj.size(); }
  std::int64_t as_int() const {
    if (type != Type::number) throw ParseError("expected number");
    if (is_int) return i;
    auto v = static_cast<std::int64_t>(num);
    if (static_cast<double>(v) != num) throw ParseError("expected integer");
    return v;
  }
  double as_double() const {
    if (type != Type::number) throw ParseError("expected number");
    return is_int ? static_cast<double>(i) : num;
  }
  bool as_bool() const {
    if (type != Type::boolean) throw ParseError("expected boolean");
    return b;
  }
  const std::string& as_string() const {
    if (type != Type::string) throw ParseError("expected string");
    return str;
  }
};

Value parse(const std::string& text);

}  // namespace json
}  // namespace planc_b200
