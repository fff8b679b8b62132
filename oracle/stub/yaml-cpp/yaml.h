// Compile-only stand-in for yaml-cpp (absent from this image).
//
// TEST INFRASTRUCTURE: used only to build the reference planc library under
// oracle/_ref/. The reference's sole yaml use is parse_strategy_yaml /
// parse_cluster_yaml (reference proj/src/strategies.cpp:714-775); the oracle
// harness builds StrategyConfig / ClusterSpec in C++ instead, so every entry
// point here throws at run time and nothing else is exercised.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

namespace YAML {

struct Exception : std::runtime_error {
  explicit Exception(const std::string& m) : std::runtime_error(m) {}
};

class Node {
 public:
  Node operator[](const char*) const { return Node(); }
  Node operator[](const std::string&) const { return Node(); }
  explicit operator bool() const { return false; }
  template <typename T>
  T as() const {
    throw Exception("yaml-cpp stub: YAML parsing is not available");
  }
  const Node* begin() const { return nullptr; }
  const Node* end() const { return nullptr; }
};

inline Node Load(const std::string&) {
  throw Exception("yaml-cpp stub: YAML parsing is not available");
}

}  // namespace YAML
