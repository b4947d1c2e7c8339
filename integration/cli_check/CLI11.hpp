// COMPILE-CHECK STUB ONLY: the declarations of the CLI11 API that the
// reference's tools/cacesim_main.cpp uses, so `make -C integration cli-check`
// can type-check cacesim_main_gpu.patch applied to it (CLI11 is not in this
// image).  Never linked into anything.
#pragma once
#include <functional>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Validator {};
inline Validator IsMember(std::initializer_list<const char*>) { return {}; }
struct Option {
  Option* check(const Validator&) { return this; }
  Option* required(bool = true) { return this; }
};
struct App {
  explicit App(std::string = {}) {}
  void require_subcommand(int) {}
  template <class T>
  Option* add_option(const std::string&, T&, const std::string& = {}) { return &opt_; }
  Option* add_flag(const std::string&, bool&, const std::string& = {}) { return &opt_; }
  App* add_subcommand(const std::string&, const std::string& = {}) { return this; }
  void parse(int, char**) {}
  int exit(const ParseError&) const { return 0; }
  bool parsed() const { return false; }
  std::size_t count(const std::string&) const { return 0; }
  std::string help() const { return {}; }
  Option opt_;
};
}  // namespace CLI
