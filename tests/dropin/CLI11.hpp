// CLI11.hpp -- minimal CLI11-compatible argument parser (TEST INFRASTRUCTURE).
//
// The reference CLI (proj/tools/sparseconv_main.cpp) is written against
// CLI11, which is not vendored in the reference tree and not installed here.
// This header implements the subset it uses -- App, add_subcommand,
// require_subcommand, add_option(name, var, desc) with ->required() and
// ->capture_default_str(), parsed(), parse(argc, argv), exit(e), ParseError --
// so that file compiles unmodified against either the reference library or
// the GPU drop-in (tests/dropin/Makefile).  Behaviour kept from CLI11: a
// missing required option, an unknown option, a missing or non-numeric value
// or a missing subcommand throws a ParseError whose exit code is non-zero;
// --help / -h prints the usage and exits 0.
#pragma once

#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& msg, int code) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

class Option {
 public:
  Option(std::string name, std::string desc, bool (*set)(void*, const std::string&), void* target)
      : name_(std::move(name)), desc_(std::move(desc)), set_(set), target_(target) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* capture_default_str() { return this; }
  const std::string& name() const { return name_; }
  const std::string& description() const { return desc_; }
  bool is_required() const { return required_; }
  bool seen() const { return seen_; }
  void set(const std::string& v) {
    if (!set_(target_, v))
      throw ParseError("Could not convert: " + name_ + " = " + v, 106);
    seen_ = true;
  }

 private:
  std::string name_, desc_;
  bool (*set_)(void*, const std::string&);
  void* target_;
  bool required_ = false, seen_ = false;
};

namespace detail {
template <typename T>
bool assign(void* p, const std::string& s) {
  T& v = *static_cast<T*>(p);
  if constexpr (std::is_same_v<T, std::string>) {
    v = s;
    return true;
  } else if constexpr (std::is_floating_point_v<T>) {
    if (s.empty()) return false;
    char* end = nullptr;
    errno = 0;
    const double d = std::strtod(s.c_str(), &end);
    if (*end != '\0' || errno == ERANGE) return false;
    v = static_cast<T>(d);
    return true;
  } else if constexpr (std::is_integral_v<T> && std::is_unsigned_v<T>) {
    if (s.empty() || s[0] == '-') return false;
    char* end = nullptr;
    errno = 0;
    const unsigned long long u = std::strtoull(s.c_str(), &end, 10);
    if (*end != '\0' || errno == ERANGE) return false;
    v = static_cast<T>(u);
    return static_cast<unsigned long long>(v) == u;
  } else if constexpr (std::is_integral_v<T>) {
    if (s.empty()) return false;
    char* end = nullptr;
    errno = 0;
    const long long i = std::strtoll(s.c_str(), &end, 10);
    if (*end != '\0' || errno == ERANGE) return false;
    v = static_cast<T>(i);
    return static_cast<long long>(v) == i;
  } else {
    static_assert(sizeof(T) == 0, "CLI11 shim: unsupported option type");
    return false;
  }
}
}  // namespace detail

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  void require_subcommand(int n) { require_subs_ = n; }

  template <typename T>
  Option* add_option(const std::string& name, T& var, const std::string& desc = "") {
    opts_.push_back(std::make_unique<Option>(name, desc, &detail::assign<T>, &var));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, const char* const* argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    size_t i = 0;
    if (i < args.size() && (args[i] == "--help" || args[i] == "-h"))
      throw ParseError(help(), 0);
    App* sub = nullptr;
    if (i < args.size()) {
      for (auto& s : subs_)
        if (s->name_ == args[i]) sub = s.get();
      if (!sub && !subs_.empty()) throw ParseError("The following argument was not expected: " + args[i], 109);
      if (sub) ++i;
    }
    if (!sub) {
      if (require_subs_ > 0) throw ParseError("A subcommand is required", 106);
      parsed_ = true;
      return;
    }
    sub->parse_options(args, i);
    parsed_ = true;
  }
  void parse(int argc, char** argv) { parse(argc, const_cast<const char* const*>(argv)); }

  int exit(const ParseError& e) const {
    if (e.get_exit_code() == 0) {
      std::cout << e.what();
      return 0;
    }
    std::cerr << e.what() << "\n"
              << "Run with --help for more information.\n";
    return e.get_exit_code();
  }

 private:
  void parse_options(const std::vector<std::string>& args, size_t i) {
    for (; i < args.size(); ++i) {
      std::string a = args[i];
      if (a == "--help" || a == "-h") throw ParseError(help(), 0);
      std::string value;
      bool has_value = false;
      const size_t eq = a.find('=');
      if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_value = true;
      }
      Option* opt = nullptr;
      for (auto& o : opts_)
        if (o->name() == a) opt = o.get();
      if (!opt) throw ParseError("The following argument was not expected: " + a, 109);
      if (!has_value) {
        if (i + 1 >= args.size()) throw ParseError(a + ": 1 required value missing", 107);
        value = args[++i];
      }
      opt->set(value);
    }
    for (auto& o : opts_)
      if (o->is_required() && !o->seen()) throw ParseError(o->name() + " is required", 106);
    parsed_ = true;
  }

  std::string help() const {
    std::string h = desc_ + "\n";
    for (auto& s : subs_) h += "  " + s->name_ + "  " + s->desc_ + "\n";
    for (auto& o : opts_) h += "  " + o->name() + "  " + o->description() + "\n";
    return h;
  }

  std::string desc_, name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  int require_subs_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI
