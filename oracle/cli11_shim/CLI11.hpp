// Minimal CLI11-compatible shim (TEST INFRASTRUCTURE ONLY).
//
// The reference CLI (/root/reference/proj/tools/octohull_main.cpp) is
// written against CLI11, which is not vendored (proj/README.md:34).  This
// header provides the subset it uses -- App with subcommands,
// require_subcommand, add_option on string / integer / double / vector
// targets, Option::required / check(PositiveNumber) / delimiter, parsed(),
// CLI11_PARSE -- so the UNMODIFIED CLI compiles against the B200 library
// (oracle/Makefile target `cli`) and acceptance criterion 9 can run.
// Parse errors print a message and exit with a nonzero status, as CLI11
// does.
#pragma once

#include <charconv>
#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};

struct Validator {
  std::function<std::string(const std::string&)> fn;
};

inline const Validator PositiveNumber{[](const std::string& s) -> std::string {
  double v = 0.0;
  try {
    std::size_t used = 0;
    v = std::stod(s, &used);
    if (used != s.size()) return "not a number: " + s;
  } catch (const std::exception&) {
    return "not a number: " + s;
  }
  return v > 0 ? std::string() : "value must be positive: " + s;
}};

namespace detail {

template <class T>
bool convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
    return true;
  } else if constexpr (std::is_floating_point_v<T>) {
    try {
      std::size_t used = 0;
      out = static_cast<T>(std::stod(s, &used));
      return used == s.size();
    } catch (const std::exception&) {
      return false;
    }
  } else {
    const auto r = std::from_chars(s.data(), s.data() + s.size(), out);
    return r.ec == std::errc{} && r.ptr == s.data() + s.size();
  }
}

}  // namespace detail

class Option {
 public:
  Option(std::string name, std::function<bool(const std::string&)> set, bool vec)
      : name_(std::move(name)), set_(std::move(set)), vector_(vec) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* check(const Validator& v) {
    checks_.push_back(v);
    return this;
  }
  Option* delimiter(char d) {
    delim_ = d;
    return this;
  }
  const std::string& name() const { return name_; }
  bool is_required() const { return required_; }
  bool seen() const { return seen_; }

  void apply(const std::string& raw) {
    seen_ = true;
    std::vector<std::string> parts;
    if (vector_ && delim_) {
      std::size_t b = 0;
      for (std::size_t e; (e = raw.find(delim_, b)) != std::string::npos; b = e + 1)
        parts.push_back(raw.substr(b, e - b));
      parts.push_back(raw.substr(b));
    } else {
      parts.push_back(raw);
    }
    for (const auto& p : parts) {
      for (const auto& c : checks_) {
        const std::string err = c.fn(p);
        if (!err.empty()) throw ParseError(name_ + ": " + err, 105);
      }
      if (!set_(p)) throw ParseError(name_ + ": could not convert '" + p + "'", 105);
    }
  }

 private:
  std::string name_;
  std::function<bool(const std::string&)> set_;
  bool vector_;
  bool required_ = false;
  bool seen_ = false;
  char delim_ = 0;
  std::vector<Validator> checks_;
};

class App {
 public:
  explicit App(std::string description = "", std::string name = "")
      : desc_(std::move(description)), name_(std::move(name)) {}

  App* require_subcommand(int n = 1) {
    require_subs_ = n;
    return this;
  }
  App* add_subcommand(const std::string& name, const std::string& description = "") {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }
  template <class T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    std::function<bool(const std::string&)> set;
    bool vec = false;
    if constexpr (requires { typename T::value_type; } && !std::is_same_v<T, std::string>) {
      vec = true;
      set = [&target, first = std::make_shared<bool>(true)](const std::string& s) {
        if (*first) {
          target.clear();
          *first = false;
        }
        typename T::value_type v{};
        if (!detail::convert(s, v)) return false;
        target.push_back(v);
        return true;
      };
    } else {
      set = [&target](const std::string& s) { return detail::convert(s, target); };
    }
    opts_.push_back(std::make_unique<Option>(name, std::move(set), vec));
    return opts_.back().get();
  }
  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parse_args(args, 0);
  }

  int exit(const ParseError& e) const {
    std::cerr << e.what() << "\n";
    return e.code;
  }

 private:
  void parse_args(const std::vector<std::string>& a, std::size_t i) {
    parsed_ = true;
    while (i < a.size()) {
      const std::string& tok = a[i];
      if (tok.rfind("--", 0) == 0) {
        std::string key = tok, val;
        bool inline_val = false;
        if (const auto eq = tok.find('='); eq != std::string::npos) {
          key = tok.substr(0, eq);
          val = tok.substr(eq + 1);
          inline_val = true;
        }
        Option* o = find(key);
        if (!o) throw ParseError("unknown option " + key, 109);
        if (!inline_val) {
          if (i + 1 >= a.size()) throw ParseError(key + " needs a value", 105);
          val = a[++i];
        }
        o->apply(val);
        ++i;
        continue;
      }
      App* sub = nullptr;
      for (auto& s : subs_)
        if (s->name_ == tok) sub = s.get();
      if (!sub) throw ParseError("unexpected argument " + tok, 109);
      check_required();
      sub->parse_args(a, i + 1);
      return;
    }
    check_required();
    if (require_subs_ > 0) throw ParseError("a subcommand is required", 106);
  }
  void check_required() const {
    for (const auto& o : opts_)
      if (o->is_required() && !o->seen()) throw ParseError(o->name() + " is required", 106);
  }
  Option* find(const std::string& key) {
    for (auto& o : opts_)
      if (o->name() == key) return o.get();
    return nullptr;
  }

  std::string desc_, name_;
  int require_subs_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)       \
  try {                                    \
    (app).parse((argc), (argv));           \
  } catch (const CLI::ParseError& e) {     \
    return (app).exit(e);                  \
  }
