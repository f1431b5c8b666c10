// CLI11.hpp — a minimal, self-contained stand-in for the subset of the CLI11
// command-line library that the reference's tools/slicesim_main.cpp uses
// (CLI11 is a header-only dependency the reference expects in proj/vendor/,
// absent here).  It lets that file compile UNCHANGED into the `slicesim`
// CLI, both against the reference core and against the B200 drop-in.
//
// Supported: App with subcommands, require_subcommand(n), add_option for
// std::string / integral / floating / std::vector<T> targets ("--name value",
// "--name=value"; vector options take every following non-option token and
// repeat), Option::required() / each(fn) / delimiter(c), App::parsed(),
// --help, and CLI11_PARSE with CLI11's exit codes (RequiredError 106,
// ExtrasError 109, ConversionError 104, ArgumentMismatch 114).
#pragma once

#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
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
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("help requested", 0) {}
};
struct ConversionError : ParseError {
  explicit ConversionError(const std::string& m) : ParseError(m, 104) {}
};
struct RequiredError : ParseError {
  explicit RequiredError(const std::string& m) : ParseError(m, 106) {}
};
struct ExtrasError : ParseError {
  explicit ExtrasError(const std::string& m) : ParseError(m, 109) {}
};
struct ArgumentMismatch : ParseError {
  explicit ArgumentMismatch(const std::string& m) : ParseError(m, 114) {}
};

namespace detail {

template <class T>
struct is_vector : std::false_type {};
template <class T, class A>
struct is_vector<std::vector<T, A>> : std::true_type {};

template <class T>
T convert(const std::string& name, const std::string& s) {
  if constexpr (std::is_same_v<T, std::string>) {
    return s;
  } else {
    std::istringstream in(s);
    T v{};
    in >> v;
    if (in.fail() || !in.eof()) throw ConversionError("could not convert '" + s + "' for " + name);
    if constexpr (std::is_unsigned_v<T>)
      if (!s.empty() && s[0] == '-') throw ConversionError("negative value '" + s + "' for " + name);
    return v;
  }
}

}  // namespace detail

class Option {
 public:
  Option(std::string name, std::string desc, bool multi, std::function<void(const std::string&)> add)
      : name_(std::move(name)), desc_(std::move(desc)), multi_(multi), add_(std::move(add)) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* each(std::function<void(const std::string&)> fn) {
    each_ = std::move(fn);
    return this;
  }
  Option* delimiter(char c) {
    delim_ = c;
    return this;
  }

 private:
  friend class App;
  void take(const std::string& raw) {
    std::vector<std::string> parts;
    if (delim_) {
      std::string cur;
      for (char ch : raw) {
        if (ch == delim_) {
          parts.push_back(cur);
          cur.clear();
        } else {
          cur += ch;
        }
      }
      parts.push_back(cur);
    } else {
      parts.push_back(raw);
    }
    for (const std::string& p : parts) {
      add_(p);
      if (each_) each_(p);
    }
    ++count_;
  }
  std::string name_, desc_;
  bool multi_ = false, required_ = false;
  char delim_ = 0;
  int count_ = 0;
  std::function<void(const std::string&)> add_, each_;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  void require_subcommand(int n) { require_sub_ = n; }

  App* add_subcommand(const std::string& name, const std::string& desc = "") {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }

  template <class T>
  Option* add_option(const std::string& name, T& target, const std::string& desc = "") {
    std::function<void(const std::string&)> add;
    bool multi = false;
    if constexpr (detail::is_vector<T>::value) {
      using V = typename T::value_type;
      multi = true;
      add = [&target, name](const std::string& s) { target.push_back(detail::convert<V>(name, s)); };
      // CLI11 replaces a vector's defaults with the parsed values
      opts_reset_.push_back([&target]() { target.clear(); });
    } else {
      add = [&target, name](const std::string& s) { target = detail::convert<T>(name, s); };
    }
    opts_.push_back(std::make_unique<Option>(name, desc, multi, std::move(add)));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, const char* const* argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    parse_tokens(args, 0);
  }

  int exit(const ParseError& e) const {
    if (e.get_exit_code() == 0) {
      print_help(std::cout);
      return 0;
    }
    std::cerr << e.what() << "\n";
    if (!name_.empty() || !subs_.empty()) std::cerr << "Run with --help for more information.\n";
    return e.get_exit_code();
  }

 private:
  void print_help(std::ostream& out) const {
    out << desc_ << "\n";
    for (const auto& s : subs_) out << "  " << s->name_ << "  " << s->desc_ << "\n";
    for (const auto& o : opts_) out << "  " << o->name_ << "  " << o->desc_ << "\n";
  }

  Option* find(const std::string& name) const {
    for (const auto& o : opts_)
      if (o->name_ == name) return o.get();
    return nullptr;
  }

  void parse_tokens(const std::vector<std::string>& a, size_t i) {
    parsed_ = true;
    while (i < a.size()) {
      const std::string& tok = a[i];
      if (tok == "--help" || tok == "-h") throw CallForHelp();
      if (!subs_.empty() && tok.rfind("-", 0) != 0) {
        for (const auto& s : subs_) {
          if (s->name_ == tok) {
            check_required();
            s->parse_tokens(a, i + 1);
            sub_count_ = 1;
            return;
          }
        }
        throw ExtrasError("The following argument was not expected: " + tok);
      }
      if (tok.rfind("--", 0) != 0) throw ExtrasError("The following argument was not expected: " + tok);
      std::string name = tok, inline_value;
      bool has_inline = false;
      const auto eq = tok.find('=');
      if (eq != std::string::npos) {
        name = tok.substr(0, eq);
        inline_value = tok.substr(eq + 1);
        has_inline = true;
      }
      Option* o = find(name);
      if (!o) throw ExtrasError("The following argument was not expected: " + tok);
      if (o->multi_ && o->count_ == 0) reset_vector(o);
      ++i;
      if (has_inline) {
        o->take(inline_value);
        continue;
      }
      if (i >= a.size() || (a[i].rfind("--", 0) == 0 && a[i].size() > 2))
        throw ArgumentMismatch(name + ": 1 required TEXT missing");
      o->take(a[i++]);
      if (o->multi_)  // a vector option takes every following plain token
        while (i < a.size() && a[i].rfind("-", 0) != 0 && !is_sub(a[i])) o->take(a[i++]);
    }
    check_required();
    if (require_sub_ > 0 && sub_count_ < require_sub_) throw RequiredError("A subcommand is required");
  }

  bool is_sub(const std::string& tok) const {
    for (const auto& s : subs_)
      if (s->name_ == tok) return true;
    return false;
  }

  void reset_vector(Option* o) {
    for (size_t k = 0; k < opts_.size(); ++k)
      if (opts_[k].get() == o) {
        size_t v = 0;
        for (size_t m = 0; m < k; ++m) v += opts_[m]->multi_ ? 1 : 0;
        if (v < opts_reset_.size()) opts_reset_[v]();
      }
  }

  void check_required() const {
    for (const auto& o : opts_)
      if (o->required_ && o->count_ == 0) throw RequiredError(o->name_ + " is required");
  }

  std::string desc_, name_;
  int require_sub_ = 0, sub_count_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::function<void()>> opts_reset_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)       \
  try {                                    \
    (app).parse((argc), (argv));           \
  } catch (const CLI::ParseError& e) {     \
    return (app).exit(e);                  \
  }
