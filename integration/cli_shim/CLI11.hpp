// CLI11.hpp — minimal stand-in for the CLI11 subset that the reference's
// command line (tools/dagsplit_main.cpp:294-333) uses, so that file compiles
// UNCHANGED here (CLI11 is not in this image).  Written for this
// repo; supports exactly:
//   CLI::App{desc}; app.require_subcommand(n); app.add_subcommand(name, desc)
//   sub->add_option("input" | "-o,--output" | "--flag", T& var, desc)->required()
//   sub->add_flag("--flag", bool& var, desc); sub->parsed(); CLI11_PARSE(app, argc, argv)
// Parse errors print to stderr and exit with CLI11's codes (106 for a missing
// required option, 109 for extras, 0 for --help).
#pragma once

#include <cstdlib>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& what, int c) : std::runtime_error(what), code(c) {}
};

class Option {
 public:
  Option(std::string names, std::function<bool(const std::string&)> set, bool flag)
      : set_(std::move(set)), flag_(flag) {
    std::stringstream ss(names);
    std::string part;
    while (std::getline(ss, part, ',')) {
      if (part.rfind("-", 0) == 0) dashed_.push_back(part);
      else positional_ = part;
    }
  }
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }

 private:
  friend class App;
  bool matches(const std::string& arg) const {
    for (const auto& n : dashed_)
      if (n == arg) return true;
    return false;
  }
  std::string display() const { return positional_.empty() ? dashed_.back() : positional_; }

  std::vector<std::string> dashed_;
  std::string positional_;
  std::function<bool(const std::string&)> set_;
  bool flag_ = false;
  bool required_ = false;
  bool seen_ = false;
};

template <class T>
bool convert(const std::string& s, T& out) {
  std::istringstream is(s);
  is >> out;
  return !is.fail() && is.peek() == std::char_traits<char>::eof();
}
inline bool convert(const std::string& s, std::string& out) {
  out = s;
  return true;
}

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  void require_subcommand(int n) { require_sub_ = n; }

  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }

  template <class T>
  Option* add_option(const std::string& names, T& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        names, [&var](const std::string& s) { return convert(s, var); }, false));
    return opts_.back().get();
  }

  Option* add_flag(const std::string& names, bool& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        names, [&var](const std::string&) { var = true; return true; }, true));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    size_t i = 0;
    App* cur = this;
    parsed_ = true;
    if (i < args.size() && (args[i] == "-h" || args[i] == "--help")) throw ParseError(help(), 0);
    if (i < args.size()) {
      for (auto& s : subs_)
        if (s->name_ == args[i]) {
          cur = s.get();
          cur->parsed_ = true;
          ++i;
          break;
        }
    }
    if (cur == this && require_sub_ > 0)
      throw ParseError("A subcommand is required\n" + help(), 109);
    size_t next_pos = 0;
    for (; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "-h" || a == "--help") throw ParseError(cur->help(), 0);
      std::string key = a, val;
      bool has_eq = false;
      if (a.rfind("--", 0) == 0 && a.find('=') != std::string::npos) {
        key = a.substr(0, a.find('='));
        val = a.substr(a.find('=') + 1);
        has_eq = true;
      }
      if (key.size() > 1 && key[0] == '-') {
        Option* o = nullptr;
        for (auto& p : cur->opts_)
          if (p->matches(key)) o = p.get();
        if (!o) throw ParseError("The following argument was not expected: " + a, 109);
        if (!o->flag_ && !has_eq) {
          if (i + 1 >= args.size()) throw ParseError(key + ": 1 required argument missing", 107);
          val = args[++i];
        }
        if (!o->set_(val)) throw ParseError(key + ": could not convert '" + val + "'", 105);
        o->seen_ = true;
        continue;
      }
      Option* o = nullptr;
      size_t k = 0;
      for (auto& p : cur->opts_) {
        if (p->positional_.empty()) continue;
        if (k++ == next_pos) o = p.get();
      }
      if (!o) throw ParseError("The following argument was not expected: " + a, 109);
      ++next_pos;
      if (!o->set_(a)) throw ParseError(o->positional_ + ": could not convert '" + a + "'", 105);
      o->seen_ = true;
    }
    for (auto& p : cur->opts_)
      if (p->required_ && !p->seen_) throw ParseError(p->display() + " is required", 106);
  }

  int exit(const ParseError& e) const {
    (e.code == 0 ? std::cout : std::cerr) << e.what() << "\n";
    return e.code;
  }

  std::string help() const {
    std::ostringstream os;
    os << desc_ << "\n";
    for (auto& s : subs_) os << "  " << s->name_ << "  " << s->desc_ << "\n";
    return os.str();
  }

 private:
  std::string desc_, name_;
  int require_sub_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)       \
  try {                                    \
    (app).parse((argc), (argv));           \
  } catch (const CLI::ParseError& e) {     \
    return (app).exit(e);                  \
  }
