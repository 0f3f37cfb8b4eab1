// Minimal stand-in for the CLI11 header the reference CLI includes
// (/root/reference/proj/tools/streamgnn_cli.cpp:18). CLI11 lives in the
// reference's git-ignored vendor/ directory and is not in this image, so this
// file implements only the subset that CLI uses: one level of subcommands,
// `--name value` options, flags, one positional vector, required(),
// PositiveNumber / IsMember checks and CLI11_PARSE. Written for this repo.
//
// TEST INFRASTRUCTURE: it lets oracle/ref.mk build the reference's own CLI
// (oracle/_ref/streamgnn_ref_cli) so `report` output can pin the product's
// stats-report restatement byte for byte.
#pragma once

#include <cstdio>
#include <functional>
#include <initializer_list>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Validator {
  std::function<std::string(const std::string&)> fn;
};

inline const Validator PositiveNumber{[](const std::string& s) -> std::string {
  try {
    return std::stod(s) > 0 ? "" : "value must be positive";
  } catch (...) {
    return "not a number";
  }
}};

inline Validator IsMember(std::initializer_list<const char*> names) {
  std::set<std::string> set(names.begin(), names.end());
  return Validator{[set](const std::string& s) -> std::string { return set.count(s) ? "" : "not a member: " + s; }};
}

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set, bool flag, bool multi)
      : name_(std::move(name)), set_(std::move(set)), flag_(flag), multi_(multi) {}
  Option* required() {
    required_ = true;
    return this;
  }
  Option* check(const Validator& v) {
    checks_.push_back(v);
    return this;
  }

 private:
  friend class App;
  std::string name_;
  std::function<void(const std::string&)> set_;
  bool flag_, multi_, required_ = false, seen_ = false;
  std::vector<Validator> checks_;
};

template <typename T>
void assign(T& out, const std::string& s) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
  } else {
    std::istringstream in(s);
    in >> out;
    if (in.fail()) throw Error("bad value: " + s);
  }
}

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
  void require_subcommand(int n) { require_sub_ = n; }
  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  template <typename T>
  Option* add_option(const std::string& name, T& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, [&var](const std::string& s) { assign(var, s); }, false, false));
    return opts_.back().get();
  }
  template <typename T>
  Option* add_option(const std::string& name, std::vector<T>& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name, [&var](const std::string& s) { var.emplace_back(); assign(var.back(), s); }, false, true));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& var, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(name, [&var](const std::string&) { var = true; }, true, false));
    return opts_.back().get();
  }
  bool parsed() const { return parsed_; }

  // argv[1] selects the subcommand; then `--opt value`, flags, positionals.
  void parse(int argc, char** argv) {
    if (argc < 2) throw Error("a subcommand is required");
    App* sub = nullptr;
    for (auto& s : subs_)
      if (s->name_ == argv[1]) sub = s.get();
    if (!sub) throw Error(std::string("unknown subcommand: ") + argv[1]);
    sub->parsed_ = true;
    parsed_ = true;
    for (int i = 2; i < argc; ++i) {
      std::string a = argv[i];
      Option* o = nullptr;
      if (a.rfind("--", 0) == 0) {
        for (auto& p : sub->opts_)
          if (p->name_ == a) o = p.get();
        if (!o) throw Error("unknown option: " + a);
        if (o->flag_) {
          o->set_("");
          o->seen_ = true;
          continue;
        }
        if (++i >= argc) throw Error("missing value for " + a);
        a = argv[i];
      } else {
        for (auto& p : sub->opts_)
          if (p->name_.rfind("--", 0) != 0) o = p.get();
        if (!o) throw Error("unexpected argument: " + a);
      }
      for (const Validator& v : o->checks_) {
        const std::string why = v.fn(a);
        if (!why.empty()) throw Error(o->name_ + ": " + why);
      }
      o->set_(a);
      o->seen_ = true;
    }
    for (auto& p : sub->opts_)
      if (p->required_ && !p->seen_) throw Error("missing required option " + p->name_);
  }

 private:
  std::string desc_, name_;
  int require_sub_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)                  \
  try {                                               \
    (app).parse((argc), (argv));                      \
  } catch (const CLI::Error& e) {                     \
    std::fprintf(stderr, "%s\n", e.what());           \
    return 106;                                       \
  }
