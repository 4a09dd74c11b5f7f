// Builder-written subset of the CLI11 command-line API, just what the
// reference's tools/shlr_cli.cpp uses (CLI11 is git-ignored vendor code,
// absent from /root/reference: proj/.gitignore:2), so that the reference CLI
// builds unmodified against the B200 drop-in.
//
// Covered: App{description}, require_subcommand(n), option_defaults()->
// multi_option_policy(TakeLast), add_subcommand, add_option(name, T&, desc)
// for strings and arithmetic types, ->required(), add_flag(name, bool&,
// desc), parse(std::vector<std::string>&) (arguments in reverse order, as
// CLI11 takes them), parsed(), ParseError and exit(e) with CLI11's exit-code
// numbering.  Options are "--name value" or "--name=value"; a repeated
// option keeps its last value (TakeLast); unknown options, missing values,
// failed conversions and missing required options are parse errors.
#pragma once

#include <cstdint>
#include <iostream>
#include <limits>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

enum class MultiOptionPolicy { Throw, TakeLast, TakeFirst };

// exit codes follow CLI11's ExitCodes
struct ParseError : std::runtime_error {
  ParseError(const std::string& name, const std::string& msg, int code)
      : std::runtime_error(msg), name_(name), code_(code) {}
  int get_exit_code() const { return code_; }
  const std::string& get_name() const { return name_; }

 private:
  std::string name_;
  int code_;
};
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("CallForHelp", "This should be caught in your main function, see examples", 0) {}
};
struct ConversionError : ParseError {
  explicit ConversionError(const std::string& m) : ParseError("ConversionError", m, 104) {}
};
struct RequiredError : ParseError {
  explicit RequiredError(const std::string& m) : ParseError("RequiredError", m, 106) {}
};
struct ExtrasError : ParseError {
  explicit ExtrasError(const std::string& m) : ParseError("ExtrasError", m, 109) {}
};
struct ArgumentMismatch : ParseError {
  explicit ArgumentMismatch(const std::string& m) : ParseError("ArgumentMismatch", m, 114) {}
};

class Option {
 public:
  Option(std::string name, std::string desc, bool flag) : name_(std::move(name)), desc_(std::move(desc)), flag_(flag) {}
  virtual ~Option() = default;
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* multi_option_policy(MultiOptionPolicy p) {
    policy_ = p;
    return this;
  }
  const std::string& get_name() const { return name_; }
  const std::string& get_description() const { return desc_; }
  bool get_required() const { return required_; }
  bool is_flag() const { return flag_; }
  std::size_t count() const { return count_; }
  void add_result(const std::string& v) {
    if (count_ > 0 && policy_ == MultiOptionPolicy::Throw)
      throw ArgumentMismatch(name_ + ": only one value allowed");
    if (count_ > 0 && policy_ == MultiOptionPolicy::TakeFirst) {
      ++count_;
      return;
    }
    assign(v);
    ++count_;
  }

 protected:
  virtual void assign(const std::string& v) = 0;

 private:
  std::string name_, desc_;
  bool flag_ = false, required_ = false;
  MultiOptionPolicy policy_ = MultiOptionPolicy::Throw;
  std::size_t count_ = 0;
};

namespace detail {
template <typename T>
bool convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
    return true;
  } else if constexpr (std::is_same_v<T, bool>) {
    if (s == "1" || s == "true" || s == "on" || s == "yes" || s.empty()) out = true;
    else if (s == "0" || s == "false" || s == "off" || s == "no") out = false;
    else return false;
    return true;
  } else if constexpr (std::is_integral_v<T> && std::is_unsigned_v<T>) {
    if (s.empty() || s[0] == '-') return false;
    std::size_t pos = 0;
    try {
      const unsigned long long v = std::stoull(s, &pos, 0);
      if (pos != s.size() || v > static_cast<unsigned long long>(std::numeric_limits<T>::max())) return false;
      out = static_cast<T>(v);
    } catch (...) {
      return false;
    }
    return true;
  } else if constexpr (std::is_integral_v<T>) {
    std::size_t pos = 0;
    try {
      const long long v = std::stoll(s, &pos, 0);
      if (pos != s.size() || v > static_cast<long long>(std::numeric_limits<T>::max()) ||
          v < static_cast<long long>(std::numeric_limits<T>::min()))
        return false;
      out = static_cast<T>(v);
    } catch (...) {
      return false;
    }
    return true;
  } else if constexpr (std::is_floating_point_v<T>) {
    std::size_t pos = 0;
    try {
      const long double v = std::stold(s, &pos);
      if (pos != s.size()) return false;
      out = static_cast<T>(v);
    } catch (...) {
      return false;
    }
    return true;
  } else {
    std::istringstream in(s);
    in >> out;
    return static_cast<bool>(in) && in.peek() == EOF;
  }
}

template <typename T>
class TypedOption : public Option {
 public:
  TypedOption(std::string name, T& target, std::string desc, bool flag)
      : Option(std::move(name), std::move(desc), flag), target_(target) {}

 protected:
  void assign(const std::string& v) override {
    if (!convert(v, target_)) throw ConversionError("The value " + v + " is not an allowed value for " + get_name());
  }

 private:
  T& target_;
};
}  // namespace detail

class App {
 public:
  App() = default;
  explicit App(std::string description, std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}
  App(const App&) = delete;
  App& operator=(const App&) = delete;

  App* require_subcommand(int n = -1) {
    require_sub_ = n;
    return this;
  }
  // option defaults: the policy applies to options added afterwards
  App* option_defaults() { return this; }
  App* multi_option_policy(MultiOptionPolicy p) {
    policy_ = p;
    return this;
  }

  App* add_subcommand(const std::string& name, const std::string& desc = "") {
    subs_.push_back(std::make_unique<App>(desc, name));
    subs_.back()->policy_ = policy_;
    subs_.back()->parent_ = this;
    return subs_.back().get();
  }

  template <typename T>
  Option* add_option(const std::string& name, T& target, const std::string& desc = "") {
    opts_.push_back(std::make_unique<detail::TypedOption<T>>(name, target, desc, false));
    opts_.back()->multi_option_policy(policy_);
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& target, const std::string& desc = "") {
    opts_.push_back(std::make_unique<detail::TypedOption<bool>>(name, target, desc, true));
    opts_.back()->multi_option_policy(policy_);
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }
  const std::string& get_name() const { return name_; }

  // args in reverse order (CLI11's vector overload): args.back() is first
  void parse(std::vector<std::string>& args) {
    std::vector<std::string> in(args.rbegin(), args.rend());
    args.clear();
    std::size_t i = 0;
    parse_tokens(in, i);
  }
  void parse(int argc, const char* const* argv) {
    std::vector<std::string> in;
    for (int k = argc - 1; k > 0; --k) in.push_back(argv[k]);
    parse(in);
  }

  int exit(const ParseError& e, std::ostream& out = std::cout, std::ostream& err = std::cerr) const {
    if (e.get_exit_code() == 0) {
      out << help();
      return 0;
    }
    err << e.what() << "\n";
    if (e.get_name() == "RequiredError" || e.get_name() == "ExtrasError") err << "Run with --help for more information.\n";
    return e.get_exit_code();
  }

  std::string help() const {
    std::ostringstream o;
    o << desc_ << "\n";
    if (!subs_.empty()) {
      o << "Subcommands:\n";
      for (const auto& s : subs_) o << "  " << s->name_ << "  " << s->desc_ << "\n";
    }
    if (!opts_.empty()) {
      o << "Options:\n";
      for (const auto& op : opts_)
        o << "  " << op->get_name() << (op->get_required() ? " (required)" : "") << "  " << op->get_description()
          << "\n";
    }
    return o.str();
  }

 private:
  Option* find(const std::string& n) {
    for (auto& o : opts_)
      if (o->get_name() == n) return o.get();
    return nullptr;
  }
  App* find_sub(const std::string& n) {
    for (auto& s : subs_)
      if (s->name_ == n) return s.get();
    return nullptr;
  }

  void parse_tokens(const std::vector<std::string>& in, std::size_t& i) {
    parsed_ = true;
    int nsub = 0;
    while (i < in.size()) {
      const std::string& tok = in[i];
      if (tok == "--help" || tok == "-h") throw CallForHelp();
      if (tok.rfind("--", 0) == 0) {
        const auto eq = tok.find('=');
        const std::string name = tok.substr(0, eq);
        Option* o = find(name);
        if (!o) throw ExtrasError("The following arguments were not expected: " + tok);
        ++i;
        if (eq != std::string::npos) {
          o->add_result(tok.substr(eq + 1));
        } else if (o->is_flag()) {
          o->add_result("1");
        } else {
          if (i >= in.size()) throw ArgumentMismatch(name + ": 1 required TEXT missing");
          o->add_result(in[i++]);
        }
        continue;
      }
      if (App* s = find_sub(tok)) {
        ++i;
        ++nsub;
        s->parse_tokens(in, i);
        continue;
      }
      throw ExtrasError("The following argument was not expected: " + tok);
    }
    for (auto& o : opts_)
      if (o->get_required() && o->count() == 0) throw RequiredError(o->get_name() + " is required");
    if (require_sub_ > 0 && nsub != require_sub_)
      throw RequiredError(nsub < require_sub_ ? "A subcommand is required" : "Too many subcommands");
  }

  std::string desc_, name_;
  App* parent_ = nullptr;
  int require_sub_ = 0;
  bool parsed_ = false;
  MultiOptionPolicy policy_ = MultiOptionPolicy::Throw;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
