// Minimal CLI11-compatible command-line parser: the subset of the CLI11 API that the reference's
// tools/fdsolve.cpp uses (CLI11 itself is not vendored in the reference, proj/.gitignore:2, and
// is absent from this image). With it the reference's fdsolve.cpp compiles unmodified, both
// against the reference library (oracle/_ref/fdsolve) and against the B200 adapter
// (adapter/_build/fdsolve_b200), so the two binaries can be compared byte for byte.
//
// Supported: App{desc}, require_subcommand(n), add_subcommand(name, desc), add_option(name,
// value, desc) for positionals ("file") and "--long" options (string / integral / floating),
// add_flag("--name", bool&, desc), ->required(), ->check(validator), IsMember, PositiveNumber,
// Range, parsed(), CLI11_PARSE. Errors print "<message>" and "Run with --help for more
// information." to stderr, with CLI11's exit codes (105 validation, 106 required, 109 extras,
// 114 conversion); --help prints usage and exits 0.
#pragma once

#include <cstdint>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
    int code;
    ParseError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};
struct CallForHelp : ParseError {
    CallForHelp() : ParseError("help", 0) {}
};

using Validator = std::function<std::string(const std::string&)>; // "" = ok

inline Validator IsMember(std::initializer_list<const char*> items) {
    std::vector<std::string> v(items.begin(), items.end());
    return [v](const std::string& s) -> std::string {
        for (const auto& x : v)
            if (x == s) return "";
        std::string all;
        for (const auto& x : v) all += (all.empty() ? "" : ",") + x;
        return s + " not in {" + all + "}";
    };
}

inline const Validator PositiveNumber = [](const std::string& s) -> std::string {
    try {
        size_t pos = 0;
        double d = std::stod(s, &pos);
        if (pos != s.size() || !(d > 0)) return "Value " + s + " not a positive number";
    } catch (...) {
        return "Value " + s + " not a positive number";
    }
    return "";
};

inline Validator Range(double lo, double hi) {
    return [lo, hi](const std::string& s) -> std::string {
        try {
            size_t pos = 0;
            double d = std::stod(s, &pos);
            if (pos != s.size() || d < lo || d > hi) throw 0;
        } catch (...) {
            std::ostringstream os;
            os << "Value " << s << " not in range [" << lo << " - " << hi << "]";
            return os.str();
        }
        return "";
    };
}

class Option {
  public:
    Option(std::string name, std::function<bool(const std::string&)> set, bool flag)
        : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    Option* check(Validator v) {
        checks_.push_back(std::move(v));
        return this;
    }
    const std::string& name() const { return name_; }
    bool positional() const { return name_.rfind("--", 0) != 0; }
    bool flag() const { return flag_; }
    void apply(const std::string& value) {
        for (auto& c : checks_) {
            std::string err = c(value);
            if (!err.empty()) throw ParseError(name_ + ": " + err, 105);
        }
        if (!set_(value)) throw ParseError("Could not convert: " + name_ + " = " + value, 114);
        seen_ = true;
    }
    bool seen() const { return seen_; }
    bool is_required() const { return required_; }

  private:
    std::string name_;
    std::function<bool(const std::string&)> set_;
    bool flag_;
    bool required_ = false;
    bool seen_ = false;
    std::vector<Validator> checks_;
};

template <class T>
bool convert(const std::string& s, T& out) {
    try {
        size_t pos = 0;
        if constexpr (std::is_same_v<T, std::string>) {
            out = s;
            return true;
        } else if constexpr (std::is_same_v<T, bool>) {
            out = !(s == "0" || s == "false");
            return true;
        } else if constexpr (std::is_floating_point_v<T>) {
            out = static_cast<T>(std::stod(s, &pos));
        } else if constexpr (std::is_unsigned_v<T>) {
            if (!s.empty() && s[0] == '-') return false;
            out = static_cast<T>(std::stoull(s, &pos));
        } else {
            out = static_cast<T>(std::stoll(s, &pos));
        }
        return pos == s.size();
    } catch (...) {
        return false;
    }
}

class App {
  public:
    explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

    App* require_subcommand(int n) {
        require_sub_ = n;
        return this;
    }
    App* add_subcommand(const std::string& name, const std::string& desc) {
        subs_.push_back(std::make_unique<App>(desc, name));
        return subs_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, T& value, const std::string& desc = "") {
        (void)desc;
        opts_.push_back(std::make_unique<Option>(name, [&value](const std::string& s) { return convert(s, value); },
                                                 false));
        return opts_.back().get();
    }
    Option* add_flag(const std::string& name, bool& value, const std::string& desc = "") {
        (void)desc;
        opts_.push_back(std::make_unique<Option>(name, [&value](const std::string&) {
            value = true;
            return true;
        }, true));
        return opts_.back().get();
    }
    bool parsed() const { return parsed_; }

    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        parse_tokens(args, 0);
    }

    int exit(const ParseError& e) const {
        if (e.code == 0) {
            std::cout << usage();
            return 0;
        }
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return e.code;
    }

  private:
    std::string usage() const {
        std::ostringstream os;
        os << desc_ << "\nUsage: " << (name_.empty() ? "fdsolve" : name_) << " [OPTIONS]";
        if (!subs_.empty()) os << " SUBCOMMAND";
        os << "\n";
        for (const auto& o : opts_) os << "  " << o->name() << "\n";
        for (const auto& s : subs_) os << "  " << s->name_ << "  " << s->desc_ << "\n";
        return os.str();
    }

    void parse_tokens(const std::vector<std::string>& a, size_t i) {
        parsed_ = true;
        size_t pos_index = 0;
        for (; i < a.size(); ++i) {
            const std::string& t = a[i];
            if (t == "--help" || t == "-h") throw CallForHelp();
            if (t.rfind("--", 0) == 0) {
                std::string key = t, val;
                const size_t eq = t.find('=');
                if (eq != std::string::npos) {
                    key = t.substr(0, eq);
                    val = t.substr(eq + 1);
                }
                Option* o = find(key);
                if (!o) throw ParseError("The following argument was not expected: " + t, 109);
                if (o->flag()) {
                    o->apply("1");
                } else {
                    if (eq == std::string::npos) {
                        if (i + 1 >= a.size()) throw ParseError(key + " requires an argument", 114);
                        val = a[++i];
                    }
                    o->apply(val);
                }
                continue;
            }
            if (!subs_.empty() && pos_index == 0) {
                for (auto& s : subs_)
                    if (s->name_ == t) {
                        s->parse_tokens(a, i + 1);
                        check_required();
                        return;
                    }
            }
            Option* p = positional(pos_index++);
            if (!p) throw ParseError("The following argument was not expected: " + t, 109);
            p->apply(t);
        }
        check_required();
        if (require_sub_ > 0 && !subs_.empty()) {
            bool any = false;
            for (auto& s : subs_) any = any || s->parsed_;
            if (!any) throw ParseError("A subcommand is required", 106);
        }
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

    Option* positional(size_t k) {
        size_t seen = 0;
        for (auto& o : opts_)
            if (o->positional() && seen++ == k) return o.get();
        return nullptr;
    }

    std::string desc_, name_;
    int require_sub_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<Option>> opts_;
    std::vector<std::unique_ptr<App>> subs_;
};

} // namespace CLI

#define CLI11_PARSE(app, argc, argv)                                                                \
    try {                                                                                           \
        (app).parse((argc), (argv));                                                                \
    } catch (const CLI::ParseError& e_) {                                                           \
        return (app).exit(e_);                                                                      \
    }
