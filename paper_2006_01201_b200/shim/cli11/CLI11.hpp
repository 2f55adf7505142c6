// Minimal command-line parser with the subset of the CLI11 API that the
// reference's tools/flowstitch_cli.cpp uses (App, add_option / add_flag /
// add_subcommand, required(), envname(), require_subcommand, fallthrough,
// parse, exit, ParseError).  CLI11 itself is a third-party header the
// reference expects under vendor/ (proj/.gitignore:2) and it is not on this
// image; this stand-in lets the reference's CLI, unchanged, be relinked
// against the B200 drop-in.  Behaviour the CLI relies on:
// "--opt value" / "--opt=value", counted / boolean flags, an environment
// fallback, required options and a required subcommand (errors exit 1 via
// App::exit), global options accepted after the subcommand.
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

class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, int code) : std::runtime_error(what), code_(code) {}
    int get_exit_code() const { return code_; }

private:
    int code_;
};

class Option {
public:
    Option(std::vector<std::string> names, std::function<bool(const std::string&)> set, bool flag)
        : names_(std::move(names)), set_(std::move(set)), flag_(flag) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    Option* envname(const std::string& e) {
        env_ = e;
        return this;
    }
    bool matches(const std::string& n) const {
        for (const auto& x : names_)
            if (x == n) return true;
        return false;
    }
    const std::string& name() const { return names_.back(); }

private:
    friend class App;
    std::vector<std::string> names_;
    std::function<bool(const std::string&)> set_;
    bool flag_ = false, required_ = false, seen_ = false;
    std::string env_;
};

namespace detail {
inline std::vector<std::string> split_names(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string t;
    while (std::getline(ss, t, ','))
        if (!t.empty()) out.push_back(t);
    return out;
}
template <class T>
bool convert(const std::string& s, T& v) {
    std::istringstream is(s);
    is >> v;
    return !is.fail() && is.eof();
}
inline bool convert(const std::string& s, std::string& v) {
    v = s;
    return true;
}
}  // namespace detail

class App {
public:
    explicit App(std::string description = "", std::string name = "")
        : description_(std::move(description)), name_(std::move(name)) {}

    template <class T>
    Option* add_option(const std::string& names, T& var, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(
            detail::split_names(names), [&var](const std::string& s) { return detail::convert(s, var); },
            false));
        return opts_.back().get();
    }
    Option* add_flag(const std::string& names, int& count, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(
            detail::split_names(names), [&count](const std::string&) { ++count; return true; }, true));
        return opts_.back().get();
    }
    Option* add_flag(const std::string& names, bool& flag, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(
            detail::split_names(names), [&flag](const std::string&) { flag = true; return true; },
            true));
        return opts_.back().get();
    }
    App* add_subcommand(const std::string& name, const std::string& description = "") {
        subs_.push_back(std::make_unique<App>(description, name));
        subs_.back()->parent_ = this;
        return subs_.back().get();
    }
    App* require_subcommand(int n = 1) {
        require_sub_ = n;
        return this;
    }
    App* fallthrough(bool f = true) {
        fallthrough_ = f;
        return this;
    }
    explicit operator bool() const { return parsed_; }

    void parse(int argc, const char* const* argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        App* cur = this;
        parsed_ = true;
        for (size_t i = 0; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a == "-h" || a == "--help") throw ParseError(cur->help(), 0);
            if (a.size() > 1 && a[0] == '-') {
                std::string name = a, value;
                const size_t eq = a.find('=');
                const bool has_eq = a.rfind("--", 0) == 0 && eq != std::string::npos;
                if (has_eq) {
                    name = a.substr(0, eq);
                    value = a.substr(eq + 1);
                }
                Option* o = cur->find(name);
                if (!o && fallthrough_)  // global options may follow the subcommand
                    for (App* s = cur->parent_; s && !o; s = s->parent_) o = s->find(name);
                if (!o) throw ParseError("The following argument was not expected: " + a, 109);
                if (!o->flag_ && !has_eq) {
                    if (i + 1 >= args.size()) throw ParseError(name + " requires an argument", 106);
                    value = args[++i];
                }
                if (!o->set_(value)) throw ParseError("Could not convert: " + name + " = " + value, 105);
                o->seen_ = true;
                continue;
            }
            App* sub = nullptr;
            for (auto& s : cur->subs_)
                if (s->name_ == a) sub = s.get();
            if (!sub) throw ParseError("The following argument was not expected: " + a, 109);
            sub->parsed_ = true;
            cur = sub;
        }
        for (App* s = cur; s; s = s->parent_) s->finish();
    }
    void parse(int argc, char** argv) { parse(argc, const_cast<const char* const*>(argv)); }

    int exit(const ParseError& e, std::ostream& out = std::cout, std::ostream& err = std::cerr) const {
        if (e.get_exit_code() == 0)
            out << e.what() << "\n";
        else
            err << e.what() << "\n";
        return e.get_exit_code();
    }

private:
    Option* find(const std::string& n) {
        for (auto& o : opts_)
            if (o->matches(n)) return o.get();
        return nullptr;
    }
    void finish() {
        for (auto& o : opts_) {
            if (!o->seen_ && !o->env_.empty())
                if (const char* v = std::getenv(o->env_.c_str())) {
                    if (!o->set_(v)) throw ParseError("Could not convert: " + o->env_, 105);
                    o->seen_ = true;
                }
            if (o->required_ && !o->seen_) throw ParseError(o->name() + " is required", 106);
        }
        if (require_sub_ > 0) {
            int n = 0;
            for (auto& s : subs_) n += s->parsed_;
            if (n < require_sub_) throw ParseError("A subcommand is required", 106);
        }
    }
    std::string help() const {
        std::string h = description_ + "\n";
        for (auto& s : subs_) h += "  " + s->name_ + "  " + s->description_ + "\n";
        for (auto& o : opts_) h += "  " + o->name() + "\n";
        return h;
    }

    std::string description_, name_;
    App* parent_ = nullptr;
    std::vector<std::unique_ptr<Option>> opts_;
    std::vector<std::unique_ptr<App>> subs_;
    int require_sub_ = 0;
    bool fallthrough_ = false, parsed_ = false;
};

}  // namespace CLI
