// CLI11.hpp — the subset of CLI11 the reference's front end uses
// (proj/tools/sdtw.cpp: App, add_subcommand, add_option / add_flag on
// scalars, strings and vectors, positional options, IsMember checks,
// require_subcommand, parse / exit, CallForHelp / ParseError, parsed()),
// so that tool compiles unchanged without the vendored header (absent from
// the reference).  Built with include/softdtw_redirect first on the include
// path, the reference's CLI then runs on the B200 engine.
#pragma once
#include <cstdlib>
#include <functional>
#include <iostream>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class Error : public std::runtime_error {
  public:
    Error(const std::string &m, int code) : std::runtime_error(m), code_(code) {}
    int get_exit_code() const { return code_; }

  private:
    int code_;
};
class ParseError : public Error {
  public:
    explicit ParseError(const std::string &m) : Error(m, 2) {}
};
class CallForHelp : public ParseError {
  public:
    CallForHelp() : ParseError("help") {}
};

struct IsMember {
    std::set<std::string> allowed;
    IsMember(std::initializer_list<std::string> l) : allowed(l) {}
};

namespace detail {
template <class T>
void assign(T &dst, const std::string &s)
{
    if constexpr (std::is_same_v<T, std::string>) {
        dst = s;
    } else if constexpr (std::is_same_v<T, bool>) {
        dst = !(s == "0" || s == "false");
    } else if constexpr (std::is_floating_point_v<T>) {
        std::size_t pos = 0;
        dst = (T)std::stod(s, &pos);
        if (pos != s.size()) throw ParseError("not a number: " + s);
    } else {
        std::size_t pos = 0;
        const long long v = std::stoll(s, &pos);
        if (pos != s.size() || (std::is_unsigned_v<T> && v < 0)) throw ParseError("not an integer: " + s);
        dst = (T)v;
    }
}
template <class T>
struct is_vector : std::false_type {};
template <class T>
struct is_vector<std::vector<T>> : std::true_type {};
}  // namespace detail

class Option {
  public:
    std::vector<std::string> names;  // "--x", "-o", or a positional name
    bool positional = false, flag = false, multi = false, seen = false;
    std::function<void(const std::string &)> set;
    std::function<void()> reset;
    std::set<std::string> allowed;
    Option *check(const IsMember &m)
    {
        allowed = m.allowed;
        return this;
    }
    void take(const std::string &v)
    {
        if (!allowed.empty() && !allowed.count(v)) throw ParseError("value '" + v + "' not allowed for " + names[0]);
        if (multi && !seen) reset();
        seen = true;
        set(v);
    }
};

class App {
  public:
    explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
    App *add_subcommand(const std::string &name, const std::string &desc)
    {
        subs_.push_back(std::make_unique<App>(desc, name));
        return subs_.back().get();
    }
    void require_subcommand(int n) { require_ = n; }
    bool parsed() const { return parsed_; }

    template <class T>
    Option *add_option(const std::string &spec, T &dst, const std::string & = "")
    {
        auto o = std::make_unique<Option>();
        std::stringstream ss(spec);
        for (std::string n; std::getline(ss, n, ',');) o->names.push_back(n);
        o->positional = o->names[0][0] != '-';
        if constexpr (detail::is_vector<T>::value) {
            o->multi = true;
            o->reset = [&dst] { dst.clear(); };
            o->set = [&dst](const std::string &v) {
                typename T::value_type e{};
                detail::assign(e, v);
                dst.push_back(e);
            };
        } else {
            o->set = [&dst](const std::string &v) { detail::assign(dst, v); };
        }
        opts_.push_back(std::move(o));
        return opts_.back().get();
    }
    Option *add_flag(const std::string &spec, bool &dst, const std::string & = "")
    {
        Option *o = add_option(spec, dst);
        o->flag = true;
        return o;
    }

    void parse(int argc, char **argv)
    {
        std::vector<std::string> args(argv + 1, argv + argc);
        std::size_t i = 0;
        parse_args(args, i);
    }
    int exit(const Error &e) const
    {
        if (dynamic_cast<const CallForHelp *>(&e)) {
            help(std::cout);
            return 0;
        }
        std::cerr << e.what() << "\n";
        return e.get_exit_code();
    }

  private:
    Option *find(const std::string &n)
    {
        for (auto &o : opts_)
            for (auto &nm : o->names)
                if (nm == n) return o.get();
        return nullptr;
    }
    void parse_args(const std::vector<std::string> &a, std::size_t &i)
    {
        parsed_ = true;
        while (i < a.size()) {
            const std::string &s = a[i];
            if (s == "--help" || s == "-h") throw CallForHelp();
            App *sub = nullptr;
            for (auto &c : subs_)
                if (c->name_ == s) sub = c.get();
            if (sub) {
                ++i;
                sub->parse_args(a, i);
                ++nsubs_;
                continue;
            }
            if (s.size() > 1 && s[0] == '-') {
                std::string key = s, val;
                const auto eq = s.find('=');
                if (eq != std::string::npos) {
                    key = s.substr(0, eq);
                    val = s.substr(eq + 1);
                }
                Option *o = find(key);
                if (!o) throw ParseError("unknown option " + key);
                ++i;
                if (o->flag) {
                    o->take(eq != std::string::npos ? val : "1");
                } else if (eq != std::string::npos) {
                    o->take(val);
                } else {
                    if (i >= a.size()) throw ParseError("missing value for " + key);
                    o->take(a[i++]);
                    while (o->multi && i < a.size() && !(a[i].size() > 1 && a[i][0] == '-') && !is_sub(a[i]))
                        o->take(a[i++]);
                }
                continue;
            }
            Option *pos = nullptr;
            for (auto &o : opts_)
                if (o->positional && (o->multi || !o->seen)) {
                    pos = o.get();
                    break;
                }
            if (!pos) throw ParseError("unexpected argument " + s);
            pos->take(s);
            ++i;
        }
        if (require_ > 0 && nsubs_ < require_) throw ParseError("a subcommand is required (--help for the list)");
    }
    bool is_sub(const std::string &s) const
    {
        for (auto &c : subs_)
            if (c->name_ == s) return true;
        return false;
    }
    void help(std::ostream &os) const
    {
        os << desc_ << "\n";
        for (auto &c : subs_) os << "  " << c->name_ << "  " << c->desc_ << "\n";
    }
    std::string desc_, name_;
    std::vector<std::unique_ptr<App>> subs_;
    std::vector<std::unique_ptr<Option>> opts_;
    int require_ = 0, nsubs_ = 0;
    bool parsed_ = false;
};

}  // namespace CLI
