// CLI11.hpp -- a minimal, independently written stand-in for the CLI11
// command-line parser (the real header is not available in this image) with
// just what the reference CLI (proj/tools/fembatch.cpp) uses: App with
// subcommands, add_option / add_flag bound to variables (scalars and
// delimiter-separated lists), validators IsMember / PositiveNumber / Range,
// count(), got_subcommand(), CLI11_PARSE.  Used only to build the reference
// CLI from its sources against the reference library and against the B200
// engine (oracle/Makefile `cli`).
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <initializer_list>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  ParseError(const std::string& m, int code) : std::runtime_error(m), exit_code(code) {}
  int exit_code;
};

// A validator returns "" for an accepted value, else the reason.
struct Validator {
  std::function<std::string(const std::string&)> check;
};

namespace detail {
template <class T>
bool parse(const std::string& s, T& out)
{
  if constexpr (std::is_same_v<T, std::string>)
  {
    out = s;
    return true;
  }
  else
  {
    std::istringstream is(s);
    T v{};
    is >> v;
    if (!is || !(is >> std::ws).eof())
      return false;
    out = v;
    return true;
  }
}
inline std::string to_text(const char* s) { return s; }
inline std::string to_text(const std::string& s) { return s; }
template <class T>
std::string to_text(T v)
{
  return std::to_string(v);
}
}  // namespace detail

template <class T>
Validator IsMember(std::initializer_list<T> items)
{
  std::vector<std::string> set;
  for (const T& i : items)
    set.push_back(detail::to_text(i));
  return {[set](const std::string& v) -> std::string
          {
            for (const std::string& s : set)
              if (s == v)
                return "";
            return v + " not in {" + [&] { std::string o; for (const auto& s : set) o += (o.empty() ? "" : ",") + s; return o; }() + "}";
          }};
}
inline Validator Range(double lo, double hi)
{
  return {[lo, hi](const std::string& v) -> std::string
          {
            double x = 0;
            if (!detail::parse(v, x) || x < lo || x > hi)
              return "value " + v + " not in range [" + std::to_string(lo) + " - " + std::to_string(hi) + "]";
            return "";
          }};
}
inline const Validator PositiveNumber{[](const std::string& v) -> std::string
                                      {
                                        double x = 0;
                                        if (!detail::parse(v, x) || !(x > 0))
                                          return "value " + v + " is not a positive number";
                                        return "";
                                      }};

class Option {
 public:
  Option(std::string name, std::function<bool(const std::string&)> set, bool list, bool flag)
      : name_(std::move(name)), set_(std::move(set)), list_(list), flag_(flag)
  {
  }
  Option* check(const Validator& v)
  {
    validators_.push_back(v);
    return this;
  }
  Option* capture_default_str() { return this; }
  Option* default_str(const std::string&) { return this; }
  Option* delimiter(char d)
  {
    delim_ = d;
    return this;
  }
  const std::string& name() const { return name_; }
  bool is_flag() const { return flag_; }
  std::size_t count() const { return count_; }
  void take(const std::string& raw)
  {
    std::vector<std::string> parts;
    if (list_ && delim_)
    {
      std::string cur;
      std::istringstream is(raw);
      while (std::getline(is, cur, delim_))
        parts.push_back(cur);
    }
    else
      parts.push_back(raw);
    for (const std::string& p : parts)
    {
      for (const Validator& v : validators_)
      {
        const std::string why = v.check(p);
        if (!why.empty())
          throw ParseError(name_ + ": " + why, 105);
      }
      if (!set_(p))
        throw ParseError(name_ + ": could not convert '" + p + "'", 106);
    }
    ++count_;
  }

 private:
  std::string name_;
  std::function<bool(const std::string&)> set_;
  bool list_, flag_;
  char delim_ = 0;
  std::vector<Validator> validators_;
  std::size_t count_ = 0;
};

class App {
 public:
  explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}
  void require_subcommand(int n) { require_ = n; }
  App* add_subcommand(const std::string& name, const std::string& description = "")
  {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }
  template <class T>
  Option* add_option(const std::string& name, T& ref, const std::string& = "")
  {
    std::function<bool(const std::string&)> set;
    bool list = false;
    if constexpr (std::is_same_v<T, std::vector<int>> || std::is_same_v<T, std::vector<std::string>>)
    {
      list = true;
      set = [&ref, first = std::make_shared<bool>(true)](const std::string& s)
      {
        typename T::value_type v{};
        if (!detail::parse(s, v))
          return false;
        ref.push_back(v);
        return true;
      };
    }
    else
      set = [&ref](const std::string& s) { return detail::parse(s, ref); };
    opts_.push_back(std::make_unique<Option>(name, set, list, false));
    return opts_.back().get();
  }
  Option* add_flag(const std::string& name, bool& ref, const std::string& = "")
  {
    opts_.push_back(std::make_unique<Option>(name, [&ref](const std::string&) { ref = true; return true; }, false, true));
    return opts_.back().get();
  }
  std::size_t count(const std::string& name) const
  {
    for (const auto& o : opts_)
      if (o->name() == name)
        return o->count();
    return 0;
  }
  bool got_subcommand(const App* sub) const { return sub == chosen_; }
  void parse(int argc, char** argv)
  {
    App* target = this;
    int i = 1;
    if (!subs_.empty())
    {
      if (argc < 2)
      {
        if (require_ > 0)
          throw ParseError("a subcommand is required", 106);
      }
      else
      {
        for (auto& s : subs_)
          if (s->name_ == argv[1])
            target = chosen_ = s.get();
        if (!chosen_)
          throw ParseError(std::string("unknown subcommand ") + argv[1], 109);
        i = 2;
      }
    }
    for (; i < argc; ++i)
    {
      std::string a = argv[i], value;
      const bool has_eq = a.find('=') != std::string::npos;
      if (has_eq)
      {
        value = a.substr(a.find('=') + 1);
        a = a.substr(0, a.find('='));
      }
      Option* o = nullptr;
      for (auto& p : target->opts_)
        if (p->name() == a)
          o = p.get();
      if (!o)
        throw ParseError("the following argument was not expected: " + a, 109);
      if (o->is_flag())
        o->take("");
      else
      {
        if (!has_eq)
        {
          if (i + 1 >= argc)
            throw ParseError(a + " requires a value", 106);
          value = argv[++i];
        }
        o->take(value);
      }
    }
  }
  int exit(const ParseError& e) const
  {
    std::fprintf(stderr, "%s\n", e.what());
    return e.exit_code;
  }

 private:
  std::string desc_, name_;
  int require_ = 0;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  App* chosen_ = nullptr;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv) \
  try                                \
  {                                  \
    (app).parse((argc), (argv));     \
  }                                  \
  catch (const CLI::ParseError& e)   \
  {                                  \
    return (app).exit(e);            \
  }
