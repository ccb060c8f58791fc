// CLI11.hpp -- COMPILE-ONLY stand-in for CLI11 (absent from the reference
// tree).  Used only by integration/check_patch.sh to type-check the patched
// tools/coopcg.cpp; it declares the subset of CLI::App / CLI::Option the
// reference's CLI calls and parses nothing.
#pragma once
#include <cstddef>
#include <deque>
#include <string>

namespace CLI {
class Option {
public:
    Option* required(bool = true) { return this; }
};
class App {
public:
    explicit App(std::string = "") {}
    App* add_subcommand(const std::string&, const std::string& = "") { return &subs_.emplace_back(); }
    template <class T>
    Option* add_option(const std::string&, T&, const std::string& = "") { return &opt_; }
    template <class T>
    Option* add_flag(const std::string&, T&, const std::string& = "") { return &opt_; }
    void require_subcommand(int = 1) {}
    std::size_t count(const std::string&) const { return 0; }
    explicit operator bool() const { return false; }
    int parse(int, char**) { return 0; }

private:
    std::deque<App> subs_;
    Option opt_;
};
}  // namespace CLI

#define CLI11_PARSE(app, argc, argv) (app).parse((argc), (argv))
