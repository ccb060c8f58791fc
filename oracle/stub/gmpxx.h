// Compile-only stand-in for GMP's C++ header.  TEST INFRASTRUCTURE.
//
// The reference's coopcg/scalar.hpp:5 includes <gmpxx.h> unconditionally,
// but only its exact-rational mode uses it.  GMP's development headers are
// not installed in this image, so this stub declares the names the float
// path's translation unit needs to parse; every body aborts.  The float
// (double) path never calls any of them.
#pragma once
#include <cstdlib>
#include <string>

struct __mpz_struct_stub { int unused; };
inline void mpz_ui_pow_ui(__mpz_struct_stub*, unsigned long, unsigned long) { std::abort(); }

class mpz_class {
public:
    mpz_class() = default;
    mpz_class(long) { std::abort(); }
    mpz_class(const std::string&, int) { std::abort(); }
    __mpz_struct_stub* get_mpz_t() { std::abort(); }
    std::string get_str(int = 10) const { std::abort(); }
};
inline mpz_class operator+(const mpz_class&, const mpz_class&) { std::abort(); }
inline mpz_class operator-(const mpz_class&, const mpz_class&) { std::abort(); }
inline mpz_class operator*(const mpz_class&, const mpz_class&) { std::abort(); }
inline mpz_class operator/(const mpz_class&, const mpz_class&) { std::abort(); }
inline int sgn(const mpz_class&) { std::abort(); }

class mpq_class {
public:
    mpq_class() = default;
    mpq_class(long) { std::abort(); }
    mpq_class(int) { std::abort(); }
    mpq_class(long, long) { std::abort(); }
    mpq_class(const mpz_class&, const mpz_class&) { std::abort(); }
    mpq_class(const mpz_class&, long) { std::abort(); }
    mpq_class(long, const mpz_class&) { std::abort(); }
    void canonicalize() { std::abort(); }
    double get_d() const { std::abort(); }
    mpz_class get_num() const { std::abort(); }
    mpz_class get_den() const { std::abort(); }
    int set_str(const std::string&, int) { std::abort(); }
    mpq_class operator-() const { std::abort(); }
    mpq_class& operator+=(const mpq_class&) { std::abort(); }
    mpq_class& operator-=(const mpq_class&) { std::abort(); }
    mpq_class& operator*=(const mpq_class&) { std::abort(); }
    mpq_class& operator/=(const mpq_class&) { std::abort(); }
    bool operator==(const mpq_class&) const { std::abort(); }
};
inline mpq_class operator+(const mpq_class&, const mpq_class&) { std::abort(); }
inline mpq_class operator-(const mpq_class&, const mpq_class&) { std::abort(); }
inline mpq_class operator*(const mpq_class&, const mpq_class&) { std::abort(); }
inline mpq_class operator/(const mpq_class&, const mpq_class&) { std::abort(); }
inline bool operator<(const mpq_class&, const mpq_class&) { std::abort(); }
inline bool operator>(const mpq_class&, const mpq_class&) { std::abort(); }
inline bool operator<=(const mpq_class&, const mpq_class&) { std::abort(); }
inline bool operator>=(const mpq_class&, const mpq_class&) { std::abort(); }
inline bool operator!=(const mpq_class&, const mpq_class&) { std::abort(); }
inline int sgn(const mpq_class&) { std::abort(); }
inline mpq_class abs(const mpq_class&) { std::abort(); }
