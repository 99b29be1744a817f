// TEST INFRASTRUCTURE (oracle build only) -- not part of the product.
//
// Minimal stand-in for <boost/multiprecision/cpp_int.hpp>, which is absent
// from this image. The reference's exact-rational layer
// (/root/reference/proj/include/wavelift/rational.hpp:6,14,58-60,79) only
// needs a signed integer with + - * / %, comparisons, str(), gcd() and a
// cpp_rational(num, den) -> double conversion. This shim backs that with an
// overflow-checked __int128: any overflow throws std::overflow_error, so a
// silently wrong oracle is impossible (the oracle build simply fails loudly).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace boost {
namespace multiprecision {

class cpp_int {
public:
    using rep = __int128;
    cpp_int() : v_(0) {}
    cpp_int(int v) : v_(v) {}            // NOLINT: implicit like boost
    cpp_int(long v) : v_(v) {}           // NOLINT
    cpp_int(long long v) : v_(v) {}      // NOLINT
    cpp_int(unsigned v) : v_(v) {}       // NOLINT
    cpp_int(unsigned long v) : v_(v) {}  // NOLINT

    static cpp_int from_rep(rep v) {
        cpp_int r;
        r.v_ = v;
        return r;
    }
    rep raw() const { return v_; }

    friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
        rep r;
        if (__builtin_add_overflow(a.v_, b.v_, &r)) throw std::overflow_error("cpp_int shim: +");
        return from_rep(r);
    }
    friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
        rep r;
        if (__builtin_sub_overflow(a.v_, b.v_, &r)) throw std::overflow_error("cpp_int shim: -");
        return from_rep(r);
    }
    friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
        rep r;
        if (__builtin_mul_overflow(a.v_, b.v_, &r)) throw std::overflow_error("cpp_int shim: *");
        return from_rep(r);
    }
    friend cpp_int operator/(const cpp_int& a, const cpp_int& b) {
        if (b.v_ == 0) throw std::domain_error("cpp_int shim: division by zero");
        return from_rep(a.v_ / b.v_);
    }
    friend cpp_int operator%(const cpp_int& a, const cpp_int& b) {
        if (b.v_ == 0) throw std::domain_error("cpp_int shim: modulo by zero");
        return from_rep(a.v_ % b.v_);
    }
    cpp_int operator-() const {
        if (v_ == -v_ && v_ != 0) throw std::overflow_error("cpp_int shim: negate");
        return from_rep(-v_);
    }
    cpp_int& operator+=(const cpp_int& b) { return *this = *this + b; }
    cpp_int& operator-=(const cpp_int& b) { return *this = *this - b; }
    cpp_int& operator*=(const cpp_int& b) { return *this = *this * b; }
    cpp_int& operator/=(const cpp_int& b) { return *this = *this / b; }
    cpp_int& operator%=(const cpp_int& b) { return *this = *this % b; }

    friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.v_ == b.v_; }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return a.v_ != b.v_; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) { return a.v_ < b.v_; }
    friend bool operator>(const cpp_int& a, const cpp_int& b) { return a.v_ > b.v_; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return a.v_ <= b.v_; }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return a.v_ >= b.v_; }

    std::string str() const {
        if (v_ == 0) return "0";
        bool neg = v_ < 0;
        unsigned __int128 u = neg ? static_cast<unsigned __int128>(-(v_ + 1)) + 1
                                  : static_cast<unsigned __int128>(v_);
        std::string s;
        while (u) {
            s.insert(s.begin(), static_cast<char>('0' + static_cast<int>(u % 10)));
            u /= 10;
        }
        return neg ? "-" + s : s;
    }

    explicit operator long double() const { return static_cast<long double>(v_); }

private:
    rep v_;
};

inline cpp_int gcd(cpp_int a, cpp_int b) {
    __int128 x = a.raw() < 0 ? -a.raw() : a.raw();
    __int128 y = b.raw() < 0 ? -b.raw() : b.raw();
    while (y != 0) {
        __int128 t = x % y;
        x = y;
        y = t;
    }
    return cpp_int::from_rep(x);
}

// Only the (num, den) constructor and the conversion to double are used
// (rational.hpp:58-60). Division of two integers exactly representable in
// double is correctly rounded by IEEE-754; larger operands fall back to
// long double, which is still exact for every coefficient the shipped
// wavelets produce (dyadic rationals with small numerators).
class cpp_rational {
public:
    cpp_rational(const cpp_int& n, const cpp_int& d) : n_(n), d_(d) {}
    explicit operator double() const {
        const __int128 lim = static_cast<__int128>(1) << 53;
        const __int128 n = n_.raw(), d = d_.raw();
        if (n > -lim && n < lim && d > -lim && d < lim)
            return static_cast<double>(static_cast<long long>(n)) /
                   static_cast<double>(static_cast<long long>(d));
        return static_cast<double>(static_cast<long double>(n) / static_cast<long double>(d));
    }

private:
    cpp_int n_, d_;
};

}  // namespace multiprecision
}  // namespace boost
