// Minimal stand-in for boost/multiprecision/cpp_int.hpp, used ONLY to compile
// the read-only reference (/root/reference/proj/src/fd.cpp and its tests) into
// oracle/_ref/. Boost is not installed in this image and there is no network.
//
// TEST INFRASTRUCTURE: nothing on the product path includes this header.
//
// Surface covered (everything fd.cpp:14-72, acceptance.cpp:52-87 and
// test_fd.cpp:21-55 use): cpp_rational from integers, + - * /, += -= *=,
// comparisons with 0, mp::numerator / mp::denominator returning cpp_int,
// cpp_int comparisons against int64 limits and convert_to<long long>().
//
// Storage is __int128 with every operation overflow-checked: the exact
// Gauss-Jordan intermediates of fd_weights peak at 60 bits for accuracy
// order 16, so 127 bits leave ample headroom. Any overflow aborts loudly
// instead of silently losing exactness.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

namespace boost {
namespace multiprecision {

namespace shim_detail {

using i128 = __int128;

[[noreturn]] inline void overflow(const char* what) {
    std::fprintf(stderr, "boost shim: 128-bit overflow in %s\n", what);
    std::abort();
}

inline i128 mul(i128 a, i128 b) {
    i128 r;
    if (__builtin_mul_overflow(a, b, &r)) overflow("mul");
    return r;
}
inline i128 add(i128 a, i128 b) {
    i128 r;
    if (__builtin_add_overflow(a, b, &r)) overflow("add");
    return r;
}
inline i128 sub(i128 a, i128 b) {
    i128 r;
    if (__builtin_sub_overflow(a, b, &r)) overflow("sub");
    return r;
}
inline i128 abs128(i128 a) { return a < 0 ? -a : a; }
inline i128 gcd(i128 a, i128 b) {
    a = abs128(a);
    b = abs128(b);
    while (b != 0) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a == 0 ? 1 : a;
}

} // namespace shim_detail

class cpp_int {
  public:
    cpp_int() : v_(0) {}
    cpp_int(shim_detail::i128 v) : v_(v) {}
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
    cpp_int(T v) : v_(static_cast<shim_detail::i128>(v)) {}

    template <typename T>
    T convert_to() const {
        return static_cast<T>(v_);
    }
    shim_detail::i128 raw() const { return v_; }

    friend bool operator>(const cpp_int& a, const cpp_int& b) { return a.v_ > b.v_; }
    friend bool operator<(const cpp_int& a, const cpp_int& b) { return a.v_ < b.v_; }
    friend bool operator>=(const cpp_int& a, const cpp_int& b) { return a.v_ >= b.v_; }
    friend bool operator<=(const cpp_int& a, const cpp_int& b) { return a.v_ <= b.v_; }
    friend bool operator==(const cpp_int& a, const cpp_int& b) { return a.v_ == b.v_; }
    friend bool operator!=(const cpp_int& a, const cpp_int& b) { return a.v_ != b.v_; }

  private:
    shim_detail::i128 v_;
};

class cpp_rational {
  public:
    cpp_rational() : n_(0), d_(1) {}
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
    cpp_rational(T v) : n_(static_cast<shim_detail::i128>(v)), d_(1) {}
    cpp_rational(shim_detail::i128 n, shim_detail::i128 d) : n_(n), d_(d) {
        normalize();
    }

    shim_detail::i128 num() const { return n_; }
    shim_detail::i128 den() const { return d_; }

    friend cpp_rational operator+(const cpp_rational& a, const cpp_rational& b) {
        using namespace shim_detail;
        i128 g = gcd(a.d_, b.d_);
        i128 da = a.d_ / g, db = b.d_ / g;
        return cpp_rational(add(mul(a.n_, db), mul(b.n_, da)), mul(a.d_, db));
    }
    friend cpp_rational operator-(const cpp_rational& a, const cpp_rational& b) {
        using namespace shim_detail;
        i128 g = gcd(a.d_, b.d_);
        i128 da = a.d_ / g, db = b.d_ / g;
        return cpp_rational(sub(mul(a.n_, db), mul(b.n_, da)), mul(a.d_, db));
    }
    friend cpp_rational operator*(const cpp_rational& a, const cpp_rational& b) {
        using namespace shim_detail;
        // cross-reduce first to keep intermediates small
        i128 g1 = gcd(a.n_, b.d_);
        i128 g2 = gcd(b.n_, a.d_);
        return cpp_rational(mul(a.n_ / g1, b.n_ / g2), mul(a.d_ / g2, b.d_ / g1));
    }
    friend cpp_rational operator/(const cpp_rational& a, const cpp_rational& b) {
        if (b.n_ == 0) {
            std::fprintf(stderr, "boost shim: rational division by zero\n");
            std::abort();
        }
        return a * cpp_rational(b.d_, b.n_);
    }
    cpp_rational operator-() const { return cpp_rational(-n_, d_); }

    cpp_rational& operator+=(const cpp_rational& o) { return *this = *this + o; }
    cpp_rational& operator-=(const cpp_rational& o) { return *this = *this - o; }
    cpp_rational& operator*=(const cpp_rational& o) { return *this = *this * o; }
    cpp_rational& operator/=(const cpp_rational& o) { return *this = *this / o; }

    friend bool operator==(const cpp_rational& a, const cpp_rational& b) {
        return a.n_ == b.n_ && a.d_ == b.d_;
    }
    friend bool operator!=(const cpp_rational& a, const cpp_rational& b) {
        return !(a == b);
    }

  private:
    void normalize() {
        using namespace shim_detail;
        if (d_ == 0) {
            std::fprintf(stderr, "boost shim: zero denominator\n");
            std::abort();
        }
        if (d_ < 0) {
            n_ = -n_;
            d_ = -d_;
        }
        i128 g = gcd(n_, d_);
        n_ /= g;
        d_ /= g;
    }

    shim_detail::i128 n_;
    shim_detail::i128 d_;
};

inline cpp_int numerator(const cpp_rational& r) { return cpp_int(r.num()); }
inline cpp_int denominator(const cpp_rational& r) { return cpp_int(r.den()); }

} // namespace multiprecision
} // namespace boost
