/*
 * TEST INFRASTRUCTURE ONLY (oracle build shim) -- never linked into the product.
 *
 * Stand-in for the slice of Boost.Multiprecision the reference's
 * src/fc_core.cpp:5,22,58 uses: number<mpfr_float_backend<120>> with + - * /,
 * compound assignment, comparisons, abs/cos/sin, explicit double conversion,
 * and boost::math::constants::pi<T>(). Boost is absent from this image; the
 * MPFR runtime (libmpfr.so.6, MPFR 4.2.1) is present, so this header declares
 * the handful of MPFR prototypes it needs by hand and links that library.
 * Precision: Boost maps 120 decimal digits to 400 bits (digits10*1000/301+2).
 */
#ifndef ORACLE_SHIM_BOOST_MP_MPFR_HPP
#define ORACLE_SHIM_BOOST_MP_MPFR_HPP

#include <type_traits>
#include <utility>

extern "C" {
typedef struct {
    long _mpfr_prec;
    int _mpfr_sign;
    long _mpfr_exp;
    unsigned long* _mpfr_d;
} oracle_mpfr_struct;
typedef oracle_mpfr_struct* oracle_mpfr_ptr;
typedef const oracle_mpfr_struct* oracle_mpfr_srcptr;
void mpfr_init2(oracle_mpfr_ptr, long);
void mpfr_clear(oracle_mpfr_ptr);
int mpfr_set(oracle_mpfr_ptr, oracle_mpfr_srcptr, int);
int mpfr_set_si(oracle_mpfr_ptr, long, int);
int mpfr_set_d(oracle_mpfr_ptr, double, int);
double mpfr_get_d(oracle_mpfr_srcptr, int);
int mpfr_add(oracle_mpfr_ptr, oracle_mpfr_srcptr, oracle_mpfr_srcptr, int);
int mpfr_sub(oracle_mpfr_ptr, oracle_mpfr_srcptr, oracle_mpfr_srcptr, int);
int mpfr_mul(oracle_mpfr_ptr, oracle_mpfr_srcptr, oracle_mpfr_srcptr, int);
int mpfr_div(oracle_mpfr_ptr, oracle_mpfr_srcptr, oracle_mpfr_srcptr, int);
int mpfr_abs(oracle_mpfr_ptr, oracle_mpfr_srcptr, int);
int mpfr_cos(oracle_mpfr_ptr, oracle_mpfr_srcptr, int);
int mpfr_sin(oracle_mpfr_ptr, oracle_mpfr_srcptr, int);
int mpfr_const_pi(oracle_mpfr_ptr, int);
int mpfr_cmp(oracle_mpfr_srcptr, oracle_mpfr_srcptr);
}

namespace boost {
namespace multiprecision {

template <unsigned Digits10>
struct mpfr_float_backend {
    static constexpr long bits = Digits10 * 1000L / 301L + ((Digits10 * 1000L) % 301 ? 2 : 1);
};

template <class Backend>
class number;

template <unsigned D>
class number<mpfr_float_backend<D>> {
  public:
    static constexpr long kBits = mpfr_float_backend<D>::bits;
    static constexpr int kRnd = 0;  // MPFR_RNDN

    number() { mpfr_init2(v_, kBits); mpfr_set_si(v_, 0, kRnd); }
    number(const number& o) { mpfr_init2(v_, kBits); mpfr_set(v_, o.v_, kRnd); }
    number(number&& o) noexcept { mpfr_init2(v_, kBits); mpfr_set(v_, o.v_, kRnd); }
    template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
    number(T x, int = 0) { mpfr_init2(v_, kBits); mpfr_set_si(v_, static_cast<long>(x), kRnd); }
    number(double x) { mpfr_init2(v_, kBits); mpfr_set_d(v_, x, kRnd); }
    ~number() { mpfr_clear(v_); }

    number& operator=(const number& o) { if (this != &o) mpfr_set(v_, o.v_, kRnd); return *this; }
    number& operator=(number&& o) noexcept { if (this != &o) mpfr_set(v_, o.v_, kRnd); return *this; }
    template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
    number& operator=(T x) { *this = number(x); return *this; }

    explicit operator double() const { return mpfr_get_d(v_, kRnd); }

    number& operator+=(const number& o) { mpfr_add(v_, v_, o.v_, kRnd); return *this; }
    number& operator-=(const number& o) { mpfr_sub(v_, v_, o.v_, kRnd); return *this; }
    number& operator*=(const number& o) { mpfr_mul(v_, v_, o.v_, kRnd); return *this; }
    number& operator/=(const number& o) { mpfr_div(v_, v_, o.v_, kRnd); return *this; }

    friend number operator+(number a, const number& b) { a += b; return a; }
    friend number operator-(number a, const number& b) { a -= b; return a; }
    friend number operator*(number a, const number& b) { a *= b; return a; }
    friend number operator/(number a, const number& b) { a /= b; return a; }
    number operator-() const { number r; mpfr_sub(r.v_, r.v_, v_, kRnd); return r; }

    friend int cmp(const number& a, const number& b) { return mpfr_cmp(a.v_, b.v_); }
    friend bool operator<(const number& a, const number& b) { return cmp(a, b) < 0; }
    friend bool operator>(const number& a, const number& b) { return cmp(a, b) > 0; }
    friend bool operator<=(const number& a, const number& b) { return cmp(a, b) <= 0; }
    friend bool operator>=(const number& a, const number& b) { return cmp(a, b) >= 0; }
    friend bool operator==(const number& a, const number& b) { return cmp(a, b) == 0; }
    friend bool operator!=(const number& a, const number& b) { return cmp(a, b) != 0; }

    friend number abs(const number& a) { number r; mpfr_abs(r.v_, a.v_, kRnd); return r; }
    friend number cos(const number& a) { number r; mpfr_cos(r.v_, a.v_, kRnd); return r; }
    friend number sin(const number& a) { number r; mpfr_sin(r.v_, a.v_, kRnd); return r; }

    static number pi() { number r; mpfr_const_pi(r.v_, kRnd); return r; }

  private:
    oracle_mpfr_struct v_[1];
};

// mixed arithmetic with built-in scalars (int * MP, MP / int, MP > double ...)
#define ORACLE_MP_MIXED(OP)                                                              \
    template <unsigned D, class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>   \
    number<mpfr_float_backend<D>> operator OP(const number<mpfr_float_backend<D>>& a, T b) { \
        return a OP number<mpfr_float_backend<D>>(b);                                    \
    }                                                                                    \
    template <unsigned D, class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>   \
    number<mpfr_float_backend<D>> operator OP(T a, const number<mpfr_float_backend<D>>& b) { \
        return number<mpfr_float_backend<D>>(a) OP b;                                    \
    }
ORACLE_MP_MIXED(+)
ORACLE_MP_MIXED(-)
ORACLE_MP_MIXED(*)
ORACLE_MP_MIXED(/)
#undef ORACLE_MP_MIXED

#define ORACLE_MP_CMP(OP)                                                               \
    template <unsigned D, class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>  \
    bool operator OP(const number<mpfr_float_backend<D>>& a, T b) {                     \
        return a OP number<mpfr_float_backend<D>>(b);                                   \
    }                                                                                   \
    template <unsigned D, class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>  \
    bool operator OP(T a, const number<mpfr_float_backend<D>>& b) {                     \
        return number<mpfr_float_backend<D>>(a) OP b;                                   \
    }
ORACLE_MP_CMP(<)
ORACLE_MP_CMP(>)
ORACLE_MP_CMP(<=)
ORACLE_MP_CMP(>=)
ORACLE_MP_CMP(==)
ORACLE_MP_CMP(!=)
#undef ORACLE_MP_CMP

}  // namespace multiprecision

namespace math {
namespace constants {
template <class T>
T pi() {
    return T::pi();
}
}  // namespace constants
}  // namespace math
}  // namespace boost

#endif
