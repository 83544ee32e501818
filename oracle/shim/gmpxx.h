// Minimal gmpxx.h stand-in for building the reference oracle (test
// infrastructure only).  The image ships the GMP runtime (libgmp.so.10) but
// neither gmp.h nor gmpxx.h, so this header declares the handful of
// libgmp entry points the reference's ExactValue (proj/src/oracle.cpp:88-214)
// and its doctest suites use, and wraps them in tiny mpz_class / mpq_class
// value types.  Written from the public GMP ABI; nothing here is copied.
#ifndef OZ_ORACLE_SHIM_GMPXX_H
#define OZ_ORACLE_SHIM_GMPXX_H

#include <cstddef>
#include <ostream>
#include <stdexcept>
#include <string>

extern "C" {
typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef unsigned long mp_bitcnt_t;
typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t* _mp_d;
} __mpz_struct;
typedef struct {
  __mpz_struct _mp_num;
  __mpz_struct _mp_den;
} __mpq_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpq_struct mpq_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;
typedef __mpq_struct* mpq_ptr;
typedef const __mpq_struct* mpq_srcptr;

void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_si(mpz_ptr, long);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_si(mpz_ptr, mpz_srcptr, long);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
mp_bitcnt_t __gmpz_scan1(mpz_srcptr, mp_bitcnt_t);
long __gmpz_get_si(mpz_srcptr);
int __gmpz_fits_slong_p(mpz_srcptr);
char* __gmpz_get_str(char*, int, mpz_srcptr);

void __gmpq_init(mpq_ptr);
void __gmpq_clear(mpq_ptr);
void __gmpq_set(mpq_ptr, mpq_srcptr);
void __gmpq_set_d(mpq_ptr, double);
void __gmpq_set_si(mpq_ptr, long, unsigned long);
void __gmpq_add(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_sub(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_mul(mpq_ptr, mpq_srcptr, mpq_srcptr);
double __gmpq_get_d(mpq_srcptr);
}

// C-level names the reference calls directly.
inline size_t mpz_sizeinbase(mpz_srcptr z, int base) { return __gmpz_sizeinbase(z, base); }
inline mp_bitcnt_t mpz_scan1(mpz_srcptr z, mp_bitcnt_t from) { return __gmpz_scan1(z, from); }
inline unsigned long mpz_get_ui(mpz_srcptr z) { return z->_mp_size != 0 ? z->_mp_d[0] : 0UL; }
inline bool mpz_even_p(mpz_srcptr z) { return z->_mp_size == 0 || (z->_mp_d[0] & 1UL) == 0; }

class mpz_class {
 public:
  mpz_class() { __gmpz_init(v_); }
  mpz_class(int x) { __gmpz_init_set_si(v_, x); }
  mpz_class(long x) { __gmpz_init_set_si(v_, x); }
  mpz_class(unsigned long x) { __gmpz_init_set_ui(v_, x); }
  mpz_class(unsigned int x) { __gmpz_init_set_ui(v_, x); }
  mpz_class(const mpz_class& o) { __gmpz_init_set(v_, o.v_); }
  ~mpz_class() { __gmpz_clear(v_); }
  mpz_class& operator=(const mpz_class& o) {
    if (this != &o) __gmpz_set(v_, o.v_);
    return *this;
  }
  mpz_class& operator=(int x) { __gmpz_set_si(v_, x); return *this; }
  mpz_class& operator=(long x) { __gmpz_set_si(v_, x); return *this; }
  mpz_class& operator=(unsigned long x) { __gmpz_set_ui(v_, x); return *this; }

  mpz_class& operator+=(const mpz_class& o) { __gmpz_add(v_, v_, o.v_); return *this; }
  mpz_class& operator-=(const mpz_class& o) { __gmpz_sub(v_, v_, o.v_); return *this; }
  mpz_class& operator*=(const mpz_class& o) { __gmpz_mul(v_, v_, o.v_); return *this; }
  mpz_class& operator+=(long x) { mpz_class t(x); return *this += t; }
  mpz_class& operator-=(long x) { mpz_class t(x); return *this -= t; }
  mpz_class& operator+=(int x) { return *this += static_cast<long>(x); }
  mpz_class& operator-=(int x) { return *this -= static_cast<long>(x); }
  mpz_class& operator+=(unsigned long x) { mpz_class t(x); return *this += t; }
  mpz_class& operator*=(long x) { __gmpz_mul_si(v_, v_, x); return *this; }
  mpz_class& operator*=(int x) { __gmpz_mul_si(v_, v_, x); return *this; }
  mpz_class& operator<<=(unsigned long s) { __gmpz_mul_2exp(v_, v_, s); return *this; }
  mpz_class& operator<<=(unsigned int s) { return *this <<= static_cast<unsigned long>(s); }
  mpz_class& operator<<=(int s) { return *this <<= static_cast<unsigned long>(s); }
  mpz_class& operator>>=(unsigned long s) { __gmpz_fdiv_q_2exp(v_, v_, s); return *this; }
  mpz_class& operator>>=(int s) { return *this >>= static_cast<unsigned long>(s); }
  mpz_class operator-() const { mpz_class r; __gmpz_neg(r.v_, v_); return r; }

  bool fits_slong_p() const { return __gmpz_fits_slong_p(v_) != 0; }
  long get_si() const { return __gmpz_get_si(v_); }
  std::string get_str(int base = 10) const {
    char* s = __gmpz_get_str(nullptr, base, v_);
    std::string out(s);
    std::free(s);
    return out;
  }
  mpz_ptr get_mpz_t() { return v_; }
  mpz_srcptr get_mpz_t() const { return v_; }

  friend int cmp(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_); }
  friend int cmp(const mpz_class& a, long b) { return __gmpz_cmp_si(a.v_, b); }

 private:
  mpz_t v_;
};

inline mpz_class abs(const mpz_class& a) {
  mpz_class r;
  __gmpz_abs(r.get_mpz_t(), a.get_mpz_t());
  return r;
}
inline int sgn(const mpz_class& a) { return a.get_mpz_t()->_mp_size < 0 ? -1 : (a.get_mpz_t()->_mp_size > 0 ? 1 : 0); }
inline mpz_class operator+(mpz_class a, const mpz_class& b) { return a += b; }
inline mpz_class operator-(mpz_class a, const mpz_class& b) { return a -= b; }
inline mpz_class operator*(mpz_class a, const mpz_class& b) { return a *= b; }
inline mpz_class operator*(mpz_class a, long b) { return a *= b; }
inline mpz_class operator*(mpz_class a, int b) { return a *= static_cast<long>(b); }
inline mpz_class operator<<(mpz_class a, unsigned long s) { return a <<= s; }
inline mpz_class operator<<(mpz_class a, int s) { return a <<= static_cast<unsigned long>(s); }
inline mpz_class operator>>(mpz_class a, unsigned long s) { return a >>= s; }
inline bool operator==(const mpz_class& a, const mpz_class& b) { return cmp(a, b) == 0; }
inline bool operator!=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) != 0; }
inline bool operator<(const mpz_class& a, const mpz_class& b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpz_class& a, const mpz_class& b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) >= 0; }
inline bool operator==(const mpz_class& a, long b) { return cmp(a, b) == 0; }
inline bool operator!=(const mpz_class& a, long b) { return cmp(a, b) != 0; }
inline bool operator<(const mpz_class& a, long b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpz_class& a, long b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpz_class& a, long b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpz_class& a, long b) { return cmp(a, b) >= 0; }
inline bool operator==(const mpz_class& a, int b) { return cmp(a, static_cast<long>(b)) == 0; }
inline bool operator!=(const mpz_class& a, int b) { return cmp(a, static_cast<long>(b)) != 0; }
inline bool operator<(const mpz_class& a, int b) { return cmp(a, static_cast<long>(b)) < 0; }
inline bool operator>(const mpz_class& a, int b) { return cmp(a, static_cast<long>(b)) > 0; }
inline std::ostream& operator<<(std::ostream& os, const mpz_class& a) { return os << a.get_str(); }

class mpq_class {
 public:
  mpq_class() { __gmpq_init(v_); }
  mpq_class(int x) { __gmpq_init(v_); __gmpq_set_si(v_, x, 1UL); }
  mpq_class(long x) { __gmpq_init(v_); __gmpq_set_si(v_, x, 1UL); }
  mpq_class(double x) { __gmpq_init(v_); __gmpq_set_d(v_, x); }
  mpq_class(const mpq_class& o) { __gmpq_init(v_); __gmpq_set(v_, o.v_); }
  ~mpq_class() { __gmpq_clear(v_); }
  mpq_class& operator=(const mpq_class& o) {
    if (this != &o) __gmpq_set(v_, o.v_);
    return *this;
  }
  mpq_class& operator+=(const mpq_class& o) { __gmpq_add(v_, v_, o.v_); return *this; }
  mpq_class& operator-=(const mpq_class& o) { __gmpq_sub(v_, v_, o.v_); return *this; }
  mpq_class& operator*=(const mpq_class& o) { __gmpq_mul(v_, v_, o.v_); return *this; }
  double get_d() const { return __gmpq_get_d(v_); }
  mpq_ptr get_mpq_t() { return v_; }
  mpq_srcptr get_mpq_t() const { return v_; }

 private:
  mpq_t v_;
};

inline mpq_class operator+(mpq_class a, const mpq_class& b) { return a += b; }
inline mpq_class operator-(mpq_class a, const mpq_class& b) { return a -= b; }
inline mpq_class operator*(mpq_class a, const mpq_class& b) { return a *= b; }

#endif  // OZ_ORACLE_SHIM_GMPXX_H
