// hadacodec-b200: on-disk / wire formats of the hot path's data,
// produced on the GPU.
//
//   print_g17 ("%.17g", io.cpp:108-112) of every code / weight value, and the codes CSV
//   (write_codes_csv, io.cpp:312-330: "id,c0,...,c{k-1}\n" then "id,v0,...\n" per row).
//
// %.17g is the exact decimal value of the double rounded to 17 significant digits
// (round half to even on the exact binary value, as glibc's printf does), printed in
// the %g style: exponent form when the decimal exponent is < -4 or >= 17, else fixed;
// trailing zeros and a bare point removed.  The digits are generated exactly with
// multi-limb integers (32-bit limbs): the integer part by repeated division by 10^9,
// the fraction (left-aligned) by repeated multiplication by 10^9, whose carry-out is
// the next nine digits.  One thread formats one value; the CSV writer is a length pass,
// an exclusive scan of the row lengths and a write pass.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cctype>
#include <cstring>
#include <string>
#include <vector>

#include "hadacodec_b200.h"
#include "hc_internal.h"

namespace hcb {
namespace {

constexpr int kLimbs = 36;     // 1152 bits: the largest integer part (2^1024) / fraction (2^-1074)
constexpr int kSlot = 32;      // bytes per formatted value slot (%.17g needs <= 24)

struct Digits {
  char d[20];  // 17 significant digits (plus room)
  int exp10;   // decimal exponent of d[0]
};

// Exact decimal digits of a finite positive double, rounded half-even to 17 digits.
__device__ Digits digits17(double v) {
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
  const int be = static_cast<int>((bits >> 52) & 0x7ff);
  uint64_t m = bits & 0xfffffffffffffull;
  int e2;
  if (be == 0) {
    e2 = -1074;
  } else {
    m |= 1ull << 52;
    e2 = be - 1075;
  }
  // All significant digits we need: 17 + 1 rounding digit, plus a sticky flag.
  char buf[24];
  int nbuf = 0;   // digits collected (significant, i.e. after the first non-zero)
  int exp10 = 0;  // decimal exponent of the first significant digit
  bool sticky = false;
  uint32_t limb[kLimbs];

  // ---- integer part: I = m * 2^e2 (e2 >= 0) or m >> -e2
  int nl = 0;  // limbs in use
  if (e2 >= 0) {
    const int w = e2 >> 5, b = e2 & 31;
    for (int i = 0; i < kLimbs; ++i) limb[i] = 0;
    const uint64_t lo = m << b;                                     // bits [b, b + 53)
    const uint64_t hi = b ? (m >> (64 - b)) : 0;                    // spill
    limb[w] = static_cast<uint32_t>(lo);
    limb[w + 1] = static_cast<uint32_t>(lo >> 32);
    if (w + 2 < kLimbs) limb[w + 2] = static_cast<uint32_t>(hi);
    nl = w + 3 < kLimbs ? w + 3 : kLimbs;
  } else if (-e2 < 64) {
    const uint64_t ip = m >> (-e2);
    limb[0] = static_cast<uint32_t>(ip);
    limb[1] = static_cast<uint32_t>(ip >> 32);
    nl = 2;
  }
  while (nl > 0 && limb[nl - 1] == 0) --nl;
  const bool has_int = nl > 0;
  if (has_int) {
    // decimal chunks of 9 digits, least significant first
    uint32_t chunk[40];
    int nc = 0;
    while (nl > 0) {
      uint64_t rem = 0;
      for (int i = nl - 1; i >= 0; --i) {
        const uint64_t cur = (rem << 32) | limb[i];
        limb[i] = static_cast<uint32_t>(cur / 1000000000ull);
        rem = cur % 1000000000ull;
      }
      chunk[nc++] = static_cast<uint32_t>(rem);
      while (nl > 0 && limb[nl - 1] == 0) --nl;
    }
    // most significant chunk without leading zeros, the rest with 9 digits each
    char top[10];
    int nt = 0;
    uint32_t c = chunk[nc - 1];
    do {
      top[nt++] = static_cast<char>('0' + c % 10);
      c /= 10;
    } while (c);
    exp10 = nt - 1 + 9 * (nc - 1);
    for (int i = nt - 1; i >= 0; --i) {
      if (nbuf < 18) buf[nbuf++] = top[i];
      else if (top[i] != '0') sticky = true;
    }
    for (int j = nc - 2; j >= 0; --j) {
      uint32_t cc = chunk[j];
      char d9[9];
      for (int i = 8; i >= 0; --i) {
        d9[i] = static_cast<char>('0' + cc % 10);
        cc /= 10;
      }
      for (int i = 0; i < 9; ++i) {
        if (nbuf < 18) buf[nbuf++] = d9[i];
        else if (d9[i] != '0') sticky = true;
      }
    }
  }
  // ---- fraction: F = (m mod 2^s) / 2^s, s = -e2 > 0, left-aligned in L limbs
  if (e2 < 0) {
    const int s = -e2;
    const int L = (s + 31) >> 5;
    const int shift = 32 * L - s;  // left-align: F * 2^(32L)
    for (int i = 0; i < L; ++i) limb[i] = 0;
    const uint64_t frac = s >= 64 ? m : (m & ((1ull << s) - 1ull));
    // place frac << shift at bit 0 of a 32L-bit number
    {
      // frac has at most 53 bits; frac << shift spans up to 53 + 31 bits
      const int w = shift >> 5, b = shift & 31;
      const uint64_t lo = frac << b;
      const uint64_t hi = b ? (frac >> (64 - b)) : 0;
      if (w < L) limb[w] = static_cast<uint32_t>(lo);
      if (w + 1 < L) limb[w + 1] = static_cast<uint32_t>(lo >> 32);
      if (w + 2 < L) limb[w + 2] = static_cast<uint32_t>(hi);
    }
    int lo_limb = 0;  // limbs below this are zero
    while (lo_limb < L && limb[lo_limb] == 0) ++lo_limb;
    int zeros = 0;    // leading zero digits of the fraction (when there is no integer part)
    while (lo_limb < L && nbuf < 18) {
      uint64_t carry = 0;
      for (int i = lo_limb; i < L; ++i) {
        const uint64_t cur = static_cast<uint64_t>(limb[i]) * 1000000000ull + carry;
        limb[i] = static_cast<uint32_t>(cur);
        carry = cur >> 32;
      }
      while (lo_limb < L && limb[lo_limb] == 0) ++lo_limb;
      uint32_t c = static_cast<uint32_t>(carry);  // next nine digits
      char d9[9];
      for (int i = 8; i >= 0; --i) {
        d9[i] = static_cast<char>('0' + c % 10);
        c /= 10;
      }
      for (int i = 0; i < 9; ++i) {
        if (nbuf == 0 && d9[i] == '0') {
          ++zeros;
          continue;
        }
        if (nbuf < 18) buf[nbuf++] = d9[i];
        else if (d9[i] != '0') sticky = true;
      }
    }
    if (lo_limb < L) sticky = true;
    if (!has_int) exp10 = -(zeros + 1);
  }
  while (nbuf < 18) buf[nbuf++] = '0';
  // ---- round half to even at 17 digits
  Digits out;
  for (int i = 0; i < 17; ++i) out.d[i] = buf[i];
  out.exp10 = exp10;
  const int r = buf[17] - '0';
  const bool up = r > 5 || (r == 5 && (sticky || ((buf[16] - '0') & 1)));
  if (up) {
    int i = 16;
    while (i >= 0 && out.d[i] == '9') out.d[i--] = '0';
    if (i >= 0) {
      ++out.d[i];
    } else {
      out.d[0] = '1';
      for (int j = 1; j < 17; ++j) out.d[j] = '0';
      ++out.exp10;
    }
  }
  return out;
}

// %.17g of v into out; returns the length (<= 24).
__device__ int format_g17(double v, char* out) {
  int n = 0;
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
  const bool neg = bits >> 63;
  if (isnan(v)) {
    if (neg) out[n++] = '-';
    out[n++] = 'n';
    out[n++] = 'a';
    out[n++] = 'n';
    return n;
  }
  if (neg) out[n++] = '-';
  if (isinf(v)) {
    out[n++] = 'i';
    out[n++] = 'n';
    out[n++] = 'f';
    return n;
  }
  if (v == 0.0) {
    out[n++] = '0';
    return n;
  }
  const Digits dg = digits17(fabs(v));
  int last = 16;  // strip trailing zeros
  while (last > 0 && dg.d[last] == '0') --last;
  const int X = dg.exp10;
  if (X < -4 || X >= 17) {  // exponent style
    out[n++] = dg.d[0];
    if (last > 0) {
      out[n++] = '.';
      for (int i = 1; i <= last; ++i) out[n++] = dg.d[i];
    }
    out[n++] = 'e';
    int ex = X;
    out[n++] = ex < 0 ? '-' : '+';
    if (ex < 0) ex = -ex;
    if (ex >= 100) {
      out[n++] = static_cast<char>('0' + ex / 100);
      ex %= 100;
      out[n++] = static_cast<char>('0' + ex / 10);
      out[n++] = static_cast<char>('0' + ex % 10);
    } else {
      out[n++] = static_cast<char>('0' + ex / 10);
      out[n++] = static_cast<char>('0' + ex % 10);
    }
    return n;
  }
  if (X >= 0) {  // fixed, integer digits X + 1
    for (int i = 0; i <= X; ++i) out[n++] = dg.d[i];
    if (last > X) {
      out[n++] = '.';
      for (int i = X + 1; i <= last; ++i) out[n++] = dg.d[i];
    }
    return n;
  }
  out[n++] = '0';  // fixed, 0.000ddd
  out[n++] = '.';
  for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
  for (int i = 0; i <= last; ++i) out[n++] = dg.d[i];
  return n;
}


// ---------------------------------------------------------------- parse_double (io.cpp:78-88)
// std::stod on a trimmed cell, which must be consumed entirely: optional sign; decimal
// digits with optional point and exponent; "inf" / "infinity" / "nan[(...)]" in any case;
// hexadecimal "0x..[p..]".  Results that glibc's strtod flags with ERANGE (overflow to
// infinity, any subnormal or zero result of non-zero digits) make std::stod throw, which
// the reference reports as "expected a number" — status 2 here.  Decimal conversion is
// exact: a double estimate is corrected against the exact midpoints with multi-limb
// integer comparisons (all significant digits kept, up to kMaxDigits), i.e. the correctly
// rounded (round-half-even) result that glibc returns.
constexpr int kBig = 96;         // 32-bit limbs: 3072 bits
constexpr int kMaxDigits = 700;  // significant decimal digits kept exactly

struct Big {
  uint32_t w[kBig];
  int n;  // limbs in use
};
__device__ inline void big_set(Big& a, uint64_t v) {
  a.w[0] = static_cast<uint32_t>(v);
  a.w[1] = static_cast<uint32_t>(v >> 32);
  a.n = a.w[1] ? 2 : (a.w[0] ? 1 : 0);
}
__device__ inline void big_mul_small(Big& a, uint32_t m, uint32_t add = 0) {
  uint64_t carry = add;
  for (int i = 0; i < a.n; ++i) {
    const uint64_t cur = static_cast<uint64_t>(a.w[i]) * m + carry;
    a.w[i] = static_cast<uint32_t>(cur);
    carry = cur >> 32;
  }
  if (carry && a.n < kBig) a.w[a.n++] = static_cast<uint32_t>(carry);
}
__device__ inline void big_mul_pow10(Big& a, int k) {
  while (k >= 9) {
    big_mul_small(a, 1000000000u);
    k -= 9;
  }
  static const uint32_t p10[9] = {1, 10, 100, 1000, 10000, 100000, 1000000, 10000000, 100000000};
  if (k > 0) big_mul_small(a, p10[k]);
}
__device__ inline void big_shl(Big& a, int s) {
  if (a.n == 0 || s == 0) return;
  const int w = s >> 5, b = s & 31;
  int n = a.n + w + 1;
  if (n > kBig) n = kBig;
  for (int i = n - 1; i >= 0; --i) {
    const int src = i - w;
    uint32_t v = 0;
    if (src >= 0 && src < a.n) v = a.w[src] << b;
    if (b && src - 1 >= 0 && src - 1 < a.n) v |= a.w[src - 1] >> (32 - b);
    a.w[i] = v;
  }
  a.n = n;
  while (a.n > 0 && a.w[a.n - 1] == 0) --a.n;
}
__device__ inline int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

// sign of (D * 10^q) - (num * 2^p)
__device__ int cmp_dec_bin(const Big& D, int q, uint64_t num, int p) {
  Big A = D, B;
  big_set(B, num);
  if (q >= 0) big_mul_pow10(A, q);
  else big_mul_pow10(B, -q);
  if (p >= 0) big_shl(B, p);
  else big_shl(A, -p);
  return big_cmp(A, B);
}

__device__ inline char lower(char c) { return (c >= 'A' && c <= 'Z') ? static_cast<char>(c + 32) : c; }

// Correctly rounded D * 10^q (D > 0); status 2 when glibc would set ERANGE.
__device__ double dec_to_double(const Big& D, uint64_t top19, int ntop, int nd, int q, int* status) {
  // nd significant digits in total, the leading min(nd, 19) of them in top19 (ntop digits)
  const int e10 = nd + q;  // value in [10^(e10-1), 10^e10)
  if (e10 > 310) {
    *status = 2;
    return INFINITY;
  }
  if (e10 < -324) {
    *status = 2;
    return 0.0;
  }
  // estimate: top19 * 10^(q + nd - ntop)
  double x = static_cast<double>(top19);
  int k = q + nd - ntop;
  while (k > 22) {
    x *= 1e22;
    k -= 22;
  }
  while (k < -22) {
    x /= 1e22;
    k += 22;
  }
  const double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                          1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
  x = k >= 0 ? x * p10[k] : x / p10[-k];
  if (!(x < INFINITY)) x = 1.7976931348623157e308;
  if (x < 4.9406564584124654e-324) x = 4.9406564584124654e-324;
  for (int iter = 0; iter < 64; ++iter) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
    const int be = static_cast<int>(bits >> 52);
    uint64_t m = bits & 0xfffffffffffffull;
    int e;
    if (be == 0) {
      e = -1074;
    } else {
      m |= 1ull << 52;
      e = be - 1075;
    }
    // upper midpoint (2m + 1) * 2^(e - 1)
    const int cu = cmp_dec_bin(D, q, 2 * m + 1, e - 1);
    if (cu > 0 || (cu == 0 && (m & 1))) {
      if (be == 0x7fe && m == 0x1fffffffffffffull) {
        *status = 2;
        return INFINITY;
      }
      x = __longlong_as_double(static_cast<long long>(bits + 1));
      if (cu == 0) break;
      continue;
    }
    // lower midpoint: (2m - 1) * 2^(e - 1), or (4m - 1) * 2^(e - 2) below a power of two
    const bool pow2 = be > 1 && m == (1ull << 52);
    const int cl = pow2 ? cmp_dec_bin(D, q, 4 * m - 1, e - 2) : cmp_dec_bin(D, q, 2 * m - 1, e - 1);
    if (cl < 0 || (cl == 0 && (m & 1))) {
      if (bits == 1) {  // below half the smallest subnormal: rounds to zero
        *status = 2;
        return 0.0;
      }
      x = __longlong_as_double(static_cast<long long>(bits - 1));
      if (cl == 0) break;
      continue;
    }
    break;
  }
  if (x < 2.2250738585072014e-308) {  // glibc: ERANGE on an inexact subnormal result
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
    if (cmp_dec_bin(D, q, bits, -1074) != 0) *status = 2;
  }
  return x;
}

// Hexadecimal float body after "0x": mantissa hex digits [. hex digits] [p exp]; exact.
__device__ double hex_to_double(const char* s, int len, int* used, int* status) {
  int i = 0;
  uint64_t mant = 0;
  int shift = 0;       // binary exponent adjustment
  bool sticky = false, any = false, point = false;
  int sig_bits = 0;
  for (; i < len; ++i) {
    const char c = lower(s[i]);
    int d;
    if (c >= '0' && c <= '9') d = c - '0';
    else if (c >= 'a' && c <= 'f') d = c - 'a' + 10;
    else if (c == '.' && !point) {
      point = true;
      continue;
    } else break;
    any = true;
    if (mant == 0 && d == 0) {
      if (point) shift -= 4;
      continue;
    }
    if (sig_bits <= 60) {
      mant = (mant << 4) | static_cast<uint64_t>(d);
      sig_bits += 4;
      if (point) shift -= 4;
    } else {
      if (d) sticky = true;
      if (!point) shift += 4;
    }
  }
  if (!any) {
    *used = 0;
    return 0.0;
  }
  if (i < len && lower(s[i]) == 'p') {
    int j = i + 1;
    bool neg = false;
    if (j < len && (s[j] == '+' || s[j] == '-')) neg = s[j++] == '-';
    int ex = 0;
    bool dig = false;
    while (j < len && s[j] >= '0' && s[j] <= '9') {
      if (ex < 100000) ex = ex * 10 + (s[j] - '0');
      ++j;
      dig = true;
    }
    if (dig) {
      shift += neg ? -ex : ex;
      i = j;
    }
  }
  *used = i;
  if (mant == 0) return 0.0;
  // value = mant * 2^shift (+ sticky); normalise mant to 64 bits
  const int lz = __clzll(static_cast<long long>(mant));
  mant <<= lz;
  shift -= lz;
  int e = shift + 63;  // value = 1.xxx * 2^e
  if (e > 1023) {
    *status = 2;
    return INFINITY;
  }
  int keep = 53;  // significant bits the result can hold
  if (e < -1022) keep = 53 - (-1022 - e);
  if (keep <= 0) {
    // below the smallest subnormal: rounds to zero or to 2^-1074
    const bool up = keep == 0 && (((mant << 1) != 0) || sticky);
    *status = 2;
    return up ? 4.9406564584124654e-324 : 0.0;
  }
  const int drop = 64 - keep;
  uint64_t q = mant >> drop;
  const uint64_t rem = mant & ((1ull << drop) - 1ull);
  const uint64_t half = 1ull << (drop - 1);
  const bool inexact = rem != 0 || sticky;
  if (rem > half || (rem == half && (sticky || (q & 1)))) ++q;
  if (q >> keep) {  // carry into a new bit
    q >>= 1;
    ++e;
    if (e > 1023) {
      *status = 2;
      return INFINITY;
    }
  }
  const double r = ldexp(static_cast<double>(q), e - (keep - 1));
  if (r < 2.2250738585072014e-308 && inexact) *status = 2;  // glibc: ERANGE on inexact underflow
  return r;
}

// Parse a trimmed cell [s, s + len); returns status 0 ok, 1 not a number / trailing junk,
// 2 out of range (ERANGE).
__device__ double parse_cell(const char* s, int len, int* status) {
  *status = 0;
  int i = 0;
  while (i < len && (s[i] == ' ' || (s[i] >= '\t' && s[i] <= '\r'))) ++i;  // strtod skips isspace
  bool neg = false;
  if (i < len && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  const int rest = len - i;
  // inf / infinity / nan[(...)]
  if (rest >= 3 && lower(s[i]) == 'i' && lower(s[i + 1]) == 'n' && lower(s[i + 2]) == 'f') {
    int end = i + 3;
    if (rest >= 8) {
      const char* w = "inity";
      bool ok = true;
      for (int j = 0; j < 5; ++j) ok &= lower(s[i + 3 + j]) == w[j];
      if (ok) end = i + 8;
    }
    if (end != len) *status = 1;
    return neg ? -INFINITY : INFINITY;
  }
  if (rest >= 3 && lower(s[i]) == 'n' && lower(s[i + 1]) == 'a' && lower(s[i + 2]) == 'n') {
    int end = i + 3;
    if (end < len && s[end] == '(') {
      int j = end + 1;
      while (j < len && (s[j] == '_' || (s[j] >= '0' && s[j] <= '9') || (lower(s[j]) >= 'a' && lower(s[j]) <= 'z'))) ++j;
      if (j < len && s[j] == ')') end = j + 1;
    }
    if (end != len) *status = 1;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    return neg ? -nan : nan;
  }
  if (rest >= 2 && s[i] == '0' && lower(s[i + 1]) == 'x') {
    int used = 0;
    const double v = hex_to_double(s + i + 2, len - i - 2, &used, status);
    if (used == 0) {  // "0x" without digits: strtod reads "0"
      if (i + 1 != len) *status = 1;
      return neg ? -0.0 : 0.0;
    }
    if (i + 2 + used != len) *status = 1;
    return neg ? -v : v;
  }
  // decimal
  Big D;
  D.n = 0;
  uint64_t top = 0;
  int ntop = 0, nd = 0, q = 0;
  bool any = false, point = false, dropped = false;
  for (; i < len; ++i) {
    const char c = s[i];
    if (c == '.' && !point) {
      point = true;
      continue;
    }
    if (c < '0' || c > '9') break;
    any = true;
    const uint32_t d = static_cast<uint32_t>(c - '0');
    if (nd == 0 && d == 0) {
      if (point) --q;
      continue;
    }
    if (nd < kMaxDigits) {
      big_mul_small(D, 10u, d);
      if (ntop < 19) {
        top = top * 10 + d;
        ++ntop;
      }
      ++nd;
      if (point) --q;
    } else {
      if (d) dropped = true;  // beyond kMaxDigits: too long to be exact
      if (!point) ++q;
    }
  }
  if (!any) {
    *status = 1;
    return 0.0;
  }
  if (i < len && lower(s[i]) == 'e') {
    int j = i + 1;
    bool eneg = false;
    if (j < len && (s[j] == '+' || s[j] == '-')) eneg = s[j++] == '-';
    int ex = 0;
    bool dig = false;
    while (j < len && s[j] >= '0' && s[j] <= '9') {
      if (ex < 100000) ex = ex * 10 + (s[j] - '0');
      ++j;
      dig = true;
    }
    if (dig) {
      q += eneg ? -ex : ex;
      i = j;
    }
  }
  if (i != len || dropped) *status = 1;
  if (nd == 0) return neg ? -0.0 : 0.0;
  int st = 0;
  const double v = dec_to_double(D, top, ntop, nd, q - 0, &st);
  if (st) *status = *status ? *status : st;
  return neg ? -v : v;
}

__global__ void g17_kernel(const double* __restrict__ v, int64_t n, char* __restrict__ slots,
                           uint8_t* __restrict__ lens) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    char buf[kSlot];
    const int len = format_g17(v[i], buf);
    char* o = slots + i * kSlot;
    for (int j = 0; j < len; ++j) o[j] = buf[j];
    lens[i] = static_cast<uint8_t>(len);
  }
}

__global__ void parse_slots_kernel(const char* __restrict__ slots, const uint8_t* __restrict__ lens, int64_t n,
                                   int stride, double* __restrict__ out, int8_t* __restrict__ status) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    int st = 0;
    out[i] = parse_cell(slots + i * stride, lens[i], &st);
    status[i] = static_cast<int8_t>(st);
  }
}

// ---------------------------------------------------------------- codes CSV
__device__ inline int uint_digits(uint64_t x) {
  int d = 1;
  while (x >= 10) {
    x /= 10;
    ++d;
  }
  return d;
}

// Pass 1: byte length of each data row ("id,v0,...,v{k-1}\n"), codes widened to double.
__global__ void csv_row_len_kernel(const float* __restrict__ Z, int64_t rows, int k, uint64_t first_id,
                                   int64_t* __restrict__ len) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    int64_t n = uint_digits(first_id + static_cast<uint64_t>(r)) + 1;  // id + '\n'
    char buf[kSlot];
    for (int j = 0; j < k; ++j) n += 1 + format_g17(static_cast<double>(Z[r * k + j]), buf);
    len[r] = n;
  }
}

// Exclusive scan of row lengths, single CTA (rows are few thousand to a few million;
// this is a small fraction of the formatting work).
__global__ void __launch_bounds__(1024) csv_scan_kernel(int64_t* __restrict__ len, int64_t rows, int64_t base,
                                                        int64_t* __restrict__ total) {
  __shared__ int64_t carry_s;
  __shared__ int64_t warp_tot[32];
  if (threadIdx.x == 0) carry_s = base;
  __syncthreads();
  for (int64_t b0 = 0; b0 < rows; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t x = i < rows ? len[i] : 0;
    int64_t incl = x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    int64_t wb = 0;
    for (int j = 0; j < w; ++j) wb += warp_tot[j];
    const int64_t carry = carry_s;
    if (i < rows) len[i] = carry + wb + incl - x;  // exclusive offset
    __syncthreads();
    if (threadIdx.x == 1023) carry_s = carry + wb + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry_s;
}

__global__ void csv_write_kernel(const float* __restrict__ Z, int64_t rows, int k, uint64_t first_id,
                                 const int64_t* __restrict__ off, char* __restrict__ out) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    char* o = out + off[r];
    uint64_t id = first_id + static_cast<uint64_t>(r);
    const int nd = uint_digits(id);
    for (int i = nd - 1; i >= 0; --i) {
      o[i] = static_cast<char>('0' + id % 10);
      id /= 10;
    }
    o += nd;
    char buf[kSlot];
    for (int j = 0; j < k; ++j) {
      *o++ = ',';
      const int len = format_g17(static_cast<double>(Z[r * k + j]), buf);
      for (int i = 0; i < len; ++i) o[i] = buf[i];
      o += len;
    }
    *o = '\n';
  }
}


// ---------------------------------------------------------------- codes CSV reader (io.cpp:267-310)
// Newline index (chunk counts -> scan -> positions), header parsed on the host from the
// first non-empty line, then one thread per physical line: trim, split on ',', cell count,
// id span, parse_double of every value cell.  Row numbers of the non-empty data lines come
// from an exclusive scan, so rows keep the file order.  The first failing physical line
// (1-based, as the reference's FormatError) is reported.
constexpr int kChunk = 16384;  // bytes per block in the newline passes

__device__ inline bool is_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

__global__ void nl_count_kernel(const char* __restrict__ text, int64_t len, int64_t* __restrict__ counts) {
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kChunk;
  int64_t cnt = 0;
  for (int64_t i = b0 + threadIdx.x; i < b0 + kChunk && i < len; i += blockDim.x) cnt += text[i] == '\n';
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ int64_t ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += ws[w];
    counts[blockIdx.x] = t;
  }
}

// newline positions: block b writes its chunk's '\n' offsets from offset[b], in order
__global__ void nl_write_kernel(const char* __restrict__ text, int64_t len, const int64_t* __restrict__ offset,
                                int64_t* __restrict__ pos) {
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kChunk;
  __shared__ int64_t base;
  __shared__ int ws[32];
  if (threadIdx.x == 0) base = offset[blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c0 = b0; c0 < b0 + kChunk && c0 < len; c0 += blockDim.x) {  // block-uniform
    const int64_t i = c0 + threadIdx.x;
    const bool nl = i < len && i < b0 + kChunk && text[i] == '\n';
    const unsigned int ball = __ballot_sync(0xffffffffu, nl);
    if (lane == 0) ws[warp] = __popc(ball);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      if (w < warp) before += ws[w];
      total += ws[w];
    }
    if (nl) pos[base + before + __popc(ball & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (threadIdx.x == 0) base += total;
    __syncthreads();
  }
}

// single-CTA exclusive scan (in place), total in *sum
__global__ void __launch_bounds__(1024) scan_excl_kernel(int64_t* __restrict__ a, int64_t n, int64_t* __restrict__ sum) {
  __shared__ int64_t carry_s;
  __shared__ int64_t warp_tot[32];
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < n; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t x = i < n ? a[i] : 0;
    int64_t incl = x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    int64_t wb = 0;
    for (int j = 0; j < w; ++j) wb += warp_tot[j];
    const int64_t carry = carry_s;
    if (i < n) a[i] = carry + wb + incl - x;
    __syncthreads();
    if (threadIdx.x == 1023) carry_s = carry + wb + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0 && sum) *sum = carry_s;
}

__device__ inline void line_span(const int64_t* pos, int64_t nnl, int64_t len, int64_t li, int64_t* a, int64_t* b) {
  *a = li == 0 ? 0 : pos[li - 1] + 1;
  *b = li < nnl ? pos[li] : len;
}

// flag[l] = 1 for non-empty data lines (after the header line)
__global__ void line_flag_kernel(const char* __restrict__ text, int64_t len, const int64_t* __restrict__ pos,
                                 int64_t nnl, int64_t first, int64_t nlines, int64_t* __restrict__ flag) {
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < nlines; l += int64_t(gridDim.x) * blockDim.x) {
    int64_t a, b;
    line_span(pos, nnl, len, first + l, &a, &b);
    bool nonempty = false;
    for (int64_t i = a; i < b && !nonempty; ++i) nonempty = !is_space(text[i]);
    flag[l] = nonempty ? 1 : 0;
  }
}

__global__ void line_parse_kernel(const char* __restrict__ text, int64_t len, const int64_t* __restrict__ pos,
                                  int64_t nnl, int64_t first, int64_t nlines, const int64_t* __restrict__ row_of,
                                  int k, double* __restrict__ codes, int64_t* __restrict__ ids,
                                  unsigned long long* __restrict__ bad_line) {
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < nlines; l += int64_t(gridDim.x) * blockDim.x) {
    int64_t a, b;
    line_span(pos, nnl, len, first + l, &a, &b);
    while (a < b && is_space(text[a])) ++a;  // trim(line)
    while (b > a && is_space(text[b - 1])) --b;
    if (a == b) continue;
    const int64_t row = row_of[l];
    const unsigned long long lineno = static_cast<unsigned long long>(first + l + 1);
    // cell count first (split keeps empty cells)
    int cells = 1;
    for (int64_t i = a; i < b; ++i) cells += text[i] == ',';
    if (cells != k + 1) {
      atomicMin(bad_line, lineno);
      continue;
    }
    int64_t c0 = a;
    for (int cell = 0; cell <= k; ++cell) {
      int64_t c1 = c0;
      while (c1 < b && text[c1] != ',') ++c1;
      int64_t x = c0, y = c1;  // trim(cell)
      while (x < y && is_space(text[x])) ++x;
      while (y > x && is_space(text[y - 1])) --y;
      if (cell == 0) {
        if (ids) {
          ids[2 * row] = x;
          ids[2 * row + 1] = y - x;
        }
      } else {
        int st = 0;
        const double v = parse_cell(text + x, static_cast<int>(y - x < 1 << 30 ? y - x : 1 << 30), &st);
        if (st) atomicMin(bad_line, lineno);
        if (codes) codes[row * k + cell - 1] = v;
      }
      c0 = c1 + 1;
    }
  }
}

int grid_for(hc_ctx ctx, int64_t n) {
  const int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : (g > int64_t(ctx->sm_count) * 16 ? int64_t(ctx->sm_count) * 16 : g));
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int hc_format_g17(hc_ctx ctx, const double* v, int64_t n, char* slots, uint8_t* lens) {
  HC_REQUIRE(ctx, HC_EINVAL, "format_g17: null context");
  HC_REQUIRE(n >= 0, HC_EINVAL, "format_g17: negative count");
  if (n == 0) return HC_OK;
  HC_REQUIRE(v && slots && lens, HC_EINVAL, "format_g17: null buffer");
  g17_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(v, n, slots, lens);
  HC_CHECK_LAUNCH(ctx, "g17_kernel");
  return HC_OK;
}

int hc_parse_doubles(hc_ctx ctx, const char* slots, const uint8_t* lens, int64_t n, int stride, double* out,
                     int8_t* status) {
  HC_REQUIRE(ctx, HC_EINVAL, "parse_doubles: null context");
  HC_REQUIRE(n >= 0 && stride > 0, HC_EINVAL, "parse_doubles: bad shape");
  if (n == 0) return HC_OK;
  HC_REQUIRE(slots && lens && out && status, HC_EINVAL, "parse_doubles: null buffer");
  parse_slots_kernel<<<grid_for(ctx, n), 128, 0, ctx->stream>>>(slots, lens, n, stride, out, status);
  HC_CHECK_LAUNCH(ctx, "parse_slots_kernel");
  return HC_OK;
}

int hc_codes_csv_write(hc_ctx ctx, const float* codes, int64_t rows, int k, uint64_t first_id, char* out,
                       int64_t capacity, int64_t* length) {
  HC_REQUIRE(ctx && length, HC_EINVAL, "codes_csv: null argument");
  HC_REQUIRE(rows >= 0 && k > 0 && k <= 64, HC_EINVAL, "codes_csv: bad shape");
  HC_REQUIRE(rows == 0 || codes, HC_EINVAL, "codes_csv: null codes");
  // header "id,c0,...,c{k-1}\n" (io.cpp:319-321)
  char header[512];
  int h = 0;
  header[h++] = 'i';
  header[h++] = 'd';
  for (int j = 0; j < k; ++j) h += std::snprintf(header + h, sizeof(header) - h, ",c%d", j);
  header[h++] = '\n';
  int rc = ensure_scratch(ctx, sizeof(int64_t) * (static_cast<size_t>(rows) + 2));
  if (rc != HC_OK) return rc;
  int64_t* off = static_cast<int64_t*>(ctx->scratch);
  int64_t* total = off + rows;
  if (rows > 0) {
    csv_row_len_kernel<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(codes, rows, k, first_id, off);
    HC_CHECK_LAUNCH(ctx, "csv_row_len_kernel");
  }
  csv_scan_kernel<<<1, 1024, 0, ctx->stream>>>(off, rows, h, total);
  HC_CHECK_LAUNCH(ctx, "csv_scan_kernel");
  HC_CUDA_TRY(cudaMemcpyAsync(length, total, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (!out) return HC_OK;  // size query
  HC_REQUIRE(*length <= capacity, HC_EINVAL, "codes_csv: output buffer too small");
  HC_CUDA_TRY(cudaMemcpyAsync(out, header, h, cudaMemcpyHostToDevice, ctx->stream));
  if (rows > 0) {
    csv_write_kernel<<<grid_for(ctx, rows), 256, 0, ctx->stream>>>(codes, rows, k, first_id, off, out);
    HC_CHECK_LAUNCH(ctx, "csv_write_kernel");
  }
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HC_OK;
}


int hc_codes_csv_read(hc_ctx ctx, const char* text, int64_t len, int* k_out, int64_t* rows_out, double* codes,
                      int64_t* ids, int64_t capacity_rows) {
  HC_REQUIRE(ctx && k_out && rows_out, HC_EINVAL, "codes_csv_read: null argument");
  HC_REQUIRE(len >= 0 && (len == 0 || text), HC_EINVAL, "codes_csv_read: bad text");
  const int64_t nblocks = (len + kChunk - 1) / kChunk;
  // scratch: counts[nblocks + 1] | newline positions | flags / row numbers
  // (newlines <= len; lines <= newlines + 1)
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  int rc = ensure_scratch(ctx, up(sizeof(int64_t) * (nblocks + 2)) + 2 * up(sizeof(int64_t) * (len + 2)) + 256);
  if (rc != HC_OK) return rc;
  char* base = static_cast<char*>(ctx->scratch);
  int64_t* counts = reinterpret_cast<int64_t*>(base);
  int64_t* pos = reinterpret_cast<int64_t*>(base + up(sizeof(int64_t) * (nblocks + 2)));
  int64_t* flag = reinterpret_cast<int64_t*>(base + up(sizeof(int64_t) * (nblocks + 2)) + up(sizeof(int64_t) * (len + 2)));
  int64_t* misc = counts + nblocks;  // [0] newline count, [1] row count
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(pos + len + 1);  // spare slot after positions
  int64_t nnl = 0;
  if (nblocks > 0) {
    nl_count_kernel<<<static_cast<int>(nblocks), 256, 0, ctx->stream>>>(text, len, counts);
    HC_CHECK_LAUNCH(ctx, "nl_count_kernel");
    scan_excl_kernel<<<1, 1024, 0, ctx->stream>>>(counts, nblocks, misc);
    HC_CHECK_LAUNCH(ctx, "scan_excl_kernel");
    nl_write_kernel<<<static_cast<int>(nblocks), 256, 0, ctx->stream>>>(text, len, counts, pos);
    HC_CHECK_LAUNCH(ctx, "nl_write_kernel");
    HC_CUDA_TRY(cudaMemcpyAsync(&nnl, misc, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  }
  const int64_t total_lines = len > 0 ? nnl + 1 : 0;  // the segment after the last '\n' may be empty
  // header: first non-empty line, parsed on the host (io.cpp:276-288); searched among the
  // first 4096 lines
  int64_t hline = -1;
  std::vector<int64_t> hpos(static_cast<size_t>(nnl < 4096 ? nnl : 4096));
  if (!hpos.empty())
    HC_CUDA_TRY(cudaMemcpy(hpos.data(), pos, sizeof(int64_t) * hpos.size(), cudaMemcpyDeviceToHost));
  std::string line;
  for (int64_t li = 0; li < total_lines && li <= static_cast<int64_t>(hpos.size()); ++li) {
    const int64_t a = li == 0 ? 0 : hpos[static_cast<size_t>(li - 1)] + 1;
    int64_t b = len;
    if (li < nnl) {
      if (li >= static_cast<int64_t>(hpos.size())) break;
      b = hpos[static_cast<size_t>(li)];
    }
    if (b - a > (1 << 20)) return set_error(HC_EINVAL, "codes_csv_read: header line too long");
    line.assign(static_cast<size_t>(b - a), '\0');
    if (b > a) HC_CUDA_TRY(cudaMemcpy(&line[0], text + a, static_cast<size_t>(b - a), cudaMemcpyDeviceToHost));
    size_t x = 0, y = line.size();
    while (x < y && std::isspace(static_cast<unsigned char>(line[x]))) ++x;
    while (y > x && std::isspace(static_cast<unsigned char>(line[y - 1]))) --y;
    if (x == y) continue;
    line = line.substr(x, y - x);
    hline = li;
    break;
  }
  if (hline < 0) return set_error(HC_EINVAL, "codes_csv_read: missing codes header");
  {
    std::vector<std::string> cells(1);
    for (char ch : line) {
      if (ch == ',') cells.emplace_back();
      else cells.back().push_back(ch);
    }
    auto trim = [](const std::string& t) {
      size_t x = 0, y = t.size();
      while (x < y && std::isspace(static_cast<unsigned char>(t[x]))) ++x;
      while (y > x && std::isspace(static_cast<unsigned char>(t[y - 1]))) --y;
      return t.substr(x, y - x);
    };
    const std::string where = " (line " + std::to_string(hline + 1) + ")";
    if (cells.size() < 2 || trim(cells[0]) != "id")
      return set_error(HC_EINVAL, "codes_csv_read: bad codes header (expected id,c0,...)" + where);
    for (size_t i = 1; i < cells.size(); ++i)
      if (trim(cells[i]) != "c" + std::to_string(i - 1))
        return set_error(HC_EINVAL, "codes_csv_read: bad codes header column " + std::to_string(i - 1) + where);
    *k_out = static_cast<int>(cells.size()) - 1;
  }
  const int k = *k_out;
  const int64_t first = hline + 1, nlines = total_lines - first;
  int64_t rows = 0;
  if (nlines > 0) {
    line_flag_kernel<<<grid_for(ctx, nlines), 256, 0, ctx->stream>>>(text, len, pos, nnl, first, nlines, flag);
    HC_CHECK_LAUNCH(ctx, "line_flag_kernel");
    scan_excl_kernel<<<1, 1024, 0, ctx->stream>>>(flag, nlines, misc + 1);
    HC_CHECK_LAUNCH(ctx, "scan_excl_kernel");
    HC_CUDA_TRY(cudaMemcpyAsync(&rows, misc + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  }
  *rows_out = rows;
  if (!codes && !ids) return HC_OK;  // size query
  HC_REQUIRE(rows <= capacity_rows, HC_EINVAL, "codes_csv_read: output capacity too small");
  if (nlines > 0) {
    const unsigned long long none = ~0ull;
    HC_CUDA_TRY(cudaMemcpyAsync(bad, &none, sizeof(none), cudaMemcpyHostToDevice, ctx->stream));
    line_parse_kernel<<<grid_for(ctx, nlines), 128, 0, ctx->stream>>>(text, len, pos, nnl, first, nlines, flag, k,
                                                                        codes, ids, bad);
    HC_CHECK_LAUNCH(ctx, "line_parse_kernel");
    unsigned long long bad_line = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&bad_line, bad, sizeof(bad_line), cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (bad_line != ~0ull)
      return set_error(HC_EINVAL, "codes_csv_read: malformed data (line " + std::to_string(bad_line) + ")");
  }
  return HC_OK;
}

}  // extern "C"
