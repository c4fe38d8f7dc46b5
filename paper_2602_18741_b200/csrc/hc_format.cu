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
#include <cstring>

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

}  // extern "C"
