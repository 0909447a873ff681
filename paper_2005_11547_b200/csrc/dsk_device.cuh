// dsk_device.cuh -- device building blocks shared by every kernel.
//
// Bit-exactness rules: the whole library is
// compiled with -fmad=false so no fp64 add/mul pair is contracted to DFMA;
// critical expressions additionally spell out __dadd_rn/__dmul_rn so the
// reference's evaluation order is visible.
#pragma once
#include <stdint.h>

#define DSK_FULL 0xffffffffu

namespace dsk {

constexpr uint64_t kMul1 = 0xBF58476D1CE4E5B9ULL;  // ref/randomness.py:51
constexpr uint64_t kMul2 = 0x94D049BB133111EBULL;  // ref/randomness.py:52
constexpr int kStreamV = 1, kStreamU = 2, kStreamPoisson = 3, kStreamFp = 4, kStreamBucket = 5,
              kStreamKeyMix = 12;  // ref/randomness.py:28-39
constexpr double kMaxAreas = 134217728.0;  // 2^27, ref/darthash.py:32
constexpr double kCandClip = 1099511627776.0;  // 2^40, ref/darthash.py:36
constexpr uint64_t kEmptyRank = ~0ULL;

#ifndef DSK_FZ_HI
#define DSK_FZ_HI 0  // 1: the high word's shifts as mul.hi (FMA pipe) instead of SHF (ALU pipe)
#endif
#if DSK_FZ_HI && defined(__CUDA_ARCH__)
__device__ __forceinline__ uint64_t xorshr(uint64_t h, int s) {
  const uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
  uint32_t hs;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(hs) : "r"(hi), "r"(1u << (32 - s)));
  const uint32_t l2 = __funnelshift_r(lo, hi, s) ^ lo, h2 = hs ^ hi;
  return ((uint64_t)h2 << 32) | l2;
}
#endif

// splitmix64 finalizer, ref/randomness.py:58-63
__host__ __device__ __forceinline__ uint64_t finalize(uint64_t h) {
#if DSK_FZ_HI && defined(__CUDA_ARCH__)
  h = xorshr(h, 30);
  h *= kMul1;
  h = xorshr(h, 27);
  h *= kMul2;
  return xorshr(h, 31);
#else
  h ^= h >> 30;
  h *= kMul1;
  h ^= h >> 27;
  h *= kMul2;
  return h ^ (h >> 31);
#endif
}

// 2^e for e in [-1022, 1023], exact
__device__ __forceinline__ double pow2(int e) {
  return __longlong_as_double((long long)(1023 + e) << 52);
}

// (h >> 11) * 2^-53, ref/randomness.py:143 -- the 53-bit integer converts exactly
__device__ __forceinline__ double u53(uint64_t h) {
  return __dmul_rn(__ull2double_rn(h >> 11), 0x1p-53);
}

// floor(math.log2(y)) for y >= 1 using the host-probed threshold table:
// thr[n] = smallest double below 2^n whose host log2 floors to n (else 2^n).
// Returns kDepthHuge for finite y >= 2^256 (the reference's depth > 255
// ValidationError) and kDepthInf for y = inf (math.floor(inf) raises
// OverflowError there, ref/darthash.py:154-156); see depth_status().
constexpr int kDepthHuge = 1024, kDepthInf = 2048;

__device__ __forceinline__ int floor_log2_host(double y, const double *thr) {
  if (!(y >= 1.0)) return 0;  // only reachable for invalid weights (status DSK_WEIGHT)
  uint64_t b = (uint64_t)__double_as_longlong(y);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  if (e >= 256) return e == 1024 ? kDepthInf : kDepthHuge;
  return e + (y >= thr[e + 1] ? 1 : 0);
}

// Status of a step's depths (ref/darthash.py:154-160): an element depth of
// inf raises OverflowError while the depths are computed, before the
// range check; then any depth or rank depth > 255 is a ValidationError.
__device__ __forceinline__ int depth_status(int maxd, int rank_depth) {
  if (maxd >= kDepthInf) return 9;  // DSK_OVERFLOW
  if (maxd > 255 || rank_depth > 255) return 3;  // DSK_DEPTH
  return 0;
}

// _largest_passing, ref/darthash.py:80-95, for the rank side:
// largest c in [0, 2^nu - 1] with r0 + c*drho <= limit, searched in the window
// floor(min(q, cap)) + {2, 1, 0, -1, -2}; q = (limit - r0) / drho computed as
// a multiplication by the exact power of two 1/drho = 2^(nu - rho).
__device__ __forceinline__ int64_t rank_window(double limit, int nu, int rho, double r0,
                                               double drho) {
  double q = limit >= r0 ? __dmul_rn(__dadd_rn(limit, -r0), pow2(nu - rho)) : -1.0;
  int64_t lim_idx = nu >= 62 ? INT64_MAX : (((int64_t)1 << nu) - 1);
  double cap = nu <= 40 ? (double)lim_idx : kCandClip;
  q = q < cap ? q : cap;
  int64_t base = (int64_t)floor(q);
#pragma unroll
  for (int delta = 2; delta >= -2; --delta) {
    int64_t c = base + delta;
    if (c < 0 || c > lim_idx) continue;
    if (__dadd_rn(r0, __dmul_rn((double)c, drho)) <= limit) return c;
  }
  return -1;
}

// weight side of the window, ref/darthash.py:200-213 (vectorised there):
// largest c in [0, 2^rho - 1] with w0 + c*dnu <= x, searched in the window
// clamp(floor((x - w0) / dnu)) + {2, 1, 0, -1, -2}.
//
// The estimate uses a multiplication by tpow = t * 2^(rho - nu) instead of
// the IEEE division by dnu = fl(1/t) * 2^(nu - rho).  Both quotients are
// within 3 ulps of the true (x - w0)/dnu, so for every legal step (area
// count <= 2^27, hence quotients < 2^50) their floors differ by at most one
// and both windows contain the true largest passing c; the predicate is
// monotone in c, so the first passing candidate is that same c.  Steps where
// the quotient is >= 2^50 clamp both estimates identically (wmax or 2^40).
__device__ __forceinline__ int64_t weight_window(double x, double w0, double dnu, double tpow,
                                                 int rho) {
  if (rho == 0) return w0 <= x ? 0 : -1;  // wmax = 0: only candidate 0, w0 + 0*dnu == w0
  if (rho == 1) {
    // wmax = 1: the clamped base is 0 or 1, so the +-2 window covers both
    // candidates and the result is the largest passing one (no estimate needed)
    if (__dadd_rn(w0, dnu) <= x) return 1;
    return w0 <= x ? 0 : -1;
  }
  double wmax = __dadd_rn(pow2(rho), -1.0);  // float(2^rho - 1) as numpy compares it
  double capw = wmax < kCandClip ? wmax : kCandClip;
  double base = floor(__dmul_rn(__dadd_rn(x, -w0), tpow));
  base = base < capw ? base : capw;  // np.minimum
  base = base > 0.0 ? base : 0.0;    // np.maximum
  // The reference takes the first passing candidate of base+2, ..., base-2;
  // the predicate is monotone in c, so that is the largest passing one --
  // found here from base outwards (usually two evaluations instead of three).
  auto pass = [&](double cand) {
    return cand >= 0.0 && cand <= wmax && __dadd_rn(w0, __dmul_rn(cand, dnu)) <= x;
  };
  if (pass(base)) {
    if (!pass(base + 1.0)) return (int64_t)base;
    return pass(base + 2.0) ? (int64_t)(base + 2.0) : (int64_t)(base + 1.0);
  }
  if (pass(base - 1.0)) return (int64_t)(base - 1.0);
  if (pass(base - 2.0)) return (int64_t)(base - 2.0);
  return -1;
}

// numpy pairwise summation (pairwise_sum_DOUBLE, PW_BLOCKSIZE 128), i.e.
// float(np.sum(weights)) of ref/core.py:44, warp-cooperative and without
// local memory.  (`sexp` != 0 sums the values rescaled by 2^sexp, i.e.
// np.sum(np.ldexp(a, sexp)).)
//
// numpy's recursion on n elements: n < 8 -> sequential sum; n <= 128 ->
// eight strided accumulators r[j] = a[j] + a[j+8] + ... (sequential per j),
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail
// added in order; otherwise split at n2 = n/2 - (n/2 mod 8) and add the two
// halves' sums.
__device__ __forceinline__ double pw_ld(const double *a, int64_t i, int sexp) {
  return sexp ? scalbn(a[i], sexp) : a[i];
}

// A leaf (n <= 128) of the recursion, by the whole warp: lane j < 8 runs
// accumulator j's chain; the result is returned to every lane.
__device__ __forceinline__ double warp_pw_leaf(const double *a, int64_t n, int lane, int sexp) {
  double res = 0.0;
  if (n < 8) {
    if (lane == 0)
      for (int64_t i = 0; i < n; i++) res = __dadd_rn(res, pw_ld(a, i, sexp));
    return __shfl_sync(DSK_FULL, res, 0);
  }
  const int64_t body = n - (n % 8);
  double r = 0.0;
  if (lane < 8) {
    double v[16];  // <= 16 terms per chain (n <= 128); loads first, then the in-order adds
#pragma unroll
    for (int q = 0; q < 16; q++) v[q] = 8 * q + lane < body ? pw_ld(a, 8 * q + lane, sexp) : 0.0;
    r = v[0];
#pragma unroll
    for (int q = 1; q < 16; q++)
      if (8 * q + lane < body) r = __dadd_rn(r, v[q]);
  }
  // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)): pairs at distance 1, 2, 4
  r = __dadd_rn(r, __shfl_down_sync(DSK_FULL, r, 1));
  r = __dadd_rn(r, __shfl_down_sync(DSK_FULL, r, 2));
  r = __dadd_rn(r, __shfl_down_sync(DSK_FULL, r, 4));
  if (lane == 0)
    for (int64_t i = body; i < n; i++) r = __dadd_rn(r, pw_ld(a, i, sexp));
  return __shfl_sync(DSK_FULL, r, 0);
}

// Warp-cooperative float(np.sum(a)) for any n.  The recursion is walked in
// post order by the whole warp (warp-uniform control flow); its stack lives
// in registers across the lanes -- lane d holds the node at depth d (start,
// length, state, left sum) -- so nothing spills to local memory.  Depth <=
// log2(n / 64) + 1 < 32 for every n < 2^31.  (`scratch` is unused; kept for
// the callers' signature.)
__device__ __forceinline__ double warp_np_sum(const double *a, int64_t n, double *scratch,
                                           int lane, int sexp) {
  (void)scratch;
  if (n <= 128) return warp_pw_leaf(a, n, lane, sexp);
  int64_t nstart = 0, nlen = n;  // this lane's stack entry
  int nstate = 0;                // 0 fresh, 1 left child pending, 2 right child pending
  double nleft = 0.0;
  int sp = 1;                    // warp-uniform stack depth; lane 0 holds the root
  double ret = 0.0;
  while (sp > 0) {
    const int top = sp - 1;
    const int64_t len = __shfl_sync(DSK_FULL, nlen, top);
    const int64_t start = __shfl_sync(DSK_FULL, nstart, top);
    if (len <= 128) {
      ret = warp_pw_leaf(a + start, len, lane, sexp);
      sp--;
      while (sp > 0) {  // deliver to the parents
        const int p = sp - 1;
        if (__shfl_sync(DSK_FULL, nstate, p) == 1) {  // left child returned: push the right
          const int64_t plen = __shfl_sync(DSK_FULL, nlen, p);
          const int64_t pstart = __shfl_sync(DSK_FULL, nstart, p);
          int64_t n2 = plen / 2;
          n2 -= n2 % 8;
          if (lane == p) { nleft = ret; nstate = 2; }
          if (lane == sp) { nstart = pstart + n2; nlen = plen - n2; nstate = 0; }
          sp++;
          break;
        }
        ret = __dadd_rn(__shfl_sync(DSK_FULL, nleft, p), ret);  // right child returned
        sp--;
      }
    } else {
      int64_t n2 = len / 2;
      n2 -= n2 % 8;
      if (lane == top) nstate = 1;
      if (lane == sp) { nstart = start; nlen = n2; nstate = 0; }
      sp++;
    }
  }
  return ret;
}

// x mod d for 64-bit x, 32-bit d >= 1 (bucket_array's uint64 %, ref/randomness.py:219)
struct ModU32 {
  uint64_t m;     // floor(2^64 / d) for non-powers of two
  uint32_t d;
  uint32_t mask;  // d - 1 when d is a power of two, else 0
  int pow2;
};

__host__ __device__ inline ModU32 make_mod(uint32_t d) {
  ModU32 r;
  r.d = d;
  r.pow2 = (d & (d - 1)) == 0;
  r.mask = d - 1;
  r.m = r.pow2 ? 0 : (~0ULL) / d;  // floor((2^64-1)/d) == floor(2^64/d) for non-powers of 2
  return r;
}

__device__ __forceinline__ uint32_t mod_u32(uint64_t x, const ModU32 &md) {
  if (md.pow2) return (uint32_t)(x & md.mask);
  uint64_t q = __umul64hi(x, md.m);
  uint64_t r = x - q * md.d;
  if (r >= md.d) r -= md.d;
  if (r >= md.d) r -= md.d;
  return (uint32_t)r;
}

// inclusive warp scan of 32-bit counts
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(DSK_FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// largest lane s with excl[s] <= pos (excl non-decreasing over lanes)
__device__ __forceinline__ int warp_owner(uint32_t excl, uint32_t pos) {
  int s = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    uint32_t e = __shfl_sync(DSK_FULL, excl, s + step);
    if (e <= pos) s += step;
  }
  return s;
}

// 128-bit shared-memory compare-and-swap (native ATOMS.CAS.128 on sm_90+)
__device__ __forceinline__ void cas128_shared(uint64_t *addr, uint64_t cmp_lo, uint64_t cmp_hi,
                                              uint64_t val_lo, uint64_t val_hi, uint64_t &old_lo,
                                              uint64_t &old_hi) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(addr);
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.shared.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(val_lo), "l"(val_hi), "r"(a)
      : "memory");
}

__device__ __forceinline__ void ld128_shared(const uint64_t *addr, uint64_t &lo, uint64_t &hi) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(addr);
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(a) : "memory");
}

// Invalidate one 128-byte L2 line (128-byte aligned) without writing it back:
// for scratch whose contents are dead, so dirty lines never reach HBM.
__device__ __forceinline__ void l2_discard(const void *line) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
}

// generic-address forms (slot arrays in global memory for large k)
__device__ __forceinline__ void cas128_generic(uint64_t *addr, uint64_t cmp_lo, uint64_t cmp_hi,
                                               uint64_t val_lo, uint64_t val_hi, uint64_t &old_lo,
                                               uint64_t &old_hi) {
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(val_lo), "l"(val_hi), "l"(addr)
      : "memory");
}

// a stale (older) pair is harmless: slot values only decrease, and a failed
// CAS returns the current pair
__device__ __forceinline__ void ld128_generic(const uint64_t *addr, uint64_t &lo, uint64_t &hi) {
  asm volatile("ld.relaxed.gpu.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(addr) : "memory");
}

}  // namespace dsk
