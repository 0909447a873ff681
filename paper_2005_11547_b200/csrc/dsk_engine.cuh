// dsk_engine.cuh -- the DartHash enumeration engine (one warp's pipeline).
//
// Restates DartHasher.dart_batch (ref/darthash.py:142-295) for the GPU.  One
// warp walks the elements of its share of a set and expands work through four
// load-balanced levels, each backed by a 64-entry shared-memory queue so every
// stage runs on full 32-lane batches:
//
//   element chunk --(depth+1)(rank_depth+1)--> regions (nu, rho)   [region queue]
//   region  --(w_hi+1)(r_hi-r_lo+1)--> areas (w, r) + Poisson count [area queue]
//   area    --count--> candidate darts, rank/weight filter       -> [hit queue]
//   hit     --> fingerprint, bucket hash, Sink (slot minimum / LSH buffer)
//
// Hashing is tabulation + splitmix64 (ref/randomness.py:121-131) with the
// constant key bytes hoisted: the element's 8-byte XOR once per element, nu
// and rho once per region, w/r low bytes once per area, and (j, stream) from a
// folded 64x4 table, so a dart hash is one XOR with a shared-memory word plus
// the finalizer.
//
// Rank bands: a pass enumerates only darts with L_lo < rank <= L_hi.  Area
// rows r < r_hi(L_lo) lie wholly below L_lo (their computed upper edge is
// the next row's corner) and are skipped; the shared row r_lo is filtered on
// the computed rank.  The union of the bands 1..phi equals the reference's
// from-scratch recompute at phi (prefix property).
//
// Queue records are 16-byte words in structure-of-arrays layout so each
// field group moves with one conflict-free LDS.128 / STS.128.
#pragma once
#include "dsk_device.cuh"

namespace dsk {

constexpr int kWarps = 24;   // warps per CTA (one CTA per SM)
constexpr int kQ = 64;       // queue capacity per level
constexpr int kJs = 64;      // folded (j, stream) table rows; Poisson counts < 64
constexpr int kRwin = 128;   // per-pass rank-window table entries per warp

struct SmemTables {
  uint64_t tE[8][256];    // T0..T7  element bytes
  uint64_t tNu[256];      // T8
  uint64_t tRho[256];     // T9
  uint64_t tW[2][256];    // T10, T11 (w bytes 0, 1)
  uint64_t tR[2][256];    // T14, T15 (r bytes 0, 1)
  uint64_t js[kJs][4];    // T18[j]^T19[0]^T20[s]^T21[0], s = 1..4 (V, U, Poisson, fp)
  uint64_t pthr[64];      // ceil(cdf[m] * 2^53): count = #{m : X >= pthr[m]}
  double w0[256];         // (2^nu - 1) / t
  double l2thr[258];
  uint64_t cfold;         // T12[0]^T13[0]^T16[0]^T17[0] (w, r < 2^16)
  uint64_t nfold;         // T11[0]^T15[0]               (w, r < 2^8)
  uint64_t bconst;        // bucket hash constant: T8..T19 at 0, stream 5
  uint64_t pad;
};

struct WarpQueues {
  ulonglong2 rgA[kQ];   // region: {P_R, x}
  uint4 rgB[kQ];        //         {w_hi, r_lo, r_hi, meta}
  ulonglong2 arA[kQ];   // area:   {P_A, x}
  uint4 arB[kQ];        //         {w, r, meta, element index (materialising sink)}
  ulonglong2 ht[kQ];    // hit:    {P_A ^ js[j][fp], rank bits}
  ulonglong2 el[32];    // element chunk: {E, x}
  uint32_t elIdx[32];
};

// region meta: nu | rho << 8 | flags << 16 (| element index << 19, materialising sink)
constexpr uint32_t kRgHasPrev = 1u << 16, kRgWide = 1u << 17, kRgNarrow = 1u << 18;
// area meta: nu | rho << 8 | count << 16 | flags << 24
constexpr uint32_t kArWb = 1u << 24, kArRb = 1u << 25, kArLb = 1u << 26;

struct PassParams {
  const uint64_t *gtab;  // global 22x256 tables (rare wide-key bytes)
  double inv_t;          // fl(1 / t)
  double tf;             // t
  double L_hi, L_lo;     // band (L_lo < 0: first pass)
  int RD, RD_lo;         // rank depths of L_hi and L_lo
  int maxd;              // max element depth of the set (rank-window table extent)
  uint64_t pt0, pt1, pt2, pt3;  // first Poisson thresholds (registers)
};

// A hit that survived the rank/weight filters.
struct HitInfo {
  double rank;
  uint64_t fp;
  uint64_t bhash;  // hash64(fp, stream 5) before the modulo
};

// Full DartBatch row (ref/darthash.py:39-53), for the materialising sink.
struct DartRow {
  uint32_t elem;  // element index within the set
  int nu, rho;
  uint32_t w, r, j;
  double weight, rank;
  uint64_t fp;
};

// Poisson(1) count: #{m : X >= thr[m]} (inverse CDF, ref/randomness.py:145-147);
// counts >= 4 (2% of areas) finish in a loop over the shared table.
__device__ __forceinline__ uint32_t poisson_count(uint64_t X, const PassParams &P,
                                                  const SmemTables &T) {
  uint32_t c = (X >= P.pt0) + (X >= P.pt1) + (X >= P.pt2) + (X >= P.pt3);
  if (c == 4) {
    while (X >= T.pthr[c]) c++;
  }
  return c;
}

template <class Sink, bool kFull>
struct Engine {
  const SmemTables &T;
  WarpQueues &Q;
  uint2 *rwin;          // per-pass rank windows by (nu, rho): {r_hi + 1, r_lo | hasprev << 31}
  Sink &sink;
  const PassParams P;
  int lane;
  int rg_head = 0, rg_cnt = 0, ar_head = 0, ar_cnt = 0, ht_head = 0, ht_cnt = 0;
  bool use_table = false;
  bool abort = false;       // warp-uniform: area cap exceeded by one lane's share
  double lane_full = 0.0;   // per lane: areas of the full (non-band) step (area cap)
  uint32_t n_darts = 0;     // per lane: candidate darts first seen in this band
  uint32_t n_hits = 0;      // per lane

  __device__ Engine(const SmemTables &t, WarpQueues &q, uint2 *rw, Sink &s, const PassParams &p,
                    int ln)
      : T(t), Q(q), rwin(rw), sink(s), P(p), lane(ln) {
    // rank windows depend on (nu, rho, limit) only: tabulate them per pass
    const int rdp1 = P.RD + 1;
    const int entries = (P.maxd + 1) * rdp1;
    use_table = entries <= kRwin;
    if (use_table) {
      for (int e = lane; e < entries; e += 32) {
        int nu = e / rdp1, rho = e - nu * rdp1;
        double r0 = __dadd_rn(pow2(rho), -1.0);
        double drho = pow2(rho - nu);
        int64_t r_hi = rank_window(P.L_hi, nu, rho, r0, drho);
        uint32_t lo = 0;
        if (P.L_lo >= 0.0 && rho <= P.RD_lo) {
          int64_t rp = rank_window(P.L_lo, nu, rho, r0, drho);
          if (rp >= 0) lo = (uint32_t)rp | 0x80000000u;
        }
        // r_hi <= 2^27 whenever the step is legal; larger values saturate and
        // the area cap rejects the step
        uint32_t hi1 = r_hi < 0 ? 0u : (r_hi >= 0x7fffffff ? 0x7fffffffu : (uint32_t)r_hi + 1);
        rwin[e] = make_uint2(hi1, lo);  // team warps write identical values
      }
    }
    __syncwarp();
  }

  // ---------------------------------------------------------------- hits
  __device__ void process_hits(int m) {
    int idx = (ht_head + lane) & (kQ - 1);
    bool valid = lane < m;
    HitInfo h;
    h.rank = 0.0; h.fp = 0; h.bhash = 0;
    if (valid) {
      ulonglong2 rec = Q.ht[idx];
      h.rank = __longlong_as_double((long long)rec.y);
      h.fp = finalize(rec.x);  // fingerprint, ref/randomness.py:149-152
      uint64_t f = h.fp;
      uint64_t x = T.bconst;   // hash64(fp, stream=5), ref/randomness.py:154-158
#pragma unroll
      for (int p = 0; p < 8; p++) x ^= T.tE[p][(f >> (8 * p)) & 0xff];
      h.bhash = finalize(x);
      n_hits++;
    }
    ht_head = (ht_head + m) & (kQ - 1);
    ht_cnt -= m;
    sink.hit(valid, h, lane);
  }

  __device__ void drain_hits(bool force) {
    while (ht_cnt >= 32 || (force && ht_cnt > 0)) process_hits(ht_cnt < 32 ? ht_cnt : 32);
  }

  __device__ void push_hit(bool valid, double rank, uint64_t fpkey) {
    unsigned b = __ballot_sync(DSK_FULL, valid);
    if (b == 0) return;
    if (valid) {
      int idx = (ht_head + ht_cnt + __popc(b & ((1u << lane) - 1))) & (kQ - 1);
      Q.ht[idx] = make_ulonglong2(fpkey, (unsigned long long)__double_as_longlong(rank));
    }
    ht_cnt += __popc(b);
    __syncwarp();
    if (ht_cnt >= 32) drain_hits(false);
  }

  // --------------------------------------------------------------- darts
  // Expand up to 32 queued areas into their Poisson(1) darts
  // (ref/darthash.py:264-292).
  __device__ void process_areas(int m) {
    int head = ar_head;
    ar_head = (ar_head + m) & (kQ - 1);
    ar_cnt -= m;
    uint32_t c = 0;
    if (lane < m) c = (Q.arB[(head + lane) & (kQ - 1)].z >> 16) & 0xff;
    uint32_t incl = warp_incl_scan(c, lane);
    uint32_t total = __shfl_sync(DSK_FULL, incl, 31);
    uint32_t excl = incl - c;
    for (uint32_t base = 0; base < total; base += 32) {
      uint32_t pos = base + lane;
      bool valid = pos < total;
      int src = warp_owner(excl, pos);
      uint32_t j = pos - __shfl_sync(DSK_FULL, excl, src);
      bool hit = false;
      double rank = 0.0, weight = 0.0;
      uint64_t pa = 0;
      uint4 B = make_uint4(0, 0, 0, 0);
      if (valid) {
        int ai = (head + src) & (kQ - 1);
        ulonglong2 A = Q.arA[ai];
        B = Q.arB[ai];
        pa = A.x;
        uint32_t meta = B.z;
        int nu = meta & 0xff, rho = (meta >> 8) & 0xff;
        // rank = r0 + (r + u) * drho, ref/darthash.py:282 (separately rounded)
        double u = u53(finalize(pa ^ T.js[j][kStreamU - 1]));
        double r0 = __dadd_rn(pow2(rho), -1.0);
        rank = __dadd_rn(r0, __dmul_rn(__dadd_rn((double)B.y, u), pow2(rho - nu)));
        hit = true;
        if (meta & kArRb) hit = rank <= P.L_hi;        // interior rows pass by monotonicity
        if (meta & kArLb) hit = hit && rank > P.L_lo;  // band: exclude darts seen before
        if (kFull || (hit && (meta & kArWb))) {        // only the w_hi column can miss
          double v = u53(finalize(pa ^ T.js[j][kStreamV - 1]));
          double dnu = __dmul_rn(P.inv_t, pow2(nu - rho));
          // weight = w0 + (w + v) * dnu, ref/darthash.py:281
          weight = __dadd_rn(T.w0[nu], __dmul_rn(__dadd_rn((double)B.x, v), dnu));
          double x = __longlong_as_double((long long)A.y);
          if (meta & kArWb) hit = hit && weight <= x;  // ref/darthash.py:284 (inclusive)
        }
      }
      if (kFull) {  // materialising sink: every hit with its full index tuple
        if (hit) {
          DartRow d;
          d.elem = B.w;
          d.nu = B.z & 0xff;
          d.rho = (B.z >> 8) & 0xff;
          d.w = B.x;
          d.r = B.y;
          d.j = j;
          d.weight = weight;
          d.rank = rank;
          d.fp = finalize(pa ^ T.js[j][kStreamFp - 1]);
          sink.row(d);
          n_hits++;
        }
      } else {
        push_hit(hit, rank, pa ^ T.js[j][kStreamFp - 1]);
      }
    }
  }

  __device__ void drain_areas(bool force) {
    while (ar_cnt >= 32 || (force && ar_cnt > 0)) process_areas(ar_cnt < 32 ? ar_cnt : 32);
  }

  __device__ void push_area(bool valid, uint64_t pa, double x, uint32_t w, uint32_t r,
                            uint32_t meta, uint32_t elem) {
    unsigned b = __ballot_sync(DSK_FULL, valid);
    if (b == 0) return;
    if (valid) {
      int idx = (ar_head + ar_cnt + __popc(b & ((1u << lane) - 1))) & (kQ - 1);
      Q.arA[idx] = make_ulonglong2(pa, (unsigned long long)__double_as_longlong(x));
      Q.arB[idx] = make_uint4(w, r, meta, elem);
    }
    ar_cnt += __popc(b);
    __syncwarp();
    if (ar_cnt >= 32) drain_areas(false);
  }

  // --------------------------------------------------------------- areas
  // Expand up to 32 queued regions into their (w, r) areas, w-major
  // (ref/darthash.py:248-262), with the Poisson(1) count of each.
  __device__ void process_regions(int m) {
    int head = rg_head;
    rg_head = (rg_head + m) & (kQ - 1);
    rg_cnt -= m;
    uint32_t c = 0;
    if (lane < m) {
      uint4 B = Q.rgB[(head + lane) & (kQ - 1)];
      c = (B.x + 1) * (B.z - B.y + 1);
    }
    uint32_t incl = warp_incl_scan(c, lane);
    uint32_t total = __shfl_sync(DSK_FULL, incl, 31);
    uint32_t excl = incl - c;
    for (uint32_t base = 0; base < total; base += 32) {
      uint32_t pos = base + lane;
      bool valid = pos < total;
      int src = warp_owner(excl, pos);
      uint32_t off = pos - __shfl_sync(DSK_FULL, excl, src);
      bool keep = false;
      uint64_t pa = 0;
      double x = 0.0;
      uint32_t w = 0, r = 0, meta = 0, elem = 0;
      if (valid) {
        int gi = (head + src) & (kQ - 1);
        ulonglong2 A = Q.rgA[gi];
        uint4 B = Q.rgB[gi];
        uint32_t whi = B.x, rlo = B.y, rhi = B.z, rmeta = B.w;
        if (whi == 0) {
          w = 0;
          r = rlo + off;
        } else {
          uint32_t rc = rhi - rlo + 1;
          w = off / rc;
          r = rlo + (off - w * rc);
        }
        pa = A.x;
        if (rmeta & kRgNarrow) {
          pa ^= T.tW[0][w] ^ T.tR[0][r];
        } else {
          pa ^= T.tW[0][w & 0xff] ^ T.tW[1][(w >> 8) & 0xff] ^ T.tR[0][r & 0xff] ^
                T.tR[1][(r >> 8) & 0xff];
          if (rmeta & kRgWide)
            pa ^= __ldg(&P.gtab[12 * 256 + ((w >> 16) & 0xff)]) ^
                  __ldg(&P.gtab[13 * 256 + (w >> 24)]) ^
                  __ldg(&P.gtab[16 * 256 + ((r >> 16) & 0xff)]) ^
                  __ldg(&P.gtab[17 * 256 + (r >> 24)]);
        }
        // poisson1, ref/randomness.py:145-147 / :209-211 (j = 0, stream 3)
        uint32_t cnt = poisson_count(finalize(pa ^ T.js[0][kStreamPoisson - 1]) >> 11, P, T);
        bool lb = (rmeta & kRgHasPrev) && r == rlo;
        if (!lb) n_darts += cnt;
        keep = cnt > 0;
        meta = (rmeta & 0xffff) | (cnt << 16) | (w == whi ? kArWb : 0) | (r == rhi ? kArRb : 0) |
               (lb ? kArLb : 0);
        x = __longlong_as_double((long long)A.y);
        if (kFull) elem = rmeta >> 19;  // materialising sink: element index
      }
      push_area(keep, pa, x, w, r, meta, elem);
    }
  }

  __device__ void drain_regions(bool force) {
    while (rg_cnt >= 32 || (force && rg_cnt > 0)) process_regions(rg_cnt < 32 ? rg_cnt : 32);
  }

  __device__ void push_region(bool valid, uint64_t pr, double x, uint32_t whi, uint32_t rlo,
                              uint32_t rhi, uint32_t meta) {
    unsigned b = __ballot_sync(DSK_FULL, valid);
    if (b == 0) return;
    if (valid) {
      int idx = (rg_head + rg_cnt + __popc(b & ((1u << lane) - 1))) & (kQ - 1);
      Q.rgA[idx] = make_ulonglong2(pr, (unsigned long long)__double_as_longlong(x));
      Q.rgB[idx] = make_uint4(whi, rlo, rhi, meta);
    }
    rg_cnt += __popc(b);
    __syncwarp();
    if (rg_cnt >= 32) drain_regions(false);
  }

  // ------------------------------------------------------------- regions
  // One element chunk (<= 32 elements, lane i holds element i): expand each
  // element into its (nu, rho) regions and compute the surviving rectangle
  // (ref/darthash.py:180-225).  Sets `abort` when the area cap trips.
  __device__ void element_chunk(bool valid, uint64_t id, double x, int depth, uint32_t eidx) {
    uint64_t E = 0;
    if (valid) {
#pragma unroll
      for (int p = 0; p < 8; p++) E ^= T.tE[p][(id >> (8 * p)) & 0xff];
    }
    __syncwarp();
    Q.el[lane] = make_ulonglong2(E, (unsigned long long)__double_as_longlong(x));
    if (kFull) Q.elIdx[lane] = eidx;
    __syncwarp();
    const int rdp1 = P.RD + 1;
    const float inv_rdp1 = 1.0f / (float)rdp1;
    uint32_t c = valid ? (uint32_t)(depth + 1) * (uint32_t)rdp1 : 0;
    uint32_t incl = warp_incl_scan(c, lane);
    uint32_t total = __shfl_sync(DSK_FULL, incl, 31);
    uint32_t excl = incl - c;
    for (uint32_t base = 0; base < total; base += 32) {
      uint32_t pos = base + lane;
      bool ok = pos < total;
      int src = warp_owner(excl, pos);
      uint32_t idx = pos - __shfl_sync(DSK_FULL, excl, src);
      uint64_t pr = 0;
      double xs = 0.0;
      uint32_t whi = 0, rlo = 0, rhi = 0, meta = 0;
      if (ok) {
        int nu, rho;
        if (rdp1 == 1) {
          nu = (int)idx;
          rho = 0;
        } else {  // fp32 quotient, off by at most one: corrected below
          nu = (int)(((float)idx + 0.5f) * inv_rdp1);
          rho = (int)idx - nu * rdp1;
          if (rho < 0) { nu--; rho += rdp1; }
          else if (rho >= rdp1) { nu++; rho -= rdp1; }
        }
        ulonglong2 el = Q.el[src];
        xs = __longlong_as_double((long long)el.y);
        int64_t r_hi, r_lo = 0;
        uint32_t flags = 0;
        if (use_table) {
          uint2 rw = rwin[nu * rdp1 + rho];
          r_hi = (int64_t)rw.x - 1;
          if (rw.y & 0x80000000u) { r_lo = rw.y & 0x7fffffffu; flags |= kRgHasPrev >> 16; }
        } else {
          double r0 = __dadd_rn(pow2(rho), -1.0);
          double drho = pow2(rho - nu);
          r_hi = rank_window(P.L_hi, nu, rho, r0, drho);
          if (P.L_lo >= 0.0 && rho <= P.RD_lo) {
            int64_t rp = rank_window(P.L_lo, nu, rho, r0, drho);
            if (rp >= 0) { r_lo = rp; flags |= kRgHasPrev >> 16; }
          }
        }
        int64_t w_hi = -1;
        if (r_hi >= 0) {
          double dnu = __dmul_rn(P.inv_t, pow2(nu - rho));
          w_hi = weight_window(xs, T.w0[nu], dnu, __dmul_rn(P.tf, pow2(rho - nu)), rho);
        }
        ok = w_hi >= 0 && r_lo <= r_hi;
        if (w_hi >= 0) {
          double full = (double)(w_hi + 1) * (double)(r_hi + 1);
          lane_full += full;
          // a region over the cap makes the step illegal (ref/darthash.py:242-244)
          if (full > kMaxAreas) ok = false;
        }
        if (ok) {
          whi = (uint32_t)w_hi; rlo = (uint32_t)r_lo; rhi = (uint32_t)r_hi;
          pr = el.x ^ T.tNu[nu] ^ T.tRho[rho];
          if (w_hi >= 65536 || r_hi >= 65536) flags |= kRgWide >> 16;
          else pr ^= T.cfold;
          if (w_hi < 256 && r_hi < 256) { flags |= kRgNarrow >> 16; pr ^= T.nfold; }
          meta = (uint32_t)nu | ((uint32_t)rho << 8) | (flags << 16);
          if (kFull) meta |= Q.elIdx[src] << 19;
        }
      }
      // Any lane whose share exceeds the cap proves the step illegal; the exact
      // team-wide sum is checked after the pass.  Every queued region then
      // holds <= 2^27 areas.
      if (__any_sync(DSK_FULL, lane_full > kMaxAreas)) { abort = true; return; }
      push_region(ok, pr, xs, whi, rlo, rhi, meta);
    }
  }

  __device__ void finish() {
    drain_regions(true);
    drain_areas(true);
    drain_hits(true);
  }

  __device__ double warp_full() const {
    double s = lane_full;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(DSK_FULL, s, o);
    return s;
  }
};

}  // namespace dsk
