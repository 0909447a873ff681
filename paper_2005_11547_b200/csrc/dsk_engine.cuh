// dsk_engine.cuh -- the DartHash enumeration engine (one warp's pipeline).
//
// Restates DartHasher.dart_batch (ref/darthash.py:142-295) for the GPU.  One
// warp walks the elements of its share of a set and expands work through four
// load-balanced levels, each backed by a shared-memory ring so every stage
// runs on full batches:
//
//   element chunk --(depth+1)(rank_depth+1)--> regions (nu, rho)   [region ring]
//   region  --(w_hi+1)(r_hi-r_lo+1)--> areas (w, r) + Poisson count [area ring]
//   area    --count--> candidate darts, rank/weight filter       -> [hit ring]
//   hit     --> fingerprint, bucket hash, Sink (slot minimum / LSH buffer)
//
// Scheduling is a flat, warp-uniform "pull" loop: each iteration runs the
// deepest stage that has a full batch ready (hits >= 64, areas >= 32,
// regions >= 32, else the next 64 regions of the element chunk).  A stage
// consumes at most 64 children of the parents at the head of its ring,
// keeping a child cursor, and produces at most 64 items downstream; with
// downstream-first priority every ring stays below its capacity.  Each stage
// body exists once in the code (small I-cache footprint) and evaluates two
// independent children per lane (positions lo+lane and lo+32+lane) in
// straight-line code, so their dependent hash / fp64 chains interleave.
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
#pragma once
#include "dsk_device.cuh"

// DSK_DEBUG builds check the ring-capacity and indexing invariants the
// scheduler relies on (compute-sanitizer is unavailable on this pool).
#ifdef DSK_DEBUG
#include <assert.h>
#define DSK_CHECK(c) assert(c)
#else
#define DSK_CHECK(c) ((void)0)
#endif

namespace dsk {

// build-time tunables (profiles/sweep.sh builds variants)
#ifndef DSK_WARPS
#define DSK_WARPS 24
#endif
#ifndef DSK_RUN
#define DSK_RUN 3  // areas per walker run (the minhash sink: DSK_RUN_MH)
#endif
#ifndef DSK_RUN_MH
#define DSK_RUN_MH 2  // cfg3 k = 64: 22.9 -> 22.4 ms, cfg5 -0.6 %; the LSH sink prefers 3
#endif
#ifndef DSK_RUN_MH_DEEP
#define DSK_RUN_MH_DEEP 1  // minhash passes of rank depth >= 1 (general engine)
#endif
#ifndef DSK_DIRECT
#define DSK_DIRECT 2  // 0: off, 1: only when the rank depth is 0, 2: always when tables fit (cfg2 on 24 x 3: 23.4 -> 22.4 ms)
#endif
#ifndef DSK_REFILL
#define DSK_REFILL 8
#endif
#ifndef DSK_SEEK_TAB
#define DSK_SEEK_TAB 1  // walker seeks by table lookup for the first 256 areas of an element
#endif
#ifndef DSK_PT_IMM
#define DSK_PT_IMM 1  // Poisson thresholds as immediates instead of shared-memory loads
#endif
// scheduler thresholds (<= 32: a stage runs once this many items are queued)
#ifndef DSK_TH_HIT
#define DSK_TH_HIT 32
#endif
#ifndef DSK_TH_AREA
#define DSK_TH_AREA 32
#endif
#ifndef DSK_TH_REG
#define DSK_TH_REG 32
#endif
#ifndef DSK_FUSE
#define DSK_FUSE 2  // dart 0 finished at area creation: 0 never, 1 direct walkers, 2 both paths
#endif
// (per sink: the LSH sink measured faster without the fusion, Sink::kFuse)

constexpr int kILP = 1;      // children per lane per stage step (independent chains)
constexpr int kStep = 32 * kILP;
constexpr int kWarps = DSK_WARPS;  // warps per CTA (one CTA per SM)
constexpr int kQR = 64 * kILP;  // region / area ring capacity (>= 31 + kStep); power of two
constexpr int kQ = 64 * kILP;   // hit ring capacity (>= kStep - 1 + kStep); power of two
constexpr int kJs = 64;      // folded (j, stream) table rows; Poisson counts < 64
constexpr int kRwin = 64;    // per-pass rank-window table entries (nu, rho)
// (areas per walker run on the direct (rho = 0) path: Sink::kRun)
constexpr int kSeekTab = 256;  // walker seek table entries (per team, after the rank-window table)
constexpr int kRwinStride = kRwin + kSeekTab / 16;  // uint4 units per rank-window block incl. the seek table

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
  uint64_t dfold;         // T9[0]^T10[0]^T11[0]^cfold: the constant bytes of a rho = 0, w = 0 area
};

struct WarpQueues {
  ulonglong2 rgA[kQR];  // region: {P_R, x}
  uint4 rgB[kQR];       //         {w_hi, r_lo, r_hi, meta}
  ulonglong2 arA[kQR];  // area:   {P_A, x}
  uint4 arB[kQR];       //         {w, r, meta, element index (materialising sink)}
  ulonglong2 ht[kQ];    // hit:    {P_A ^ js[j][fp], rank bits}
  ulonglong2 el[32];    // element chunk: {E, x}
  uint2 elD[32];        // direct path: {rho=0 areas of the element, top nu | first V nu << 8}
  uint32_t elIdx[32];
};

// region meta: nu | rho << 8 | flags << 16 (| element index << 20, materialising sink)
constexpr uint32_t kRgHasPrev = 1u << 16, kRgWide = 1u << 17, kRgNarrow = 1u << 18,
                   kRgWEdge = 1u << 19;  // the w_hi column can hold darts heavier than x
// area meta: nu | rho << 8 | count << 16 | flags << 24
constexpr uint32_t kArWb = 1u << 24, kArRb = 1u << 25, kArLb = 1u << 26,
                   kArJ1 = 1u << 27;  // dart 0 was evaluated when the area was made

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

// The first six integer thresholds ceil(cdf[m] * 2^53) of the reference's
// POISSON1_CDF (ref/randomness.py:66-85) as immediates, pre-shifted to the
// 64-bit hash domain: X = h >> 11 >= t  <=>  h >= t << 11 (t < 2^53), so the
// count needs no shift.  dsk_ctx_create checks that the CDF it is given
// reproduces them (and rejects any other CDF).
constexpr uint64_t kPt0 = 0xbc5ab1b16779cULL, kPt1 = 0x178b56362cef38ULL,
                   kPt2 = 0x1d6e2bc3b82b06ULL, kPt3 = 0x1f6472f2e6944bULL,
                   kPt4 = 0x1fe204beb22e9cULL, kPt5 = 0x1ffb21e77480acULL;

// Poisson(1) count of the area whose Poisson hash (stream 3, j = 0) is h:
// #{m : (h >> 11) >= thr[m]} (inverse CDF, ref/randomness.py:145-147);
// counts >= 6 (0.06 % of areas) finish in a loop over the shared table.
__device__ __forceinline__ uint32_t poisson_count(uint64_t h, const PassParams &P,
                                                  const SmemTables &T) {
#if DSK_PT_IMM
  uint32_t c = (h >= (kPt0 << 11)) + (h >= (kPt1 << 11)) + (h >= (kPt2 << 11)) +
               (h >= (kPt3 << 11)) + (h >= (kPt4 << 11)) + (h >= (kPt5 << 11));
  (void)P;
  if (c == 6) {
    const uint64_t X = h >> 11;
    while (X >= T.pthr[c]) c++;
  }
#else
  const uint64_t X = h >> 11;
  uint32_t c = (X >= P.pt0) + (X >= P.pt1) + (X >= P.pt2) + (X >= P.pt3);
  if (c == 4) {
    while (X >= T.pthr[c]) c++;
  }
#endif
  return c;
}

// Parents at the head of a ring, expanded into children in steps of <= 64:
// scan of the first <= 32 parents' child counts.
struct HeadScan {
  uint32_t excl, incl, total;
  int mp;
};

__device__ __forceinline__ HeadScan head_scan(uint32_t c, int mp, int lane) {
  HeadScan h;
  h.mp = mp;
  h.incl = warp_incl_scan(c, lane);
  h.total = __shfl_sync(DSK_FULL, h.incl, 31);
  h.excl = h.incl - c;
  return h;
}

// After consuming children [cursor, hi) of the head parents: how many parents
// are exhausted, and the cursor into the first remaining one.
__device__ __forceinline__ void head_pop(const HeadScan &h, uint32_t hi, int lane, int &npop,
                                         uint32_t &cursor) {
  unsigned done = __ballot_sync(DSK_FULL, lane < h.mp && h.incl <= hi);
  npop = __popc(done);
  uint32_t consumed = __shfl_sync(DSK_FULL, h.incl, npop > 0 ? npop - 1 : 0);
  cursor = hi - (npop > 0 ? consumed : 0);
}

__device__ __forceinline__ int ringR(uint32_t x) { return (int)(x & (uint32_t)(kQR - 1)); }

// rank windows of one (nu, rho) for the rare sets whose (depth, rank depth)
// grid exceeds the per-pass table (kept out of line: cold code)
__device__ __noinline__ void rank_windows_slow(const PassParams &P, int nu, int rho,
                                               int64_t &r_hi, int64_t &r_lo, uint32_t &flags) {
  double r0 = __dadd_rn(pow2(rho), -1.0);
  double drho = pow2(rho - nu);
  r_hi = rank_window(P.L_hi, nu, rho, r0, drho);
  r_lo = 0;
  if (P.L_lo >= 0.0 && rho <= P.RD_lo) {
    int64_t rp = rank_window(P.L_lo, nu, rho, r0, drho);
    if (rp >= 0) { r_lo = rp; flags |= kRgHasPrev >> 16; }
  }
}

__device__ __forceinline__ uint32_t add_sat(uint32_t a, uint32_t b) {
  uint32_t r = a + b;
  return (r < a || r > 0x80000000u) ? 0x80000000u : r;
}

// kDirect: a specialisation for passes whose rank depth is 0 (every area
// has rho = 0: the direct walkers only); the region stages and their state
// compile away.  A pass that does not qualify sets `not_direct` and runs
// nothing (the caller redoes the set with the general engine).
template <class Sink, bool kFull, bool kDirect = false>
struct Engine {
  static constexpr int kRun = Sink::kRun;
  // Walker run length of this pass: passes of rank depth >= 1 (cfg2: elements
  // with a handful of rho = 0 areas each) hand out single areas when the sink
  // asks for it (Sink::kRunDeep; cfg2 22.4 -> 21.6 ms), rank depth 0 runs of kRun
  __device__ __forceinline__ uint32_t run_len() const {
    return (!kDirect && Sink::kRunDeep != kRun && P.RD > 0) ? (uint32_t)Sink::kRunDeep
                                                            : (uint32_t)kRun;
  }
  const SmemTables &T;
  WarpQueues &Q;
  // per-pass rank windows by (nu, rho): {r_hi + 1, r_lo | hasprev << 31,
  // inclusive prefix over nu of rho=0 in-band areas, inclusive prefix of
  // rho=0 full-step areas}
  uint4 *rwin;
  Sink &sink;
  const PassParams &P;  // in shared memory: read on use instead of pinning ~20 registers
  int lane;
  int rg_head = 0, rg_cnt = 0, ar_head = 0, ar_cnt = 0, ht_head = 0, ht_cnt = 0;
  uint32_t rg_cur = 0, ar_cur = 0;
  bool use_table = false;
  bool direct = false;      // rho = 0 areas come from per-lane walkers, not the region ring
  bool abort = false;       // warp-uniform: area cap exceeded by one lane's share
  bool not_direct = false;  // kDirect: this pass needs the general engine
  // per lane: areas of the full (non-band) step (area cap); saturates at
  // 2^31, far above the 2^27 cap, so sums stay exact wherever they matter
  uint32_t lane_full = 0;
  uint32_t n_darts = 0;     // per lane: candidate darts first seen in this band
  uint32_t n_hits = 0;      // per lane
  // element chunk state: lane i holds element i's region-count scan
  uint32_t el_excl = 0, el_total = 0, el_cur = 0;
  // direct path: chunk run scan (lane i: element i's first run) and cursor
  uint32_t run_excl = 0, run_total = 0, run_cur = 0;
  // direct path walker of this lane: areas [wk_a, wk_end) of element wk_slot
  uint32_t wk_a = 0, wk_end = 0, wk_r = 0, wk_rhi = 0, wk_rlo = 0;
  int wk_slot = 0, wk_nu = 0;

  __device__ Engine(const SmemTables &t, WarpQueues &q, uint4 *rw, Sink &s, const PassParams &p,
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
        // team warps write identical values into every field, and each warp
        // writes the whole table before reading it: no transient values
        reinterpret_cast<uint2 *>(&rwin[e])[0] = make_uint2(hi1, lo);
      }
      __syncwarp();
      // direct path tables: prefix sums over nu of the rho = 0 row counts
      uint32_t carry_a = 0, carry_f = 0;
      bool narrow = true;
      for (int nu0 = 0; nu0 <= P.maxd; nu0 += 32) {
        int nu = nu0 + lane;
        uint32_t ca = 0, cf = 0;
        if (nu <= P.maxd) {
          uint4 rw = rwin[nu * rdp1];
          uint32_t hi1 = rw.x, rlo = rw.y & 0x7fffffffu;
          cf = hi1;                                 // r_hi + 1 rows in the full step
          ca = hi1 > rlo ? hi1 - rlo : 0;           // rows r_lo .. r_hi in this band
          narrow = narrow && hi1 <= 65536;
        }
        uint32_t ia = warp_incl_scan(ca, lane) + carry_a;
        uint32_t fi = warp_incl_scan(cf, lane) + carry_f;
        if (nu <= P.maxd) reinterpret_cast<uint2 *>(&rwin[nu * rdp1])[1] = make_uint2(ia, fi);
        carry_a = __shfl_sync(DSK_FULL, ia, 31);
        carry_f = __shfl_sync(DSK_FULL, fi, 31);
      }
      // row counts stay far below 2^31 for every legal step
      direct = DSK_DIRECT && (P.RD == 0 || DSK_DIRECT == 2) && __all_sync(DSK_FULL, narrow) &&
               carry_a < (1u << 30) &&
               carry_f < (1u << 30);
#if DSK_SEEK_TAB
      if (direct) {
        // walker seek table: the nu of in-band area a of an element, for
        // a < kSeekTab (smallest nu with inclusive prefix > a; the element's
        // own dtop bounds a, so one table serves every element)
        __syncwarp();
        uint8_t *tab = seek_tab();
        for (uint32_t a = lane; a < (uint32_t)kSeekTab && a < carry_a; a += 32) {
          int lo = 0, hi = P.maxd;
          while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (rwin[mid * rdp1].z > a) hi = mid; else lo = mid + 1;
          }
          tab[a] = (uint8_t)lo;
        }
      }
#endif
    }
    if (kDirect) {
      not_direct = !(use_table && direct && P.RD == 0);
      direct = true;
    }
    __syncwarp();
  }

  // ---------------------------------------------------------------- pushes
  // (no draining here: the scheduler keeps every ring below capacity)
  __device__ __forceinline__ void push_hit(bool valid, double rank, uint64_t fpkey) {
    unsigned b = __ballot_sync(DSK_FULL, valid);
    if (valid) {
      int idx = (ht_head + ht_cnt + __popc(b & ((1u << lane) - 1))) & (kQ - 1);
      Q.ht[idx] = make_ulonglong2(fpkey, (unsigned long long)__double_as_longlong(rank));
    }
    ht_cnt += __popc(b);
    DSK_CHECK(ht_cnt <= kQ);
  }

  __device__ __forceinline__ void push_area(bool valid, uint64_t pa, double x, uint32_t w,
                                            uint32_t r, uint32_t meta, uint32_t elem) {
    unsigned b = __ballot_sync(DSK_FULL, valid);
    if (valid) {
      int idx = ringR(ar_head + ar_cnt + __popc(b & ((1u << lane) - 1)));
      Q.arA[idx] = make_ulonglong2(pa, (unsigned long long)__double_as_longlong(x));
      Q.arB[idx] = make_uint4(w, r, meta, elem);
    }
    ar_cnt += __popc(b);
    DSK_CHECK(ar_cnt <= kQR);
  }

  __device__ __forceinline__ void push_region(bool valid, uint64_t pr, double x, uint32_t whi,
                                              uint32_t rlo, uint32_t rhi, uint32_t meta) {
    unsigned b = __ballot_sync(DSK_FULL, valid);
    if (valid) {
      int idx = ringR(rg_head + rg_cnt + __popc(b & ((1u << lane) - 1)));
      Q.rgA[idx] = make_ulonglong2(pr, (unsigned long long)__double_as_longlong(x));
      Q.rgB[idx] = make_uint4(whi, rlo, rhi, meta);
    }
    rg_cnt += __popc(b);
    DSK_CHECK(rg_cnt <= kQR);
  }

  // ----------------------------------------------------------------- hits
  __device__ __forceinline__ void hit_keys(int idx, HitInfo &h) {
    ulonglong2 rec = Q.ht[idx];
    h.rank = __longlong_as_double((long long)rec.y);
    h.fp = finalize(rec.x);  // fingerprint, ref/randomness.py:149-152
    uint64_t x = T.bconst;   // hash64(fp, stream=5), ref/randomness.py:154-158
#pragma unroll
    for (int p = 0; p < 8; p++) x ^= T.tE[p][(h.fp >> (8 * p)) & 0xff];
    h.bhash = finalize(x);
  }

  __device__ void hits_step() {
    const int m = ht_cnt < kStep ? ht_cnt : kStep;
    HitInfo h[kILP];
#pragma unroll
    for (int q = 0; q < kILP; q++) hit_keys((ht_head + 32 * q + lane) & (kQ - 1), h[q]);
#pragma unroll
    for (int q = 0; q < kILP; q++) n_hits += (uint32_t)(lane + 32 * q < m);
    ht_head = (ht_head + m) & (kQ - 1);
    ht_cnt -= m;
#pragma unroll
    for (int q = 0; q < kILP; q++)
      if (m > 32 * q) sink.hit(lane + 32 * q < m, h[q], lane);
  }

  // ---------------------------------------------------------------- darts
  // Dart j of an area with uniform u (U stream) already drawn: rank, the
  // rank / weight tests (ref/darthash.py:264-292), and the hit (warp-collective).
  __device__ __forceinline__ void finish_dart(bool valid, uint64_t pa, uint32_t meta, uint32_t w,
                                              uint32_t r, double x, uint32_t j, double u,
                                              uint32_t elem) {
    const int nu = meta & 0xff, rho = (meta >> 8) & 0xff;
    // rank = r0 + (r + u) * drho, ref/darthash.py:282 (separately rounded)
    const double r0 = __dadd_rn(pow2(rho), -1.0);
    const double rank = __dadd_rn(r0, __dmul_rn(__dadd_rn((double)r, u), pow2(rho - nu)));
    bool hit = valid;
    if (meta & kArRb) hit = hit && rank <= P.L_hi;  // interior rows pass by monotonicity
    if (meta & kArLb) hit = hit && rank > P.L_lo;   // band: exclude darts seen before
    const bool needv = hit && (kFull || (meta & kArWb));  // only the w_hi column can miss
    double weight = 0.0;
    if (__any_sync(DSK_FULL, needv)) {
      double v = u53(finalize(pa ^ T.js[j][kStreamV - 1]));
      double dnu = __dmul_rn(P.inv_t, pow2(nu - rho));
      // weight = w0 + (w + v) * dnu, ref/darthash.py:281
      weight = __dadd_rn(T.w0[nu], __dmul_rn(__dadd_rn((double)w, v), dnu));
      if (needv && (meta & kArWb)) hit = weight <= x;  // inclusive, ref/darthash.py:284
    }
    if (kFull) {  // materialising sink: every hit with its full index tuple
      if (hit) {
        DartRow d;
        d.elem = elem;
        d.nu = nu;
        d.rho = rho;
        d.w = w;
        d.r = r;
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

  // Area (w, r) with key prefix pa: its Poisson(1) count (ref/randomness.py:
  // 145-147, j = 0, stream 3) and, from the same key, the U draw of dart 0
  // (an independent hash chain); dart 0 is finished here and only areas with
  // further darts enter the area ring (count - 1 darts, starting at j = 1).
  template <bool kFuse>
  __device__ __forceinline__ void emit_area(bool valid, uint64_t pa, double x, uint32_t w,
                                            uint32_t r, uint32_t meta, bool lb, uint32_t elem) {
    if (!kFuse) {
      const uint32_t k = poisson_count(finalize(pa ^ T.js[0][kStreamPoisson - 1]), P, T);
      const uint32_t cnt = valid ? k : 0;
      if (!lb) n_darts += cnt;
      push_area(cnt > 0, pa, x, w, r, meta | (cnt << 16), elem);
      return;
    }
    const uint64_t hp = finalize(pa ^ T.js[0][kStreamPoisson - 1]);
    const uint64_t hu = finalize(pa ^ T.js[0][kStreamU - 1]);
    const uint32_t k = poisson_count(hp, P, T);
    const uint32_t cnt = valid ? k : 0;
    if (!lb) n_darts += cnt;
    finish_dart(cnt > 0, pa, meta, w, r, x, 0, u53(hu), elem);
    push_area(cnt > 1, pa, x, w, r, meta | ((cnt - 1) << 16) | kArJ1, elem);
  }

  // darts [ar_cur, ar_cur + 32) of the head areas, j >= 1 (dart 0 was
  // finished when the area was made)
  __device__ void areas_step() {
    DSK_CHECK(ht_cnt < kStep);
    const int mp = ar_cnt < 32 ? ar_cnt : 32;
    uint32_t c = lane < mp ? (Q.arB[ringR(ar_head + lane)].z >> 16) & 0xff : 0;
    HeadScan hs = head_scan(c, mp, lane);
    const uint32_t lo = ar_cur, hi = lo + kStep < hs.total ? lo + kStep : hs.total;
    const uint32_t pos = lo + lane;
    const bool valid = pos < hi;
    const int src = warp_owner(hs.excl, pos);
    const int ai = ringR(ar_head + src);
    const ulonglong2 A = Q.arA[ai];
    const uint4 B = Q.arB[ai];
    const uint32_t meta = B.z;
    const uint32_t j = ((pos - __shfl_sync(DSK_FULL, hs.excl, src)) +
                        ((meta & kArJ1) ? 1u : 0u)) & (kJs - 1);
    const double u = u53(finalize(A.x ^ T.js[j][kStreamU - 1]));
    finish_dart(valid, A.x, meta, B.x, B.y, __longlong_as_double((long long)A.y), j, u, B.w);
    int npop;
    head_pop(hs, hi, lane, npop, ar_cur);
    ar_head = ringR(ar_head + npop);
    ar_cnt -= npop;
    __syncwarp();
  }

  // ---------------------------------------------------------------- areas
  // areas [rg_cur, rg_cur + 64) of the head regions, w-major
  // (ref/darthash.py:248-262), with the Poisson(1) count of each
  // (ref/randomness.py:145-147, :209-211: j = 0, stream 3)
  __device__ void regions_step() {
    DSK_CHECK(ar_cnt < 32 && ht_cnt < kStep);
    const int mp = rg_cnt < 32 ? rg_cnt : 32;
    uint32_t c = 0;
    if (lane < mp) {
      uint4 b = Q.rgB[ringR(rg_head + lane)];
      c = (b.x + 1) * (b.z - b.y + 1);
    }
    HeadScan hs = head_scan(c, mp, lane);
    const uint32_t lo = rg_cur, hi = lo + kStep < hs.total ? lo + kStep : hs.total;
    bool valid[kILP];
    uint32_t w[kILP], r[kILP], rmeta[kILP], rlo[kILP], whi[kILP], rhi[kILP];
    uint64_t pa[kILP];
    double x[kILP];
#pragma unroll
    for (int q = 0; q < kILP; q++) {
      uint32_t pos = lo + lane + 32 * q;
      valid[q] = pos < hi;
      int src = warp_owner(hs.excl, pos);
      uint32_t base = __shfl_sync(DSK_FULL, hs.excl, src);
      uint32_t off = valid[q] ? pos - base : 0;
      int gi = ringR(rg_head + src);
      ulonglong2 A = Q.rgA[gi];
      uint4 B = Q.rgB[gi];
      whi[q] = B.x; rlo[q] = B.y; rhi[q] = B.z; rmeta[q] = B.w;
      pa[q] = A.x;
      x[q] = __longlong_as_double((long long)A.y);
      uint32_t rc = rhi[q] - rlo[q] + 1;
      uint32_t ww;
      if (whi[q] == 0 || !valid[q]) {
        ww = 0;
      } else if (off < (1u << 20)) {  // fp32 quotient, off by at most one: corrected
        ww = (uint32_t)(((float)off + 0.5f) * __frcp_rn((float)rc));
        if (ww * rc > off) ww--;
        else if ((ww + 1) * rc <= off) ww++;
      } else {
        ww = off / rc;
      }
      w[q] = ww;
      r[q] = rlo[q] + (off - ww * rc);
    }
#pragma unroll
    for (int q = 0; q < kILP; q++) {
      uint64_t p = pa[q];
      if (rmeta[q] & kRgNarrow) {
        p ^= T.tW[0][w[q] & 0xff] ^ T.tR[0][r[q] & 0xff];
      } else {
        p ^= T.tW[0][w[q] & 0xff] ^ T.tW[1][(w[q] >> 8) & 0xff] ^ T.tR[0][r[q] & 0xff] ^
             T.tR[1][(r[q] >> 8) & 0xff];
        if (rmeta[q] & kRgWide)
          p ^= __ldg(&P.gtab[12 * 256 + ((w[q] >> 16) & 0xff)]) ^
               __ldg(&P.gtab[13 * 256 + (w[q] >> 24)]) ^
               __ldg(&P.gtab[16 * 256 + ((r[q] >> 16) & 0xff)]) ^
               __ldg(&P.gtab[17 * 256 + (r[q] >> 24)]);
      }
      const bool lb = (rmeta[q] & kRgHasPrev) && r[q] == rlo[q];
      const uint32_t meta = (rmeta[q] & 0xffff) |
                            (w[q] == whi[q] && (rmeta[q] & kRgWEdge) ? kArWb : 0) |
                            (r[q] == rhi[q] ? kArRb : 0) | (lb ? kArLb : 0);
      emit_area<Sink::kFuse && DSK_FUSE >= 2>(valid[q], p, x[q], w[q], r[q], meta, lb,
                               kFull ? rmeta[q] >> 20 : 0);
    }
    int npop;
    head_pop(hs, hi, lane, npop, rg_cur);
    rg_head = ringR(rg_head + npop);
    rg_cnt -= npop;
    __syncwarp();
  }

  // -------------------------------------------------------------- regions
  __device__ void load_chunk(bool valid, uint64_t id, double x, int depth, uint32_t eidx) {
    uint64_t E = 0;
    if (valid) {
#pragma unroll
      for (int p = 0; p < 8; p++) E ^= T.tE[p][(id >> (8 * p)) & 0xff];
    }
    uint32_t c;
    uint32_t nruns = 0, cnt0 = 0, dmeta = 0;
    if (direct) {
      // rho = 0 regions (nu, 0) have w_hi = 0 iff w0[nu] <= x (wmax = 0); w0
      // grows with nu, so they are exactly nu <= dtop.  Column 0 is the w_hi
      // column; its darts can miss only where the region's upper weight edge
      // fl(w0 + fl(1 * dnu)) exceeds x, i.e. from nu_v up (edges grow with nu).
      int dtop = valid ? depth : -1;
      while (dtop >= 0 && T.w0[dtop] > x) dtop--;
      int nu_v = dtop + 1;
      while (nu_v > 0 && __dadd_rn(T.w0[nu_v - 1], __dmul_rn(P.inv_t, pow2(nu_v - 1))) > x) nu_v--;
      if (dtop >= 0) {
        uint4 rw = rwin[dtop * (P.RD + 1)];
        cnt0 = rw.z;
        lane_full = add_sat(lane_full, rw.w);
      }
      nruns = (!kDirect && Sink::kRunDeep != kRun && P.RD > 0)
                  ? (cnt0 + Sink::kRunDeep - 1) / Sink::kRunDeep
                  : (cnt0 + kRun - 1) / kRun;
      dmeta = (uint32_t)(dtop & 0xff) | ((uint32_t)nu_v << 8);
      c = valid ? (uint32_t)(depth + 1) * (uint32_t)P.RD : 0;  // rho >= 1 regions
    } else {
      c = valid ? (uint32_t)(depth + 1) * (uint32_t)(P.RD + 1) : 0;
    }
    __syncwarp();
    Q.el[lane] = make_ulonglong2(E, (unsigned long long)__double_as_longlong(x));
    Q.elD[lane] = make_uint2(cnt0, dmeta);
    if (kFull) Q.elIdx[lane] = eidx;
    __syncwarp();
    uint32_t incl = warp_incl_scan(c, lane);
    el_total = __shfl_sync(DSK_FULL, incl, 31);
    el_excl = incl - c;
    el_cur = 0;
    uint32_t rincl = warp_incl_scan(nruns, lane);
    run_total = __shfl_sync(DSK_FULL, rincl, 31);
    run_excl = rincl - nruns;
    run_cur = 0;
  }

  // ------------------------------------------------------- direct (rho = 0)
  // Each lane walks a run of <= kRun consecutive rho = 0 areas of one element
  // (nu ascending, r ascending: the same areas the region ring would yield,
  // in any order), one area per step; idle lanes take the chunk's next runs.
  __device__ __forceinline__ uint8_t *seek_tab() const {
    return reinterpret_cast<uint8_t *>(rwin + kRwin);
  }

  __device__ __forceinline__ void walker_seek(uint32_t a, int dtop) {
    // smallest nu <= dtop with inclusive prefix > a
    const int rdp1 = P.RD + 1;
    int lo = 0, hi = dtop;
#if DSK_SEEK_TAB
    if (a < (uint32_t)kSeekTab) {
      lo = seek_tab()[a];
    } else
#endif
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (rwin[mid * rdp1].z > a) hi = mid; else lo = mid + 1;
    }
    uint4 rw = rwin[lo * rdp1];
    uint32_t rows = rw.x > (rw.y & 0x7fffffffu) ? rw.x - (rw.y & 0x7fffffffu) : 0;
    wk_nu = lo;
    wk_rlo = rw.y;
    wk_rhi = rw.x - 1;
    wk_r = (rw.y & 0x7fffffffu) + (a - (rw.z - rows));
  }

  __device__ void direct_step() {
    DSK_CHECK(ar_cnt < 32 && ht_cnt < kStep);
    // refill idle walkers with the chunk's next runs
    bool idle = wk_a >= wk_end;
    unsigned idle_mask = __ballot_sync(DSK_FULL, idle);
    if ((run_cur < run_total && __popc(idle_mask) >= DSK_REFILL) || idle_mask == DSK_FULL) {
      uint32_t q = run_cur + __popc(idle_mask & ((1u << lane) - 1));
      int src = warp_owner(run_excl, q);
      uint32_t first = __shfl_sync(DSK_FULL, run_excl, src);
      if (idle && q < run_total) {
        uint2 d = Q.elD[src];
        const uint32_t rl = run_len();
        uint32_t a0 = (q - first) * rl;
        wk_slot = src;
        wk_a = a0;
        wk_end = a0 + rl < d.x ? a0 + rl : d.x;
        walker_seek(a0, (int)(d.y & 0xff));
      }
      uint32_t took = (uint32_t)__popc(idle_mask);
      run_cur = run_cur + took < run_total ? run_cur + took : run_total;
    }
    const bool act = wk_a < wk_end;
    ulonglong2 el = Q.el[wk_slot];
    uint2 d = Q.elD[wk_slot];
    const int nu = wk_nu;
    const uint32_t r = wk_r;
    uint64_t p = el.x ^ T.tNu[nu] ^ T.dfold ^ T.tR[0][r & 0xff] ^ T.tR[1][(r >> 8) & 0xff];
    const bool hp = (wk_rlo & 0x80000000u) != 0;
    const bool lb = hp && r == (wk_rlo & 0x7fffffffu);
    const uint32_t meta = (uint32_t)nu | (nu >= (int)(d.y >> 8) ? kArWb : 0) |
                          (r == wk_rhi ? kArRb : 0) | (lb ? kArLb : 0);
    emit_area<Sink::kFuse && DSK_FUSE >= 1>(act, p, __longlong_as_double((long long)el.y), 0, r, meta, lb,
                             kFull ? Q.elIdx[wk_slot] : 0);
    // advance: next row, else the next non-empty nu
    if (act) {
      wk_a++;
      if (wk_a < wk_end) {
        if (r < wk_rhi) {
          wk_r = r + 1;
        } else {
          const int rdp1 = P.RD + 1;
          int nn = nu + 1;
          uint4 rw = rwin[nn * rdp1];
          while (rw.x <= (rw.y & 0x7fffffffu)) {  // empty band row range
            nn++;
            rw = rwin[nn * rdp1];
          }
          wk_nu = nn;
          wk_rlo = rw.y;
          wk_rhi = rw.x - 1;
          wk_r = rw.y & 0x7fffffffu;
        }
      }
    }
    __syncwarp();
  }

  __device__ __forceinline__ bool walkers_busy() const {
    return __any_sync(DSK_FULL, wk_a < wk_end) || run_cur < run_total;
  }

  // regions [el_cur, el_cur + 64) of the element chunk: the surviving
  // rectangle of each (nu, rho) (ref/darthash.py:180-225)
  __device__ void element_step() {
    DSK_CHECK(rg_cnt < 32);
    const int rdp1 = P.RD + 1;
    const float inv_rdp1 = 1.0f / (float)rdp1;
    const float inv_rd = P.RD > 0 ? 1.0f / (float)P.RD : 0.0f;
    const uint32_t lo = el_cur, hi = lo + kStep < el_total ? lo + kStep : el_total;
    bool ok[kILP];
    uint64_t pr[kILP];
    double xs[kILP];
    uint32_t owhi[kILP], orlo[kILP], orhi[kILP], ometa[kILP];
#pragma unroll
    for (int q = 0; q < kILP; q++) {
      uint32_t pos = lo + lane + 32 * q;
      const bool valid = pos < hi;
      int src = warp_owner(el_excl, pos);
      uint32_t idx = pos - __shfl_sync(DSK_FULL, el_excl, src);
      int nu, rho;
      if (direct) {  // rho = 0 comes from the walkers: idx covers rho in [1, RD]
        const int rd = P.RD;
        nu = (int)(((float)idx + 0.5f) * inv_rd);
        rho = (int)idx - nu * rd;
        if (rho < 0) { nu--; rho += rd; }
        else if (rho >= rd) { nu++; rho -= rd; }
        rho += 1;
      } else if (rdp1 == 1) {
        nu = (int)idx;
        rho = 0;
      } else {  // fp32 quotient, off by at most one: corrected below
        nu = (int)(((float)idx + 0.5f) * inv_rdp1);
        rho = (int)idx - nu * rdp1;
        if (rho < 0) { nu--; rho += rdp1; }
        else if (rho >= rdp1) { nu++; rho -= rdp1; }
      }
      nu &= 255;
      rho &= 255;
      ulonglong2 el = Q.el[src];
      xs[q] = __longlong_as_double((long long)el.y);
      ok[q] = false;
      pr[q] = 0; owhi[q] = 0; orlo[q] = 0; orhi[q] = 0; ometa[q] = 0;
      if (valid) {
        int64_t r_hi, r_lo = 0;
        uint32_t flags = 0;
        if (use_table) {
          DSK_CHECK(nu * rdp1 + rho < kRwin);
          uint4 rw = rwin[nu * rdp1 + rho];
          r_hi = (int64_t)rw.x - 1;
          if (rw.y & 0x80000000u) { r_lo = rw.y & 0x7fffffffu; flags |= kRgHasPrev >> 16; }
        } else {
          rank_windows_slow(P, nu, rho, r_hi, r_lo, flags);
        }
        int64_t w_hi = -1;
        bool wedge = true;
        if (r_hi >= 0) {
          double dnu = __dmul_rn(P.inv_t, pow2(nu - rho));
          w_hi = weight_window(xs[q], T.w0[nu], dnu, __dmul_rn(P.tf, pow2(rho - nu)), rho);
          // every dart of column w_hi weighs <= fl(w0 + fl((w_hi+1)*dnu)) by monotone
          // rounding; when that edge is <= x no dart of the region can miss
          wedge = __dadd_rn(T.w0[nu], __dmul_rn((double)(w_hi + 1), dnu)) > xs[q];
        }
        bool okq = w_hi >= 0 && r_lo <= r_hi;
        if (w_hi >= 0) {
          double full = (double)(w_hi + 1) * (double)(r_hi + 1);
          lane_full = add_sat(lane_full, full >= 2147483648.0 ? 0x80000000u : (uint32_t)full);
          // a region over the cap makes the step illegal (ref/darthash.py:242-244)
          if (full > kMaxAreas) okq = false;
        }
        if (okq) {
          owhi[q] = (uint32_t)w_hi; orlo[q] = (uint32_t)r_lo; orhi[q] = (uint32_t)r_hi;
          uint64_t p = el.x ^ T.tNu[nu] ^ T.tRho[rho];
          if (w_hi >= 65536 || r_hi >= 65536) flags |= kRgWide >> 16;
          else p ^= T.cfold;
          if (w_hi < 256 && r_hi < 256) { flags |= kRgNarrow >> 16; p ^= T.nfold; }
          if (wedge) flags |= kRgWEdge >> 16;
          pr[q] = p;
          ometa[q] = (uint32_t)nu | ((uint32_t)rho << 8) | (flags << 16);
          if (kFull) ometa[q] |= Q.elIdx[src] << 20;
        }
        ok[q] = okq;
      }
    }
    // Any lane whose share exceeds the cap proves the step illegal; the exact
    // team-wide sum is checked after the pass.  Every queued region then
    // holds <= 2^27 areas.
    if (__any_sync(DSK_FULL, lane_full > kMaxAreas)) {
      abort = true;
      return;
    }
#pragma unroll
    for (int q = 0; q < kILP; q++)
      push_region(ok[q], pr[q], xs[q], owhi[q], orlo[q], orhi[q], ometa[q]);
    el_cur = hi;
    __syncwarp();
  }

  // ------------------------------------------------------------ scheduler
  // `next_chunk(valid, id, x, depth, eidx)` loads this lane's element of the
  // warp's next chunk and returns false (warp-uniformly) when none is left.
  template <class ChunkFn>
  __device__ void run(ChunkFn next_chunk) {
    if (kDirect && not_direct) return;
    bool el_done = false;
    for (;;) {
      const bool up_area_empty = el_done && rg_cnt == 0;
      const bool up_hit_empty = up_area_empty && ar_cnt == 0;
      if (ht_cnt >= DSK_TH_HIT || (up_hit_empty && ht_cnt > 0)) {
        hits_step();
      } else if (ar_cnt >= DSK_TH_AREA || (up_area_empty && ar_cnt > 0)) {
        areas_step();
      } else if (!kDirect && (rg_cnt >= DSK_TH_REG || (el_done && rg_cnt > 0))) {
        regions_step();
      } else if (!el_done) {
        if (direct && walkers_busy()) {
          direct_step();
        } else if (!kDirect && el_cur < el_total) {
          element_step();
          if (abort) return;
        } else {
          bool valid;
          uint64_t id;
          double x;
          int depth;
          uint32_t eidx;
          if (!next_chunk(valid, id, x, depth, eidx)) {
            el_done = true;
          } else {
            load_chunk(valid, id, x, depth, eidx);
            if (__any_sync(DSK_FULL, lane_full > kMaxAreas)) {  // direct rows' cap share
              abort = true;
              return;
            }
          }
        }
      } else {
        return;
      }
    }
  }

  __device__ double warp_full() const {
    double s = (double)lane_full;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(DSK_FULL, s, o);
    return s;
  }
};

}  // namespace dsk
