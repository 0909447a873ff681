// dsk_lsh_kernel.cuh -- K5: (L, K) LSH table keys (included by dsk_kernels.cu).
#ifndef DSK_LSH_CLOSE
#define DSK_LSH_CLOSE 1  // drop hits of buckets already full when the band began
#endif
#ifndef DSK_LSH_DISCARD
#define DSK_LSH_DISCARD 0  // 1: discard spent hit-slot / selection lines from L2 (no write-back; measured -40 % DRAM traffic, +2 % time)
#endif
#ifndef DSK_LSH_SSEL
#define DSK_LSH_SSEL 1  // selections staged in the team's idle warp queues (shared memory; 5 % faster on cfg4)
#endif
#ifndef DSK_LSH_SEL32
#define DSK_LSH_SEL32 0  // 1: buckets of 33..64 entries: threshold + compaction, then a 32-wide sort (-0.5 % at 24 warps in teams of 2, +2.3 % in 28 single-warp teams at 72 registers)
#endif
#ifndef DSK_LSH_FAST
#define DSK_LSH_FAST 1  // 0: exact sort only; 1: float-key sort + exact fallback; 2: timing only
#endif
//
// lsh_key (ref/annindex.py:64-82): density t = L*K; darts are bucketed by
// hash64(fp, stream 5) mod L; at the first phi step where every bucket holds
// >= K darts (and >= L*K darts in total), each table's key is the K
// smallest darts of its bucket by (rank, index), in order.  LshIndex folds
// each key with HashFamily.mix64 (ref/annindex.py:135, ref/randomness.py:
// 160-166); that fold is fused here as the epilogue.
//
// Per team (G warps on one set):
//   enumeration  the shared engine, phi bands 1, 2, ... as for minhash; the
//                sink writes every hit {fp, rank} into its bucket's slots of
//                the team's global scratch (overflow list past S slots) and
//                counts hits per bucket;
//   check        after each band: all L buckets >= K (counter of buckets
//                that reached K);
//   selection    per bucket, a register bitonic sort (<= 64 entries) or a
//                counting rank by (rank bits, fp) -- positions < K are the
//                key, in order;
//   epilogue     one lane per table folds the K fingerprints with mix64.

#ifndef DSK_RUN_LSH_DEEP
#define DSK_RUN_LSH_DEEP DSK_RUN  // walker run length of LSH passes of rank depth >= 1 (general engine: normalised sets)
#endif
#ifndef DSK_LSH_FUSE
#define DSK_LSH_FUSE 1  // dart-0 fusion for the LSH sink (1.8 % faster since the per-bucket slots)
#endif
struct LshSink {
  static constexpr bool kFuse = DSK_LSH_FUSE != 0;
  static constexpr int kRun = DSK_RUN;
  static constexpr int kRunDeep = DSK_RUN_LSH_DEEP;
  ulonglong2 *buf;      // global: {fp, rank bits}, bucket b's first S hits at b*S
  ulonglong2 *ovf;      // global: hits beyond a bucket's S slots
  uint32_t *ovf_b;      // global: their buckets
  uint32_t S;           // slots per bucket
  uint32_t cap;         // overflow capacity
  ModU32 md;
  uint32_t K;
  unsigned int *total;  // smem: overflow entries
  unsigned int *cnt;    // buffered hits per bucket
  const unsigned int *prev;  // cnt at the start of this band
  unsigned int *full;   // buckets holding >= K hits
  int *overflow;

  // Bands are rank-ordered, so a bucket that held >= K darts when this band
  // began can never take a dart of this band into its K smallest: those hits
  // are not buffered (they still count toward H(phi*) in the engine).
  // (phi* = 1 inside a phi0 = 2 first band is recovered at selection time
  // from each bucket's K-th smallest rank, so nothing else is counted here.)
  __device__ void hit(bool valid, const HitInfo &h, int lane) {
    if (valid) {
      const uint32_t bucket = mod_u32(h.bhash, md);
      if (!(DSK_LSH_CLOSE && prev[bucket] >= K)) {
        const unsigned slot = atomicAdd(&cnt[bucket], 1u);
        if (slot == K - 1) atomicAdd(full, 1u);
        const ulonglong2 e =
            make_ulonglong2(h.fp, (unsigned long long)__double_as_longlong(h.rank));
        if (slot < S) {
          buf[(size_t)bucket * S + slot] = e;
        } else {  // rare: the bucket's slots are full
          const unsigned o = atomicAdd(total, 1u);
          if (o < cap) {
            ovf[o] = e;
            ovf_b[o] = bucket;
          } else {
            atomicOr(overflow, 1);
          }
        }
      }
    }
    (void)lane;
  }
  __device__ void row(const DartRow &) {}
};

struct LshArgs {
  const int64_t *indptr;
  const uint64_t *ids;
  const double *w;
  int64_t n;
  int32_t L, K;
  int32_t normalize;
  int32_t exact_sort;  // 1: skip the float-key fast path (env DSK_LSH_EXACT=1; tests)
  int32_t qshift;      // tests (env DSK_LSH_QSHIFT): coarser fixed-point sort keys, forcing collisions
  int32_t phi0;        // first band (0, phi0 / l1]; 2 when phi* = 1 is unlikely (large L)
  const uint32_t *retry_rows;  // second launch: rows whose first band failed (phi0 = 1)
  const unsigned *retry_n;
  int32_t force_retry;  // tests (env DSK_LSH_FORCE_RETRY=1): every first band is handed back
  double tf, inv_t;
  ModU32 md;
  int G;
  uint64_t *out_keys;
  uint64_t *out_fps;
  int32_t *status;
  int32_t *phi;
  uint32_t *stats;
  unsigned long long *counter;
  unsigned char *scratch;  // per-team global scratch
  size_t team_scratch;     // bytes per team
  uint32_t cap;            // overflow capacity per team
  uint32_t S;              // slots per bucket
  TableArgs tabs;
};


__host__ __device__ inline size_t lsh_team_bytes(int L) {
  return kTeamCtlBytes + align16((size_t)3 * L * sizeof(unsigned int)) + 16;
}

// (the direct-only kernel packs its queue blocks: q_stride / off_team_x in dsk_kernels.cu)
__host__ __device__ inline size_t lsh_smem(int L, int G, int nw, bool direct = false) {
  int teams = nw / G;
  return off_team_x(nw, direct) + (size_t)teams * lsh_team_bytes(L);
}

// Selection + epilogue of one set (ref/annindex.py:77-81, :135), kept out
// of line so its registers do not perturb the allocation of the enumeration
// engine (the kernel runs at the 80-register limit).
struct LshSel {
  const SmemTables *T;
  unsigned char *smem;
  TeamCtl *C;
  const unsigned *cnt;
  unsigned *fullc;
  const ulonglong2 *buf, *ovf;
  const uint32_t *ovf_b;
  uint64_t *sel;
  const uint64_t *gtab;
  uint64_t *out_fps, *out_keys;
  long long s;
  double Lsel;
  int L, K, G, team, wit, lane, tt, exact_sort, qshift, phi0, phi_star;
  uint32_t S, cap;
  uint32_t sq_off, qstride;  // the team's staging area: the used part of its warps' queue blocks
};

#ifndef DSK_LSH_SEL_NOINLINE
#define DSK_LSH_SEL_NOINLINE 0
#endif
#if DSK_LSH_SEL_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
int lsh_select(const LshSel &x) {
  const SmemTables &T = *x.T;
  unsigned char *smem = x.smem;
  TeamCtl &C = *x.C;
  const unsigned *cnt = x.cnt;
  unsigned *fullc = x.fullc;
  const ulonglong2 *buf = x.buf, *ovf = x.ovf;
  const uint32_t *ovf_b = x.ovf_b;
  uint64_t *sel = x.sel;
  const long long s = x.s;
  const double Lsel = x.Lsel;
  const int L = x.L, K = x.K, G = x.G, team = x.team, wit = x.wit, lane = x.lane, tt = x.tt;
  const uint32_t S = x.S;
  int phi_star = x.phi_star;
    // ---- selection (ref/annindex.py:77-81): bucket b's hits sit in its S
    // slots (plus, past S, in the overflow list).  K smallest of each
    // bucket by (rank bits, fp); bit-identical ranks with different
    // fingerprints flag a tie (the reference orders them by index tuple).
    //
    // Buckets of <= 64 entries (nearly all: ~40 per bucket at cfg4's
    // stopping step) are sorted in registers.  With K <= 32 the sort key is
    // 32 bits: a 26-bit fixed-point rank q = floor(rank * 2^26 / limit)
    // (monotone in the rank, every buffered rank is <= the final limit)
    // above the entry's 6-bit index, so the sorted position names its entry
    // directly; when two of the first K + 1 sorted keys share q the bucket
    // is redone on the exact (rank bits, fp) pair.  Larger buckets rank
    // each entry by counting.  (Fetching the next bucket's entries ahead --
    // into registers, by L1/L2 prefetch or by cp.async into shared memory --
    // measured slower: profiles/r02/experiments.md.)
    //
    // phi* = 1 inside a phi0 = 2 first band: bucket b held >= K hits with
    // rank <= L1 = fl(1 / l1) iff its K-th smallest rank is <= L1; when all
    // L buckets do, phi* = 1 (the K smallest are the same darts) and H(1)
    // is recounted from the buffer.
    const unsigned ovf_n = C.total < x.cap ? C.total : x.cap;
    const bool chk1 = phi_star == x.phi0 && x.phi0 > 1;
    const double L1 = chk1 ? __ddiv_rn(1.0, C.l1) : -1.0;
    const double qscale = __ddiv_rn(67108864.0, Lsel);  // 2^26 / limit
    const bool fastK = K <= 32 && DSK_LSH_FAST != 0 && !x.exact_sort && qscale < 1e300;
    const bool fast64 = DSK_LSH_FAST != 0 && !x.exact_sort;
    unsigned *full1 = fullc + 1;
    // selections of up to TB tables at a time in the team's (now idle) warp
    // queues, row stride K | 1 words (conflict-free column reads in the
    // epilogue); the global `sel` when one table does not fit
    const int KS = K | 1;
    // (the last 128 B of each warp's share are its compaction scratch words)
    const int cap_s = (int)((size_t)G * (x.qstride - 128) / 8);
    const bool in_smem = DSK_LSH_SSEL && cap_s >= KS;
    // (a multiple of the team's thread count, so no epilogue round is partial)
    const int TB = in_smem ? (cap_s / KS >= G * 32 ? cap_s / KS / (G * 32) * (G * 32) : cap_s / KS) : L;
    const int rs = in_smem ? KS : K;
    uint64_t *sq = reinterpret_cast<uint64_t *>(smem + x.sq_off);
    uint32_t *scr = reinterpret_cast<uint32_t *>(smem + x.sq_off + (size_t)G * x.qstride -
                                                 (size_t)(wit + 1) * 128);
    bool tie = false;
    auto fetch = [&](int b, ulonglong2 (&e)[2]) {
      const unsigned nb = cnt[b];
      const ulonglong2 *src = buf + (size_t)b * S;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const unsigned i = lane + 32 * h;
        e[h] = (nb <= 64 && i < nb) ? src[i] : make_ulonglong2(~0ULL, ~0ULL);
      }
    };
    for (int c0 = 0; c0 < L; c0 += TB) {
      const int c1 = c0 + TB < L ? c0 + TB : L;
      uint64_t *selp = in_smem ? sq : sel + (size_t)c0 * K;
      ulonglong2 e[2];
      for (int b = c0 + wit; b < c1; b += G) {
        const unsigned nb = cnt[b];
        const size_t o = (size_t)b * S;  // bucket b's slots (nb <= 64 <= S on the register paths)
        uint64_t *row = selp + (size_t)(b - c0) * rs;
        if (fastK) fetch(b, e);
        bool exact = nb > 64 || !fast64;
        if (!exact && fastK) {
          uint32_t key[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const unsigned i = lane + 32 * h;
            double qd = __dmul_rn(__longlong_as_double((long long)e[h].y), qscale);
            uint32_t q = qd < 67108863.0 ? (uint32_t)qd : 67108863u;
            key[h] = i < nb ? ((q >> x.qshift) << 6) | i : 0xffffffffu;
          }
          auto sort32 = [&](uint32_t &v) {
            for (int kk = 2; kk <= 32; kk <<= 1) {
              for (int j = kk >> 1; j > 0; j >>= 1) {
                uint32_t y = __shfl_xor_sync(DSK_FULL, v, j);
                bool take_min = ((lane & j) == 0) == ((lane & kk) == 0);
                if (take_min == (y < v)) v = y;
              }
            }
          };
          bool sorted = false;
          if (nb <= 32) {
            sort32(key[0]);
            sorted = true;
          }
#if DSK_LSH_SEL32
          else if (K <= 31) {
            // Only the K + 1 smallest keys matter: keep the keys below a q
            // threshold sized from the bucket (one band's ranks are uniform:
            // ~K + 6 of nb expected, widened / narrowed once), and when
            // K + 1..32 survive, compact them into one register (through the
            // warp's scratch words) and sort 32 instead of 64
            float fq = (float)(K + 6) / (float)nb * 67108864.0f;
            for (int att = 0; att < 2 && !sorted; att++) {
              const uint32_t tq = fq < 67108863.0f ? (uint32_t)fq : 67108863u;
              const uint32_t thr = ((tq >> x.qshift) << 6) | 63u;
              const bool s0 = key[0] <= thr, s1 = key[1] <= thr;
              const unsigned b0 = __ballot_sync(DSK_FULL, s0), b1 = __ballot_sync(DSK_FULL, s1);
              const int n0 = __popc(b0), c = n0 + __popc(b1);
              if (c >= K + 1 && c <= 32) {
                const unsigned lt = (1u << lane) - 1u;
                if (s0) scr[__popc(b0 & lt)] = key[0];
                if (s1) scr[n0 + __popc(b1 & lt)] = key[1];
                __syncwarp();
                uint32_t v = lane < c ? scr[lane] : 0xffffffffu;
                __syncwarp();
                sort32(v);
                key[0] = v;
                key[1] = 0xffffffffu;  // positions 0..K all lie below the threshold
                sorted = true;
              } else {
                fq = c < K + 1 ? fq * 1.5f : fq * 0.7f;
              }
            }
          }
#endif
          if (!sorted) {
            for (int kk = 2; kk <= 64; kk <<= 1) {
              for (int j = kk >> 1; j > 0; j >>= 1) {
                if (j == 32) {
                  if (key[1] < key[0]) { uint32_t t0 = key[0]; key[0] = key[1]; key[1] = t0; }
                } else {
#pragma unroll
                  for (int h = 0; h < 2; h++) {
                    int p = lane + 32 * h;
                    uint32_t y = __shfl_xor_sync(DSK_FULL, key[h], j);
                    bool take_min = ((p & j) == 0) == ((p & kk) == 0);
                    if (take_min == (y < key[h])) key[h] = y;
                  }
                }
              }
            }
          }
          // positions 0..K (K <= 32): lane p holds position p, position 32
          // is lane 0 of key[1]; equal q among them -> exact path
          uint32_t nx = __shfl_down_sync(DSK_FULL, key[0], 1);
          uint32_t f1 = __shfl_sync(DSK_FULL, key[1], 0);
          if (lane == 31) nx = f1;
          const bool coll = (unsigned)lane < (unsigned)K && (unsigned)lane + 1 < nb &&
                            (nx >> 6) == (key[0] >> 6);
          exact = __any_sync(DSK_FULL, coll);
          if (!exact) {
            const uint32_t idx = key[0] & 63u;
            const int srcl = (int)(idx & 31u);
            const uint64_t fa = __shfl_sync(DSK_FULL, e[0].x, srcl);
            const uint64_t fb = __shfl_sync(DSK_FULL, e[1].x, srcl);
            if (lane < K) row[lane] = idx >= 32 ? fb : fa;
            if (chk1) {
              const uint64_t ra = __shfl_sync(DSK_FULL, e[0].y, srcl);
              const uint64_t rb = __shfl_sync(DSK_FULL, e[1].y, srcl);
              const double rk = __longlong_as_double((long long)(idx >= 32 ? rb : ra));
              if (lane == K - 1 && rk <= L1) atomicAdd(full1, 1u);
            }
          }
        } else if (!exact) {
          // K > 32: bitonic sort of one 64-bit key per entry, the rank
          // rounded to float (monotone) above the entry's buffer index; when
          // the first K + 1 sorted keys have distinct float ranks their order
          // and the K-set equal the exact (rank, fp) order, else the bucket
          // takes the exact path below
          unsigned long long key[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            unsigned i = lane + 32 * h;
            if (i < nb) {
              uint32_t ei = (uint32_t)(o + i);
              double rk = __longlong_as_double((long long)buf[ei].y);
              key[h] = ((unsigned long long)__float_as_uint(__double2float_rn(rk)) << 32) | ei;
            } else {
              key[h] = ~0ULL;
            }
          }
          for (int kk = 2; kk <= 64; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
              if (j == 32) {
                if (key[1] < key[0]) { unsigned long long t0 = key[0]; key[0] = key[1]; key[1] = t0; }
              } else {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                  int p = lane + 32 * h;
                  unsigned long long y = __shfl_xor_sync(DSK_FULL, key[h], j);
                  bool take_min = ((p & j) == 0) == ((p & kk) == 0);
                  if (take_min == (y < key[h])) key[h] = y;
                }
              }
            }
          }
          unsigned long long d0 = __shfl_down_sync(DSK_FULL, key[0], 1);
          unsigned long long f1 = __shfl_sync(DSK_FULL, key[1], 0);
          unsigned long long d1 = __shfl_down_sync(DSK_FULL, key[1], 1);
          unsigned long long nx[2] = {lane < 31 ? d0 : f1, d1};
          bool coll = false;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            unsigned p = lane + 32 * h;
            if (p < (unsigned)K && p + 1 < nb && (nx[h] >> 32) == (key[h] >> 32)) coll = true;
          }
          exact = __any_sync(DSK_FULL, coll);
          if (!exact) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
              unsigned p = lane + 32 * h;
              if (p < (unsigned)K && p < nb) {
                const ulonglong2 ent = buf[(uint32_t)key[h]];
                row[p] = ent.x;
                if (chk1 && p == (unsigned)K - 1 &&
                    __longlong_as_double((long long)ent.y) <= L1)
                  atomicAdd(full1, 1u);
              }
            }
          }
        }
        if (exact && nb <= 64) {
          unsigned long long kr[2], kf[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            unsigned i = lane + 32 * h;
            if (i < nb) {
              ulonglong2 ent = buf[o + i];
              kr[h] = ent.y;
              kf[h] = ent.x;
            } else {
              kr[h] = ~0ULL;
              kf[h] = ~0ULL;
            }
          }
          for (int kk = 2; kk <= 64; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
              if (j == 32) {  // partner of position lane is lane + 32
                bool sw = kr[1] < kr[0] || (kr[1] == kr[0] && kf[1] < kf[0]);
                if (sw) {
                  unsigned long long t0 = kr[0], t1 = kf[0];
                  kr[0] = kr[1]; kf[0] = kf[1]; kr[1] = t0; kf[1] = t1;
                }
              } else {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                  int p = lane + 32 * h;
                  unsigned long long yr = __shfl_xor_sync(DSK_FULL, kr[h], j);
                  unsigned long long yf = __shfl_xor_sync(DSK_FULL, kf[h], j);
                  bool y_less = yr < kr[h] || (yr == kr[h] && yf < kf[h]);
                  bool take_min = ((p & j) == 0) == ((p & kk) == 0);
                  if (take_min == y_less) { kr[h] = yr; kf[h] = yf; }
                }
              }
            }
          }
          // successor in sorted order (position p + 1) for the tie check
          unsigned long long d0r = __shfl_down_sync(DSK_FULL, kr[0], 1);
          unsigned long long d0f = __shfl_down_sync(DSK_FULL, kf[0], 1);
          unsigned long long d1r = __shfl_down_sync(DSK_FULL, kr[1], 1);
          unsigned long long d1f = __shfl_down_sync(DSK_FULL, kf[1], 1);
          unsigned long long f1r = __shfl_sync(DSK_FULL, kr[1], 0);
          unsigned long long f1f = __shfl_sync(DSK_FULL, kf[1], 0);
          unsigned long long nxr[2] = {lane < 31 ? d0r : f1r, d1r};
          unsigned long long nxf[2] = {lane < 31 ? d0f : f1f, d1f};
#pragma unroll
          for (int h = 0; h < 2; h++) {
            unsigned p = lane + 32 * h;
            if (p + 1 < nb && nxr[h] == kr[h] && nxf[h] != kf[h]) tie = true;
            if (p < (unsigned)K) row[p] = kf[h];
            if (chk1 && p == (unsigned)K - 1 && __longlong_as_double((long long)kr[h]) <= L1)
              atomicAdd(full1, 1u);
          }
        } else if (exact) {
          // > 64 entries: rank every entry by counting; entry m of the bucket
          // is slot m (m < S) or the (m - S)-th overflow entry of bucket b
          const unsigned ns = nb < S ? nb : S;
          auto entry = [&](unsigned m, uint32_t &id) -> ulonglong2 {
            if (m < ns) { id = (uint32_t)m; return buf[o + m]; }
            unsigned seen = ns;
            for (unsigned q = 0; q < ovf_n; q++)
              if (ovf_b[q] == (uint32_t)b && seen++ == m) { id = S + q; return ovf[q]; }
            id = 0xffffffffu;
            return make_ulonglong2(~0ULL, ~0ULL);
          };
          for (unsigned i = lane; i < nb; i += 32) {
            uint32_t ei;
            ulonglong2 en2 = entry(i, ei);
            unsigned pos = 0;
            for (unsigned m = 0; m < nb; m++) {
              uint32_t mi;
              ulonglong2 f = entry(m, mi);
              bool less = f.y < en2.y || (f.y == en2.y && (f.x < en2.x || (f.x == en2.x && mi < ei)));
              pos += less;
              if (f.y == en2.y && mi != ei && f.x != en2.x) tie = true;
            }
            if (pos < (unsigned)K) row[pos] = en2.x;
            if (chk1 && pos == (unsigned)K - 1 && __longlong_as_double((long long)en2.y) <= L1)
              atomicAdd(full1, 1u);
          }
        }
        // the bucket's slots are spent: drop their L2 lines without a write-back
        // (the next set rewrites them), so the hit buffer never round-trips to HBM
#if DSK_LSH_DISCARD
        const unsigned lines = ((nb < S ? nb : S) * 16 + 127) / 128;
        for (unsigned q = lane; q < lines; q += 32) l2_discard(buf + o + 8 * q);
#endif
      }
      __threadfence_block();
      team_sync(G, team);
      // ---- epilogue: mix64 per table (ref/randomness.py:160-166):
      // mixed = hash64(element = v ^ mixed, w = position, stream 12)
      const uint64_t mconst = T.tNu[0] ^ T.tRho[0] ^ __ldg(&x.gtab[12 * 256]) ^
                              __ldg(&x.gtab[13 * 256]) ^ T.tR[0][0] ^ T.tR[1][0] ^
                              __ldg(&x.gtab[16 * 256]) ^ __ldg(&x.gtab[17 * 256]) ^
                              __ldg(&x.gtab[18 * 256]) ^ __ldg(&x.gtab[19 * 256]) ^
                              __ldg(&x.gtab[20 * 256 + kStreamKeyMix]) ^
                              __ldg(&x.gtab[21 * 256]);
      for (int b = c0 + tt; b < c1; b += G * 32) {
        const uint64_t *row = selp + (size_t)(b - c0) * rs;
        uint64_t mixed = 0;
        for (int p = 0; p < K; p++) {
          uint64_t v = row[p];
          if (x.out_fps) x.out_fps[((size_t)s * L + b) * K + p] = v;
          uint64_t e2 = v ^ mixed;
          uint64_t h = mconst ^ T.tW[0][p & 0xff] ^ T.tW[1][(p >> 8) & 0xff];
#pragma unroll
          for (int q = 0; q < 8; q++) h ^= T.tE[q][(e2 >> (8 * q)) & 0xff];
          mixed = finalize(h);
        }
        if (x.out_keys) x.out_keys[(size_t)s * L + b] = mixed;
      }
#if DSK_LSH_DISCARD
      if (!in_smem) {
        team_sync(G, team);  // every table's selection has been read
        const unsigned sel_lines = ((unsigned)(c1 - c0) * K * 8 + 127) / 128;
        for (unsigned q = tt; q < sel_lines; q += G * 32) l2_discard(selp + 16 * q);
      }
#endif
      team_sync(G, team);  // the next chunk overwrites the selections
    }
    if (__any_sync(DSK_FULL, tie) && lane == 0) atomicOr(&C.tie, 1);
    if (chk1) {
      team_sync(G, team);
      if (fullc[1] == (unsigned)L) {
        // phi* = 1: H(1) = the buffered hits with rank <= L1 (every hit of
        // the first band is buffered: no bucket was closed before it)
        phi_star = 1;
        unsigned c = 0;
        for (int b = wit; b < L; b += G) {
          const unsigned nb = cnt[b], ns = nb < S ? nb : S;
          for (unsigned i = lane; i < ns; i += 32)
            c += __longlong_as_double((long long)buf[(size_t)b * S + i].y) <= L1;
        }
        for (unsigned q = tt; q < ovf_n; q += G * 32)
          c += __longlong_as_double((long long)ovf[q].y) <= L1;
        c = __reduce_add_sync(DSK_FULL, c);
        team_sync(G, team);
        if (tt == 0) C.hits = 0;
        team_sync(G, team);
        if (lane == 0) atomicAdd(&C.hits, c);
      }
    }
  return phi_star;
}

// kGC: the per-bucket counters live in the team's global scratch instead of
// shared memory (L too large for shared memory; instantiated for NW = 20)
// kDirect: the first launch of a batch without normalisation runs the
// direct-only engine (rank depth 0 in every band: cfg4's (0, 2/l1] with
// l1 ~ 200); a set with a band that needs the region stages is handed to the
// retry launch (general engine, from phi = 1) like a failed first band.
template <int NW, bool kGC = false, bool kDirect = false>
__global__ void __launch_bounds__(NW * 32, 1) lsh_kernel(LshArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  SmemTables &T = g_tabs;
  load_tables(T, a.tabs);
  const int warp = opaque_int(threadIdx.x >> 5), lane = opaque_int(threadIdx.x & 31);
  const int G = a.G, team = opaque_team(warp / G), wit = opaque_team(warp % G),
            tt = opaque_team(wit * 32 + lane);
  const int L = a.L, K = a.K;
  WarpQueues &Q = *reinterpret_cast<WarpQueues *>(smem + kOffQueues + warp * q_stride(kDirect));
  const size_t tbytes = kGC ? kTeamCtlBytes : lsh_team_bytes(L);
#if DSK_OPAQUE_TB
  unsigned char *tb = smem + opaque_int((int)(off_team_x(NW, kDirect) + team * tbytes));
#else
  unsigned char *tb = smem + off_team_x(NW, kDirect) + team * tbytes;
#endif
  TeamCtl &C = *reinterpret_cast<TeamCtl *>(tb);
  // global scratch of this team
  const int teams = NW / G;
#if DSK_OPAQUE_TB
  unsigned char *gs = a.scratch + opaque_size(((size_t)blockIdx.x * teams + team) * a.team_scratch);
#else
  unsigned char *gs = a.scratch + ((size_t)blockIdx.x * teams + team) * a.team_scratch;
#endif
  // team scratch (128-byte aligned regions, so spent lines can be discarded):
  // slots L*S*16 | overflow cap*16 | overflow buckets cap*4 | selection
  // L*K*8 | (kGC) counters
  const size_t o_ovf = align128((size_t)L * a.S * 16), o_ovb = o_ovf + align128((size_t)a.cap * 16);
  const size_t o_sel = o_ovb + align128((size_t)a.cap * 4), o_cnt = o_sel + align128((size_t)L * K * 8);
  unsigned char *cb = kGC ? gs + o_cnt : tb + kTeamCtlBytes;
  unsigned int *cnt = reinterpret_cast<unsigned int *>(cb);
  unsigned int *off = cnt + L;
  unsigned int *fullc =
      reinterpret_cast<unsigned int *>(cb + align16((size_t)3 * L * sizeof(unsigned)));
  ulonglong2 *buf = reinterpret_cast<ulonglong2 *>(gs);
  ulonglong2 *ovf = reinterpret_cast<ulonglong2 *>(gs + o_ovf);
  uint32_t *ovf_b = reinterpret_cast<uint32_t *>(gs + o_ovb);
  uint64_t *sel = reinterpret_cast<uint64_t *>(gs + o_sel);
  const uint32_t S = a.S;
  __syncthreads();

  LshSink sink;
  sink.buf = buf;
  sink.ovf = ovf;
  sink.ovf_b = ovf_b;
  sink.S = S;
  sink.cap = a.cap;
  sink.md = a.md;
  sink.K = (uint32_t)K;
  sink.total = &C.total;
  sink.cnt = cnt;
  sink.prev = off;  // band-start snapshot of cnt
  sink.full = fullc;
  sink.overflow = &C.overflow;

  for (;;) {
    if (tt == 0) {
      long long q = (long long)atomicAdd(a.counter, 1ULL);
      if (a.retry_rows)  // retry launch: the rows the first launch handed back
        q = q < (long long)*a.retry_n ? (long long)a.retry_rows[q] : a.n;
      C.set = q;
    }
    team_sync(G, team);
    const long long s = C.set;
    if (s >= a.n) break;
    const int64_t lo = a.indptr[s], nnz = a.indptr[s + 1] - lo;
    for (int i = tt; i < L; i += G * 32) cnt[i] = off[i] = 0;
    if (tt == 0) {
      C.filled = 0; C.tie = 0; C.abort = 0; C.status = 0;
      C.areas[0] = C.areas[1] = 0.0; C.chunk[0] = C.chunk[1] = 0;
      C.darts = 0; C.hits = 0; C.total = 0; C.sexp = 0; C.overflow = 0;
      fullc[0] = fullc[1] = 0;
    }
    team_sync(G, team);
    if (wit == 0)
      set_prologue(a.w, a.tf, T, C, lo, nnz, reinterpret_cast<double *>(&Q), lane,
                   a.normalize != 0);
    team_sync(G, team);
    int status = C.status;
    int phi_star = 0;
    double final_areas = 0.0, Lsel = 0.0;
    uint32_t n_darts = 0, n_hits = 0;
    if (status == 0) {
      const double l1 = C.l1;
      const int maxd = C.maxdepth;
      const int sexp = C.sexp;
      // The first band is (0, phi0 / l1]: the keys do not depend on the phi
      // schedule, and phi* = 1 is recovered at
      // selection time (every bucket's K-th smallest rank <= fl(1 / l1)).  A first band that
      // fails (limit, depth or area cap at phi0 that phi = 1 might not hit)
      // is redone from phi = 1 by a second launch, stepping exactly as the
      // reference does.
      const int phi0 = a.phi0;
      status = DSK_NOCONV;
      double L_prev = -1.0;
      int RD_prev = 0;
      for (int phi = phi0; phi <= 64; phi++) {  // ref/annindex.py:70
        int err = 0;
        double Lim = __ddiv_rn((double)phi, l1);
        int RD = 0;
        if (!(Lim > 0.0) || isinf(Lim)) {
          err = DSK_LIMIT;
        } else {
          RD = floor_log2_host(__dadd_rn(1.0, Lim), T.l2thr);
          err = depth_status(maxd, RD);
        }
        if (!err) {
          PassParams P;
          P.gtab = a.tabs.tab;
          P.inv_t = a.inv_t;
          P.tf = a.tf;
          P.L_hi = Lim;
          P.L_lo = L_prev;
          P.RD = RD;
          P.RD_lo = RD_prev;
          P.maxd = maxd;
          poisson_regs(P, T);
          const int par = phi & 1;
          team_sync(G, team);
          if (!run_pass<LshSink, kDirect>(T, Q, sink, P, a.ids, a.w, lo, nnz, G, wit, lane, a.tf, C,
                                          n_darts, n_hits, par, sexp) &&
              tt == 0)
            atomicOr(&C.abort, 2);  // kDirect: this band needs the general engine
          team_sync(G, team);
          const double areas = C.areas[par];
          const bool ab = C.abort != 0;
          const unsigned full = fullc[0];
          const bool ovf = C.overflow != 0;
          if (tt == 0) { C.areas[par ^ 1] = 0.0; C.chunk[par ^ 1] = 0; }
          for (int i = tt; i < L; i += G * 32) off[i] = cnt[i];  // band snapshot
          team_sync(G, team);
          if (kDirect && (C.abort & 2)) err = DSK_RETRY;  // needs the general engine
          else if (ab || areas > kMaxAreas) err = DSK_AREAS;  // ref/darthash.py:243
          else if (ovf) err = DSK_SCRATCH;
          else if (a.force_retry && phi == phi0 && phi0 > 1) err = DSK_RETRY;  // tests
          if (!err) {
            final_areas = areas;
            // ref/annindex.py:72-76: >= L*K darts and every bucket >= K
            if (full == (unsigned)L) {  // implies >= L*K darts
              status = DSK_OK;
              phi_star = phi;
              Lsel = Lim;
              break;
            }
          }
        }
        if (err) {
          // a failing first band at phi0 > 1: the host's retry launch redoes
          // the set from phi = 1 (dsk_lsh_csr)
          status = ((phi == phi0 && phi0 > 1) || err == DSK_RETRY) ? DSK_RETRY : err;
          break;
        }
        L_prev = Lim;
        RD_prev = RD;
      }
    }
    unsigned wd = __reduce_add_sync(DSK_FULL, n_darts), wh = __reduce_add_sync(DSK_FULL, n_hits);
    if (lane == 0) { atomicAdd(&C.darts, wd); atomicAdd(&C.hits, wh); }
    team_sync(G, team);
    if (status == 0) {
      LshSel x;
      x.T = &T; x.smem = smem; x.C = &C; x.cnt = cnt; x.fullc = fullc; x.buf = buf; x.ovf = ovf;
      x.ovf_b = ovf_b; x.sel = sel; x.gtab = a.tabs.tab; x.out_fps = a.out_fps;
      x.out_keys = a.out_keys; x.s = s; x.Lsel = Lsel; x.L = L; x.K = K; x.G = G; x.team = team;
      x.wit = wit; x.lane = lane; x.tt = tt; x.exact_sort = a.exact_sort; x.qshift = a.qshift; x.phi0 = a.phi0;
      x.phi_star = phi_star; x.S = S; x.cap = a.cap;
      x.qstride = (uint32_t)q_stride(kDirect);
      x.sq_off = (uint32_t)(kOffQueues + (size_t)team * G * q_stride(kDirect) +
                            (kDirect ? kQDirectSkip : 0));
      phi_star = lsh_select(x);
    } else {
      for (int b = tt; b < L; b += G * 32) {
        if (a.out_keys) a.out_keys[(size_t)s * L + b] = 0;
        if (a.out_fps)
          for (int p = 0; p < K; p++) a.out_fps[((size_t)s * L + b) * K + p] = 0;
      }
    }
    team_sync(G, team);
    if (tt == 0) {
      a.status[s] = status | (C.tie ? DSK_STATUS_TIE : 0);
      if (a.phi) a.phi[s] = phi_star;
      if (a.stats) {
        uint32_t *st = a.stats + (size_t)s * 4;
        st[0] = (uint32_t)fmin(final_areas, 4294967295.0);
        st[1] = C.darts;
        st[2] = C.hits;
        st[3] = (uint32_t)phi_star;
      }
    }
    team_sync(G, team);
  }
}


// Rows of a phi0 = 2 launch whose first band failed (DSK_RETRY), for the
// retry launch that redoes them from phi = 1.
__global__ void lsh_retry_compact_kernel(const int32_t *status, int64_t n, uint32_t *rows,
                                         unsigned *count) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    if (status[r] == DSK_RETRY) rows[atomicAdd(count, 1u)] = (uint32_t)r;
}
