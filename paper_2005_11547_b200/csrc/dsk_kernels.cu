// dsk_kernels.cu -- sm_100a kernels and the C ABI of libdsk_b200.so.
//
//   K1+K2+K3+K4  minhash_kernel   CSR ingest, l1, validation, DartHash
//                                 enumeration, k-slot (rank, index) minimum,
//                                 in-kernel phi-band retry, 1-bit epilogue
//   K5           lsh_kernel       (dsk_lsh_kernel.cuh) bottom-K per table + mix64
//   K6           darts_kernel     DartBatch materialisation (tests)
//   K0           hash_peak_kernel hash-rate microbenchmark (roofline peak)
//   utilities    hash64 / mix64 / pack_onebit kernels
//
// Persistent grid: one 512-thread CTA per SM, 16 warps grouped into teams of
// G warps; a team sketches one set at a time, pulling set indices from a
// global atomic counter (load balance under Zipf-skewed nnz).  The 45 KB of
// hash tables live once per CTA in shared memory.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <thread>
#include <mutex>
#include <string>

#include "../../include/dsk_b200.h"
#include "dsk_device.cuh"
#include "dsk_engine.cuh"

#ifndef DSK_OPAQUE
#define DSK_OPAQUE 2  // 1: thread coordinates opaque; 2: team coordinates too (no re-derived warp / G: cfg4 -0.8 %, cfg2 -1.8 %)
#endif
#ifndef DSK_LPT
#define DSK_LPT 1  // largest-first row order for multi-wave minhash launches
#endif
#ifndef DSK_LSH_DIRECT_KERNEL
#define DSK_LSH_DIRECT_KERNEL 1  // LSH first launch on the direct-only engine specialisation
#endif
#ifndef DSK_MH_SPLIT_DEFAULT
#define DSK_MH_SPLIT_DEFAULT 1  // size split of single-warp-team minhash launches (DSK_MH_SPLIT)
#endif
#ifndef DSK_OPAQUE_TB
#define DSK_OPAQUE_TB 1  // LSH team block offsets opaque to the compiler (no rematerialisation)
#endif

using namespace dsk;

// ------------------------------------------------------------- context

constexpr int kMaxChunks = 64;  // host-buffer pipeline chunks per call

struct dsk_ctx {
  int device;
  int num_sms;
  uint64_t *d_tab;     // 22*256
  uint64_t *d_pthr;    // 64
  double *d_l2thr;     // 258
  unsigned long long *d_counter;  // kCounterSlots work counters, one per in-flight launch
  unsigned *d_hint = nullptr, *h_hint = nullptr;  // dsk_minhash_hints: device counters, pinned copy
  std::mutex hint_mu;
  std::atomic<unsigned> next_slot{0};
  size_t max_smem;
  // host-buffer path: device staging owned by the context
  std::mutex host_mu;
  void *stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t hs[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_in[kMaxChunks] = {}, ev_k[kMaxChunks] = {};
  // pageable host inputs are staged through two pinned buffers (ids and
  // weights of one chunk each), reused once their copy-out event fired
  unsigned char *pin_stage[2] = {nullptr, nullptr};
  size_t pin_bytes = 0;
  cudaEvent_t ev_pin[2] = {nullptr, nullptr};
  // pageable outputs: chunk results land in one of four pinned buffers and
  // are copied out by the host threads four chunks later
  static constexpr int kOutSlots = 4;
  unsigned char *out_stage[kOutSlots] = {};
  size_t out_bytes = 0;
  cudaEvent_t ev_out[kOutSlots] = {};
  // global scratch of the kernels (LSH hit buffers, large-k minhash slot
  // arrays): a small pool of slots reused in stream order, a launch waits for
  // the previous user of its slot (scratch_acquire / scratch_release)
  std::mutex scratch_mu;
  static constexpr int kScratchSlots = 4;
  void *scratch[kScratchSlots] = {};
  size_t scratch_bytes[kScratchSlots] = {};
  cudaEvent_t scratch_last[kScratchSlots] = {};
  cudaStream_t scratch_stream[kScratchSlots] = {};  // stream of the slot's last launch
  unsigned scratch_next = 0;
};

constexpr int kCounterSlots = 256;

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};  // kernels launched by this library

static inline void count_launch(unsigned k = 1) { g_launches.fetch_add(k); }

extern "C" uint64_t dsk_launch_count(void) { return g_launches.load(); }

static int set_err(int code, const char *msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                              \
  do {                                                                           \
    cudaError_t e__ = (x);                                                       \
    if (e__ != cudaSuccess) {                                                    \
      g_err = std::string(#x) + ": " + cudaGetErrorString(e__);                  \
      return DSK_ECUDA;                                                          \
    }                                                                            \
  } while (0)

extern "C" const char *dsk_last_error(void) { return g_err.c_str(); }

// SM count of the current device (grid caps of the context-free entry points)
static int c_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cache[dev].load();
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev].store(v);
  }
  return v;
}

extern "C" int64_t dsk_minhash_density(int64_t k) {
  if (k < 1) return -1;
  if (k == 1) return 1;
  return (int64_t)ceil((double)k * log((double)k)) + k;  // ref/core.py:156
}

// ----------------------------------------------------------- smem setup

struct TableArgs {
  const uint64_t *tab;
  const uint64_t *pthr;
  const double *l2thr;
  double tf;
};

// The hash tables live in STATIC shared memory: their addresses are link-time
// constants, so every table lookup is one LDS with an immediate offset (in
// dynamic shared memory the compiler rematerialises the window base,
// S2R + LEA, and adds it to every lookup address).  Dynamic shared memory
// (warp queues, team blocks, slots) follows it.
__shared__ __align__(16) SmemTables g_tabs;

__device__ void load_tables(SmemTables &T, const TableArgs &a) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < 8 * 256; i += nt) (&T.tE[0][0])[i] = a.tab[i];
  for (int i = tid; i < 256; i += nt) {
    T.tNu[i] = a.tab[8 * 256 + i];
    T.tRho[i] = a.tab[9 * 256 + i];
    T.tW[0][i] = a.tab[10 * 256 + i];
    T.tW[1][i] = a.tab[11 * 256 + i];
    T.tR[0][i] = a.tab[14 * 256 + i];
    T.tR[1][i] = a.tab[15 * 256 + i];
    // w0 = (2^nu - 1) / t, ref/darthash.py:189 (IEEE division)
    T.w0[i] = __ddiv_rn(__dadd_rn(pow2(i), -1.0), a.tf);
  }
  for (int i = tid; i < kJs * 4; i += nt) {
    int j = i / 4, s = i % 4 + 1;
    T.js[j][s - 1] = a.tab[18 * 256 + j] ^ a.tab[19 * 256] ^ a.tab[20 * 256 + s] ^ a.tab[21 * 256];
  }
  for (int i = tid; i < 64; i += nt) T.pthr[i] = a.pthr[i];
  for (int i = tid; i < 258; i += nt) T.l2thr[i] = a.l2thr[i];
  if (tid == 0) {
    T.cfold = a.tab[12 * 256] ^ a.tab[13 * 256] ^ a.tab[16 * 256] ^ a.tab[17 * 256];
    T.nfold = a.tab[11 * 256] ^ a.tab[15 * 256];
    uint64_t b = a.tab[20 * 256 + kStreamBucket] ^ a.tab[21 * 256];
    for (int p = 8; p < 20; p++) b ^= a.tab[p * 256];
    T.bconst = b;
    T.dfold = a.tab[9 * 256] ^ a.tab[10 * 256] ^ a.tab[11 * 256] ^ T.cfold;
  }
}

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ constexpr size_t align128(size_t x) { return (x + 127) & ~(size_t)127; }

constexpr size_t kOffQueues = 0;  // dynamic shared memory begins with the warp queues (tables: g_tabs)
constexpr size_t kQBytes = align16(sizeof(WarpQueues));
constexpr size_t kOffTeam = kOffQueues + kWarps * kQBytes;
// minhash / LSH kernels are instantiated for several CTA widths (warps per
// CTA); the host picks per launch the width whose team size is smallest.
__host__ __device__ constexpr size_t off_team(int nw) { return kOffQueues + nw * kQBytes; }
// The direct-only engine never touches the region ring (the first
// kQDirectSkip bytes of WarpQueues), so its kernels pack the warps' queue
// blocks at a stride of kQBytes - kQDirectSkip: warp w's (unused) region ring
// overlaps the tail of warp w - 1's block, and 28 warps fit where 22-24 did.
constexpr size_t kQDirectSkip = offsetof(WarpQueues, arA);
__host__ __device__ constexpr size_t q_stride(bool direct) {
  return direct ? kQBytes - kQDirectSkip : kQBytes;
}
__host__ __device__ constexpr size_t off_team_x(int nw, bool direct) {
  return direct ? kOffQueues + nw * q_stride(true) + kQDirectSkip : off_team(nw);
}
constexpr int kWidths[] = {24, 22, 20};

struct TeamCtl {
  long long set;
  double l1;
  double areas[2];        // per-pass area counts, double-buffered by phi parity
  unsigned int chunk[2];  // per-pass element-chunk cursor, double-buffered
  unsigned int filled;
  int tie;
  int abort;
  int status;
  int maxdepth;
  unsigned int darts;
  unsigned int hits;
  int sexp;       // weight rescaling exponent (LSH normalisation), 0 otherwise
  unsigned int total;  // LSH: buffered hits
  int overflow;        // LSH: hit buffer overflow
  PassParams pp;       // parameters of the current pass (identical writes by the team's warps)
};
// per-team block: control word + the per-pass rank-window table + walker seek table
constexpr size_t kTeamCtlBytes = align16(sizeof(TeamCtl)) + kRwin * sizeof(uint4) + kSeekTab;
__device__ __forceinline__ uint4 *team_rwin(TeamCtl *C) {
  return reinterpret_cast<uint4 *>(reinterpret_cast<unsigned char *>(C) + align16(sizeof(TeamCtl)));
}

__device__ __forceinline__ void team_sync(int G, int team) {
  if (G == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(G * 32) : "memory");
  }
}

// ------------------------------------------------------------- minhash

template <bool kGlobal>  // slots in global memory (k too large for shared memory)
struct MinhashSink {
  static constexpr bool kFuse = true;
  static constexpr int kRun = DSK_RUN_MH;
  static constexpr int kRunDeep = DSK_RUN_MH_DEEP;
  uint64_t *slots;  // 2*k words: {rank bits, fingerprint} per slot, 16-B aligned
  ModU32 md;
  unsigned int *filled;
  int *tie;

  // Slot minimum by (rank, index) (ref/sketching.py:93-99): ranks are
  // positive doubles, so their IEEE bits order as uint64.  Bit-identical
  // ranks with different fingerprints flag a tie (resolved by full index
  // tuple on the host-requested tie path).
  __device__ void hit(bool valid, const HitInfo &h, int lane) {
    unsigned newly = 0;
    bool t = false;
    if (valid) {
      uint32_t b = mod_u32(h.bhash, md);
      uint64_t *sl = slots + 2 * (size_t)b;
      uint64_t rb = (uint64_t)__double_as_longlong(h.rank);
      uint64_t cr, cf;
      if (kGlobal) ld128_generic(sl, cr, cf);
      else ld128_shared(sl, cr, cf);
      while (true) {
        if (rb > cr || (rb == cr && h.fp >= cf)) {
          if (rb == cr && h.fp != cf) t = true;
          break;
        }
        if (rb == cr) t = true;
        uint64_t orr, off;
        if (kGlobal) cas128_generic(sl, cr, cf, rb, h.fp, orr, off);
        else cas128_shared(sl, cr, cf, rb, h.fp, orr, off);
        if (orr == cr && off == cf) {
          if (cr == kEmptyRank) newly = 1;
          break;
        }
        cr = orr;
        cf = off;
      }
    }
    unsigned nf = __reduce_add_sync(DSK_FULL, newly);
    bool anyt = __any_sync(DSK_FULL, t);
    if (lane == 0) {
      if (nf) atomicAdd(filled, nf);
      if (anyt) atomicOr(tie, 1);
    }
  }
  __device__ void row(const DartRow &) {}
};

struct MinhashArgs {
  const int64_t *indptr;
  const uint64_t *ids;
  const double *w;
  int64_t n;
  int32_t k;
  int32_t t;
  double tf, inv_t;
  ModU32 md;
  int G;  // warps per team
  uint64_t *out_values;
  uint64_t *out_bits;
  int32_t *status;
  int32_t *phi;
  uint32_t *stats;
  unsigned long long *counter;
  uint64_t *gslots;  // non-null: slot arrays in global memory, 2*k words per team
  const uint32_t *order;  // non-null: rows in processing order (largest first)
  const unsigned *order_on;  // device flag: the order differs from the identity
  // direct-only first launch: rows whose bands need the general engine are
  // appended to retry_out; the second (general) launch works through them
  uint32_t *retry_out;
  unsigned *retry_out_n;
  const uint32_t *retry_rows;
  const unsigned *retry_n;
  // size split: this launch takes positions [*q_begin, *q_end) of the order
  // (device values written by order_scatter_kernel; null: 0 / n)
  const unsigned *q_begin;
  const unsigned *q_end;
  TableArgs tabs;
};

// Per-set validation and l1 by warp 0 of the team: empty set (ref/sketching.py:86-88),
// finite positive weights (ref/core.py:38-41), l1 = np.sum (ref/core.py:44),
// max element depth (ref/darthash.py:154-158).  With `normalize`, the set is
// first rescaled by 2^-weight_class(l1) as LshIndex.insert does
// (ref/annindex.py:130-131, ref/core.py:57-60): C.sexp = -c and l1 is the
// np.sum of the rescaled weights.
__device__ void set_prologue(const double *w, double tf, const SmemTables &T, TeamCtl &C,
                             int64_t lo, int64_t nnz, double *scratch, int lane, bool normalize) {
  if (nnz == 0) {
    if (lane == 0) C.status = DSK_EMPTY;
    return;
  }
  bool bad = false;
  for (int64_t i = lane; i < nnz; i += 32) {
    double x = w[lo + i];
    bad |= !(isfinite(x) && x > 0.0);
  }
  bad = __any_sync(DSK_FULL, bad);
  double l1 = warp_np_sum(w + lo, nnz, scratch, lane, 0);
  int sexp = 0;
  if (normalize && !bad) {
    int e;
    frexp(l1, &e);  // weight_class, ref/annindex.py:39-44
    sexp = -(e - 1);
    l1 = warp_np_sum(w + lo, nnz, scratch, lane, sexp);
  }
  int maxd = 0;
  for (int64_t i = lane; i < nnz; i += 32) {
    double x = sexp ? scalbn(w[lo + i], sexp) : w[lo + i];
    int d = floor_log2_host(__dadd_rn(1.0, __dmul_rn(tf, x)), T.l2thr);
    maxd = d > maxd ? d : maxd;
  }
  maxd = __reduce_max_sync(DSK_FULL, (unsigned)maxd);
  if (lane == 0) {
    C.l1 = l1;
    C.maxdepth = maxd;
    C.sexp = sexp;
    if (bad) C.status = DSK_WEIGHT;
  }
}

template <class Sink, bool kDirect = false>
__device__ bool run_pass(const SmemTables &T, WarpQueues &Q, Sink &sink, const PassParams &P,
                         const uint64_t *ids, const double *w, int64_t lo, int64_t nnz, int G,
                         int wit, int lane, double tf, TeamCtl &C, uint32_t &n_darts,
                         uint32_t &n_hits, int par, int sexp = 0) {
  int64_t next_chunk = 0;
  C.pp = P;
  __syncwarp();
  Engine<Sink, false, kDirect> eng(T, Q, team_rwin(&C), sink, C.pp, lane);
  if (kDirect && eng.not_direct) return false;  // (same verdict in every warp of the team)
  // element chunks are handed out dynamically to the team's warps; small sets
  // use narrower chunks so every warp of the team gets elements
  const int CH = (G == 1 || nnz >= 64 * G) ? 32 : (32 / G > 4 ? 32 / G : 4);
  eng.run([&](bool &valid, uint64_t &id, double &x, int &depth, uint32_t &eidx) -> bool {
    int64_t c;
    if (G > 1) {
      unsigned got = 0;
      if (lane == 0) got = atomicAdd(&C.chunk[par], 1u);
      c = __shfl_sync(DSK_FULL, got, 0);
    } else {
      c = next_chunk++;
    }
    if (c * CH >= nnz) return false;
    int64_t e = c * CH + lane;
    valid = lane < CH && e < nnz;
    id = 0;
    x = 0.0;
    depth = 0;
    eidx = (uint32_t)e;
    if (valid) {
      id = ids[lo + e];
      x = w[lo + e];
      if (sexp) x = scalbn(x, sexp);
      depth = floor_log2_host(__dadd_rn(1.0, __dmul_rn(tf, x)), T.l2thr);
    }
    return true;
  });
  n_darts += eng.n_darts;
  n_hits += eng.n_hits;
  double wf = eng.warp_full();
  if (lane == 0) {
    atomicAdd(&C.areas[par], wf);
    if (eng.abort) atomicOr(&C.abort, 1);
  }
  return true;
}

__device__ __forceinline__ void poisson_regs(PassParams &P, const SmemTables &T) {
  P.pt0 = T.pthr[0];
  P.pt1 = T.pthr[1];
  P.pt2 = T.pthr[2];
  P.pt3 = T.pthr[3];
}

// Thread coordinates the compiler cannot rematerialise from special
// registers (at 80 registers it otherwise re-derives them, S2R included, at
// many uses); it keeps or spills them instead.
__device__ __forceinline__ int opaque_int(int v) {
#if DSK_OPAQUE
  asm volatile("" : "+r"(v));
#endif
  return v;
}
__device__ __forceinline__ size_t opaque_size(size_t v) {
#if DSK_OPAQUE
  asm volatile("" : "+l"(v));
#endif
  return v;
}
__device__ __forceinline__ int opaque_team(int v) {
#if DSK_OPAQUE >= 2
  asm volatile("" : "+r"(v));
#endif
  return v;
}

// kDirect: the direct-only engine specialisation (rank depth 0 in every
// band) on packed queue blocks; a set with a band that needs the region
// stages is appended to a.retry_out for the general-engine launch.
// kSingle: single-warp teams known at compile time (team = warp: no team
// barriers or divisions by the team size left in the code; cfg5 -1.7 %)
template <int NW, bool kGlobal = false, bool kDirect = false, bool kSingle = false>
__global__ void __launch_bounds__(NW * 32, 1) minhash_kernel(MinhashArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  SmemTables &T = g_tabs;
  load_tables(T, a.tabs);
  const int warp = opaque_int(threadIdx.x >> 5), lane = opaque_int(threadIdx.x & 31);
  const int G = kSingle ? 1 : a.G, team = kSingle ? warp : opaque_team(warp / G),
            wit = kSingle ? 0 : opaque_team(warp % G),
            tt = kSingle ? lane : opaque_team(wit * 32 + lane);
  const int k = a.k;
  WarpQueues &Q = *reinterpret_cast<WarpQueues *>(smem + kOffQueues + warp * q_stride(kDirect));
  TeamCtl &C =
      *reinterpret_cast<TeamCtl *>(smem + off_team_x(NW, kDirect) + team * kTeamCtlBytes);
  const int teams = NW / G;
  uint64_t *slots =
      kGlobal ? a.gslots + ((size_t)blockIdx.x * teams + team) * 2 * (size_t)k
              : reinterpret_cast<uint64_t *>(smem + off_team_x(NW, kDirect) +
                                             teams * kTeamCtlBytes) +
                    (size_t)team * 2 * k;
  __syncthreads();

  MinhashSink<kGlobal> sink;
  sink.slots = slots;
  sink.md = a.md;
  sink.filled = &C.filled;
  sink.tie = &C.tie;

  for (;;) {
    if (tt == 0) {
      long long q = (long long)atomicAdd(a.counter, 1ULL);
      if (a.retry_rows) {  // second launch: the rows the direct-only launch handed back
        C.set = q < (long long)*a.retry_n ? (long long)a.retry_rows[q] : a.n;
      } else {
        if (a.q_begin) q += (long long)*a.q_begin;
        if (a.q_end && q >= (long long)*a.q_end) q = a.n;
        C.set = (a.order && q < a.n && *a.order_on) ? (long long)a.order[q] : q;
      }
    }
    team_sync(G, team);
    const long long s = C.set;
    if (s >= a.n) break;
    const int64_t lo = a.indptr[s], nnz = a.indptr[s + 1] - lo;
    for (int i = tt; i < k; i += G * 32) {
      slots[2 * i] = kEmptyRank;
      slots[2 * i + 1] = 0;
    }
    if (tt == 0) {
      C.filled = 0; C.tie = 0; C.abort = 0; C.status = 0;
      C.areas[0] = C.areas[1] = 0.0; C.chunk[0] = C.chunk[1] = 0;
      C.darts = 0; C.hits = 0;
    }
    team_sync(G, team);
    if (wit == 0)
      set_prologue(a.w, a.tf, T, C, lo, nnz, reinterpret_cast<double *>(&Q), lane, false);
    team_sync(G, team);
    int status = C.status;
    int phi_star = 0;
    double final_areas = 0.0;
    uint32_t n_darts = 0, n_hits = 0;
    if (status == 0) {
      const double l1 = C.l1;
      const int maxd = C.maxdepth;
      status = DSK_NOCONV;
      double L_prev = -1.0;
      int RD_prev = 0;
      for (int phi = 1; phi <= 64; phi++) {  // ref/sketching.py:105
        // limit = phi / l1 and the checks of DartHasher.dart_batch
        // (ref/darthash.py:136-138, 157-160)
        double L = __ddiv_rn((double)phi, l1);
        if (!(L > 0.0) || isinf(L)) { status = DSK_LIMIT; break; }
        int RD = floor_log2_host(__dadd_rn(1.0, L), T.l2thr);
        if (depth_status(maxd, RD)) { status = depth_status(maxd, RD); break; }
        PassParams P;
        P.gtab = a.tabs.tab;
        P.inv_t = a.inv_t;
        P.tf = a.tf;
        P.L_hi = L;
        P.L_lo = L_prev;
        P.RD = RD;
        P.RD_lo = RD_prev;
        P.maxd = maxd;
        poisson_regs(P, T);
        const int par = phi & 1;
        // (both engine specialisations inlined here, direct-only for rank
        // depth 0 passes, measured cfg3 -2.5 % but cfg2 / cfg5 +16 %: the
        // minhash kernel keeps the general engine)
        if (!run_pass<MinhashSink<kGlobal>, kDirect>(T, Q, sink, P, a.ids, a.w, lo, nnz, G, wit,
                                                     lane, a.tf, C, n_darts, n_hits, par) &&
            tt == 0)
          atomicOr(&C.abort, 2);  // kDirect: this band needs the general engine
        team_sync(G, team);
        const double areas = C.areas[par];
        const bool ab = C.abort != 0;
        const bool handoff = kDirect && (C.abort & 2);
        const unsigned filled = C.filled;
        // the other parity's counters were last read before the previous
        // barrier and are next written in the following pass
        if (tt == 0) { C.areas[par ^ 1] = 0.0; C.chunk[par ^ 1] = 0; }
        team_sync(G, team);
        if (handoff) { status = DSK_RETRY; break; }
        if (ab || areas > kMaxAreas) { status = DSK_AREAS; break; }  // ref/darthash.py:243
        final_areas = areas;
        if (filled == (unsigned)k) {  // every bucket non-empty, ref/sketching.py:110
          status = DSK_OK;
          phi_star = phi;
          break;
        }
        L_prev = L;
        RD_prev = RD;
      }
    }
    // statistics
    unsigned wd = __reduce_add_sync(DSK_FULL, n_darts), wh = __reduce_add_sync(DSK_FULL, n_hits);
    if (lane == 0) { atomicAdd(&C.darts, wd); atomicAdd(&C.hits, wh); }
    team_sync(G, team);
    // epilogue: values, packed bits (ref/sketching.py:164-167, :229), status
    if (a.out_values) {
      uint64_t *o = a.out_values + (size_t)s * k;
      for (int i = tt; i < k; i += G * 32) o[i] = status == 0 ? slots[2 * i + 1] : 0;
    }
    if (a.out_bits) {
      const int words = (k + 63) / 64;
      uint64_t *o = a.out_bits + (size_t)s * words;
      for (int m = wit; m < words; m += G) {
        int i0 = 64 * m + lane, i1 = i0 + 32;
        bool b0 = status == 0 && i0 < k && (slots[2 * i0 + 1] & 1);
        bool b1 = status == 0 && i1 < k && (slots[2 * i1 + 1] & 1);
        unsigned lo32 = __ballot_sync(DSK_FULL, b0), hi32 = __ballot_sync(DSK_FULL, b1);
        if (lane == 0) o[m] = ((uint64_t)hi32 << 32) | lo32;
      }
    }
    if (tt == 0) {
      if (kDirect && status == DSK_RETRY && a.retry_out)
        a.retry_out[atomicAdd(a.retry_out_n, 1u)] = (uint32_t)s;
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

// ---------------------------------------------------------- K6: darts

struct DartsArgs {
  const int64_t *indptr;
  const uint64_t *ids;
  const double *w;
  int64_t n;
  double tf, inv_t;
  const double *rank_limit;
  const int64_t *offsets;
  int64_t cap;
  int64_t *counts;
  int32_t *status;
  uint64_t *element;
  uint16_t *nu, *rho;
  uint32_t *ww, *rr;
  uint16_t *jj;
  double *weight, *rank;
  uint64_t *fp;
  TableArgs tabs;
};

constexpr int64_t kSliceElems = 4096;  // element index field of the row sink (12 bits)

struct RowSink {
  static constexpr bool kFuse = true;
  static constexpr int kRun = DSK_RUN;
  static constexpr int kRunDeep = DSK_RUN;
  const DartsArgs *a;
  int64_t set, lo;
  unsigned long long *cursor;  // shared per warp
  __device__ void hit(bool, const HitInfo &, int) {}
  __device__ void row(const DartRow &d) {
    unsigned long long i = atomicAdd(cursor, 1ULL);
    if (a->cap > 0) {
      int64_t o = a->offsets[set] + (int64_t)i;
      int64_t end = set + 1 < a->n ? a->offsets[set + 1] : a->cap;
      if (o < end && o < a->cap) {
        a->element[o] = a->ids[lo + d.elem];
        a->nu[o] = (uint16_t)d.nu;
        a->rho[o] = (uint16_t)d.rho;
        a->ww[o] = d.w;
        a->rr[o] = d.r;
        a->jj[o] = (uint16_t)d.j;
        a->weight[o] = d.weight;
        a->rank[o] = d.rank;
        a->fp[o] = d.fp;
      }
    }
  }
};

__global__ void __launch_bounds__(kWarps * 32, 1) darts_kernel(DartsArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  SmemTables &T = g_tabs;
  load_tables(T, a.tabs);
  const int warp = opaque_int(threadIdx.x >> 5), lane = opaque_int(threadIdx.x & 31);
  WarpQueues &Q = *reinterpret_cast<WarpQueues *>(smem + kOffQueues + warp * kQBytes);
  unsigned long long *cursors =
      reinterpret_cast<unsigned long long *>(smem + kOffTeam);
  uint4 *rwin = reinterpret_cast<uint4 *>(smem + kOffTeam +
                                          align16(kWarps * sizeof(unsigned long long))) +
                warp * kRwinStride;
  PassParams *pps = reinterpret_cast<PassParams *>(
      smem + kOffTeam + align16(kWarps * sizeof(unsigned long long)) +
      kWarps * kRwinStride * sizeof(uint4));
  __syncthreads();
  for (int64_t s = (int64_t)blockIdx.x * kWarps + warp; s < a.n; s += (int64_t)gridDim.x * kWarps) {
    const int64_t lo = a.indptr[s], nnz = a.indptr[s + 1] - lo;
    const double L = a.rank_limit[s];
    int status = 0;
    if (nnz == 0) status = DSK_EMPTY;                           // ref/darthash.py:133-134
    else if (!(L > 0.0) || isinf(L)) status = DSK_LIMIT;        // :136-138
    int maxd = 0;
    for (int64_t i = lane; i < nnz && status == 0; i += 32) {
      int d = floor_log2_host(__dadd_rn(1.0, __dmul_rn(a.tf, a.w[lo + i])), T.l2thr);
      maxd = d > maxd ? d : maxd;
    }
    maxd = __reduce_max_sync(DSK_FULL, (unsigned)maxd);
    int RD = status == 0 ? floor_log2_host(__dadd_rn(1.0, L), T.l2thr) : 0;
    if (status == 0) status = depth_status(maxd, RD);  // :154-160
    if (lane == 0) cursors[warp] = 0;
    __syncwarp();
    if (status == 0) {
      PassParams P;
      P.gtab = a.tabs.tab;
      P.inv_t = a.inv_t;
      P.tf = a.tf;
      P.L_hi = L;
      P.L_lo = -1.0;
      P.RD = RD;
      P.RD_lo = 0;
      P.maxd = maxd;
      poisson_regs(P, T);
      if (lane == 0) pps[warp] = P;
      __syncwarp();
      // the row sink carries a 12-bit element index, so large sets are
      // enumerated in slices of 4096 elements (darts of an element depend on
      // that element alone); the area cap applies to the whole set
      // (ref/darthash.py:242-244; dsk_darts_csr runs a counting pass first,
      // so a capped set produces no rows)
      double full = 0.0;
      for (int64_t base = 0; base < nnz && status == 0; base += kSliceElems) {
        const int64_t m = nnz - base < kSliceElems ? nnz - base : kSliceElems;
        RowSink sink;
        sink.a = &a;
        sink.set = s;
        sink.lo = lo + base;
        sink.cursor = &cursors[warp];
        Engine<RowSink, true> eng(T, Q, rwin, sink, pps[warp], lane);
        int64_t next = 0;
        eng.run([&](bool &valid, uint64_t &id, double &x, int &depth, uint32_t &eidx) -> bool {
          int64_t c = next++;
          if (c * 32 >= m) return false;
          int64_t e = c * 32 + lane;
          valid = e < m;
          id = valid ? a.ids[lo + base + e] : 0;
          x = valid ? a.w[lo + base + e] : 0.0;
          depth = valid ? floor_log2_host(__dadd_rn(1.0, __dmul_rn(a.tf, x)), T.l2thr) : 0;
          eidx = (uint32_t)e;
          return true;
        });
        full += eng.warp_full();
        if (eng.abort || full > kMaxAreas) status = DSK_AREAS;
      }
    }
    __syncwarp();
    if (lane == 0) {
      a.status[s] = status;
      a.counts[s] = status == 0 ? (int64_t)cursors[warp] : 0;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------- utilities

__device__ __forceinline__ uint64_t hash64_global(const uint64_t *tab, uint64_t e, uint64_t nu,
                                                  uint64_t rho, uint64_t w, uint64_t r,
                                                  uint64_t j, uint64_t s) {
  uint64_t h = 0;
#pragma unroll
  for (int p = 0; p < 8; p++) h ^= __ldg(&tab[p * 256 + ((e >> (8 * p)) & 0xff)]);
  h ^= __ldg(&tab[8 * 256 + (nu & 0xff)]) ^ __ldg(&tab[9 * 256 + (rho & 0xff)]);
#pragma unroll
  for (int p = 0; p < 4; p++) h ^= __ldg(&tab[(10 + p) * 256 + ((w >> (8 * p)) & 0xff)]);
#pragma unroll
  for (int p = 0; p < 4; p++) h ^= __ldg(&tab[(14 + p) * 256 + ((r >> (8 * p)) & 0xff)]);
  h ^= __ldg(&tab[18 * 256 + (j & 0xff)]) ^ __ldg(&tab[19 * 256 + ((j >> 8) & 0xff)]);
  h ^= __ldg(&tab[20 * 256 + (s & 0xff)]) ^ __ldg(&tab[21 * 256 + ((s >> 8) & 0xff)]);
  return finalize(h);
}

__global__ void hash64_kernel(const uint64_t *tab, const uint64_t *e, const uint64_t *nu,
                              const uint64_t *rho, const uint64_t *w, const uint64_t *r,
                              const uint64_t *j, const uint64_t *s, int64_t n, uint64_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hash64_global(tab, e[i], nu[i], rho[i], w[i], r[i], j[i], s[i]);
}

// HashFamily.mix64, ref/randomness.py:160-166
__global__ void mix64_kernel(const uint64_t *tab, const uint64_t *v, int64_t nseq, int len,
                             uint64_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nseq;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t mixed = 0;
    for (int p = 0; p < len; p++)
      mixed = hash64_global(tab, v[i * len + p] ^ mixed, 0, 0, (uint64_t)p, 0, 0, kStreamKeyMix);
    out[i] = mixed;
  }
}

__global__ void pack_onebit_kernel(const uint64_t *v, int64_t n, int k, uint64_t *out) {
  const int words = (k + 63) / 64;
  const int lane = threadIdx.x & 31;
  int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = wid; t < n * words; t += nw) {
    int64_t s = t / words;
    int m = (int)(t % words);
    int i0 = 64 * m + lane, i1 = i0 + 32;
    bool b0 = i0 < k && (v[s * k + i0] & 1);
    bool b1 = i1 < k && (v[s * k + i1] & 1);
    unsigned lo = __ballot_sync(DSK_FULL, b0), hi = __ballot_sync(DSK_FULL, b1);
    if (lane == 0) out[t] = ((uint64_t)hi << 32) | lo;
  }
}

// K0: unit-cost microbenchmarks on all SMs, four independent chains per
// thread, no enumeration bookkeeping.  Modes:
//   0  the reference's hash unit (ref/randomness.py:121-131): 22 table
//      lookups, one per key byte, from all 22 tables in shared memory, plus
//      splitmix64 (key bytes taken from the chain's previous output);
//   1  a fully hoisted hash: one shared-memory word + splitmix64;
//   2  an area (ref/darthash.py:258-262): hoisted Poisson hash + the
//      inverse-CDF count against the integer thresholds;
//   3  a candidate dart (ref/darthash.py:279-284): hoisted U hash, the exact
//      u53 -> double, rank = r0 + (r + u) * drho (three rounded fp64 ops) and
//      the inclusive rank test;
//   4  a hit (ref/darthash.py:293, ref/randomness.py:154-158,
//      ref/sketching.py:93-99): fingerprint finalizer, the 8-lookup bucket
//      hash, mod k, and a 128-bit shared-memory CAS minimum into k = 256 slots;
//   5  one mix64 step (ref/randomness.py:160-166): 8 lookups + splitmix64.
// Modes 2-5 price the work the reference's algorithm cannot avoid per unit;
// bench.py sums A/rate2 + D/rate3 + H/rate4 (+ L*K/rate5) into the
// useful-work lower bound on a step's time.
__global__ void __launch_bounds__(512) hash_peak_kernel(const uint64_t *tab, int64_t iters,
                                                        int mode, uint64_t *sink) {
  __shared__ uint64_t ts[22 * 256];
  __shared__ __align__(16) uint64_t slots[2 * 256];
  for (int i = threadIdx.x; i < 22 * 256; i += blockDim.x) ts[i] = tab[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) { slots[2 * i] = kEmptyRank; slots[2 * i + 1] = 0; }
  __syncthreads();
  uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h[4] = {g * 4 + 1, g * 4 + 2, g * 4 + 3, g * 4 + 4};
  double acc = 0.0;
  uint32_t cnt = 0;
  if (mode == 0) {
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
      for (int c = 0; c < 4; c++) {
        // 22 key bytes: the 8 bytes of h, 8 of its rotation, 6 of its byte-swap
        uint64_t a = h[c], b = (a >> 29) | (a << 35), d = __byte_perm((uint32_t)a, (uint32_t)(a >> 32), 0x0123);
        uint64_t x = 0;
#pragma unroll
        for (int p = 0; p < 8; p++) x ^= ts[p * 256 + ((a >> (8 * p)) & 0xff)];
#pragma unroll
        for (int p = 0; p < 8; p++) x ^= ts[(8 + p) * 256 + ((b >> (8 * p)) & 0xff)];
#pragma unroll
        for (int p = 0; p < 6; p++) x ^= ts[(16 + p) * 256 + ((d >> (8 * p)) & 0xff)];
        h[c] = finalize(x);
      }
    }
  } else if (mode == 1) {
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
      for (int c = 0; c < 4; c++) h[c] = finalize(h[c] ^ ts[h[c] & 0xff]);
    }
  } else if (mode == 2) {
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
      for (int c = 0; c < 4; c++) {
        uint64_t X = finalize(h[c] ^ ts[(h[c] >> 3) & 0xff]) >> 11;
        uint32_t k = (X >= 0xbc5ab1b16779cULL) + (X >= 0x178b56362cef38ULL) +
                     (X >= 0x1d6e2bc3b82b06ULL) + (X >= 0x1f6472f2e6944bULL);
        cnt += k;
        h[c] = (h[c] + 0x9e3779b97f4a7c15ULL) ^ X;
      }
    }
  } else if (mode == 3) {
    const double L = 1.0 + 1e-9;
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
      for (int c = 0; c < 4; c++) {
        uint64_t hu = finalize(h[c] ^ ts[(h[c] >> 5) & 0xff]);
        double u = u53(hu);
        uint32_t r = (uint32_t)h[c] & 7;
        double rank = __dadd_rn(0.0, __dmul_rn(__dadd_rn((double)r, u), 0.125));
        cnt += rank <= L;
        h[c] = hu;
      }
    }
  } else if (mode == 4) {
    const ModU32 md = make_mod(256);
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
      for (int c = 0; c < 4; c++) {
        uint64_t fp = finalize(h[c]);
        uint64_t x = ts[20 * 256 + 5];
#pragma unroll
        for (int p = 0; p < 8; p++) x ^= ts[p * 256 + ((fp >> (8 * p)) & 0xff)];
        uint64_t bh = finalize(x);
        uint64_t *sl = slots + 2 * mod_u32(bh, md);
        uint64_t rb = bh >> 12;  // a positive double's bit pattern stands in for the rank
        uint64_t cr, cf;
        ld128_shared(sl, cr, cf);
        while (rb < cr || (rb == cr && fp < cf)) {
          uint64_t orr, off;
          cas128_shared(sl, cr, cf, rb, fp, orr, off);
          if (orr == cr && off == cf) break;
          cr = orr;
          cf = off;
        }
        h[c] = fp + 0x9e3779b97f4a7c15ULL;
      }
    }
  } else {
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
      for (int c = 0; c < 4; c++) {
        uint64_t x = ts[10 * 256 + (i & 0xff)];
#pragma unroll
        for (int p = 0; p < 8; p++) x ^= ts[p * 256 + ((h[c] >> (8 * p)) & 0xff)];
        h[c] = finalize(x) ^ (h[c] * 3);
      }
    }
  }
  uint64_t x = h[0] ^ h[1] ^ h[2] ^ h[3] ^ cnt ^ (uint64_t)__double_as_longlong(acc);
  if (x == 0x9e3779b97f4a7c15ULL) sink[0] = x;  // practically never; keeps the work live
}

#include "dsk_lsh_kernel.cuh"

// ------------------------------------------------------------- host side

static size_t minhash_smem(int k, int G, int nw, bool global_slots = false, bool direct = false) {
  int teams = nw / G;
  return off_team_x(nw, direct) + teams * kTeamCtlBytes +
         (global_slots ? 0 : (size_t)teams * k * 16);
}

static cudaError_t bottomk_set_smem(int bytes);  // dsk_bottomk.cuh

extern "C" int dsk_ctx_create(int device, const uint64_t *tables_host, const double *cdf_host,
                              const double *log2_thr_host, dsk_ctx **out) {
  if (!tables_host || !cdf_host || !log2_thr_host || !out) return set_err(DSK_EARG, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  dsk_ctx *c = new dsk_ctx();
  c->device = device;
  CUDA_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  int smem_optin = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  // the engine kernels hold the tables in static shared memory (g_tabs); the
  // dynamic budget is the opt-in maximum minus that
  {
    cudaFuncAttributes fa;
    CUDA_TRY(cudaFuncGetAttributes(&fa, lsh_kernel<24>));
    smem_optin -= (int)fa.sharedSizeBytes;
  }
  c->max_smem = (size_t)smem_optin;
  uint64_t pthr[64];
  for (int m = 0; m < 64; m++) {
    // count = #{m : cdf[m] <= (X * 2^-53)} = #{m : X >= ceil(cdf[m] * 2^53)}
    double v = ceil(ldexp(cdf_host[m], 53));
    pthr[m] = (uint64_t)v;
  }
  pthr[63] = pthr[63] > (1ULL << 53) ? pthr[63] : (1ULL << 53);  // X < 2^53: loop sentinel
#if DSK_PT_IMM
  if (pthr[0] != kPt0 || pthr[1] != kPt1 || pthr[2] != kPt2 || pthr[3] != kPt3 ||
      pthr[4] != kPt4 || pthr[5] != kPt5) {
    delete c;
    return set_err(DSK_EUNSUPPORTED, "Poisson CDF differs from the reference's POISSON1_CDF");
  }
#endif
  CUDA_TRY(cudaMalloc(&c->d_tab, 22 * 256 * sizeof(uint64_t)));
  CUDA_TRY(cudaMalloc(&c->d_pthr, 64 * sizeof(uint64_t)));
  CUDA_TRY(cudaMalloc(&c->d_l2thr, 258 * sizeof(double)));
  CUDA_TRY(cudaMalloc(&c->d_counter, kCounterSlots * sizeof(unsigned long long)));
  CUDA_TRY(cudaMalloc(&c->d_hint, 2 * sizeof(unsigned)));
  CUDA_TRY(cudaMallocHost(&c->h_hint, 2 * sizeof(unsigned)));
  CUDA_TRY(cudaMemcpy(c->d_tab, tables_host, 22 * 256 * sizeof(uint64_t), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_pthr, pthr, sizeof(pthr), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c->d_l2thr, log2_thr_host, 258 * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<22>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<20>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<28, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<28, false, true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<20, false, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<22, false, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<24, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(minhash_kernel<20, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(darts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  CUDA_TRY(bottomk_set_smem(smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(lsh_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(lsh_kernel<24, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(lsh_kernel<26, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(lsh_kernel<28, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(lsh_kernel<20, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(lsh_kernel<22>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  CUDA_TRY(cudaFuncSetAttribute(lsh_kernel<20>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin));
  *out = c;
  return DSK_OK;
}

extern "C" int dsk_ctx_destroy(dsk_ctx *c) {
  if (!c) return DSK_OK;
  cudaSetDevice(c->device);
  cudaFree(c->d_tab);
  cudaFree(c->d_pthr);
  cudaFree(c->d_l2thr);
  cudaFree(c->d_counter);
  cudaFree(c->d_hint);
  cudaFreeHost(c->h_hint);
  if (c->stage) cudaFree(c->stage);
  for (int i = 0; i < dsk_ctx::kScratchSlots; i++) {
    if (c->scratch[i]) cudaFree(c->scratch[i]);
    if (c->scratch_last[i]) cudaEventDestroy(c->scratch_last[i]);
  }
  for (int i = 0; i < 4; i++)
    if (c->hs[i]) cudaStreamDestroy(c->hs[i]);
  for (int i = 0; i < kMaxChunks; i++) {
    if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
    if (c->ev_k[i]) cudaEventDestroy(c->ev_k[i]);
  }
  for (int i = 0; i < 2; i++) {
    if (c->pin_stage[i]) cudaFreeHost(c->pin_stage[i]);
    if (c->ev_pin[i]) cudaEventDestroy(c->ev_pin[i]);
  }
  for (int i = 0; i < dsk_ctx::kOutSlots; i++) {
    if (c->out_stage[i]) cudaFreeHost(c->out_stage[i]);
    if (c->ev_out[i]) cudaEventDestroy(c->ev_out[i]);
  }
  delete c;
  return DSK_OK;
}

extern "C" int dsk_ctx_device(const dsk_ctx *c) { return c ? c->device : -1; }

static TableArgs table_args(const dsk_ctx *c, double tf) {
  TableArgs t;
  t.tab = c->d_tab;
  t.pthr = c->d_pthr;
  t.l2thr = c->d_l2thr;
  t.tf = tf;
  return t;
}

// a team size must divide the CTA's warps; teams of > 1 warp synchronise on
// named barriers 1..15
static bool team_size_ok(int G, int nw) { return nw % G == 0 && (G == 1 || nw / G <= 15); }

// (CTA width, team size).  Large batches: the smallest team whose slot
// arrays fit beside the queues (most teams in flight), preferring the wider
// CTA on ties.  Batches that fit in one wave of teams (n <= SMs * teams, e.g.
// single-set calls): the largest team that still gives every set its own
// team, so the warps of a CTA share few sets and each set finishes sooner.
template <class SmemFn>
static bool choose_shape(const dsk_ctx *c, SmemFn smem_of, int64_t n, int &nw_out,
                         int &g_out, int wide_g = 0) {
  // wide_g > 0: the widest CTA whose smallest team is <= max(that, best)
  // wins (LSH measured faster at 24 warps in teams of 2 than 22 in teams of 1)
  int best_g = 1 << 30, best_nw = 0;       // large-batch rule
  int wide_nw = 0, wide_gm = 0;
  int wave_g = 0, wave_nw = 0;             // one-wave rule
  const char *force = getenv("DSK_NW");  // tuning: restrict to one CTA width
  for (int nw : kWidths) {
    if (force && atoi(force) != nw) continue;
    int gmin = 0;
    const char *gforce = getenv("DSK_GMIN");  // tuning: smallest team size allowed
    for (int G = gforce ? atoi(gforce) : 1; G <= nw; G++) {
      if (!team_size_ok(G, nw) || smem_of(G, nw) > c->max_smem) continue;
      if (!gmin) gmin = G;
      if ((int64_t)c->num_sms * (nw / G) >= n && G > wave_g) { wave_g = G; wave_nw = nw; }
    }
    if (gmin && gmin < best_g) { best_g = gmin; best_nw = nw; }
    if (gmin && !wide_nw && gmin <= wide_g) { wide_nw = nw; wide_gm = gmin; }
  }
  if (!best_nw) return false;
  if (wide_nw && wide_nw > best_nw) { best_nw = wide_nw; best_g = wide_gm; }
  if (wave_nw && !getenv("DSK_NO_WAVE")) {
    nw_out = wave_nw;
    g_out = wave_g;
  } else {
    nw_out = best_nw;
    g_out = best_g;
  }
  return true;
}

// Stream-ordered scratch: the caller holds c->scratch_mu from acquire until
// release (after its launch), so concurrent calls on different streams never
// share a buffer and a reused slot waits for its previous launch.
static int scratch_acquire(dsk_ctx *c, size_t need, cudaStream_t st, int &slot, void *&ptr) {
  // prefer the slot last used on this stream (stream order already
  // serialises it), then an unused slot, then an idle one, then round robin
  slot = -1;
  for (int i = 0; i < dsk_ctx::kScratchSlots && slot < 0; i++)
    if (c->scratch[i] && c->scratch_stream[i] == st) slot = i;
  for (int i = 0; i < dsk_ctx::kScratchSlots && slot < 0; i++)
    if (!c->scratch[i]) slot = i;
  for (int i = 0; i < dsk_ctx::kScratchSlots && slot < 0; i++)
    if (cudaEventQuery(c->scratch_last[i]) == cudaSuccess) slot = i;
  if (slot < 0) slot = (int)(c->scratch_next++ % dsk_ctx::kScratchSlots);
  c->scratch_stream[slot] = st;
  if (!c->scratch_last[slot])
    CUDA_TRY(cudaEventCreateWithFlags(&c->scratch_last[slot], cudaEventDisableTiming));
  else
    CUDA_TRY(cudaStreamWaitEvent(st, c->scratch_last[slot], 0));
  if (c->scratch_bytes[slot] < need) {
    CUDA_TRY(cudaEventSynchronize(c->scratch_last[slot]));
    if (c->scratch[slot]) CUDA_TRY(cudaFree(c->scratch[slot]));
    c->scratch[slot] = nullptr;
    c->scratch_bytes[slot] = 0;
    CUDA_TRY(cudaMalloc(&c->scratch[slot], need));
    c->scratch_bytes[slot] = need;
  }
  ptr = c->scratch[slot];
  return DSK_OK;
}

static int scratch_release(dsk_ctx *c, int slot, cudaStream_t st) {
  CUDA_TRY(cudaEventRecord(c->scratch_last[slot], st));
  return DSK_OK;
}

// Largest-first processing order for multi-wave launches: rows grouped by
// floor(log2(nnz)) classes, largest class first (an approximate LPT order:
// the heavy tail of Zipf-sized batches no longer finishes last).
constexpr int kSizeClasses = 32;

constexpr int kBigClass = 10;  // sets of >= 1024 elements go to the wide-team launch of a size split

__device__ __forceinline__ int size_class(int64_t nnz) {
  return nnz <= 1 ? 0 : 63 - __clzll((unsigned long long)nnz);  // < 32 for nnz < 2^32
}

__global__ void order_hist_kernel(const int64_t *indptr, int64_t n, unsigned *hist) {
  __shared__ unsigned h[kSizeClasses];
  if (threadIdx.x < kSizeClasses) h[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[size_class(indptr[r + 1] - indptr[r])], 1u);
  __syncthreads();
  if (threadIdx.x < kSizeClasses && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// cursor[kSizeClasses] receives the "skewed" flag: with all rows in one
// size class the order stays the identity (the minhash kernel ignores it)
__global__ void order_scatter_kernel(const int64_t *indptr, int64_t n, const unsigned *hist,
                                     unsigned *cursor, uint32_t *order, int big_class) {
  __shared__ unsigned start[kSizeClasses];
  __shared__ bool one_class;
  if (threadIdx.x == 0) {  // exclusive scan, largest class first
    unsigned acc = 0, mx = 0;
    for (int c = kSizeClasses - 1; c >= 0; c--) {
      start[c] = acc;
      acc += hist[c];
      mx = hist[c] > mx ? hist[c] : mx;
    }
    one_class = (int64_t)mx == n;
    if (blockIdx.x == 0) {
      cursor[kSizeClasses] = one_class ? 0u : 1u;
      // size split: rows of >= 2^kBigClass elements sit at order[0, nbig)
      cursor[kSizeClasses + 1] = one_class ? 0u : start[big_class - 1];
      cursor[kSizeClasses + 2] = (unsigned)n;
    }
  }
  __syncthreads();
  if (one_class) return;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int c = size_class(indptr[r + 1] - indptr[r]);
    order[start[c] + atomicAdd(&cursor[c], 1u)] = (uint32_t)r;
  }
}

extern "C" int dsk_minhash_csr(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                               const double *weights, int64_t n, int32_t k, uint64_t *out_values,
                               uint64_t *out_bits, int32_t *status, int32_t *phi, uint32_t *stats,
                               void *stream) {
  return dsk_minhash_csr_ex(c, indptr, ids, weights, n, k, 0, out_values, out_bits, status, phi,
                            stats, stream);
}

// bit 62 of dsk_minhash_csr_ex's nnz_hint
constexpr int64_t kMhDirectHint = DSK_HINT_DIRECT;

extern "C" int dsk_minhash_csr_ex(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                                  const double *weights, int64_t n, int32_t k, int64_t nnz_hint,
                                  uint64_t *out_values, uint64_t *out_bits, int32_t *status,
                                  int32_t *phi, uint32_t *stats, void *stream) {
  if (!c || !indptr || !status || n < 0) return set_err(DSK_EARG, "bad argument");
  if (k < 1) return set_err(DSK_EARG, "k must be positive");  // ref/sketching.py:89-90
  if (n == 0) return DSK_OK;
  int64_t t = dsk_minhash_density(k);
  if (t > INT32_MAX) return set_err(DSK_EUNSUPPORTED, "k too large");
  int NW = 0, G = 0;
  // sets of >= 96 elements on average keep two warps busy: allow teams of 2
  // in a wider CTA (uniform 1024-element sets, k = 64/128: 24 x 2 is 4-5 %
  // faster than 20 x 1; sets of 64 elements prefer single-warp teams).
  // Callers withhold the hint for batches of mostly small sets (cfg5's Zipf
  // sizes, median 2: 20 x 1 is 8-12 % faster than 24 x 2)
  const bool direct_hint = (nnz_hint & kMhDirectHint) != 0;
  nnz_hint &= ~kMhDirectHint;
  // (sets of >= 512 elements also keep teams of 3 busy: cfg2, k = 256, runs
  // 1.1 % faster on 24 x 3 than on 22 x 2)
  const int wide_g = nnz_hint >= 512 * n ? 3 : nnz_hint >= 96 * n ? 2 : 0;
  // slot arrays in shared memory; k too large for that -> global memory (L2)
  bool global_slots = false;
  const char *gsl = getenv("DSK_GLOBAL_SLOTS");  // tuning/tests: slot arrays in global memory
  if ((gsl && atoi(gsl) != 0) ||
      !choose_shape(c, [&](int g, int nw) { return minhash_smem(k, g, nw); }, n, NW, G,
                    wide_g)) {
    global_slots = true;  // (instantiated for the 20-warp CTA only)
    if (!choose_shape(c, [&](int g, int nw) {
          return nw == 20 ? minhash_smem(k, g, nw, true) : (size_t)1 << 40; }, n, NW, G))
      return set_err(DSK_EUNSUPPORTED, "no CTA shape fits shared memory");
  }
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(c->device));
  // each launch owns one counter slot; slots recycle after kCounterSlots launches,
  // far beyond the number that can be in flight
  unsigned long long *counter = c->d_counter + (c->next_slot.fetch_add(1) % kCounterSlots);
  CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  MinhashArgs a;
  a.indptr = indptr; a.ids = ids; a.w = weights; a.n = n; a.k = k; a.t = (int32_t)t;
  a.tf = (double)t; a.inv_t = 1.0 / (double)t; a.md = make_mod((uint32_t)k); a.G = G;
  a.out_values = out_values; a.out_bits = out_bits; a.status = status; a.phi = phi;
  a.stats = stats; a.counter = counter; a.tabs = table_args(c, (double)t);
  a.gslots = nullptr;
  a.order = nullptr;
  a.order_on = nullptr;
  a.retry_out = nullptr;
  a.retry_out_n = nullptr;
  a.retry_rows = nullptr;
  a.retry_n = nullptr;
  a.q_begin = nullptr;
  a.q_end = nullptr;
  size_t smem = minhash_smem(k, G, NW, global_slots);
  int grid = c->num_sms;
  if ((int64_t)grid * (NW / G) > n) grid = (int)((n + (NW / G) - 1) / (NW / G));
  // Direct-first (kMhDirectHint in nnz_hint, or DSK_MH_DIRECT=1): the batch's
  // sets mostly have l1 above their phi* (rank depth 0 in every band), so a
  // first launch runs the direct-only engine on packed queue blocks -- the
  // widest CTA in which the general shape's team size (or the next that
  // fits) fits -- and appends the sets that need the region stages to a list
  // the general-engine launch then works through.
  int DNW = 0, DG = 0;
  {
    const char *e = getenv("DSK_MH_DIRECT");
    bool want = e ? atoi(e) != 0 : direct_hint;
    if (want && !global_slots && n >= 4 * (int64_t)grid * (NW / G) && n < (1LL << 32)) {
      for (int nw : {28, 24}) {
        if (nw < NW) break;
        for (int g = G; g <= nw && !DNW; g++)
          if (team_size_ok(g, nw) && minhash_smem(k, g, nw, false, true) <= c->max_smem) {
            DNW = nw;
            DG = g;
          }
        if (DNW) break;
      }
    }
  }
  const bool direct_first = DNW != 0;
  // largest-first order when the batch spans several waves of teams
  const bool lpt = DSK_LPT && n >= 4 * (int64_t)grid * (NW / G) && n < (1LL << 32);
  std::unique_lock<std::mutex> lock(c->scratch_mu, std::defer_lock);
  int slot = -1;
  uint32_t *retry_rows = nullptr;
  unsigned *retry_cnt = nullptr;
  if (global_slots || lpt || direct_first) {
    lock.lock();
    void *p = nullptr;
    const size_t slot_bytes = global_slots ? (size_t)grid * (NW / G) * 16 * (size_t)k : 0;
    const size_t order_off = align16(slot_bytes);
    const size_t retry_off =
        order_off + (lpt ? align16((size_t)n * 4) + 2 * kSizeClasses * 4 + 16 : 0);
    const size_t need = retry_off + (direct_first ? align16((size_t)n * 4) + 16 : 0);
    int rc = scratch_acquire(c, need, st, slot, p);
    if (rc) return rc;
    if (global_slots) a.gslots = (uint64_t *)p;
    if (lpt) {
      uint32_t *order = (uint32_t *)((char *)p + order_off);
      unsigned *hist = (unsigned *)((char *)order + align16((size_t)n * 4));
      CUDA_TRY(cudaMemsetAsync(hist, 0, 2 * kSizeClasses * 4 + 16, st));
      int og = (int)((n + 255) / 256 < 4 * c->num_sms ? (n + 255) / 256 : 4 * c->num_sms);
      order_hist_kernel<<<og, 256, 0, st>>>(indptr, n, hist); count_launch();
      int big_class = kBigClass;
      if (const char *e = getenv("DSK_MH_SPLIT_CLASS"))
        big_class = atoi(e) >= 1 && atoi(e) < kSizeClasses ? atoi(e) : kBigClass;
      order_scatter_kernel<<<og, 256, 0, st>>>(indptr, n, hist, hist + kSizeClasses, order, big_class); count_launch();
      a.order = order;
      a.order_on = hist + 2 * kSizeClasses;
    }
    if (direct_first) {
      retry_rows = (uint32_t *)((char *)p + retry_off);
      retry_cnt = (unsigned *)((char *)retry_rows + align16((size_t)n * 4));
      CUDA_TRY(cudaMemsetAsync(retry_cnt, 0, sizeof(unsigned), st));
    }
  }
  if (direct_first) {
    MinhashArgs d = a;
    d.G = DG;
    d.retry_out = retry_rows;
    d.retry_out_n = retry_cnt;
    int dgrid = c->num_sms;
    if ((int64_t)dgrid * (DNW / DG) > n) dgrid = (int)((n + (DNW / DG) - 1) / (DNW / DG));
    const size_t dsm = minhash_smem(k, DG, DNW, false, true);
    if (DNW == 28 && DG == 1) minhash_kernel<28, false, true, true><<<dgrid, 28 * 32, dsm, st>>>(d);
    else if (DNW == 28) minhash_kernel<28, false, true><<<dgrid, 28 * 32, dsm, st>>>(d);
    else minhash_kernel<24, false, true><<<dgrid, 24 * 32, dsm, st>>>(d);
    count_launch();
    CUDA_TRY(cudaGetLastError());
    // the general launch below takes the rows handed back (often none)
    unsigned long long *counter2 = c->d_counter + (c->next_slot.fetch_add(1) % kCounterSlots);
    CUDA_TRY(cudaMemsetAsync(counter2, 0, sizeof(unsigned long long), st));
    a.counter = counter2;
    a.order = nullptr;
    a.order_on = nullptr;
    a.retry_rows = retry_rows;
    a.retry_n = retry_cnt;
  }
  // Size split (single-warp-team shapes over rows of mixed sizes): a set of
  // 16384 elements takes ~17 ms on one warp, which bounds the launch; the
  // rows of >= 1024 elements (the head of the largest-first order) go to a
  // first launch in teams of >= 4 warps, the rest to the single-warp launch.
  {
    const char *e = getenv("DSK_MH_SPLIT");
    const bool want = e ? atoi(e) != 0 : DSK_MH_SPLIT_DEFAULT;
    if (want && lpt && !direct_first && !global_slots && G == 1) {
      int WNW = 0, WG = 0;
      for (int nw : kWidths) {
        for (int g = getenv("DSK_MH_SPLIT_G") ? atoi(getenv("DSK_MH_SPLIT_G")) : 4; g <= nw && !WNW; g++)
          if (team_size_ok(g, nw) && minhash_smem(k, g, nw) <= c->max_smem) { WNW = nw; WG = g; }
        if (WNW) break;
      }
      if (WNW) {
        MinhashArgs b = a;
        b.G = WG;
        b.q_end = a.order_on + 1;  // nbig
        unsigned long long *cw = c->d_counter + (c->next_slot.fetch_add(1) % kCounterSlots);
        CUDA_TRY(cudaMemsetAsync(cw, 0, sizeof(unsigned long long), st));
        b.counter = cw;
        const size_t wsm = minhash_smem(k, WG, WNW);
        switch (WNW) {
          case 24: minhash_kernel<24><<<c->num_sms, 24 * 32, wsm, st>>>(b); break;
          case 22: minhash_kernel<22><<<c->num_sms, 22 * 32, wsm, st>>>(b); break;
          default: minhash_kernel<20><<<c->num_sms, 20 * 32, wsm, st>>>(b); break;
        }
        count_launch();
        CUDA_TRY(cudaGetLastError());
        a.q_begin = a.order_on + 1;
        a.q_end = a.order_on + 2;
      }
    }
  }
  if (global_slots) {
    minhash_kernel<20, true><<<grid, 20 * 32, smem, st>>>(a); count_launch();
  } else {
    switch (NW) {
      case 24: minhash_kernel<24><<<grid, 24 * 32, smem, st>>>(a); break;
      case 22:
        if (G == 1) minhash_kernel<22, false, false, true><<<grid, 22 * 32, smem, st>>>(a);
        else minhash_kernel<22><<<grid, 22 * 32, smem, st>>>(a);
        break;
      default:
        if (G == 1) minhash_kernel<20, false, false, true><<<grid, 20 * 32, smem, st>>>(a);
        else minhash_kernel<20><<<grid, 20 * 32, smem, st>>>(a);
        break;
    }
    count_launch();
  }
  CUDA_TRY(cudaGetLastError());
  if (slot >= 0) return scratch_release(c, slot, st);
  return DSK_OK;
}

extern "C" int dsk_darts_csr(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                             const double *weights, int64_t n, int64_t t, const double *rank_limit,
                             const int64_t *offsets, int64_t cap, int64_t *counts, int32_t *status,
                             uint64_t *element, uint16_t *nu, uint16_t *rho, uint32_t *w,
                             uint32_t *r, uint16_t *j, double *weight, double *rank,
                             uint64_t *fingerprint, void *stream) {
  if (!c || !indptr || !rank_limit || !counts || !status || n < 0)
    return set_err(DSK_EARG, "bad argument");
  if (t < 1) return set_err(DSK_EARG, "density parameter t must be positive");
  if (cap > 0 && (!offsets || !element || !nu || !rho || !w || !r || !j || !weight || !rank ||
                  !fingerprint))
    return set_err(DSK_EARG, "null output column");
  if (n == 0) return DSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(c->device));
  DartsArgs a;
  a.indptr = indptr; a.ids = ids; a.w = weights; a.n = n; a.tf = (double)t;
  a.inv_t = 1.0 / (double)t; a.rank_limit = rank_limit; a.offsets = offsets; a.cap = cap;
  a.counts = counts; a.status = status; a.element = element; a.nu = nu; a.rho = rho; a.ww = w;
  a.rr = r; a.jj = j; a.weight = weight; a.rank = rank; a.fp = fingerprint;
  a.tabs = table_args(c, (double)t);
  size_t smem = kOffTeam + align16(kWarps * sizeof(unsigned long long)) +
                kWarps * kRwinStride * sizeof(uint4) + kWarps * sizeof(PassParams);
  int grid = (int)((n + kWarps - 1) / kWarps);
  if (grid > c->num_sms) grid = c->num_sms;
  darts_kernel<<<grid, kWarps * 32, smem, st>>>(a); count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}

extern "C" int dsk_hash64(dsk_ctx *c, const uint64_t *element, const uint64_t *nu,
                          const uint64_t *rho, const uint64_t *w, const uint64_t *r,
                          const uint64_t *j, const uint64_t *stream_tag, int64_t n, uint64_t *out,
                          void *stream) {
  if (!c || n < 0) return set_err(DSK_EARG, "bad argument");
  if (n == 0) return DSK_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  int grid = (int)((n + 255) / 256);
  if (grid > c->num_sms * 8) grid = c->num_sms * 8;
  hash64_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(c->d_tab, element, nu, rho, w, r, j,
                                                         stream_tag, n, out); count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}

extern "C" int dsk_mix64(dsk_ctx *c, const uint64_t *values, int64_t nseq, int32_t len,
                         uint64_t *out, void *stream) {
  if (!c || nseq < 0 || len < 0) return set_err(DSK_EARG, "bad argument");
  if (nseq == 0) return DSK_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  int grid = (int)((nseq + 255) / 256);
  if (grid > c->num_sms * 8) grid = c->num_sms * 8;
  mix64_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(c->d_tab, values, nseq, len, out); count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}

extern "C" int dsk_pack_onebit(const uint64_t *values, int64_t n, int32_t k, uint64_t *out_bits,
                               void *stream) {
  if (!values || !out_bits || n < 0 || k < 1) return set_err(DSK_EARG, "bad argument");
  if (n == 0) return DSK_OK;
  int64_t warps = n * ((k + 63) / 64);
  int grid = (int)((warps * 32 + 255) / 256);
  if (grid > c_sms() * 16) grid = c_sms() * 16;
  pack_onebit_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(values, n, k, out_bits); count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}

extern "C" int dsk_hash_peak(dsk_ctx *c, int32_t mode, int64_t n_per_thread, uint64_t *sink,
                             int64_t *hashes_done, void *stream) {
  if (!c || n_per_thread < 1 || !sink) return set_err(DSK_EARG, "bad argument");
  CUDA_TRY(cudaSetDevice(c->device));
  int grid = c->num_sms * 4;
  hash_peak_kernel<<<grid, 512, 0, (cudaStream_t)stream>>>(c->d_tab, n_per_thread, mode, sink); count_launch();
  CUDA_TRY(cudaGetLastError());
  if (hashes_done) *hashes_done = (int64_t)grid * 512 * 4 * n_per_thread;
  return DSK_OK;
}

// ------------------------------------------------------ host-buffer calls
//
// dsk_*_csr_host: the drop-in for a caller holding numpy arrays.  Rows are
// cut into chunks; one copy stream issues every chunk's H2D back to back
// (the whole input is staged, so the copy engine never waits), the compute
// streams run chunk c's kernel once its input event fires, and an output
// stream copies chunk c's results back once its kernel event fires.  The
// PCIe H2D then runs without gaps and only the last chunk's kernel and D2H
// stick out, so chunks ramp up at the start (16, 32 MB) and halve towards
// the end (down to 8 MB).  Device staging is owned by the context.

static int ensure_stage(dsk_ctx *c, size_t bytes) {
  if (!c->hs[0]) {
    for (int i = 0; i < 4; i++)
      CUDA_TRY(cudaStreamCreateWithFlags(&c->hs[i], cudaStreamNonBlocking));
    for (int i = 0; i < kMaxChunks; i++) {
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming));
    }
  }
  if (c->stage_bytes >= bytes) return DSK_OK;
  if (c->stage) CUDA_TRY(cudaFree(c->stage));
  c->stage = nullptr;
  c->stage_bytes = 0;
  CUDA_TRY(cudaMalloc(&c->stage, bytes));
  c->stage_bytes = bytes;
  return DSK_OK;
}

// Row chunk boundaries: chunk i carries ~min(cap, 16 MB << i, max(8 MB,
// remaining / 2)) input bytes (16 B per nonzero + 8 B per row).
// first chunk and smallest tail chunk in MB (env DSK_RAMP_MB="first,tail")
static size_t kRampMB[2] = {16, 8};

static void plan_chunks(const int64_t *indptr, int64_t n, size_t cap, int64_t *bounds,
                        int max_chunks, int *nchunks) {
  if (const char *e = getenv("DSK_RAMP_MB")) {
    int f = 0, t = 0;
    if (sscanf(e, "%d,%d", &f, &t) == 2 && f > 0 && t > 0) { kRampMB[0] = f; kRampMB[1] = t; }
  }
  const size_t total = (size_t)indptr[n] * 16 + (size_t)n * 8;
  if (cap < total / (max_chunks - 12)) cap = total / (max_chunks - 12) + 1;
  int m = 0;
  bounds[m++] = 0;
  int64_t r = 0;
  size_t done = 0;
  while (r < n && m < max_chunks) {
    const int64_t lo = r;
    size_t target = cap;
    const size_t ramp = kRampMB[0] << (20 + (m - 1 < 6 ? m - 1 : 6));
    if (ramp < target) target = ramp;
    size_t half = (total - done) / 2;
    if (half < (kRampMB[1] << 20)) half = kRampMB[1] << 20;
    if (half < target) target = half;
    // largest r with bytes(lo, r) <= target (at least one row)
    int64_t a = lo + 1, b = n;
    while (a < b) {
      const int64_t mid = a + (b - a + 1) / 2;
      if ((size_t)((indptr[mid] - indptr[lo]) * 16 + (mid - lo) * 8) <= target) a = mid;
      else b = mid - 1;
    }
    r = a;
    done += (size_t)((indptr[r] - indptr[lo]) * 16 + (r - lo) * 8);
    bounds[m++] = r;
  }
  if (bounds[m - 1] != n) bounds[m - 1] = n;
  *nchunks = m - 1;
}

// Largest chunk in MB of input.  Minhash, measured on cfg2 (pinned / plain
// numpy): 16 MB 31.6 / 35.6 ms/step e2e, 24 MB 31.6 / 34.1, 32 MB 31.4 / 35-37,
// 48 MB 32.4 / 42.4, 64 MB 32.2 / 40.8, 128 MB 32.3 / 42.3; cfg3 k = 64: 32 MB
// 26.6 / 35.5, 64 MB 27.2 / 44.2.  Batches of skewed row sizes (cfg5) take
// 512 MB chunks: a launch lasts at least as long as its largest set takes on
// one single-warp team (~17 ms for 16384 elements), so short launches are all
// tail -- 2e6 cfg5 sets: 64 MB 499 ms, 256 MB 296, 512 MB 236, 1 GB 232
// (device-resident 152).  LSH (two launches and a compaction per
// chunk, ~85 ns of kernel time per input KB), measured on cfg4: 32 MB 186.9,
// 64 MB 183.1, 128 MB 181.3, 192 MB 180.1, 256 MB 179.5.
static size_t host_chunk_cap(size_t default_mb) {
  size_t mb = default_mb;
  if (const char *e = getenv("DSK_CHUNK_MB")) mb = atoi(e) > 0 ? (size_t)atoi(e) : default_mb;
  return mb << 20;
}

static std::atomic<unsigned long long> g_h2d_bytes{0};  // bytes copied in by host-buffer calls

extern "C" uint64_t dsk_h2d_bytes(void) { return g_h2d_bytes.load(); }

// Drive the pipeline.  launch(r0, m, stream) sketches rows [r0, r0 + m)
// reading the staged input; out(r0, m, stream) copies their results back.
// dp/di/dw are the staged indptr/ids/weights.  With two compute streams the
// CTAs of chunk c + 1 take over SMs as chunk c's persistent CTAs retire, so
// launch tails overlap (LSH launches take separate scratch slots).
//
// (Narrowing ids to u32 on the host before the copy was tried: 16 host
// threads narrowing while the DMA engine reads the same host memory made the
// cfg2 e2e step slower, 43.6 ms against 31.6 ms.)
static bool is_pinned(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// memcpy with the host's threads (pageable -> pinned staging)
static int stage_threads();

static void par_memcpy(void *dst, const void *src, size_t bytes, int threads) {
  // (re-read per copy: concurrent host-buffer calls share the cores)
  const int live = stage_threads();
  threads = live < threads ? live : threads;
  const int64_t blocks = (int64_t)threads * 4;
  const size_t step = ((bytes + blocks - 1) / blocks + 63) & ~(size_t)63;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t b = 0; b < blocks; b++) {
    const size_t o = (size_t)b * step;
    if (o < bytes) memcpy((char *)dst + o, (const char *)src + o, o + step < bytes ? step : bytes - o);
  }
}

// host-buffer calls in flight in this process (one per GPU under
// shard.minhash_host_multi): the staging threads are shared among them
static std::atomic<int> g_host_calls{0};

static int stage_threads() {
  if (const char *e = getenv("DSK_HOST_THREADS")) return atoi(e) > 0 ? atoi(e) : 1;
  unsigned hw = std::thread::hardware_concurrency();
  int t = hw ? (int)(hw < 16 ? hw : 16) : 8;
  const int calls = g_host_calls.load();
  if (calls > 1) {
    const int share = hw ? (int)hw / calls : t / calls;  // the host's cores, split between the calls
    t = share < t ? share : t;
  }
  return t > 0 ? t : 1;
}

struct HostCallScope {
  HostCallScope() { g_host_calls.fetch_add(1); }
  ~HostCallScope() { g_host_calls.fetch_sub(1); }
};

static int ensure_pin_stage(dsk_ctx *c, size_t bytes) {
  for (int b = 0; b < 2; b++)
    if (!c->ev_pin[b]) {
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_pin[b], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(c->ev_pin[b], c->hs[0]));
    }
  if (c->pin_bytes >= bytes) return DSK_OK;
  CUDA_TRY(cudaStreamSynchronize(c->hs[0]));
  for (int b = 0; b < 2; b++) {
    if (c->pin_stage[b]) CUDA_TRY(cudaFreeHost(c->pin_stage[b]));
    c->pin_stage[b] = nullptr;
  }
  c->pin_bytes = 0;
  for (int b = 0; b < 2; b++) CUDA_TRY(cudaHostAlloc((void **)&c->pin_stage[b], bytes, 0));
  c->pin_bytes = bytes;
  return DSK_OK;
}

static int ensure_out_stage(dsk_ctx *c, size_t bytes) {
  for (int b = 0; b < dsk_ctx::kOutSlots; b++)
    if (!c->ev_out[b]) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_out[b], cudaEventDisableTiming));
  if (c->out_bytes >= bytes) return DSK_OK;
  CUDA_TRY(cudaStreamSynchronize(c->hs[2]));
  for (int b = 0; b < dsk_ctx::kOutSlots; b++) {
    if (c->out_stage[b]) CUDA_TRY(cudaFreeHost(c->out_stage[b]));
    c->out_stage[b] = nullptr;
  }
  c->out_bytes = 0;
  for (int b = 0; b < dsk_ctx::kOutSlots; b++)
    CUDA_TRY(cudaHostAlloc((void **)&c->out_stage[b], bytes, 0));
  c->out_bytes = bytes;
  return DSK_OK;
}

// Device-to-host copies of one chunk's results: straight into pinned
// destinations, else into the chunk's pinned output slot, recorded for the
// host threads to copy out once the slot's event fired.
struct OutCopies {
  struct Seg { void *dst; const void *src; size_t bytes; };
  dsk_ctx *c;
  int slot = 0;
  size_t used = 0;
  int nseg[dsk_ctx::kOutSlots] = {};
  Seg seg[dsk_ctx::kOutSlots][8];
  int operator()(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return DSK_OK;
    if (is_pinned(dst) || nseg[slot] == 8 || used + bytes > c->out_bytes) {
      CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
      return DSK_OK;
    }
    unsigned char *p = c->out_stage[slot] + used;
    CUDA_TRY(cudaMemcpyAsync(p, src, bytes, cudaMemcpyDeviceToHost, st));
    seg[slot][nseg[slot]++] = {dst, p, bytes};
    used += (bytes + 255) & ~(size_t)255;
    return DSK_OK;
  }
  int finish(int b, int threads) {  // copy slot b's results out to the caller
    if (!nseg[b]) return DSK_OK;
    CUDA_TRY(cudaEventSynchronize(c->ev_out[b]));
    for (int i = 0; i < nseg[b]; i++) par_memcpy(seg[b][i].dst, seg[b][i].src, seg[b][i].bytes, threads);
    nseg[b] = 0;
    return DSK_OK;
  }
};

template <class Launch, class Out>
static int host_pipeline(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                         const double *weights, int64_t n, int64_t *dp, uint64_t *di, double *dw,
                         int compute_streams, size_t out_row_bytes, Launch launch, Out out,
                         size_t chunk_mb = 64) {
  int64_t bounds[kMaxChunks + 1];
  int nch = 0;
  plan_chunks(indptr, n, host_chunk_cap(chunk_mb), bounds, kMaxChunks + 1, &nch);
  cudaStream_t cp = c->hs[0], os = c->hs[2];
  OutCopies d2h;
  d2h.c = c;
  {
    int64_t mx = 0;
    for (int ch = 0; ch < nch; ch++) mx = bounds[ch + 1] - bounds[ch] > mx ? bounds[ch + 1] - bounds[ch] : mx;
    // (at most 256 MB per slot: larger chunk outputs fall back to direct copies)
    size_t want = (size_t)mx * out_row_bytes + 8 * 256;
    if (want > ((size_t)256 << 20)) want = (size_t)256 << 20;
    int rc = ensure_out_stage(c, want);
    if (rc) return rc;
  }
  // pageable inputs: stage each chunk through pinned buffers with the host's
  // threads while the copy engine moves the previous chunk (a direct copy
  // from pageable memory goes through the driver's own small bounce buffer
  // and measured 6x slower on cfg2)
  const bool stage = !(is_pinned(ids) && is_pinned(weights));
  HostCallScope scope;  // counted while this call runs (thread split for concurrent calls)
  const int threads = stage_threads();
  if (stage) {
    int64_t mx = 0;
    for (int ch = 0; ch < nch; ch++) {
      int64_t m = indptr[bounds[ch + 1]] - indptr[bounds[ch]];
      mx = m > mx ? m : mx;
    }
    int rc = ensure_pin_stage(c, (size_t)mx * 16);
    if (rc) return rc;
  }
  CUDA_TRY(cudaMemcpyAsync(dp, indptr, (n + 1) * 8, cudaMemcpyHostToDevice, cp));
  unsigned long long h2d = (unsigned long long)(n + 1) * 8;
  int rc = DSK_OK;
  for (int ch = 0; ch < nch && rc == DSK_OK; ch++) {
    const int64_t e0 = indptr[bounds[ch]], e1 = indptr[bounds[ch + 1]], m = e1 - e0;
    if (stage && m > 0) {
      const int b = ch & 1;
      CUDA_TRY(cudaEventSynchronize(c->ev_pin[b]));  // buffer b's previous copy is done
      unsigned char *pb = c->pin_stage[b];
      par_memcpy(pb, ids + e0, (size_t)m * 8, threads);
      par_memcpy(pb + (size_t)m * 8, weights + e0, (size_t)m * 8, threads);
      CUDA_TRY(cudaMemcpyAsync(di + e0, pb, m * 8, cudaMemcpyHostToDevice, cp));
      CUDA_TRY(cudaMemcpyAsync(dw + e0, pb + (size_t)m * 8, m * 8, cudaMemcpyHostToDevice, cp));
      CUDA_TRY(cudaEventRecord(c->ev_pin[b], cp));
    } else {
      CUDA_TRY(cudaMemcpyAsync(di + e0, ids + e0, m * 8, cudaMemcpyHostToDevice, cp));
      CUDA_TRY(cudaMemcpyAsync(dw + e0, weights + e0, m * 8, cudaMemcpyHostToDevice, cp));
    }
    h2d += (unsigned long long)m * 16;
    CUDA_TRY(cudaEventRecord(c->ev_in[ch], cp));
    const int64_t r0 = bounds[ch], rows = bounds[ch + 1] - r0;
    cudaStream_t ks = c->hs[(compute_streams > 1 && (ch & 1)) ? 3 : 1];
    CUDA_TRY(cudaStreamWaitEvent(ks, c->ev_in[ch], 0));
    rc = launch(r0, rows, ks);
    if (rc) break;
    CUDA_TRY(cudaEventRecord(c->ev_k[ch], ks));
    CUDA_TRY(cudaStreamWaitEvent(os, c->ev_k[ch], 0));
    const int b = ch % dsk_ctx::kOutSlots;
    rc = d2h.finish(b, threads);  // chunk ch - 4's results, if staged
    if (rc) break;
    d2h.slot = b;
    d2h.used = 0;
    rc = out(r0, rows, os, d2h);
    if (rc) break;
    CUDA_TRY(cudaEventRecord(c->ev_out[b], os));
  }
  for (int i = 0; i < 4; i++) CUDA_TRY(cudaStreamSynchronize(c->hs[i]));
  for (int b = 0; b < dsk_ctx::kOutSlots; b++) {
    int r2 = d2h.finish(b, threads);
    if (!rc) rc = r2;
  }
  g_h2d_bytes.fetch_add(h2d);
  return rc;
}

// Half or more of (up to) 4096 evenly spaced rows hold < 48 elements.
static bool dsk_rows_skewed(const int64_t *indptr, int64_t n) {
  const int64_t samples = n < 4096 ? n : 4096;
  int64_t small = 0;
  for (int64_t q = 0; q < samples; q++) {
    const int64_t r = q * n / samples;
    small += indptr[r + 1] - indptr[r] < 48;
  }
  return 2 * small >= samples;
}

// At least 90 % of (up to) 256 evenly spaced rows have l1 > 2 (a plain sum is
// enough for this heuristic): rank depth 0 in every band up to phi = 2, i.e.
// the direct-only first launch serves nearly every set.
static bool dsk_rows_direct(const int64_t *indptr, const double *w, int64_t n) {
  const int64_t samples = n < 256 ? n : 256;
  int64_t direct = 0;
  for (int64_t q = 0; q < samples; q++) {
    const int64_t r = q * n / samples;
    double l1 = 0.0;
    for (int64_t e = indptr[r]; e < indptr[r + 1] && !(l1 > 2.0); e++) l1 += w[e];
    direct += l1 > 2.0;
  }
  return 10 * direct >= 9 * samples;
}

extern "C" int dsk_minhash_csr_host(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                                    const double *weights, int64_t n, int32_t k,
                                    uint64_t *out_values, uint64_t *out_bits, int32_t *status,
                                    int32_t *phi, uint32_t *stats) {
  if (!c || !indptr || !status || n < 0 || k < 1) return set_err(DSK_EARG, "bad argument");
  if (n == 0) return DSK_OK;
  if (indptr[0] != 0) return set_err(DSK_EARG, "indptr[0] must be 0");
  CUDA_TRY(cudaSetDevice(c->device));
  std::lock_guard<std::mutex> lock(c->host_mu);
  const int64_t nnz = indptr[n];
  const int words = (k + 63) / 64;
  // device layout: indptr | ids | w | values | bits | status | phi | stats
  size_t off_p = 0, off_i = align16((n + 1) * 8), off_w = off_i + align16(nnz * 8);
  size_t off_v = off_w + align16(nnz * 8);
  size_t off_b = off_v + (out_values ? align16((size_t)n * k * 8) : 0);
  size_t off_s = off_b + (out_bits ? align16((size_t)n * words * 8) : 0);
  size_t off_ph = off_s + align16(n * 4);
  size_t off_st = off_ph + (phi ? align16(n * 4) : 0);
  size_t total = off_st + (stats ? align16(n * 16) : 0);
  int rc = ensure_stage(c, total);
  if (rc) return rc;
  char *base = (char *)c->stage;
  int64_t *dp = (int64_t *)(base + off_p);
  uint64_t *di = (uint64_t *)(base + off_i);
  double *dw = (double *)(base + off_w);
  uint64_t *dv = out_values ? (uint64_t *)(base + off_v) : nullptr;
  uint64_t *db = out_bits ? (uint64_t *)(base + off_b) : nullptr;
  int32_t *ds = (int32_t *)(base + off_s);
  int32_t *dph = phi ? (int32_t *)(base + off_ph) : nullptr;
  uint32_t *dst = stats ? (uint32_t *)(base + off_st) : nullptr;
  // shape hint: a batch where most sets are small (cfg5's Zipf sizes) runs
  // best on single-warp teams even when its mean is large, so the hint is
  // withheld (0) when half of ~4096 evenly spaced rows have < 48 elements
  const bool skewed = dsk_rows_skewed(indptr, n);
  // direct-first hint: nearly every sampled set has l1 > 2 (cfg3's raw
  // weights; not cfg2's normalised ones)
  const int64_t dhint = weights && dsk_rows_direct(indptr, weights, n) ? kMhDirectHint : 0;
  auto launch = [&](int64_t r0, int64_t m, cudaStream_t st) {
    return dsk_minhash_csr_ex(c, dp + r0, di, dw, m, k,
                              (skewed ? 0 : indptr[r0 + m] - indptr[r0]) | dhint,
                              dv ? dv + r0 * k : nullptr,
                           db ? db + r0 * words : nullptr, ds + r0, dph ? dph + r0 : nullptr,
                           dst ? dst + r0 * 4 : nullptr, st);
  };
  auto out = [&](int64_t r0, int64_t m, cudaStream_t st, OutCopies &d2h) -> int {
    int rc2 = DSK_OK;
    if (out_values) rc2 |= d2h(out_values + r0 * k, dv + r0 * k, (size_t)m * k * 8, st);
    if (out_bits) rc2 |= d2h(out_bits + r0 * words, db + r0 * words, (size_t)m * words * 8, st);
    rc2 |= d2h(status + r0, ds + r0, (size_t)m * 4, st);
    if (phi) rc2 |= d2h(phi + r0, dph + r0, (size_t)m * 4, st);
    if (stats) rc2 |= d2h(stats + r0 * 4, dst + r0 * 4, (size_t)m * 16, st);
    return rc2;
  };
  int streams = 2;
  if (const char *e = getenv("DSK_HOST_STREAMS")) streams = atoi(e) == 1 ? 1 : 2;
  const size_t row_bytes = (out_values ? (size_t)k * 8 : 0) + (out_bits ? (size_t)words * 8 : 0) +
                           4 + (phi ? 4 : 0) + (stats ? 16 : 0);
  return host_pipeline(c, indptr, ids, weights, n, dp, di, dw, streams, row_bytes, launch, out,
                       skewed ? 512 : 32);
}

#include "dsk_lsh_host.cuh"
#include "dsk_extra.cuh"
#include "dsk_bottomk.cuh"
#include "dsk_icws.cuh"
