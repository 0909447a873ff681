// dsk_bottomk.cuh -- bottom_k (ref/sketching.py:126-161) as one kernel
// (included by dsk_kernels.cu after the darts kernel).
//
// bottom_k: density t = k; at the first phi step (1..64) whose darts
// (rank <= phi / ||x||_1) number >= k, the k smallest by (rank, element, nu,
// rho, w, r, j) in that order (ref/sketching.py:126-143 _bottom_indices).
//
// One warp per set, as the materialising darts kernel: phi bands 1, 2, ...
// through the engine with the full-tuple sink, every hit appended to the
// warp's global buffer (sets beyond 4096 elements in element slices, the
// row sink's index width); after the band that brings the count to >= k,
// each entry's position by (rank, index tuple) is counted and positions < k
// are written in order.  A set whose darts outgrow the buffer reports
// DSK_SCRATCH and the facade recomputes it with the composed path.

struct BkEntry {
  uint64_t element, fp;
  double rank, weight;
  uint32_t w, r;
  uint16_t nu, rho, j, pad;
};

__device__ __forceinline__ bool bk_less(const BkEntry &a, const BkEntry &b) {
  const uint64_t ra = (uint64_t)__double_as_longlong(a.rank);
  const uint64_t rb = (uint64_t)__double_as_longlong(b.rank);  // ranks >= 0: bits order
  if (ra != rb) return ra < rb;
  if (a.element != b.element) return a.element < b.element;
  if (a.nu != b.nu) return a.nu < b.nu;
  if (a.rho != b.rho) return a.rho < b.rho;
  if (a.w != b.w) return a.w < b.w;
  if (a.r != b.r) return a.r < b.r;
  return a.j < b.j;
}

struct BottomKArgs {
  const int64_t *indptr;
  const uint64_t *ids;
  const double *w;
  int64_t n;
  int32_t k;
  double tf, inv_t;
  BkEntry *buf;        // per warp: cap entries
  uint32_t cap;
  uint64_t *element;   // outputs [n, k]
  uint16_t *nu, *rho, *jj;
  uint32_t *ww, *rr;
  double *weight, *rank;
  uint64_t *fp;
  int32_t *status;
  int32_t *phi;
  TableArgs tabs;
};

struct BottomKSink {
  static constexpr bool kFuse = true;
  static constexpr int kRun = DSK_RUN;
  static constexpr int kRunDeep = DSK_RUN;
  BkEntry *buf;
  uint32_t cap;
  const uint64_t *ids;  // ids of the current slice
  unsigned long long *cursor;
  __device__ void hit(bool, const HitInfo &, int) {}
  __device__ void row(const DartRow &d) {
    const unsigned long long i = atomicAdd(cursor, 1ULL);
    if (i < cap) {
      BkEntry e;
      e.element = ids[d.elem];
      e.fp = d.fp;
      e.rank = d.rank;
      e.weight = d.weight;
      e.w = d.w;
      e.r = d.r;
      e.nu = (uint16_t)d.nu;
      e.rho = (uint16_t)d.rho;
      e.j = (uint16_t)d.j;
      e.pad = 0;
      buf[i] = e;
    }
  }
};

__global__ void __launch_bounds__(kWarps * 32, 1) bottomk_kernel(BottomKArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  SmemTables &T = g_tabs;
  load_tables(T, a.tabs);
  const int warp = opaque_int(threadIdx.x >> 5), lane = opaque_int(threadIdx.x & 31);
  WarpQueues &Q = *reinterpret_cast<WarpQueues *>(smem + kOffQueues + warp * kQBytes);
  unsigned long long *cursors = reinterpret_cast<unsigned long long *>(smem + kOffTeam);
  uint4 *rwin = reinterpret_cast<uint4 *>(smem + kOffTeam +
                                          align16(kWarps * sizeof(unsigned long long))) +
                warp * kRwinStride;
  PassParams *pps = reinterpret_cast<PassParams *>(
      smem + kOffTeam + align16(kWarps * sizeof(unsigned long long)) +
      kWarps * kRwinStride * sizeof(uint4));
  BkEntry *buf = a.buf + ((size_t)blockIdx.x * kWarps + warp) * a.cap;
  const uint32_t k = (uint32_t)a.k;
  __syncthreads();
  for (int64_t s = (int64_t)blockIdx.x * kWarps + warp; s < a.n; s += (int64_t)gridDim.x * kWarps) {
    const int64_t lo = a.indptr[s], nnz = a.indptr[s + 1] - lo;
    int status = 0, phi_star = 0;
    if (nnz == 0) status = DSK_EMPTY;  // ref/sketching.py:86-88 (via _check_set)
    bool bad = false;
    for (int64_t i = lane; i < nnz; i += 32) {
      const double x = a.w[lo + i];
      bad |= !(isfinite(x) && x > 0.0);
    }
    if (status == 0 && __any_sync(DSK_FULL, bad)) status = DSK_WEIGHT;
    double l1 = 0.0;
    int maxd = 0;
    if (status == 0) {
      l1 = warp_np_sum(a.w + lo, nnz, reinterpret_cast<double *>(&Q), lane, 0);  // ref/core.py:44
      __syncwarp();
      for (int64_t i = lane; i < nnz; i += 32) {
        int d = floor_log2_host(__dadd_rn(1.0, __dmul_rn(a.tf, a.w[lo + i])), T.l2thr);
        maxd = d > maxd ? d : maxd;
      }
      maxd = (int)__reduce_max_sync(DSK_FULL, (unsigned)maxd);
    }
    if (lane == 0) cursors[warp] = 0;
    __syncwarp();
    if (status == 0) {
      status = DSK_NOCONV;
      double L_prev = -1.0;
      int RD_prev = 0;
      for (int phi = 1; phi <= 64; phi++) {  // ref/sketching.py:150
        const double L = __ddiv_rn((double)phi, l1);
        if (!(L > 0.0) || isinf(L)) { status = DSK_LIMIT; break; }
        const int RD = floor_log2_host(__dadd_rn(1.0, L), T.l2thr);
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
        if (lane == 0) pps[warp] = P;
        __syncwarp();
        double full = 0.0;
        bool capped = false;
        for (int64_t base = 0; base < nnz && !capped; base += kSliceElems) {
          const int64_t m = nnz - base < kSliceElems ? nnz - base : kSliceElems;
          BottomKSink sink;
          sink.buf = buf;
          sink.cap = a.cap;
          sink.ids = a.ids + lo + base;
          sink.cursor = &cursors[warp];
          Engine<BottomKSink, true> eng(T, Q, rwin, sink, pps[warp], lane);
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
          capped = eng.abort || full > kMaxAreas;
        }
        __syncwarp();
        if (capped) { status = DSK_AREAS; break; }  // ref/darthash.py:242-244
        const unsigned long long total = cursors[warp];
        if (total > a.cap) { status = DSK_SCRATCH; break; }
        if (total >= k) { status = DSK_OK; phi_star = phi; break; }  // ref/sketching.py:152
        L_prev = L;
        RD_prev = RD;
      }
    }
    if (status == DSK_OK) {
      // position of every buffered dart by (rank, index tuple); those < k are
      // the sketch, ascending (ref/sketching.py:126-143)
      const uint32_t total = (uint32_t)cursors[warp];
      for (uint32_t i = lane; i < total; i += 32) {
        const BkEntry e = buf[i];
        uint32_t pos = 0;
        for (uint32_t m = 0; m < total && pos < k; m++) pos += bk_less(buf[m], e);
        if (pos < k) {
          const size_t o = (size_t)s * k + pos;
          a.element[o] = e.element;
          a.nu[o] = e.nu;
          a.rho[o] = e.rho;
          a.ww[o] = e.w;
          a.rr[o] = e.r;
          a.jj[o] = e.j;
          a.weight[o] = e.weight;
          a.rank[o] = e.rank;
          a.fp[o] = e.fp;
        }
      }
    }
    if (lane == 0) {
      a.status[s] = status;
      if (a.phi) a.phi[s] = phi_star;
    }
    __syncwarp();
  }
}

static cudaError_t bottomk_set_smem(int bytes) {
  return cudaFuncSetAttribute(bottomk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

extern "C" int dsk_bottomk_csr(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                               const double *weights, int64_t n, int32_t k, uint64_t *element,
                               uint16_t *nu, uint16_t *rho, uint32_t *w, uint32_t *r, uint16_t *j,
                               double *weight, double *rank, uint64_t *fingerprint,
                               int32_t *status, int32_t *phi, void *stream) {
  if (!c || !indptr || !status || n < 0) return set_err(DSK_EARG, "bad argument");
  if (k < 1) return set_err(DSK_EARG, "k must be positive");  // ref/sketching.py:147-148
  if (!element || !nu || !rho || !w || !r || !j || !weight || !rank || !fingerprint)
    return set_err(DSK_EARG, "null output column");
  if (n == 0) return DSK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(c->device));
  int grid = (int)((n + kWarps - 1) / kWarps);
  if (grid > c->num_sms) grid = c->num_sms;
  // ~k darts per phi step: room for ~8 steps, at least 1024 entries
  const uint32_t cap = (uint32_t)(8 * (int64_t)k + 1024 < (1 << 24) ? 8 * (int64_t)k + 1024
                                                                     : (1 << 24));
  uint32_t cap_used = cap;
  if (const char *e = getenv("DSK_BOTTOMK_CAP"))  // tests: force the DSK_SCRATCH fallback
    cap_used = atoi(e) > 0 ? (uint32_t)atoi(e) : cap;
  std::lock_guard<std::mutex> lock(c->scratch_mu);
  int slot;
  void *scratch;
  int rc = scratch_acquire(c, (size_t)grid * kWarps * cap_used * sizeof(BkEntry), st, slot,
                           scratch);
  if (rc) return rc;
  BottomKArgs a;
  a.indptr = indptr; a.ids = ids; a.w = weights; a.n = n; a.k = k;
  a.tf = (double)k; a.inv_t = 1.0 / (double)k;
  a.buf = (BkEntry *)scratch; a.cap = cap_used;
  a.element = element; a.nu = nu; a.rho = rho; a.jj = j; a.ww = w; a.rr = r;
  a.weight = weight; a.rank = rank; a.fp = fingerprint; a.status = status; a.phi = phi;
  a.tabs = table_args(c, (double)k);
  size_t smem = kOffTeam + align16(kWarps * sizeof(unsigned long long)) +
                kWarps * kRwinStride * sizeof(uint4) + kWarps * sizeof(PassParams);
  bottomk_kernel<<<grid, kWarps * 32, smem, st>>>(a); count_launch();
  CUDA_TRY(cudaGetLastError());
  return scratch_release(c, slot, st);
}
