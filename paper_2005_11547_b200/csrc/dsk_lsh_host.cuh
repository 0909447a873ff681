// dsk_lsh_host.cuh -- host side of K5 (included at the end of dsk_kernels.cu).

extern "C" int dsk_lsh_csr(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                           const double *weights, int64_t n, int32_t L, int32_t K,
                           int32_t normalize, uint64_t *out_keys, uint64_t *out_fps,
                           int32_t *status, int32_t *phi, uint32_t *stats, void *stream) {
  return dsk_lsh_csr_ex(c, indptr, ids, weights, n, L, K, normalize, 0, out_keys, out_fps, status,
                        phi, stats, stream);
}

extern "C" int dsk_lsh_csr_ex(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                              const double *weights, int64_t n, int32_t L, int32_t K,
                              int32_t normalize, int64_t max_row_hint, uint64_t *out_keys,
                              uint64_t *out_fps, int32_t *status, int32_t *phi, uint32_t *stats,
                              void *stream) {
  if (!c || !indptr || !status || n < 0) return set_err(DSK_EARG, "bad argument");
  if (L < 1 || K < 1) return set_err(DSK_EARG, "L and K must be positive");  // ref/annindex.py:33-34
  if (n == 0) return DSK_OK;
  int64_t t = (int64_t)L * K;
  if (t > INT32_MAX) return set_err(DSK_EUNSUPPORTED, "L*K too large");
  int NW = 0, G = 0;
  // bucket counters in shared memory; L too large for that -> global scratch
  bool gc = false;
  if (!choose_shape(c, [&](int g, int nw) { return lsh_smem(L, g, nw); }, n, NW, G, 2)) {
    gc = true;
    if (!choose_shape(c, [&](int g, int nw) {
          return nw == 20 ? off_team(nw) + (size_t)(nw / g) * kTeamCtlBytes : (size_t)1 << 40;
        }, n, NW, G))
      return set_err(DSK_EUNSUPPORTED, "no CTA shape fits shared memory");
  }
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(c->device));
  // phi0 = 2 when every one of L >= 8 buckets rarely fills at phi = 1
  // (P(all L buckets >= K) <= 0.63^L; cfg4: phi* = 2 or 3 for every set)
  int phi0 = L >= 8 ? 2 : 1;
  if (const char *e = getenv("DSK_LSH_PHI0")) phi0 = atoi(e) == 2 ? 2 : 1;
  // the first launch runs the direct-only engine when its sets are likely to
  // qualify (no normalisation: l1 ~ sum of raw weights) and a retry launch
  // follows anyway (phi0 = 2); DSK_LSH_DIRECT=0 disables it (tests).  Without
  // the region rings its queue blocks pack tighter, so it runs on the widest
  // CTA that fits shared memory and the 16 named barriers: 28 warps (72
  // registers per thread) in teams of 2 for cfg4, against 24 for the general
  // engine (DSK_LSH_DNW: tuning)
  const char *dk = getenv("DSK_LSH_DIRECT");
  bool direct_first = DSK_LSH_DIRECT_KERNEL && !gc && NW == 24 && phi0 > 1 && !normalize &&
                      !(dk && atoi(dk) == 0);
  int DNW = NW, DG = G;  // CTA width and team size of the first launch
  if (direct_first) {
    const char *e = getenv("DSK_LSH_DNW");
    const int want = e ? atoi(e) : 28;
    // multi-wave batches: single-warp teams when they fit (no team barriers,
    // no chunk hand-out; cfg4: 28 x 1 is 3.6 % faster than 14 x 2), else the
    // general shape's team size.  DSK_LSH_DG: tuning
    const char *eg = getenv("DSK_LSH_DG");
    // ... unless a large set would bound the launch: a set takes ~1-2 us per
    // element on one warp (30 k cfg5 rows, largest 16384: 22.9 ms in
    // single-warp teams against 15.1 in teams of 2; 300 k rows: 82.7 against
    // 84.5), so single-warp teams need rows of <= 1024 elements
    // (max_row_hint) or, sizes unknown, a batch of >= 64 waves
    const int64_t wave = (int64_t)c->num_sms * 28;
    const bool single = n >= 4 * wave && (max_row_hint > 0 ? max_row_hint <= 1024 : n >= 64 * wave);
    int cand[2] = {single ? 1 : G, G};
    if (eg && atoi(eg) >= 1) cand[0] = cand[1] = atoi(eg);
    DNW = 0;
    for (int q = 0; q < 2 && !DNW; q++)
      for (int nw : {28, 26, 24})
        if (nw <= want && team_size_ok(cand[q], nw) &&
            lsh_smem(L, cand[q], nw, true) <= c->max_smem) {
          DNW = nw;
          DG = cand[q];
          break;
        }
    if (!DNW) { DNW = NW; DG = G; direct_first = lsh_smem(L, G, NW, true) <= c->max_smem; }
  }
  const int teams = DNW / DG;  // (>= the retry launch's NW / G: scratch is sized for it)
  int grid = c->num_sms;
  if ((int64_t)grid * teams > n) grid = (int)((n + teams - 1) / teams);
  // hit slots per bucket: >= 64 (the register sorts) and >= about two bands
  // of a bucket's hits past K (buffering stops once a band begins full)
  int64_t S64 = 2 * ((int64_t)K + t / L) + 32;
  S64 = S64 < 64 ? 64 : (S64 + 31) / 32 * 32;
  if (S64 > (1 << 20)) S64 = 1 << 20;
  if (const char *e = getenv("DSK_LSH_SLOTS"))  // tests: force the overflow list
    S64 = atoi(e) > 64 ? (atoi(e) + 7) / 8 * 8 : 64;  // 128-byte bucket regions
  const uint32_t S = (uint32_t)S64;
  // overflow list per team for buckets past their S slots (rare)
  uint32_t cap = (uint32_t)(2 * t > 16384 ? (2 * t < (1 << 26) ? 2 * t : (1 << 26)) : 16384);
  // 128-byte aligned regions (the kernel discards spent lines; lsh_kernel's layout)
  size_t team_bytes = align128((size_t)L * S * 16) + align128((size_t)cap * 16) +
                      align128((size_t)cap * 4) + align128((size_t)L * K * 8) +
                      (gc ? align128(align16((size_t)3 * L * sizeof(unsigned)) + 16) : 0);
  const size_t retry_off = (size_t)grid * teams * team_bytes;
  size_t need = retry_off + (phi0 > 1 ? align16((size_t)n * 4) + 16 : 0);
  // hit buffers from the context's stream-ordered scratch pool
  std::lock_guard<std::mutex> lock(c->scratch_mu);
  int slot;
  void *scratch;
  {
    int rc = scratch_acquire(c, need, st, slot, scratch);
    if (rc) return rc;
  }
  unsigned long long *counter = c->d_counter + (c->next_slot.fetch_add(1) % kCounterSlots);
  CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  LshArgs a;
  a.indptr = indptr; a.ids = ids; a.w = weights; a.n = n; a.L = L; a.K = K;
  a.normalize = normalize;
  const char *ex = getenv("DSK_LSH_EXACT");
  a.exact_sort = ex && atoi(ex) != 0;
  const char *qs = getenv("DSK_LSH_QSHIFT");
  a.qshift = qs ? (atoi(qs) < 0 ? 0 : (atoi(qs) > 26 ? 26 : atoi(qs))) : 0; a.tf = (double)t; a.inv_t = 1.0 / (double)t;
  a.phi0 = phi0;
  a.retry_rows = nullptr;
  a.retry_n = nullptr;
  const char *fr = getenv("DSK_LSH_FORCE_RETRY");
  a.force_retry = fr && atoi(fr) != 0;
  a.md = make_mod((uint32_t)L); a.G = G; a.out_keys = out_keys; a.out_fps = out_fps;
  a.status = status; a.phi = phi; a.stats = stats; a.counter = counter;
  a.scratch = (unsigned char *)scratch; a.team_scratch = team_bytes; a.cap = cap; a.S = S;
  a.tabs = table_args(c, (double)t);
  auto launch = [&]() {
    if (gc) {
      lsh_kernel<20, true><<<grid, 20 * 32, off_team(20) + (size_t)teams * kTeamCtlBytes, st>>>(a);
    } else if (direct_first) {
      const size_t sm = lsh_smem(L, DG, DNW, true);
      a.G = DG;
      switch (DNW) {
        // (a compile-time single-warp-team specialisation of this kernel
        // measured 198.2 against 180.9 ms on cfg4: worse register allocation)
        case 28: lsh_kernel<28, false, true><<<grid, 28 * 32, sm, st>>>(a); break;
        case 26: lsh_kernel<26, false, true><<<grid, 26 * 32, sm, st>>>(a); break;
        default: lsh_kernel<24, false, true><<<grid, 24 * 32, sm, st>>>(a); break;
      }
    } else {
      switch (NW) {
        case 24: lsh_kernel<24><<<grid, 24 * 32, lsh_smem(L, G, NW), st>>>(a); break;
        case 22: lsh_kernel<22><<<grid, 22 * 32, lsh_smem(L, G, NW), st>>>(a); break;
        default: lsh_kernel<20><<<grid, 20 * 32, lsh_smem(L, G, NW), st>>>(a); break;
      }
    }
    count_launch();
  };
  launch();
  CUDA_TRY(cudaGetLastError());
  if (phi0 > 1) {
    // rows whose (0, 2 / l1] first band failed are redone from phi = 1 (the
    // reference's own stepping); normally none, and the retry launch exits
    uint32_t *rows = (uint32_t *)((char *)scratch + retry_off);
    unsigned *cnt = (unsigned *)((char *)rows + align16((size_t)n * 4));
    CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned), st));
    int cg = (int)((n + 255) / 256 < 2 * c->num_sms ? (n + 255) / 256 : 2 * c->num_sms);
    lsh_retry_compact_kernel<<<cg, 256, 0, st>>>(status, n, rows, cnt);
    count_launch();
    unsigned long long *counter2 = c->d_counter + (c->next_slot.fetch_add(1) % kCounterSlots);
    CUDA_TRY(cudaMemsetAsync(counter2, 0, sizeof(unsigned long long), st));
    a.counter = counter2;
    a.phi0 = 1;
    a.G = G;  // (the general shape)
    a.retry_rows = rows;
    a.retry_n = cnt;
    direct_first = false;  // the retry launch runs the general engine
    launch();
    CUDA_TRY(cudaGetLastError());
  }
  return scratch_release(c, slot, st);
}

extern "C" int dsk_lsh_csr_host(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                                const double *weights, int64_t n, int32_t L, int32_t K,
                                int32_t normalize, uint64_t *out_keys, uint64_t *out_fps,
                                int32_t *status, int32_t *phi, uint32_t *stats) {
  if (!c || !indptr || !status || n < 0 || L < 1 || K < 1) return set_err(DSK_EARG, "bad argument");
  if (n == 0) return DSK_OK;
  if (indptr[0] != 0) return set_err(DSK_EARG, "indptr[0] must be 0");
  CUDA_TRY(cudaSetDevice(c->device));
  std::lock_guard<std::mutex> lock(c->host_mu);
  const int64_t nnz = indptr[n];
  size_t off_i = align16((n + 1) * 8), off_w = off_i + align16(nnz * 8);
  size_t off_k = off_w + align16(nnz * 8);
  size_t off_f = off_k + (out_keys ? align16((size_t)n * L * 8) : 0);
  size_t off_s = off_f + (out_fps ? align16((size_t)n * L * K * 8) : 0);
  size_t off_ph = off_s + align16(n * 4);
  size_t off_st = off_ph + (phi ? align16(n * 4) : 0);
  size_t total = off_st + (stats ? align16(n * 16) : 0);
  int rc = ensure_stage(c, total);
  if (rc) return rc;
  char *base = (char *)c->stage;
  int64_t *dp = (int64_t *)base;
  uint64_t *di = (uint64_t *)(base + off_i);
  double *dw = (double *)(base + off_w);
  uint64_t *dk = out_keys ? (uint64_t *)(base + off_k) : nullptr;
  uint64_t *df = out_fps ? (uint64_t *)(base + off_f) : nullptr;
  int32_t *ds = (int32_t *)(base + off_s);
  int32_t *dph = phi ? (int32_t *)(base + off_ph) : nullptr;
  uint32_t *dst = stats ? (uint32_t *)(base + off_st) : nullptr;
  int64_t max_row = 1;  // team-shape hint of dsk_lsh_csr_ex
  for (int64_t r = 0; r < n; r++) max_row = indptr[r + 1] - indptr[r] > max_row ? indptr[r + 1] - indptr[r] : max_row;
  auto launch = [&](int64_t r0, int64_t m, cudaStream_t st) {
    return dsk_lsh_csr_ex(c, dp + r0, di, dw, m, L, K, normalize, max_row,
                          dk ? dk + r0 * L : nullptr, df ? df + r0 * L * K : nullptr, ds + r0,
                          dph ? dph + r0 : nullptr, dst ? dst + r0 * 4 : nullptr, st);
  };
  auto out = [&](int64_t r0, int64_t m, cudaStream_t st, OutCopies &d2h) -> int {
    int rc2 = DSK_OK;
    if (out_keys) rc2 |= d2h(out_keys + r0 * L, dk + r0 * L, (size_t)m * L * 8, st);
    if (out_fps) rc2 |= d2h(out_fps + r0 * L * K, df + r0 * L * K, (size_t)m * L * K * 8, st);
    rc2 |= d2h(status + r0, ds + r0, (size_t)m * 4, st);
    if (phi) rc2 |= d2h(phi + r0, dph + r0, (size_t)m * 4, st);
    if (stats) rc2 |= d2h(stats + r0 * 4, dst + r0 * 4, (size_t)m * 16, st);
    return rc2;
  };
  const size_t row_bytes = (out_keys ? (size_t)L * 8 : 0) + (out_fps ? (size_t)L * K * 8 : 0) +
                           4 + (phi ? 4 : 0) + (stats ? 16 : 0);
  return host_pipeline(c, indptr, ids, weights, n, dp, di, dw, 2, row_bytes, launch, out, 256);
}
