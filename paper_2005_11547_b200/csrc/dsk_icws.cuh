// dsk_icws.cuh -- ICWS comparator (ref/baselines.py:84-161), included by
// dsk_kernels.cu.  Not part of DartMinHash: the paper's Table 1 baseline.
//
// Coordinate j of a set: for every element e the reference draws
//   r = -(log1p(-u1) + log1p(-u2)),  c = -(log1p(-u3) + log1p(-u4)),  beta = u5
// with u_s = uniform(element = id_e, w = j, stream = 6..10), then
//   tick = floor(log(x_e) / r + beta),  ln_a = log(c) - r * (tick - beta) - r
// and keeps (id, tick) of the first e minimising ln_a (np.argmin).
//
// One warp per set; lanes stride over the elements for each coordinate and
// the warp reduces (ln_a, index) to the first minimum.  The arithmetic is
// the reference's operation for operation (no contraction), but log / log1p
// come from CUDA's libdevice rather than the host's numpy/libm: results are
// identical except where two candidates' ln_a (or a tick's floor argument)
// differ by an ulp, which the tests measure on the reference's outputs.

constexpr int kStreamIcwsR1 = 6, kStreamIcwsBeta = 10;

__global__ void __launch_bounds__(256) icws_kernel(const uint64_t *tab, const int64_t *indptr,
                                                   const uint64_t *ids, const double *w,
                                                   int64_t n, int32_t k, uint64_t *out_elem,
                                                   int64_t *out_tick, int32_t *status) {
  __shared__ uint64_t sE[8][256];  // T0..T7
  __shared__ uint64_t sW[4][256];  // T10..T13 (coordinate bytes)
  __shared__ uint64_t sS[5];       // stream bytes for streams 6..10 (T20, T21[0])
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) sE[i >> 8][i & 255] = tab[i];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x)
    sW[i >> 8][i & 255] = tab[(10 + (i >> 8)) * 256 + (i & 255)];
  if (threadIdx.x < 5) sS[threadIdx.x] = tab[20 * 256 + kStreamIcwsR1 + threadIdx.x] ^ tab[21 * 256];
  __syncthreads();
  // fields fixed at 0: nu (T8), rho (T9), r (T14-T17), j (T18, T19)
  const uint64_t zero = tab[8 * 256] ^ tab[9 * 256] ^ tab[14 * 256] ^ tab[15 * 256] ^
                        tab[16 * 256] ^ tab[17 * 256] ^ tab[18 * 256] ^ tab[19 * 256];
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < n;
       s += warps) {
    const int64_t lo = indptr[s], nnz = indptr[s + 1] - lo;
    if (nnz == 0) {
      if (lane == 0) status[s] = DSK_EMPTY;
      continue;
    }
    for (int32_t j = 0; j < k; j++) {
      const uint64_t wj = zero ^ sW[0][j & 255] ^ sW[1][(j >> 8) & 255] ^
                          sW[2][(j >> 16) & 255] ^ sW[3][((uint32_t)j >> 24) & 255];
      double best = 0.0, best_tick = 0.0;
      int64_t best_i = -1;
      for (int64_t e = lane; e < nnz; e += 32) {
        const uint64_t id = ids[lo + e];
        uint64_t base = wj;
#pragma unroll
        for (int p = 0; p < 8; p++) base ^= sE[p][(id >> (8 * p)) & 0xff];
        double u[5];
#pragma unroll
        for (int q = 0; q < 5; q++) u[q] = u53(finalize(base ^ sS[q]));
        const double r = -__dadd_rn(log1p(-u[0]), log1p(-u[1]));
        const double c = -__dadd_rn(log1p(-u[2]), log1p(-u[3]));
        const double beta = u[4];
        const double lnx = log(w[lo + e]);
        const double tick = floor(__dadd_rn(__ddiv_rn(lnx, r), beta));
        const double ln_y = __dmul_rn(r, __dadd_rn(tick, -beta));
        const double ln_a = __dadd_rn(__dadd_rn(log(c), -ln_y), -r);
        if (best_i < 0 || ln_a < best) { best = ln_a; best_tick = tick; best_i = e; }
      }
      // first minimum over the warp (np.argmin): smaller ln_a, then index
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double ob = __shfl_xor_sync(DSK_FULL, best, o);
        const double ot = __shfl_xor_sync(DSK_FULL, best_tick, o);
        const long long oi = __shfl_xor_sync(DSK_FULL, (long long)best_i, o);
        const bool take = oi >= 0 && (best_i < 0 || ob < best || (ob == best && oi < best_i));
        if (take) { best = ob; best_tick = ot; best_i = oi; }
      }
      if (lane == 0) {
        out_elem[(size_t)s * k + j] = ids[lo + best_i];
        out_tick[(size_t)s * k + j] = (int64_t)best_tick;
      }
    }
    if (lane == 0) status[s] = DSK_OK;
  }
}

extern "C" int dsk_icws_csr(dsk_ctx *c, const int64_t *indptr, const uint64_t *ids,
                            const double *weights, int64_t n, int32_t k, uint64_t *out_element,
                            int64_t *out_tick, int32_t *status, void *stream) {
  if (!c || !indptr || !out_element || !out_tick || !status || n < 0)
    return set_err(DSK_EARG, "bad argument");
  if (k < 1) return set_err(DSK_EARG, "k must be positive");  // ref/baselines.py:98-99
  if (n == 0) return DSK_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  int64_t g = (n + 7) / 8;
  int grid = (int)(g < 16 * c->num_sms ? g : 16 * c->num_sms);
  icws_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(c->d_tab, indptr, ids, weights, n, k,
                                                       out_element, out_tick, status);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}
