// dsk_extra.cuh -- small batch kernels around the hot path (included at the
// end of dsk_kernels.cu):
//   dsk_l1_csr        float(np.sum(weights)) per set (ref/core.py:44), the
//                     rank-limit denominator of every phi step
//   dsk_dsk1_records  DSK1 sketch records (ref/sketching.py:210-231) for a
//                     batch, byte-identical to concatenated dump_sketch()

__global__ void l1_kernel(const int64_t *indptr, const double *w, int64_t n, double *out) {
  __shared__ double scratch[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t s = (int64_t)blockIdx.x * 8 + warp; s < n; s += (int64_t)gridDim.x * 8) {
    const int64_t lo = indptr[s], nnz = indptr[s + 1] - lo;
    double l1 = warp_np_sum(w + lo, nnz, scratch[warp], lane, 0);
    if (lane == 0) out[s] = l1;
  }
}

extern "C" int dsk_l1_csr(const int64_t *indptr, const double *weights, int64_t n, double *out,
                          void *stream) {
  if (!indptr || !weights || !out || n < 0) return set_err(DSK_EARG, "bad argument");
  if (n == 0) return DSK_OK;
  int grid = (int)((n + 7) / 8);
  if (grid > c_sms() * 16) grid = c_sms() * 16;
  l1_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(indptr, weights, n, out); count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}

// header <4sBBHIQ: "DSK1", version 1, kind, reserved 0, k, seed (ref/sketching.py:221)
__global__ void dsk1_kernel(int kind, uint32_t k, uint64_t seed, const uint64_t *payload,
                            int64_t words_per_set, int64_t payload_bytes, int64_t n,
                            uint8_t *out) {
  const int64_t rec = 20 + payload_bytes;
  const int64_t total = n * rec;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / rec, o = i - s * rec;
    uint8_t b;
    if (o < 4) {
      b = (uint8_t)("DSK1"[o]);
    } else if (o == 4) {
      b = 1;  // SKETCH_VERSION
    } else if (o == 5) {
      b = (uint8_t)kind;
    } else if (o < 8) {
      b = 0;  // reserved
    } else if (o < 12) {
      b = (uint8_t)(k >> (8 * (o - 8)));
    } else if (o < 20) {
      b = (uint8_t)(seed >> (8 * (o - 12)));
    } else {
      const int64_t p = o - 20;  // little-endian payload byte p of set s
      b = (uint8_t)(payload[s * words_per_set + (p >> 3)] >> (8 * (p & 7)));
    }
    out[i] = b;
  }
}

// Records whose size is a multiple of 4 bytes (every kind 1 / 3 record, and
// kind 2 when ceil(k/8) % 4 == 0): one warp per record writes it as aligned
// 32-bit words -- 5 header words, then the little-endian payload -- so the
// stores coalesce and no per-byte index arithmetic is needed (HBM-bound).
__global__ void dsk1_words_kernel(int kind, uint32_t k, uint64_t seed, const uint64_t *payload,
                                  int64_t words_per_set, int64_t payload_bytes, int64_t n,
                                  uint32_t *out) {
  const int64_t rw = (20 + payload_bytes) / 4;  // 32-bit words per record
  const int lane = threadIdx.x & 31;
  const uint32_t hdr[5] = {0x314b5344u /* "DSK1" */,
                           1u | ((uint32_t)kind << 8),  // version 1, kind, reserved 0
                           k, (uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < n;
       s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    uint32_t *o = out + s * rw;
    const uint32_t *pl = reinterpret_cast<const uint32_t *>(payload + s * words_per_set);
    for (int64_t q = lane; q < rw; q += 32) o[q] = q < 5 ? hdr[q] : pl[q - 5];
  }
}

// kind 1 (minhash) and 3 (bottom-k): payload = k uint64 values per set;
// kind 2 (one-bit): payload = ceil(k/8) bytes of the packed words
// (np.packbits(bits, bitorder="little"), ref/sketching.py:229).
extern "C" int dsk_dsk1_records(int32_t kind, int32_t k, uint64_t seed, const uint64_t *payload,
                                int64_t n, uint8_t *out, void *stream) {
  if (!payload || !out || n < 0 || k < 1 || kind < 1 || kind > 3)
    return set_err(DSK_EARG, "bad argument");
  if (n == 0) return DSK_OK;
  const int64_t words = kind == 2 ? (k + 63) / 64 : k;
  const int64_t pbytes = kind == 2 ? (k + 7) / 8 : 8 * (int64_t)k;
  int64_t total = n * (20 + pbytes);
  if ((pbytes & 3) == 0 && ((uintptr_t)out & 3) == 0) {
    int64_t wgrid = (n + 7) / 8;  // 8 warps per block
    int grid = (int)(wgrid < c_sms() * 64 ? wgrid : c_sms() * 64);
    dsk1_words_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        kind, (uint32_t)k, seed, payload, words, pbytes, n, reinterpret_cast<uint32_t *>(out)); count_launch();
    CUDA_TRY(cudaGetLastError());
    return DSK_OK;
  }
  int grid = (int)((total + 255) / 256);
  if (grid > c_sms() * 32) grid = c_sms() * 32;
  dsk1_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(kind, (uint32_t)k, seed, payload, words,
                                                      pbytes, n, out); count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}

// exact_jaccard (ref/core.py:103-120) for pairs of sets whose ids are sorted
// ascending within each row: sum of minima over sum of maxima, accumulated in
// ascending id order exactly as the reference's loop over the sorted union.
// One thread per pair merges the two rows.
__global__ void jaccard_kernel(const int64_t *a_ptr, const uint64_t *a_ids, const double *a_w,
                               const int64_t *b_ptr, const uint64_t *b_ids, const double *b_w,
                               const int64_t *pa, const int64_t *pb, int64_t npairs,
                               double *out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npairs;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = a_ptr[pa[t]], ie = a_ptr[pa[t] + 1];
    int64_t j = b_ptr[pb[t]], je = b_ptr[pb[t] + 1];
    double mn = 0.0, mx = 0.0;
    while (i < ie || j < je) {
      double wx, wy;
      if (j >= je || (i < ie && a_ids[i] < b_ids[j])) {
        wx = a_w[i++]; wy = 0.0;
      } else if (i >= ie || b_ids[j] < a_ids[i]) {
        wx = 0.0; wy = b_w[j++];
      } else {
        wx = a_w[i++]; wy = b_w[j++];
      }
      mn = __dadd_rn(mn, wx < wy ? wx : wy);  // min(wx, wy)
      mx = __dadd_rn(mx, wx < wy ? wy : wx);  // max(wx, wy)
    }
    out[t] = __ddiv_rn(mn, mx);
  }
}

extern "C" int dsk_exact_jaccard(const int64_t *a_ptr, const uint64_t *a_ids, const double *a_w,
                                 const int64_t *b_ptr, const uint64_t *b_ids, const double *b_w,
                                 const int64_t *pa, const int64_t *pb, int64_t npairs,
                                 double *out, void *stream) {
  if (npairs < 0 || (npairs > 0 && (!a_ptr || !b_ptr || !pa || !pb || !out)))
    return set_err(DSK_EARG, "bad argument");
  if (npairs == 0) return DSK_OK;
  int grid = (int)((npairs + 255) / 256);
  if (grid > c_sms() * 16) grid = c_sms() * 16;
  jaccard_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a_ptr, a_ids, a_w, b_ptr, b_ids, b_w,
                                                         pa, pb, npairs, out); count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSK_OK;
}


// ---- batch hints for dsk_minhash_csr_ex, sampled on the device ----------
// out[0]: of min(n, 4096) evenly spaced rows, those holding < 48 elements;
// out[1]: of min(n, 256) evenly spaced rows, those with l1 > 2 (plain sum of
// the row's first 4096 weights: a lower bound, enough for the heuristic).
__global__ void hint_sample_kernel(const int64_t *indptr, const double *w, int64_t n,
                                   unsigned *out) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31;
  const int64_t m = n < 4096 ? n : 4096, md = n < 256 ? n : 256;
  bool small = false;
  if (tid < m) {
    const int64_t r = (int64_t)tid * n / m;
    small = indptr[r + 1] - indptr[r] < 48;
  }
  const unsigned sb = __ballot_sync(0xffffffffu, small);
  if (lane == 0 && sb) atomicAdd(&out[0], (unsigned)__popc(sb));
  const int warp = tid >> 5;
  if (warp < md) {
    const int64_t r = (int64_t)warp * n / md, lo = indptr[r];
    int64_t len = indptr[r + 1] - lo;
    len = len < 4096 ? len : 4096;
    double s = 0.0;
    for (int64_t e = lane; e < len; e += 32) s += w[lo + e];
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && s > 2.0) atomicAdd(&out[1], 1u);
  }
}

// nnz_hint for dsk_minhash_csr_ex from device-resident CSR arrays (what
// dsk_minhash_csr_host derives from its host arrays): `nnz` or 0 for the team
// shape, DSK_HINT_DIRECT when >= 90 % of the sampled rows have l1 > 2.  One
// small launch, an 8-byte copy and a stream synchronise.
extern "C" int dsk_minhash_hints(dsk_ctx *c, const int64_t *indptr, const double *weights,
                                 int64_t n, int64_t nnz, int64_t *hint, void *stream) {
  if (!c || !indptr || !hint || n < 0) return set_err(DSK_EARG, "bad argument");
  *hint = nnz;
  if (n < 4096 || !weights) return DSK_OK;  // small batches keep the mean-based hint
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(c->device));
  std::lock_guard<std::mutex> lock(c->hint_mu);
  CUDA_TRY(cudaMemsetAsync(c->d_hint, 0, 2 * sizeof(unsigned), st));
  hint_sample_kernel<<<32, 256, 0, st>>>(indptr, weights, n, c->d_hint); count_launch();
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(c->h_hint, c->d_hint, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t m = 4096, md = 256;
  int64_t h = 2 * (int64_t)c->h_hint[0] >= m ? 0 : nnz;
  if (10 * (int64_t)c->h_hint[1] >= 9 * md) h |= kMhDirectHint;
  *hint = h;
  return DSK_OK;
}
