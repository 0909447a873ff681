/*
 * dsk_b200.h -- C ABI of the B200-native DartMinHash sketching library
 * (libdsk_b200.so, built from paper_2005_11547_b200/csrc/).
 *
 * The reference (`dartsketch`, pure Python) has no FFI; each entry point
 * below replaces one public function of its hot path, listed beside it as
 * ref/ = /root/reference/pkg/src/dartsketch/.  INTEGRATION.md shows the
 * ctypes binding a maintainer of the reference would add.
 *
 * Conventions
 *   - Return 0 on success, a negative DSK_E* code on argument / CUDA error;
 *     dsk_last_error() describes the last failure of the calling thread.
 *   - Unless a name ends in _host, array arguments are DEVICE pointers on the
 *     context's device and calls are ordered on `stream` (a cudaStream_t, NULL =
 *     legacy default stream).  The caller owns every buffer; the context owns
 *     only the uploaded hash-family constants and its scratch.
 *   - uint64 values are raw bit patterns (numpy uint64 / torch int64 views).
 *   - Per-set status: DSK_OK or one of the codes below.  Bit DSK_STATUS_TIE is
 *     OR-ed in when two darts of one slot had bit-identical fp64 ranks: such a
 *     slot holds the smaller fingerprint, while the reference orders equal
 *     ranks by index tuple (ref/sketching.py:93-99).  C callers must handle a
 *     tied row themselves (re-sketch it through the Python facade, whose
 *     minhash_batch / lsh_batch / shard.minhash_host_multi re-resolve tied rows
 *     by full index tuple on the GPU, or materialise its darts with
 *     dsk_darts_csr at phi* and take the per-bucket minimum by index tuple).
 *   - The C entry points take rows as given; duplicate element ids inside a
 *     row (rejected by ref/core.py:42-43) are checked by the Python facade.
 *   - A context is read-only after creation: concurrent calls on different
 *     streams are safe.
 */
#ifndef DSK_B200_H
#define DSK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* per-set status codes (the reference raises these as exceptions) */
#define DSK_OK 0
#define DSK_EMPTY 1    /* ValidationError "cannot sketch an empty set"   ref/sketching.py:86-88 */
#define DSK_WEIGHT 2   /* ValidationError weights not finite and > 0     ref/core.py:38-41 */
#define DSK_DEPTH 3    /* ValidationError depth/rank depth > 255         ref/darthash.py:158-160 */
#define DSK_AREAS 4    /* ValidationError > 2^27 areas in one step       ref/darthash.py:242-244 */
#define DSK_NOCONV 5   /* RuntimeError: buckets unfilled after 64 steps  ref/sketching.py:112 */
#define DSK_LIMIT 6    /* ValidationError rank limit <= 0 or infinite    ref/darthash.py:136-138 */
#define DSK_SCRATCH 7  /* LSH hit buffer overflow (library limit, not a reference error) */
#define DSK_TOOLARGE 8 /* reserved (no longer returned: large sets are enumerated in slices) */
#define DSK_OVERFLOW 9 /* OverflowError: 1 + t*x_i is inf (math.floor(inf)) ref/darthash.py:154-156 */
#define DSK_RETRY 11   /* internal: an LSH row whose phi0 = 2 first band failed; never returned */
#define DSK_STATUS_TIE 0x100

/* call-level error codes */
#define DSK_EARG (-1)
#define DSK_ECUDA (-2)
#define DSK_ENOMEM (-3)
#define DSK_EUNSUPPORTED (-4)

typedef struct dsk_ctx dsk_ctx;

/* HashFamily.__init__ (ref/randomness.py:104-112): uploads the 22x256 uint64
 * tabulation tables (built on the host by numpy exactly as the reference
 * does), the Poisson(1) CDF (ref/randomness.py:66-85, host libm exp) and the
 * 258-entry floor(log2) threshold table probed from the host libm
 * (DESIGN.md "bit-exactness"). */
int dsk_ctx_create(int device, const uint64_t *tables_host, const double *cdf_host,
                   const double *log2_thr_host, dsk_ctx **out);
int dsk_ctx_destroy(dsk_ctx *ctx);
int dsk_ctx_device(const dsk_ctx *ctx);

/* minhash_density (ref/core.py:150-156): ceil(k ln k) + k, host libm log. */
int64_t dsk_minhash_density(int64_t k);

/* dart_minhash over a CSR batch (ref/sketching.py:115-123 with
 * _minhash_values :102-112 and _bucket_minima :93-99), fused with one_bit
 * packing (ref/sketching.py:164-167; words = np.packbits(bits,
 * bitorder="little") viewed as <u8, ref/sketching.py:229).
 *   indptr int64[n+1], ids uint64[nnz], weights float64[nnz]
 *   out_values uint64[n*k] or NULL; out_bits uint64[n*ceil(k/64)] or NULL
 *   status int32[n] (required); phi int32[n] or NULL (the reference's final
 *   step); stats uint32[n*4] or NULL: {areas, candidate darts, hit darts,
 *   retry passes} at the final step (SURVEY.md §8(d) work units). */
int dsk_minhash_csr(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                    const double *weights, int64_t n, int32_t k, uint64_t *out_values,
                    uint64_t *out_bits, int32_t *status, int32_t *phi, uint32_t *stats,
                    void *stream);

/* dsk_minhash_csr with a hint for the CTA shape: nnz_hint = total nonzeros
 * of the batch (0 = unknown).  Results are identical; only the team shape
 * (warps per set) depends on it: a large mean admits two-warp teams.  Pass 0
 * for batches of mostly small sets (the facade and dsk_minhash_csr_host do so
 * when half of ~4096 sampled rows hold < 48 elements).
 * DSK_HINT_DIRECT or-ed into nnz_hint says that nearly every set has l1 > 2
 * (every band up to phi = 2 has rank depth 0): large batches then run a
 * first launch of the direct-only engine on a wider CTA and a second,
 * general launch for the sets that need the region stages (10-12 % faster
 * on cfg3; a batch of normalised sets would pay ~6 % for the hand-back, so
 * the callers set it only when 90 % of 256 sampled rows qualify). */
#define DSK_HINT_DIRECT ((int64_t)1 << 62)
int dsk_minhash_csr_ex(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                       const double *weights, int64_t n, int32_t k, int64_t nnz_hint,
                       uint64_t *out_values, uint64_t *out_bits, int32_t *status, int32_t *phi,
                       uint32_t *stats, void *stream);

/* nnz_hint for dsk_minhash_csr_ex from device-resident CSR arrays, sampled on
 * the device as dsk_minhash_csr_host samples its host arrays: `nnz` (or 0
 * when half of ~4096 evenly spaced rows hold < 48 elements), with
 * DSK_HINT_DIRECT when >= 90 % of 256 evenly spaced rows have l1 > 2.
 * Batches of < 4096 rows return `nnz`.  Synchronises `stream` (one small
 * launch and an 8-byte copy). */
int dsk_minhash_hints(dsk_ctx *ctx, const int64_t *indptr, const double *weights, int64_t n,
                      int64_t nnz, int64_t *hint, void *stream);

/* The same call with HOST buffers: copies inputs in, sketches, copies the
 * results out, synchronously.  This is the drop-in a ctypes binding of the
 * reference would call with numpy arrays.  Rows are pipelined in chunks of
 * <= 64 MB of input (env DSK_CHUNK_MB overrides): one stream copies every
 * chunk in, two compute streams alternate (so a launch's tail overlaps the
 * next chunk), one stream copies results out.  Pageable host buffers are
 * staged through context-owned pinned buffers by the host's threads (env
 * DSK_HOST_THREADS), so plain numpy arrays run at ~70 % of the pinned rate. */
int dsk_minhash_csr_host(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                         const double *weights, int64_t n, int32_t k, uint64_t *out_values,
                         uint64_t *out_bits, int32_t *status, int32_t *phi, uint32_t *stats);

/* lsh_key over a CSR batch (ref/annindex.py:64-82) fused with the per-table
 * HashFamily.mix64 fold (ref/randomness.py:160-166) that LshIndex applies
 * (ref/annindex.py:135).  normalize != 0 first rescales each set by
 * 2^-weight_class(l1) as LshIndex.insert does (ref/annindex.py:130-131).
 *   out_keys uint64[n*L] or NULL; out_fps uint64[n*L*K] or NULL (the K
 *   rank-ordered fingerprints of each table, i.e. lsh_key's tuples). */
int dsk_lsh_csr(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                const double *weights, int64_t n, int32_t L, int32_t K, int32_t normalize,
                uint64_t *out_keys, uint64_t *out_fps, int32_t *status, int32_t *phi,
                uint32_t *stats, void *stream);

/* dsk_lsh_csr with a team-shape hint: max_row_hint = the largest row's
 * element count (0 = unknown).  Results are identical.  Multi-wave batches
 * run fastest in single-warp teams, but one very large set on one warp can
 * bound the launch, so that shape is taken only for rows of <= 1024 elements
 * (or, sizes unknown, for batches of >= 64 waves of teams).
 * dsk_lsh_csr_host derives the hint from its host indptr. */
int dsk_lsh_csr_ex(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                   const double *weights, int64_t n, int32_t L, int32_t K, int32_t normalize,
                   int64_t max_row_hint, uint64_t *out_keys, uint64_t *out_fps, int32_t *status,
                   int32_t *phi, uint32_t *stats, void *stream);

/* Host-buffer form of dsk_lsh_csr (same pipeline as dsk_minhash_csr_host).
 * LSH launches draw their per-team hit buffers from a pool of context-owned
 * slots reused in stream order, so concurrent calls on different streams
 * are safe. */
int dsk_lsh_csr_host(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                     const double *weights, int64_t n, int32_t L, int32_t K, int32_t normalize,
                     uint64_t *out_keys, uint64_t *out_fps, int32_t *status, int32_t *phi,
                     uint32_t *stats);

/* DartHasher.dart_batch (ref/darthash.py:142-295) for each set of a CSR
 * batch at an absolute rank limit per set: materialises the DartBatch
 * columns (ref/darthash.py:39-53).  Darts of set s are written at
 * [offsets[s], offsets[s] + counts[s]) where offsets is an exclusive scan of
 * the counts of a previous call with cap == 0 (counting pass).  Columns may
 * be NULL when cap == 0. */
int dsk_darts_csr(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                  const double *weights, int64_t n, int64_t t, const double *rank_limit,
                  const int64_t *offsets, int64_t cap, int64_t *counts, int32_t *status,
                  uint64_t *element, uint16_t *nu, uint16_t *rho, uint32_t *w, uint32_t *r,
                  uint16_t *j, double *weight, double *rank, uint64_t *fingerprint,
                  void *stream);

/* HashFamily.hash64_array (ref/randomness.py:170-203) over explicit key
 * columns; every column is uint64[n]. */
int dsk_hash64(dsk_ctx *ctx, const uint64_t *element, const uint64_t *nu, const uint64_t *rho,
               const uint64_t *w, const uint64_t *r, const uint64_t *j, const uint64_t *stream_tag,
               int64_t n, uint64_t *out, void *stream);

/* HashFamily.mix64 (ref/randomness.py:160-166) over nseq sequences of len
 * values each (row-major). */
int dsk_mix64(dsk_ctx *ctx, const uint64_t *values, int64_t nseq, int32_t len, uint64_t *out,
              void *stream);

/* one_bit (ref/sketching.py:164-167) packed little-endian into uint64 words. */
int dsk_pack_onebit(const uint64_t *values, int64_t n, int32_t k, uint64_t *out_bits,
                    void *stream);

/* K0 hash-rate microbenchmark over a full-device grid (4 chains per thread,
 * n_per_thread hashes per chain; xor of results into sink[0]).
 * mode 0: a full hash evaluation as the reference defines it -- 22 table
 * lookups + splitmix64 (ref/randomness.py:121-131): the ALU roofline
 * denominator.  mode 1: one lookup + splitmix64, the cheapest hoisted hash. */
int dsk_hash_peak(dsk_ctx *ctx, int32_t mode, int64_t n_per_thread, uint64_t *sink,
                  int64_t *hashes_done, void *stream);

/* float(np.sum(weights)) of every set (ref/core.py:44, numpy pairwise order):
 * the denominator of each phi step's rank limit phi / ||x||_1. */
int dsk_l1_csr(const int64_t *indptr, const double *weights, int64_t n, double *out_l1,
               void *stream);

/* DSK1 records (ref/sketching.py:210-231) for n sketches, byte-identical to
 * b"".join(dump_sketch(s) for s in sketches): kind 1 = minhash (payload k
 * uint64 values per set), 2 = one-bit (payload: the packed words of
 * dsk_minhash_csr's out_bits, ceil(k/8) bytes written), 3 = bottom-k
 * fingerprints (k uint64).  out holds n * (20 + payload bytes). */
int dsk_dsk1_records(int32_t kind, int32_t k, uint64_t seed, const uint64_t *payload, int64_t n,
                     uint8_t *out, void *stream);

/* exact_jaccard (ref/core.py:103-120) for npairs (row pa[t] of set batch A,
 * row pb[t] of set batch B); rows must hold ids sorted ascending.  Sums run
 * in ascending id order like the reference, so results are bit-identical. */
int dsk_exact_jaccard(const int64_t *a_ptr, const uint64_t *a_ids, const double *a_w,
                      const int64_t *b_ptr, const uint64_t *b_ids, const double *b_w,
                      const int64_t *pa, const int64_t *pb, int64_t npairs, double *out,
                      void *stream);

/* bottom_k (ref/sketching.py:126-161) for each set of a CSR batch, fused:
 * density t = k, the first phi step with >= k darts, the k smallest darts by
 * (rank, element, nu, rho, w, r, j), ascending, as DartBatch columns of
 * shape [n, k].  Per-set status as dsk_minhash_csr, plus DSK_SCRATCH when a
 * set's darts outgrow the per-warp buffer (the caller recomputes it, e.g.
 * with dsk_darts_csr). */
int dsk_bottomk_csr(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids,
                    const double *weights, int64_t n, int32_t k, uint64_t *element, uint16_t *nu,
                    uint16_t *rho, uint32_t *w, uint32_t *r, uint16_t *j, double *weight,
                    double *rank, uint64_t *fingerprint, int32_t *status, int32_t *phi,
                    void *stream);

/* ICWS comparator (ref/baselines.py:84-161, the paper's Table 1 baseline):
 * k consistent weighted samples (element id, tick) per set of a CSR batch.
 * log / log1p come from CUDA's libdevice, so a sample can differ from the
 * host reference's where two candidates tie to within an ulp. */
int dsk_icws_csr(dsk_ctx *ctx, const int64_t *indptr, const uint64_t *ids, const double *weights,
                 int64_t n, int32_t k, uint64_t *out_element, int64_t *out_tick, int32_t *status,
                 void *stream);

/* Number of kernels this library has launched in the process so far (all
 * entry points and contexts); a caller brackets a region with two reads. */
uint64_t dsk_launch_count(void);

/* Bytes the host-buffer entry points have copied host -> device so far. */
uint64_t dsk_h2d_bytes(void);

const char *dsk_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DSK_B200_H */
