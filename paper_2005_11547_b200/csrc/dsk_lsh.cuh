// dsk_lsh.cuh -- K5: (L, K) LSH keys.  (stub, filled in below)
extern "C" int dsk_lsh_csr(dsk_ctx *, const int64_t *, const uint64_t *, const double *, int64_t,
                           int32_t, int32_t, int32_t, uint64_t *, uint64_t *, int32_t *,
                           int32_t *, uint32_t *, void *) {
  return set_err(DSK_EUNSUPPORTED, "lsh not built yet");
}
extern "C" int dsk_lsh_csr_host(dsk_ctx *, const int64_t *, const uint64_t *, const double *,
                                int64_t, int32_t, int32_t, int32_t, uint64_t *, uint64_t *,
                                int32_t *, int32_t *, uint32_t *) {
  return set_err(DSK_EUNSUPPORTED, "lsh not built yet");
}
