/* trims_oracle.h — CPU restatement of the reference's byte/integer algorithms
 * on the load-and-serve path, plus the CPU definition of the transforms the
 * reference does not have (fp32->bf16, KCRS->KRSC, block checksum, weight
 * init). TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg, never by the product path.
 *
 * Pinning (see tests/test_oracle_golden.py): the restated functions are
 * checked against the reference's own known-answer tests and against golden
 * vectors produced by the reference itself (oracle/_ref/libmrm_ref.so, built
 * from /root/reference by oracle/Makefile; tests/golden/make_golden.py).
 * The new transforms (bf16 convert, layout permute, block checksum, uniform
 * init) have no reference counterpart: "parity unpinned" for those rows — this
 * file defines them, and DESIGN.md says so.
 */
#ifndef TRIMS_ORACLE_H
#define TRIMS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FIPS 180-4 SHA-256 — follows proj/src/sha256.cpp:24-123. */
void tro_sha256(const void* data, uint64_t n, uint8_t out[32]);

/* FNV-1a-64 over a string — follows proj/src/bench/catalog.cpp:79-86. */
uint64_t tro_fnv1a_str(const char* s);

/* Splitmix64 output k (0-based) of a stream seeded with `stream_seed`:
 * next() adds 0x9e3779b97f4a7c15 then mixes (catalog.hpp:59-71), so the k-th
 * output is mix(stream_seed + (k+1)*golden). */
uint64_t tro_splitmix_at(uint64_t stream_seed, uint64_t k);
void tro_splitmix_fill(uint64_t stream_seed, uint64_t k0, uint64_t n, uint64_t* out);

/* Catalog stream seed for a model: seed ^ fnv1a(name) (catalog.cpp:142). */
uint64_t tro_catalog_stream(uint64_t seed, const char* model_name);

/* Client::touch — FNV-1a over LE u64 lanes of every tensor in manifest order,
 * tail bytes one by one, padding excluded (proj/src/client.cpp:338-359). */
uint64_t tro_touch(const uint8_t* blob, const uint64_t* offsets, const uint64_t* nbytes,
                   uint64_t ntensors);

/* share_benefit rho = b/q - n(o+s) (proj/src/client.cpp:16-18). */
double tro_share_benefit(double bytes, double n_objects, double q, double o, double s);

/* ---- transforms with no reference counterpart (parity unpinned) ---- */

/* fp32 -> bf16, round-to-nearest-even. NaN -> the canonical bf16 NaN 0x7fff
 * (what B200's cvt.rn.bf16x2.f32 produces; scripts/probe_cvt.cu); +-Inf and
 * +-0 preserved; values that round past the largest finite bf16 become +-Inf
 * (IEEE RNE overflow). f64 -> bf16 uses the same NaN encoding. */
uint16_t tro_f32_to_bf16_1(uint32_t bits);
void tro_f32_to_bf16(const uint32_t* src, uint64_t n, uint16_t* dst);
/* f64 -> f32 (IEEE RNE, the C cast; NaN -> 0x7fc00000 | sign) and f64 -> bf16 (via a single rounding
 * from f64: round-to-nearest-even at bit 48 of the f64 mantissa after
 * rebasing the exponent; subnormal results flush per IEEE RNE). */
void tro_f64_to_f32(const double* src, uint64_t n, float* dst);
void tro_f64_to_bf16(const double* src, uint64_t n, uint16_t* dst);
/* f16 -> f32 exact widening; f16 -> bf16 via f32 then RNE. */
void tro_f16_to_f32(const uint16_t* src, uint64_t n, float* dst);

/* [K][C][R][S] -> [K][R][S][C] for elements of `esize` bytes (1,2,4,8). */
void tro_permute_kcrs_krsc(const void* src, uint64_t K, uint64_t C, uint64_t R, uint64_t S,
                           uint64_t esize, void* dst);

/* TRIMS block checksum (our definition, fused into the GPU ingest): the
 * region is read as LE u64 words w_g (tail zero-padded to 8 bytes), g counted
 * from `word0`; result = sum_g w_g * K(g) mod 2^64, a multilinear hash with an
 * odd per-position key: t = (u32)g * 0x9e3779b1, K(g) = (t*0xc2b2ae3d) << 32
 * | ((t ^ t >> 16) | 1) (keys repeat every 2^32 words = 32 GiB). Any change
 * of a single word changes the sum (odd key); position enters through K.
 * Additive over disjoint word ranges, so a blob's checksum is the sum of its
 * objects' checksums. On the GPU it costs ~8 integer instructions per word
 * (32-bit IMADs), where a splitmix finaliser per word cost ~30. */
uint64_t tro_block_checksum(const uint8_t* p, uint64_t nbytes, uint64_t word0);

/* Synthetic real-valued init (our definition): element j of a tensor whose
 * stream seed is `stream` is lo + (hi-lo) * u, u = (splitmix_at(stream, j)
 * >> 40) * 2^-24, evaluated as one fmaf(hi-lo, u, lo) in fp32. */
void tro_uniform_fill_f32(uint64_t stream, uint64_t j0, uint64_t n, float lo, float hi,
                          float* dst);

#ifdef __cplusplus
}
#endif
#endif
