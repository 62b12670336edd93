/* bbmh_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's b-bit minwise-hashing preprocessing
 * path (arxiv/paper_1205_2958, /root/reference/proj/src). It exists to CHECK
 * the CUDA product (paper_1205_2958_b200/libbbmh.so); only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. It is
 * never the thing measured or shipped, and the product never falls back to it.
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement against the
 * reference itself (oracle/_ref/liboracle_bbmh.so, built from the reference
 * sources by oracle/Makefile) and against the committed golden vectors in
 * tests/golden/ that were generated from that same reference build.
 *
 * Status codes and detail messages follow proj/include/bbmh.h:27-42 and the
 * reference's fail() sites; every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).
 */
#ifndef BBMH_ORACLE_H
#define BBMH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_family orc_family;

typedef struct {
    uint64_t records;
    uint64_t chunks;
    double read_seconds;
    double compute_seconds;
    double write_seconds;
    double wall_seconds;
} orc_pipeline_stats;

const char* orc_last_error(void);

/* src/prng.hpp:10-27 */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_keyed_u64(uint64_t seed, uint64_t tag, uint64_t j, uint64_t i);
/* src/hash_family.hpp:24-32 */
uint64_t orc_mod_mersenne31(uint64_t v);

/* src/hash_family.cpp:53-119 + capi.cpp:132-140 (prime 0 -> 2^31-1, cap 0 -> 1 GiB) */
int32_t orc_family_create(int32_t scheme, uint64_t dim, uint32_t k, uint64_t seed,
                          uint64_t prime, uint64_t perm_cap_bytes, orc_family** out);
void orc_family_destroy(orc_family* f);

/* Permutation table j (dim entries) of the family with this seed. */
void orc_perm_table(uint64_t seed, uint64_t dim, uint32_t j, uint32_t* tab);
/* capi.cpp:142-151 -> hash_family.hpp:77-92 */
int32_t orc_family_map(const orc_family* f, uint32_t j, uint32_t t, uint32_t* out);
/* raw coefficients for white-box tests: 2U -> k*(a1,a2); 4U -> k*(a0..a3) */
int32_t orc_family_coeffs(const orc_family* f, uint32_t* twou_out, uint64_t* fouru_out);

/* capi.cpp:153-169 -> sketch.cpp:71-100 */
int32_t orc_sketch_set(const orc_family* f, const uint32_t* indices, size_t count, uint32_t b,
                       uint64_t* minima_out, uint8_t* codes_out, int32_t* empty_out);

/* Batched restatement of sketch_one over a CSR block (row_ptr has n+1
 * entries). codes_out: n * ceil(k*b/8) bytes; minima_out (nullable): n*k;
 * flags_out (nullable): n bytes (bit0 = empty). `threads` >= 1 splits rows. */
int32_t orc_sketch_csr(const orc_family* f, const uint64_t* row_ptr, const uint32_t* indices,
                       uint64_t n, uint32_t b, uint8_t* codes_out, uint64_t* minima_out,
                       uint8_t* flags_out, uint32_t threads);

/* capi.cpp:171-185 -> pipeline.cpp:215-226 (single-threaded restatement; the
 * reference's output bytes are independent of chunk_size/workers) */
int32_t orc_sketch_file(const orc_family* f, const char* input_path, const char* output_path,
                        uint32_t b, uint64_t chunk_size, uint32_t workers, int32_t emit_minima,
                        orc_pipeline_stats* stats_out);

/* capi.cpp:268-275 -> expansion.cpp:47-90 */
int32_t orc_expand_file(const char* sketch_path, const char* out_path, int32_t row_format);

#ifdef __cplusplus
}
#endif
#endif
