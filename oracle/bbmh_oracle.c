/* bbmh_oracle.c -- TEST INFRASTRUCTURE ONLY (see bbmh_oracle.h).
 *
 * Plain-C restatement of the reference's preprocessing path. Citations are
 * /root/reference/proj-relative file:line. Written for clarity, not speed:
 * it is the checker the CUDA product is compared against.
 */
#define _GNU_SOURCE
#include "bbmh_oracle.h"

#include <errno.h>
#include <inttypes.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* status codes: include/bbmh.h:27-42 */
enum {
    ORC_OK = 0,
    ORC_E_INVALID_ARGUMENT = -1,
    ORC_E_UNSUPPORTED_UNIVERSE = -2,
    ORC_E_PERMUTATION_TOO_LARGE = -3,
    ORC_E_MISSING_MINIMA = -5,
    ORC_E_EMPTY_SKETCH = -7,
    ORC_E_DIMENSION_EXCEEDED = -8,
    ORC_E_NON_BINARY_LABEL = -9,
    ORC_E_PARSE = -10,
    ORC_E_IO = -12,
    ORC_E_INTERNAL = -13
};

enum { SCHEME_PERM = 0, SCHEME_2U = 1, SCHEME_4U_MOD = 2, SCHEME_4U_BIT = 3 };

static const uint64_t kM31 = (1ull << 31) - 1;              /* hash_family.hpp:22 */
static const uint64_t kDefaultPermCap = 1ull << 30;          /* hash_family.hpp:69 */

/* thread-local detail message, cleared on entry like capi.cpp:46 */
static __thread char t_err[1024];

const char* orc_last_error(void) { return t_err; }

static int32_t set_err(int32_t st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_err, sizeof t_err, fmt, ap);
    va_end(ap);
    return st;
}

/* ---- prng.hpp:10-61 ----------------------------------------------------- */

uint64_t orc_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

uint64_t orc_keyed_u64(uint64_t seed, uint64_t tag, uint64_t j, uint64_t i) {
    uint64_t x = orc_mix64(seed + 0x9e3779b97f4a7c15ull * (tag + 1));
    x = orc_mix64(x ^ (j + 0xd1b54a32d192ed03ull));
    x = orc_mix64(x ^ (i + 0x8cb92ba72f3d8dd7ull));
    return x;
}

typedef struct { uint64_t state; } splitmix;

static uint64_t sm_next(splitmix* s) {
    s->state += 0x9e3779b97f4a7c15ull;
    return orc_mix64(s->state);
}

static uint64_t sm_next_below(splitmix* s, uint64_t bound) {
    if ((bound & (bound - 1)) == 0) return sm_next(s) & (bound - 1);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t v;
    do {
        v = sm_next(s);
    } while (v >= limit);
    return v % bound;
}

/* hash_family.cpp:43-49 */
static uint64_t keyed_below(uint64_t seed, uint64_t tag, uint64_t j, uint64_t i, uint64_t bound) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    for (uint64_t attempt = 0;; ++attempt) {
        uint64_t v = orc_keyed_u64(seed, tag, j, i * 64 + attempt);
        if (v < limit) return v % bound;
    }
}

/* ---- hash_family.hpp:24-63 ---------------------------------------------- */

uint64_t orc_mod_mersenne31(uint64_t v) {
    const uint64_t p = kM31;
    v = (v >> 31) + (v & p);
    if (v >= 2 * p) v = (v >> 31) + (v & p);
    if (v >= p) return v - p;
    return v;
}

/* hash_family.cpp:28-37 */
static int is_prime_u64(uint64_t n) {
    if (n < 2) return 0;
    static const uint64_t small[4] = {2, 3, 5, 7};
    for (int i = 0; i < 4; ++i)
        if (n % small[i] == 0) return n == small[i];
    for (uint64_t d = 11; d * d <= n; d += 2)
        if (n % d == 0) return 0;
    return 1;
}

struct orc_family {
    int32_t scheme;
    uint64_t dim;
    uint32_t k;
    uint64_t seed;
    uint32_t s;       /* log2(dim) when dim is a power of two */
    int dim_pow2;
    uint64_t p;
    uint32_t* twou;   /* k * {a1, a2} */
    uint64_t* fouru;  /* k * {a0, a1, a2, a3} */
    uint32_t* perm;   /* k * dim */
};

/* eval_2u, hash_family.hpp:48-51. The reference shifts a uint32 right by
 * (32 - s); for dim = 1 (s = 0) that is a shift by 32, which the x86 build
 * executes with the count masked to 0 (result h). The & 31 states that
 * observed behaviour explicitly. */
static uint32_t eval_2u(uint32_t a1, uint32_t a2, uint32_t t, uint32_t s) {
    uint32_t h = a1 + a2 * t;
    return s >= 32 ? h : h >> ((32 - s) & 31);
}

static uint32_t reduce_dim(const orc_family* f, uint64_t h) {     /* hash_family.hpp:107-109 */
    return (uint32_t)(f->dim_pow2 ? (h & (f->dim - 1)) : (h % f->dim));
}

/* HashFamily::map, hash_family.hpp:77-92 */
static uint32_t fam_map(const orc_family* f, uint32_t j, uint32_t t) {
    switch (f->scheme) {
        case SCHEME_2U:
            return eval_2u(f->twou[2 * j], f->twou[2 * j + 1], t, f->s);
        case SCHEME_4U_BIT: {   /* eval_4u with mod_mersenne31, hash_family.hpp:56-63 */
            const uint64_t* a = f->fouru + 4 * (size_t)j;
            uint64_t h = a[3];
            h = orc_mod_mersenne31(h * t + a[2]);
            h = orc_mod_mersenne31(h * t + a[1]);
            h = orc_mod_mersenne31(h * t + a[0]);
            return reduce_dim(f, h);
        }
        case SCHEME_4U_MOD: {   /* eval_4u with v % p, hash_family.hpp:84-87 */
            const uint64_t* a = f->fouru + 4 * (size_t)j;
            const uint64_t p = f->p;
            uint64_t h = a[3];
            h = (h * t + a[2]) % p;
            h = (h * t + a[1]) % p;
            h = (h * t + a[0]) % p;
            return reduce_dim(f, h);
        }
        default:
            return f->perm[(size_t)j * f->dim + t];
    }
}

/* HashFamily::build, hash_family.cpp:53-119 (+ capi.cpp:97-101 scheme_of) */
/* Permutation table j of a family (hash_family.cpp:105-114): Fisher-Yates
 * over 0..dim-1 driven by SplitMix64 seeded keyed_u64(seed, 1, j, 0). */
void orc_perm_table(uint64_t seed, uint64_t dim, uint32_t j, uint32_t* tab) {
    for (uint64_t t = 0; t < dim; ++t) tab[t] = (uint32_t)t;
    splitmix rng = {orc_keyed_u64(seed, 1, j, 0)};
    for (uint64_t t = dim - 1; t > 0; --t) {
        uint64_t r = sm_next_below(&rng, t + 1);
        uint32_t tmp = tab[t];
        tab[t] = tab[r];
        tab[r] = tmp;
    }
}

int32_t orc_family_create(int32_t scheme, uint64_t dim, uint32_t k, uint64_t seed,
                          uint64_t prime, uint64_t perm_cap_bytes, orc_family** out) {
    t_err[0] = 0;
    if (!out) return set_err(ORC_E_INVALID_ARGUMENT, "out must not be NULL");
    if (scheme < SCHEME_PERM || scheme > SCHEME_4U_BIT)
        return set_err(ORC_E_INVALID_ARGUMENT, "unknown scheme tag %d", (int)scheme);
    if (!prime) prime = kM31;
    if (!perm_cap_bytes) perm_cap_bytes = kDefaultPermCap;
    if (dim < 1) return set_err(ORC_E_INVALID_ARGUMENT, "universe size must be >= 1");
    if (k < 1) return set_err(ORC_E_INVALID_ARGUMENT, "k must be >= 1");

    orc_family* f = calloc(1, sizeof *f);
    if (!f) return set_err(ORC_E_INTERNAL, "std::bad_alloc");
    f->scheme = scheme;
    f->dim = dim;
    f->k = k;
    f->seed = seed;
    f->dim_pow2 = (dim & (dim - 1)) == 0;
    f->s = f->dim_pow2 ? (uint32_t)__builtin_ctzll(dim) : 0;
    f->p = kM31;

    if (scheme == SCHEME_2U) {
        if (!f->dim_pow2 || dim > (1ull << 32)) {
            free(f);
            return set_err(ORC_E_UNSUPPORTED_UNIVERSE,
                           "2u requires a power-of-two universe <= 2^32, got %" PRIu64, dim);
        }
        f->twou = malloc(sizeof(uint32_t) * 2 * (size_t)k);
        for (uint32_t j = 0; j < k; ++j) {
            f->twou[2 * j] = (uint32_t)orc_keyed_u64(seed, 2, j, 0);
            f->twou[2 * j + 1] = (uint32_t)orc_keyed_u64(seed, 2, j, 1) | 1u;
        }
    } else if (scheme == SCHEME_4U_MOD || scheme == SCHEME_4U_BIT) {
        const uint64_t p = prime;
        const char* msg = NULL;
        int32_t st = ORC_E_INVALID_ARGUMENT;
        if (scheme == SCHEME_4U_BIT && p != kM31) msg = "4u-bit is fixed to p = 2^31-1";
        else if (p > kM31) msg = "prime modulus must be <= 2^31-1";
        else if (!is_prime_u64(p)) msg = "modulus is not prime";
        if (msg) {
            free(f);
            return set_err(st, "%s", msg);
        }
        if (dim >= p) {
            free(f);
            return set_err(ORC_E_UNSUPPORTED_UNIVERSE,
                           "universe size %" PRIu64 " must be < p = %" PRIu64, dim, p);
        }
        f->p = p;
        f->fouru = malloc(sizeof(uint64_t) * 4 * (size_t)k);
        for (uint32_t j = 0; j < k; ++j)
            for (uint64_t i = 0; i < 4; ++i)
                f->fouru[4 * (size_t)j + i] = keyed_below(seed, 3, j, i, p);
    } else {
        const uint64_t bytes = dim * (uint64_t)k * 4u;
        if (dim > (1ull << 32) || bytes / 4u / k != dim || bytes > perm_cap_bytes) {
            free(f);
            return set_err(ORC_E_PERMUTATION_TOO_LARGE,
                           "permutation tables need %" PRIu64 " bytes, cap is %" PRIu64,
                           dim * (uint64_t)k * 4u, perm_cap_bytes);
        }
        f->perm = malloc((size_t)bytes);
        if (!f->perm) {
            free(f);
            return set_err(ORC_E_INTERNAL, "std::bad_alloc");
        }
        for (uint32_t j = 0; j < k; ++j) orc_perm_table(seed, dim, j, f->perm + (size_t)j * dim);
    }
    *out = f;
    return ORC_OK;
}

void orc_family_destroy(orc_family* f) {
    if (!f) return;
    free(f->twou);
    free(f->fouru);
    free(f->perm);
    free(f);
}

/* capi.cpp:142-151 */
int32_t orc_family_map(const orc_family* f, uint32_t j, uint32_t t, uint32_t* out) {
    t_err[0] = 0;
    if (!f || !out) return set_err(ORC_E_INVALID_ARGUMENT, "family and out must not be NULL");
    if (j >= f->k) return set_err(ORC_E_INVALID_ARGUMENT, "j out of range");
    if ((uint64_t)t >= f->dim) return set_err(ORC_E_INVALID_ARGUMENT, "t out of range");
    *out = fam_map(f, j, t);
    return ORC_OK;
}

int32_t orc_family_coeffs(const orc_family* f, uint32_t* twou_out, uint64_t* fouru_out) {
    if (!f) return ORC_E_INVALID_ARGUMENT;
    if (f->twou && twou_out) memcpy(twou_out, f->twou, sizeof(uint32_t) * 2 * (size_t)f->k);
    if (f->fouru && fouru_out) memcpy(fouru_out, f->fouru, sizeof(uint64_t) * 4 * (size_t)f->k);
    return ORC_OK;
}

/* ---- sketch.cpp:55-100 ---------------------------------------------------- */

static size_t packed_code_bytes(uint32_t k, uint32_t b) {   /* sketch.hpp:28 */
    return ((size_t)k * b + 7) / 8;
}

static uint32_t get_code(const uint8_t* codes, uint32_t j, uint32_t b) {   /* sketch.cpp:55-62 */
    uint32_t out = 0;
    size_t pos = (size_t)j * b;
    for (uint32_t i = 0; i < b; ++i, ++pos) out |= (uint32_t)((codes[pos >> 3] >> (pos & 7)) & 1u) << i;
    return out;
}

static void set_code(uint8_t* codes, uint32_t j, uint32_t b, uint32_t code) {   /* :64-69 */
    size_t pos = (size_t)j * b;
    for (uint32_t i = 0; i < b; ++i, ++pos)
        if ((code >> i) & 1u) codes[pos >> 3] |= (uint8_t)(1u << (pos & 7));
}

/* sketch_one, sketch.cpp:71-100. b already narrowed to u8 by the caller
 * (capi.cpp:163). Returns flags. */
static int sketch_one(const orc_family* f, const uint32_t* idx, size_t n, uint32_t b,
                      uint8_t* codes, uint64_t* minima) {
    const uint32_t k = f->k;
    const size_t cb = packed_code_bytes(k, b);
    memset(codes, 0, cb);
    if (n == 0) {
        memset(codes, 0xff, cb);
        size_t tail = ((size_t)k * b) & 7;
        if (tail) codes[cb - 1] = (uint8_t)(0xffu >> (8 - tail));
        if (minima)
            for (uint32_t j = 0; j < k; ++j) minima[j] = UINT64_MAX;
        return 1;
    }
    const uint32_t mask = b >= 32 ? 0xffffffffu : ((1u << b) - 1);
    for (uint32_t j = 0; j < k; ++j) {
        uint32_t mn = fam_map(f, j, idx[0]);
        for (size_t i = 1; i < n; ++i) {
            uint32_t h = fam_map(f, j, idx[i]);
            if (h < mn) mn = h;
        }
        if (minima) minima[j] = mn;
        set_code(codes, j, b, mn & mask);
    }
    return 0;
}

/* capi.cpp:153-169 */
int32_t orc_sketch_set(const orc_family* f, const uint32_t* indices, size_t count, uint32_t b,
                       uint64_t* minima_out, uint8_t* codes_out, int32_t* empty_out) {
    t_err[0] = 0;
    if (!f || !codes_out) return set_err(ORC_E_INVALID_ARGUMENT, "family and codes_out required");
    if (count > 0 && !indices) return set_err(ORC_E_INVALID_ARGUMENT, "indices must not be NULL");
    b = (uint8_t)b;
    if (b < 1 || b > 32) return set_err(ORC_E_INVALID_ARGUMENT, "b must be in 1..32");
    int fl = sketch_one(f, indices, count, b, codes_out, minima_out);
    if (empty_out) *empty_out = fl;
    return ORC_OK;
}

typedef struct {
    const orc_family* f;
    const uint64_t* row_ptr;
    const uint32_t* indices;
    uint64_t lo, hi;
    uint32_t b;
    uint8_t* codes;
    uint64_t* minima;
    uint8_t* flags;
} csr_job;

static void* csr_worker(void* arg) {
    csr_job* jb = arg;
    const size_t cb = packed_code_bytes(jb->f->k, jb->b);
    for (uint64_t r = jb->lo; r < jb->hi; ++r) {
        const uint64_t s = jb->row_ptr[r], e = jb->row_ptr[r + 1];
        int fl = sketch_one(jb->f, jb->indices + s, (size_t)(e - s), jb->b, jb->codes + r * cb,
                            jb->minima ? jb->minima + r * jb->f->k : NULL);
        if (jb->flags) jb->flags[r] = (uint8_t)fl;
    }
    return NULL;
}

int32_t orc_sketch_csr(const orc_family* f, const uint64_t* row_ptr, const uint32_t* indices,
                       uint64_t n, uint32_t b, uint8_t* codes_out, uint64_t* minima_out,
                       uint8_t* flags_out, uint32_t threads) {
    t_err[0] = 0;
    if (!f || !codes_out || (n && !row_ptr))
        return set_err(ORC_E_INVALID_ARGUMENT, "family, row_ptr and codes_out required");
    b = (uint8_t)b;
    if (b < 1 || b > 32) return set_err(ORC_E_INVALID_ARGUMENT, "b must be in 1..32");
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    csr_job jobs[256];
    for (uint32_t w = 0; w < threads; ++w) {
        jobs[w] = (csr_job){f, row_ptr, indices, n * w / threads, n * (w + 1) / threads, b,
                            codes_out, minima_out, flags_out};
        if (threads > 1) pthread_create(&tid[w], NULL, csr_worker, &jobs[w]);
        else csr_worker(&jobs[w]);
    }
    if (threads > 1)
        for (uint32_t w = 0; w < threads; ++w) pthread_join(tid[w], NULL);
    return ORC_OK;
}

/* ---- dataio.cpp / sketch.cpp byte formats -------------------------------- */

static void put_u32(FILE* f, uint32_t v) {
    uint8_t b[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16), (uint8_t)(v >> 24)};
    fwrite(b, 1, 4, f);
}

static void put_u64(FILE* f, uint64_t v) {
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(v >> (8 * i));
    fwrite(b, 1, 8, f);
}

static int get_bytes(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n; }

static int get_u32(FILE* f, uint32_t* v) {
    uint8_t b[4];
    if (!get_bytes(f, b, 4)) return 0;
    *v = (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24;
    return 1;
}

static int get_u64(FILE* f, uint64_t* v) {
    uint8_t b[8];
    if (!get_bytes(f, b, 8)) return 0;
    *v = 0;
    for (int i = 0; i < 8; ++i) *v |= (uint64_t)b[i] << (8 * i);
    return 1;
}

/* one parsed record */
typedef struct {
    uint32_t* idx;
    size_t n, cap;
    int8_t label;
} rec_t;

static void rec_push(rec_t* r, uint32_t v) {
    if (r->n == r->cap) {
        r->cap = r->cap ? r->cap * 2 : 64;
        r->idx = realloc(r->idx, r->cap * sizeof(uint32_t));
    }
    r->idx[r->n++] = v;
}

/* record source: LibsvmSource (dataio.cpp:157-190) or BinarySource (:192-245) */
typedef struct {
    FILE* f;
    int binary;
    uint64_t count, read, line_no;
    char* line;
    size_t line_cap;
    const char* path;
} source_t;

/* parse_libsvm, dataio.cpp:60-106, binary mode + accept01 (dataio.hpp:27-30) */
static int32_t parse_libsvm(const char* line, uint64_t line_no, rec_t* out) {
    const char* p = line;
    char* end = NULL;
    out->n = 0;
    double label = strtod(p, &end);
    if (end == p) return set_err(ORC_E_PARSE, "line %" PRIu64 ": missing label", line_no);
    if (label == 1 || label == -1) out->label = (int8_t)label;
    else if (label == 0) out->label = -1;
    else return set_err(ORC_E_PARSE, "line %" PRIu64 ": label must be +-1 (or 0/1)", line_no);
    p = end;
    int64_t prev = -1;
    for (;;) {
        while (*p == ' ' || *p == '\t') ++p;
        if (*p == '\0' || *p == '\n' || *p == '\r' || *p == '#') break;
        long long idx = strtoll(p, &end, 10);
        if (end == p || *end != ':')
            return set_err(ORC_E_PARSE, "line %" PRIu64 ": expected idx:val", line_no);
        if (idx < 1 || idx > (long long)UINT32_MAX)
            return set_err(ORC_E_PARSE, "line %" PRIu64 ": index out of range (1-based u32)",
                           line_no);
        if (idx - 1 <= prev)
            return set_err(ORC_E_PARSE, "line %" PRIu64 ": indices must be strictly ascending",
                           line_no);
        prev = idx - 1;
        p = end + 1;
        double val = strtod(p, &end);
        if (end == p) return set_err(ORC_E_PARSE, "line %" PRIu64 ": missing value", line_no);
        p = end;
        if (val != 1.0)   /* std::to_string(double) formats with "%f" */
            return set_err(ORC_E_PARSE, "line %" PRIu64 ": value %f in binary mode", line_no, val);
        rec_push(out, (uint32_t)(idx - 1));
    }
    return ORC_OK;
}

/* open_corpus, dataio.cpp:257-264 */
static int32_t source_open(source_t* s, const char* path) {
    memset(s, 0, sizeof *s);
    s->path = path;
    FILE* f = fopen(path, "rb");
    if (!f) return set_err(ORC_E_IO, "%s: %s", path, strerror(errno));
    char magic[4] = {0, 0, 0, 0};
    size_t got = fread(magic, 1, 4, f);
    fclose(f);
    s->f = fopen(path, "rb");
    if (!s->f) return set_err(ORC_E_IO, "%s: %s", path, strerror(errno));
    if (got == 4 && memcmp(magic, "BBCV", 4) == 0) {
        s->binary = 1;
        uint8_t version;
        uint64_t dim;
        char m[4];
        if (!get_bytes(s->f, m, 4)) return set_err(ORC_E_IO, "short read");
        if (!get_bytes(s->f, &version, 1)) return set_err(ORC_E_IO, "short read");
        if (version != 1) return set_err(ORC_E_PARSE, "%s: unknown BBCV version", path);
        if (!get_u64(s->f, &dim) || !get_u64(s->f, &s->count)) return set_err(ORC_E_IO, "short read");
    }
    return ORC_OK;
}

static void source_close(source_t* s) {
    if (s->f) fclose(s->f);
    free(s->line);
    s->f = NULL;
}

/* returns 1 = record, 0 = end, <0 = status */
static int32_t source_next(source_t* s, rec_t* out) {
    if (s->binary) {   /* BinarySource::next, dataio.cpp:211-230 */
        if (s->read >= s->count) return 0;
        int8_t label;
        uint32_t n, prev = 0, v;
        if (!get_bytes(s->f, &label, 1)) return set_err(ORC_E_IO, "short read");
        if (label != 1 && label != -1)
            return set_err(ORC_E_NON_BINARY_LABEL, "record %" PRIu64 ": bad label", s->read);
        if (!get_u32(s->f, &n)) return set_err(ORC_E_IO, "short read");
        out->n = 0;
        for (uint32_t i = 0; i < n; ++i) {
            if (!get_u32(s->f, &v)) return set_err(ORC_E_IO, "short read");
            if (i > 0 && v <= prev) return set_err(ORC_E_PARSE, "record %" PRIu64, s->read);
            prev = v;
            rec_push(out, v);
        }
        out->label = label;
        ++s->read;
        return 1;
    }
    for (;;) {   /* LibsvmSource::next, dataio.cpp:166-175 */
        size_t len = 0;
        int c;
        while ((c = fgetc(s->f)) != EOF && c != '\n') {
            if (len + 1 >= s->line_cap) {
                s->line_cap = s->line_cap ? s->line_cap * 2 : 256;
                s->line = realloc(s->line, s->line_cap);
            }
            s->line[len++] = (char)c;
        }
        if (len == 0 && c == EOF) return 0;
        ++s->line_no;
        if (len == 0) continue;   /* blank line */
        s->line[len] = 0;
        int32_t st = parse_libsvm(s->line, s->line_no, out);
        return st == ORC_OK ? 1 : st;
    }
}

/* sketch_file (pipeline.cpp:215-226) through capi.cpp:171-185 */
int32_t orc_sketch_file(const orc_family* f, const char* input_path, const char* output_path,
                        uint32_t b, uint64_t chunk_size, uint32_t workers, int32_t emit_minima,
                        orc_pipeline_stats* stats_out) {
    t_err[0] = 0;
    if (!f) return set_err(ORC_E_INVALID_ARGUMENT, "family must not be NULL");
    if (!output_path) return set_err(ORC_E_INVALID_ARGUMENT, "output_path must not be NULL");
    if (!input_path) return set_err(ORC_E_INVALID_ARGUMENT, "input_path must not be NULL");
    struct timespec w0, w1;
    clock_gettime(CLOCK_MONOTONIC, &w0);
    source_t src;
    int32_t st = source_open(&src, input_path);
    if (st) {
        source_close(&src);
        return st;
    }
    const uint8_t b8 = (uint8_t)b;
    FILE* out = fopen(output_path, "wb");   /* SketchWriter ctor, sketch.cpp:102-113 */
    if (!out) {
        st = set_err(ORC_E_IO, "%s: %s", output_path, strerror(errno));
        source_close(&src);
        return st;
    }
    fwrite("BBMH", 1, 4, out);
    uint8_t head[4] = {1, (uint8_t)f->scheme, b8, 0};
    fwrite(head, 1, 4, out);
    put_u32(out, f->k);
    put_u64(out, f->dim);
    put_u64(out, f->seed);
    put_u64(out, 0);
    FILE* fmin = NULL;
    if (emit_minima) {
        char mp[4096];
        snprintf(mp, sizeof mp, "%s.min64", output_path);
        fmin = fopen(mp, "wb");
        if (!fmin) {
            st = set_err(ORC_E_IO, "%s: %s", mp, strerror(errno));
            goto done;
        }
    }
    if (chunk_size < 1) {   /* pipeline.cpp:125-126 */
        st = set_err(ORC_E_INVALID_ARGUMENT, "chunk_size must be >= 1");
        goto done;
    }
    if (workers < 1) {
        st = set_err(ORC_E_INVALID_ARGUMENT, "workers must be >= 1");
        goto done;
    }
    uint64_t count = 0, chunks = 0, in_chunk = 0;
    rec_t r = {0};
    const size_t cb = packed_code_bytes(f->k, b8);
    uint8_t* codes = malloc(cb ? cb : 1);
    uint64_t* minima = malloc(sizeof(uint64_t) * f->k);
    for (;;) {
        int32_t got = source_next(&src, &r);
        if (got < 0) {
            st = got;
            break;
        }
        if (got == 0) break;
        if (b8 < 1 || b8 > 32) {   /* sketch.cpp:73, raised by the first record */
            st = set_err(ORC_E_INVALID_ARGUMENT, "b must be in 1..32");
            break;
        }
        int fl = sketch_one(f, r.idx, r.n, b8, codes, emit_minima ? minima : NULL);
        int8_t label = r.label;
        uint8_t flags = (uint8_t)fl;
        fwrite(&label, 1, 1, out);
        fwrite(&flags, 1, 1, out);
        fwrite(codes, 1, cb, out);
        if (fmin)
            for (uint32_t j = 0; j < f->k; ++j) put_u64(fmin, minima[j]);
        ++count;
        if (++in_chunk == chunk_size) {
            ++chunks;
            in_chunk = 0;
        }
    }
    if (in_chunk) ++chunks;
    free(r.idx);
    free(codes);
    free(minima);
    if (st == ORC_OK && stats_out) {
        clock_gettime(CLOCK_MONOTONIC, &w1);
        memset(stats_out, 0, sizeof *stats_out);
        stats_out->records = count;
        stats_out->chunks = chunks;
        stats_out->wall_seconds = (w1.tv_sec - w0.tv_sec) + 1e-9 * (w1.tv_nsec - w0.tv_nsec);
    }
    fseek(out, 28, SEEK_SET);   /* count patch, sketch.cpp:131-141 */
    put_u64(out, count);
done:
    if (out) fclose(out);
    if (fmin) fclose(fmin);
    source_close(&src);
    return st;
}

/* expand_stream, expansion.cpp:47-90 (+ SketchReader ctor sketch.cpp:143-163) */
int32_t orc_expand_file(const char* sketch_path, const char* out_path, int32_t row_format) {
    t_err[0] = 0;
    if (row_format != 0 && row_format != 1)
        return set_err(ORC_E_INVALID_ARGUMENT, "unknown row format");
    if (!out_path) return set_err(ORC_E_INVALID_ARGUMENT, "out_path must not be NULL");
    if (!sketch_path) return set_err(ORC_E_INVALID_ARGUMENT, "sketch_path must not be NULL");
    FILE* in = fopen(sketch_path, "rb");
    if (!in) return set_err(ORC_E_IO, "%s: %s", sketch_path, strerror(errno));
    int32_t st = ORC_OK;
    char magic[4];
    uint8_t head[4];
    uint32_t k = 0;
    uint64_t dim0, seed, count;
    if (!get_bytes(in, magic, 4)) { st = set_err(ORC_E_IO, "short read"); goto out_in; }
    if (memcmp(magic, "BBMH", 4) != 0) {
        st = set_err(ORC_E_PARSE, "%s: not a BBMH sketch file", sketch_path);
        goto out_in;
    }
    if (!get_bytes(in, head, 4)) { st = set_err(ORC_E_IO, "short read"); goto out_in; }
    if (head[0] != 1) { st = set_err(ORC_E_PARSE, "%s: unknown version", sketch_path); goto out_in; }
    if (head[1] > 3) { st = set_err(ORC_E_PARSE, "%s: unknown scheme tag", sketch_path); goto out_in; }
    if (!get_u32(in, &k) || !get_u64(in, &dim0) || !get_u64(in, &seed) || !get_u64(in, &count)) {
        st = set_err(ORC_E_IO, "short read");
        goto out_in;
    }
    const uint32_t b = head[2];
    if (b < 1 || b > 32) { st = set_err(ORC_E_INVALID_ARGUMENT, "b must be in 1..32"); goto out_in; }
    const uint64_t edim = (1ull << b) * k;   /* expanded_dim, expansion.cpp:9-15 */
    if (edim > (1ull << 32)) {
        st = set_err(ORC_E_DIMENSION_EXCEEDED, "2^b * k exceeds 32-bit row indices");
        goto out_in;
    }
    FILE* out = fopen(out_path, "wb");
    if (!out) {
        st = row_format == 1 ? set_err(ORC_E_IO, "%s: %s", out_path, strerror(errno))
                             : set_err(ORC_E_IO, "%s: cannot open for writing", out_path);
        goto out_in;
    }
    if (row_format == 1) {   /* CorpusWriter header, dataio.cpp:127-133 */
        fwrite("BBCV", 1, 4, out);
        uint8_t ver = 1;
        fwrite(&ver, 1, 1, out);
        put_u64(out, edim);
        put_u64(out, 0);
    }
    const size_t cb = packed_code_bytes(k, b);
    uint8_t* codes = malloc(cb ? cb : 1);
    uint64_t n = 0;
    for (uint64_t r = 0; r < count; ++r) {
        int8_t label;
        uint8_t flags;
        if (!get_bytes(in, &label, 1) || !get_bytes(in, &flags, 1) || !get_bytes(in, codes, cb)) {
            st = set_err(ORC_E_IO, "short read");
            break;
        }
        const int empty = flags & 1;
        if (row_format == 1) {
            fwrite(&label, 1, 1, out);
            put_u32(out, empty ? 0 : k);
            if (!empty)
                for (uint32_t j = 0; j < k; ++j)
                    put_u32(out, (uint32_t)((1ull << b) * j + get_code(codes, j, b)));
        } else {   /* write_libsvm, dataio.cpp:115-125 */
            fprintf(out, "%+d", (int)label);
            if (!empty)
                for (uint32_t j = 0; j < k; ++j)
                    fprintf(out, " %" PRIu32 ":1",
                            (uint32_t)((1ull << b) * j + get_code(codes, j, b)) + 1);
            fputc('\n', out);
        }
        ++n;
    }
    free(codes);
    if (row_format == 1) {
        fseek(out, 13, SEEK_SET);
        put_u64(out, n);
    }
    fclose(out);
out_in:
    fclose(in);
    return st;
}
