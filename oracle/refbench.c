/* refbench.c -- TEST/BENCH INFRASTRUCTURE ONLY.
 *
 * Times a bbmh.h-compatible CPU library (normally the unmodified reference
 * built by oracle/Makefile into oracle/_ref/liboracle_bbmh.so) on an
 * in-memory CSR block, calling the reference's own public entry point
 * bbmh_sketch_set (proj/include/bbmh.h:78-84, capi.cpp:155-169) from
 * `threads` POSIX threads, each taking rows from a shared atomic counter.
 * The library is dlopen()ed RTLD_LOCAL so its bbmh_* symbols never clash with
 * the CUDA product's identically named exports.
 */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef int32_t (*create_fn)(int32_t, uint64_t, uint32_t, uint64_t, uint64_t, uint64_t, void**);
typedef void (*destroy_fn)(void*);
typedef int32_t (*sketch_set_fn)(const void*, const uint32_t*, size_t, uint32_t, uint64_t*,
                                 uint8_t*, int32_t*);

typedef struct {
    sketch_set_fn sketch_set;
    const void* fam;
    const uint64_t* row_ptr;
    const uint32_t* indices;
    uint64_t n;
    uint32_t b;
    size_t cb;
    uint8_t* codes;
    atomic_uint_fast64_t* next;
    int32_t status;
} worker_t;

static void* worker(void* arg) {
    worker_t* w = arg;
    for (;;) {
        uint64_t r = atomic_fetch_add(w->next, 1);
        if (r >= w->n) break;
        int32_t empty = 0;
        int32_t st = w->sketch_set(w->fam, w->indices + w->row_ptr[r],
                                   (size_t)(w->row_ptr[r + 1] - w->row_ptr[r]), w->b, NULL,
                                   w->codes + r * w->cb, &empty);
        if (st) {
            w->status = st;
            break;
        }
    }
    return NULL;
}

typedef struct {
    double r_hat, r_raw, p_hat, c1b, c2b, var_theory;
} est_t;
typedef int32_t (*est_fn)(const uint8_t*, const uint8_t*, uint32_t, uint32_t, uint64_t, uint64_t,
                          uint64_t, uint64_t, est_t*);

typedef struct {
    est_fn fn;
    const uint8_t *a, *b;
    uint64_t na, nb;
    uint32_t k, bb;
    size_t cb;
    uint32_t* counts;
    atomic_uint_fast64_t* next;
} est_worker_t;

static void* est_worker(void* arg) {
    est_worker_t* w = arg;
    for (;;) {
        const uint64_t i = atomic_fetch_add(w->next, 1);
        if (i >= w->na) break;
        for (uint64_t j = 0; j < w->nb; ++j) {
            est_t e;
            w->fn(w->a + i * w->cb, w->b + j * w->cb, w->k, w->bb, 10, 10, 5, 1ull << 20, &e);
            w->counts[i * w->nb + j] = (uint32_t)(e.p_hat * w->k + 0.5);
        }
    }
    return NULL;
}

/* All pairs through the reference's bbmh_estimate_codes (estimator.cpp:53-69)
 * on `threads` threads; returns wall seconds (counts_out = p_hat * k). */
double refbench_estimate_pairs(const char* lib_path, const uint8_t* a, uint64_t na,
                               const uint8_t* b, uint64_t nb, uint32_t k, uint32_t bits,
                               uint32_t* counts_out, uint32_t threads) {
    void* h = dlopen(lib_path, RTLD_NOW | RTLD_LOCAL);
    if (!h) return -1;
    est_fn fn = (est_fn)dlsym(h, "bbmh_estimate_codes");
    if (!fn) return -1;
    if (threads < 1) threads = 1;
    pthread_t* tid = calloc(threads, sizeof *tid);
    est_worker_t* ws = calloc(threads, sizeof *ws);
    atomic_uint_fast64_t next = 0;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (uint32_t i = 0; i < threads; ++i) {
        ws[i] = (est_worker_t){fn, a, b, na, nb, k, bits, ((size_t)k * bits + 7) / 8, counts_out, &next};
        pthread_create(&tid[i], NULL, est_worker, &ws[i]);
    }
    for (uint32_t i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    free(tid);
    free(ws);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* Returns wall seconds of the sketching (family build excluded), or a
 * negative value on failure (-1 dlopen/dlsym, -2 family, -3 sketch). */
double refbench_sketch_csr(const char* lib_path, int32_t scheme, uint64_t dim, uint32_t k,
                           uint64_t seed, uint64_t perm_cap, const uint64_t* row_ptr,
                           const uint32_t* indices, uint64_t n, uint32_t b, uint8_t* codes_out,
                           uint32_t threads) {
    void* h = dlopen(lib_path, RTLD_NOW | RTLD_LOCAL);
    if (!h) return -1;
    create_fn create = (create_fn)dlsym(h, "bbmh_family_create");
    destroy_fn destroy = (destroy_fn)dlsym(h, "bbmh_family_destroy");
    sketch_set_fn sk = (sketch_set_fn)dlsym(h, "bbmh_sketch_set");
    if (!create || !destroy || !sk) return -1;
    void* fam = NULL;
    if (create(scheme, dim, k, seed, 0, perm_cap, &fam) != 0) return -2;
    if (threads < 1) threads = 1;
    pthread_t* tid = calloc(threads, sizeof *tid);
    worker_t* ws = calloc(threads, sizeof *ws);
    atomic_uint_fast64_t next = 0;
    const size_t cb = ((size_t)k * (uint8_t)b + 7) / 8;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (uint32_t i = 0; i < threads; ++i) {
        ws[i] = (worker_t){sk, fam, row_ptr, indices, n, b, cb, codes_out, &next, 0};
        pthread_create(&tid[i], NULL, worker, &ws[i]);
    }
    int32_t st = 0;
    for (uint32_t i = 0; i < threads; ++i) {
        pthread_join(tid[i], NULL);
        if (ws[i].status) st = ws[i].status;
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    destroy(fam);
    free(tid);
    free(ws);
    if (st) return -3;
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
