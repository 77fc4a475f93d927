/*
 * rk_oracle.c -- CPU restatement of the reference scan path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the checker, never the product.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_1810_01051_b200) never links or calls it and fails loudly when its CUDA
 * extension is missing.
 *
 * Each function restates, in plain C, the algorithm of one reference function of the
 * `rkmatch` package (/root/reference/pkg/src/rkmatch/...):
 *
 *   ro_hash_full        rkhash.py:21-28      h = ((h << 1) + b) mod 2^64, empty -> 0
 *   ro_scan_range       _scan.py:28-50       per-window O(m) recompute, compare, byte
 *                                            verify, bounded write, (matches, collisions)
 *   ro_scan             _scan.py:53-68       cap = min(len, 4096); rescan on overflow
 *   ro_scan_parallel    parallel.py:155-176  contiguous ranges of ceil(N/W) windows run
 *                                            on W threads, concatenated in range order
 *   ro_window_hashes    _scan.py:71-91       batched u64 hash of windows [start, stop)
 *   ro_search_multi     matcher.py:125-157   per-length hash sweep, lookup, verify
 *   ro_splitmix64_fill  datagen.py:37-77     counter-based splitmix64 corpus bytes
 *
 * Parity is pinned by tests/test_oracle.py against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RO_INITIAL_CAPACITY 4096u /* _scan.py:14 */

uint64_t ro_hash_full(const uint8_t* data, uint64_t len) {
    uint64_t h = 0;
    for (uint64_t i = 0; i < len; ++i) h = (h << 1) + (uint64_t)data[i];
    return h;
}

/* _scan.py:28-50.  Returns matches; *collisions receives the verify-fail count.
 * Offsets beyond cap are counted but not written, exactly like the reference. */
uint64_t ro_scan_range(const uint8_t* text, const uint8_t* pattern, uint64_t m, uint64_t hx,
                       uint64_t start, uint64_t stop, int64_t* out, uint64_t cap,
                       uint64_t* collisions) {
    uint64_t matches = 0, coll = 0;
    for (uint64_t x = start; x < stop; ++x) {
        uint64_t hy = 0;
        for (uint64_t i = 0; i < m; ++i) hy = (hy << 1) + (uint64_t)text[x + i];
        if (hy == hx) {
            int equal = 1;
            for (uint64_t i = 0; i < m; ++i) {
                if (text[x + i] != pattern[i]) { equal = 0; break; }
            }
            if (equal) {
                if (matches < cap) out[matches] = (int64_t)x;
                ++matches;
            } else {
                ++coll;
            }
        }
    }
    *collisions = coll;
    return matches;
}

/* _scan.py:53-68: first pass with min(len, 4096) slots, full rescan with exact room on
 * overflow.  Returns a malloc'd array (caller frees) and its length. */
int64_t* ro_scan(const uint8_t* text, const uint8_t* pattern, uint64_t m, uint64_t hx,
                 uint64_t start, uint64_t stop, uint64_t* n_out, uint64_t* collisions) {
    *n_out = 0;
    *collisions = 0;
    if (stop <= start) return NULL;
    uint64_t cap = stop - start < RO_INITIAL_CAPACITY ? stop - start : RO_INITIAL_CAPACITY;
    int64_t* out = (int64_t*)malloc(cap * sizeof(int64_t));
    uint64_t matches = ro_scan_range(text, pattern, m, hx, start, stop, out, cap, collisions);
    if (matches > cap) {
        free(out);
        out = (int64_t*)malloc(matches * sizeof(int64_t));
        matches = ro_scan_range(text, pattern, m, hx, start, stop, out, matches, collisions);
    }
    *n_out = matches;
    return out;
}

void ro_free(void* p) { free(p); }

typedef struct {
    const uint8_t* text;
    const uint8_t* pattern;
    uint64_t m, hx, start, stop;
    int64_t* offs;
    uint64_t n, coll;
} ro_job;

static void* ro_job_run(void* arg) {
    ro_job* j = (ro_job*)arg;
    j->offs = ro_scan(j->text, j->pattern, j->m, j->hx, j->start, j->stop, &j->n, &j->coll);
    return NULL;
}

/* parallel.py:155-176: range w = [w*chunk, min((w+1)*chunk, total_threads, n_windows)),
 * chunk = ceil(total_threads / workers); one pthread per non-empty range, results
 * concatenated in range order.  Writes up to cap offsets, returns total matches. */
uint64_t ro_scan_parallel(const uint8_t* text, uint64_t n, const uint8_t* pattern, uint64_t m,
                          uint64_t hx, uint64_t total_threads, int workers, int64_t* out,
                          uint64_t cap, uint64_t* collisions) {
    *collisions = 0;
    if (m == 0 || m > n || workers < 1) return 0;
    uint64_t n_windows = n - m + 1;
    uint64_t chunk = (total_threads + (uint64_t)workers - 1) / (uint64_t)workers;
    ro_job* jobs = (ro_job*)calloc((size_t)workers, sizeof(ro_job));
    pthread_t* th = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
    int nj = 0;
    for (int w = 0; w < workers; ++w) {
        uint64_t s = (uint64_t)w * chunk;
        uint64_t e = s + chunk;
        if (e > total_threads) e = total_threads;
        if (e > n_windows) e = n_windows;
        if (s < e) {
            ro_job* j = &jobs[nj++];
            j->text = text; j->pattern = pattern; j->m = m; j->hx = hx;
            j->start = s; j->stop = e;
        }
    }
    if (nj == 1) {
        ro_job_run(&jobs[0]);
    } else {
        for (int i = 0; i < nj; ++i) pthread_create(&th[i], NULL, ro_job_run, &jobs[i]);
        for (int i = 0; i < nj; ++i) pthread_join(th[i], NULL);
    }
    uint64_t total = 0;
    for (int i = 0; i < nj; ++i) {
        for (uint64_t k = 0; k < jobs[i].n; ++k) {
            if (total < cap) out[total] = jobs[i].offs[k];
            ++total;
        }
        *collisions += jobs[i].coll;
        free(jobs[i].offs);
    }
    free(jobs);
    free(th);
    return total;
}

/* _scan.py:71-91 (bounds checked by the Python wrapper). */
void ro_window_hashes(const uint8_t* text, uint64_t m, uint64_t start, uint64_t stop,
                      uint64_t* out) {
    uint64_t count = stop - start;
    for (uint64_t k = 0; k < count; ++k) out[k] = 0;
    for (uint64_t i = 0; i < m; ++i) {
        const uint8_t* t = text + start + i;
        for (uint64_t k = 0; k < count; ++k) out[k] = (out[k] << 1) + (uint64_t)t[k];
    }
}

/* matcher.py:125-157 restated for one length group.  The patterns arrive already
 * deduplicated (PatternSet, matcher.py:66-84), all of length m, concatenated in
 * `pats` (P*m bytes) with their hashes in `phash`.  For every window whose hash equals
 * some pattern hash, every pattern carrying that hash is byte-compared; a match is
 * emitted as (pattern index, offset).  Output is grouped per pattern with ascending
 * offsets (the order the reference's found[i] lists have).  counts[P] receives the
 * per-pattern totals; pairs beyond cap are counted but not written.  The reference's
 * O(P) compare per window (matcher.py:147-148) is replaced by a sort+bisect of the
 * hash keys: same result set, the checker just has to finish in seconds. */
typedef struct { uint64_t h; uint32_t idx; } ro_key;

static int ro_key_cmp(const void* a, const void* b) {
    const ro_key* x = (const ro_key*)a;
    const ro_key* y = (const ro_key*)b;
    if (x->h != y->h) return x->h < y->h ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

uint64_t ro_search_multi(const uint8_t* text, uint64_t n, const uint8_t* pats,
                         const uint64_t* phash, uint32_t P, uint64_t m,
                         int64_t* out_off, uint32_t* out_idx, uint64_t cap, uint64_t* counts) {
    for (uint32_t i = 0; i < P; ++i) counts[i] = 0;
    if (m == 0 || m > n || P == 0) return 0;
    uint64_t n_windows = n - m + 1;
    ro_key* keys = (ro_key*)malloc(sizeof(ro_key) * P);
    for (uint32_t i = 0; i < P; ++i) { keys[i].h = phash[i]; keys[i].idx = i; }
    qsort(keys, P, sizeof(ro_key), ro_key_cmp);
    /* pass 1: per-pattern counts */
    for (int pass = 0; pass < 2; ++pass) {
        uint64_t* base = NULL;
        uint64_t* fill = NULL;
        if (pass == 1) {
            base = (uint64_t*)calloc(P + 1, sizeof(uint64_t));
            fill = (uint64_t*)calloc(P, sizeof(uint64_t));
            for (uint32_t i = 0; i < P; ++i) base[i + 1] = base[i] + counts[i];
        }
        for (uint64_t x = 0; x < n_windows; ++x) {
            uint64_t hy = 0;
            for (uint64_t i = 0; i < m; ++i) hy = (hy << 1) + (uint64_t)text[x + i];
            /* lower bound */
            uint32_t lo = 0, hi = P;
            while (lo < hi) {
                uint32_t mid = (lo + hi) >> 1;
                if (keys[mid].h < hy) lo = mid + 1; else hi = mid;
            }
            for (uint32_t k = lo; k < P && keys[k].h == hy; ++k) {
                uint32_t i = keys[k].idx;
                if (memcmp(text + x, pats + (uint64_t)i * m, m) == 0) {
                    if (pass == 0) {
                        counts[i]++;
                    } else {
                        uint64_t pos = base[i] + fill[i]++;
                        if (pos < cap) { out_off[pos] = (int64_t)x; out_idx[pos] = i; }
                    }
                }
            }
        }
        if (pass == 1) { free(base); free(fill); }
    }
    free(keys);
    uint64_t total = 0;
    for (uint32_t i = 0; i < P; ++i) total += counts[i];
    return total;
}

/* datagen.py:28-48, 68-77: byte i of the corpus is alphabet[z_{skip+i+1} mod k] where
 * z_s = mix(seed + s * GOLDEN).  Fills out[0..count). */
static inline uint64_t ro_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void ro_splitmix64_fill(uint64_t seed, uint64_t skip, uint64_t count, const uint8_t* alphabet,
                        uint32_t k, uint8_t* out) {
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t z = ro_mix(seed + 0x9E3779B97F4A7C15ull * (skip + i + 1));
        out[i] = alphabet[z % (uint64_t)k];
    }
}
