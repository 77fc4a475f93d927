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
 *   ro_scan_roll_mt     _scan.py:28-50 with rkhash.py:48-60 `roll`, on pthreads (full sizes)
 *   ro_fill_mt          ro_splitmix64_fill on pthreads
 *   ro_search_multi_mt  matcher.py:139-153 per length group, rolled, on pthreads
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
    if ((k & (k - 1)) == 0) { /* z mod k == z & (k - 1) for a power of two */
        for (uint64_t i = 0; i < count; ++i)
            out[i] = alphabet[ro_mix(seed + 0x9E3779B97F4A7C15ull * (skip + i + 1)) & (k - 1)];
        return;
    }
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t z = ro_mix(seed + 0x9E3779B97F4A7C15ull * (skip + i + 1));
        out[i] = alphabet[z % (uint64_t)k];
    }
}

/* ------------------------------------------------------------------------------------
 * Full-size checkers (still TEST INFRASTRUCTURE ONLY).  The same per-window decisions as
 * ro_scan_range (_scan.py:35-49), but the window hash is carried by the reference's own
 * exact rolling update (rkhash.py:48-60, `roll`: h' = ((h - out * 2^(m-1)) * 2 + in)
 * mod 2^64) instead of being refolded per window, so a 16 GiB scan finishes in seconds
 * on the host cores.  The range split is parallel.py:155-161's contiguous partition;
 * results are concatenated in range order (parallel.py:168-172).
 */
typedef struct {
    const uint8_t* text;
    const uint8_t* pattern;
    uint64_t m, hx, start, stop;
    int64_t* offs;
    uint64_t n, cap, coll;
} ro_roll_job;

static void ro_push(int64_t** v, uint64_t* n, uint64_t* cap, int64_t x) {
    if (*n == *cap) {
        *cap = *cap ? 2 * *cap : 1024;
        *v = (int64_t*)realloc(*v, *cap * sizeof(int64_t));
    }
    (*v)[(*n)++] = x;
}

static void* ro_roll_run(void* arg) {
    ro_roll_job* j = (ro_roll_job*)arg;
    const uint8_t* t = j->text;
    const uint64_t m = j->m;
    const uint64_t top = m - 1 < 64 ? m - 1 : 64; /* out * 2^(m-1) vanishes for m > 64 */
    uint64_t h = ro_hash_full(t + j->start, m);
    for (uint64_t x = j->start; x < j->stop; ++x) {
        if (h == j->hx) {
            if (memcmp(t + x, j->pattern, m) == 0)
                ro_push(&j->offs, &j->n, &j->cap, (int64_t)x);
            else
                ++j->coll;
        }
        if (x + 1 < j->stop) {
            const uint64_t out = top < 64 ? ((uint64_t)t[x] << top) : 0;
            h = ((h - out) << 1) + (uint64_t)t[x + m];
        }
    }
    return NULL;
}

/* Windows [start, stop) of text (which holds at least stop + m - 1 bytes) on `threads`
 * pthreads.  Writes up to cap offsets (ascending), returns the match count; *collisions
 * receives the hash-equal-but-bytes-differ count. */
uint64_t ro_scan_roll_mt(const uint8_t* text, const uint8_t* pattern, uint64_t m, uint64_t hx,
                         uint64_t start, uint64_t stop, int threads, int64_t* out, uint64_t cap,
                         uint64_t* collisions) {
    *collisions = 0;
    if (m == 0 || stop <= start) return 0;
    if (threads < 1) threads = 1;
    const uint64_t total = stop - start;
    const uint64_t chunk = (total + (uint64_t)threads - 1) / (uint64_t)threads;
    ro_roll_job* jobs = (ro_roll_job*)calloc((size_t)threads, sizeof(ro_roll_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    int nj = 0;
    for (int w = 0; w < threads; ++w) {
        uint64_t s = start + (uint64_t)w * chunk, e = s + chunk;
        if (e > stop) e = stop;
        if (s >= e) break;
        ro_roll_job* j = &jobs[nj++];
        j->text = text; j->pattern = pattern; j->m = m; j->hx = hx; j->start = s; j->stop = e;
    }
    for (int i = 0; i < nj; ++i) pthread_create(&th[i], NULL, ro_roll_run, &jobs[i]);
    for (int i = 0; i < nj; ++i) pthread_join(th[i], NULL);
    uint64_t k = 0;
    for (int i = 0; i < nj; ++i) {
        for (uint64_t q = 0; q < jobs[i].n; ++q, ++k)
            if (k < cap) out[k] = jobs[i].offs[q];
        *collisions += jobs[i].coll;
        free(jobs[i].offs);
    }
    free(jobs);
    free(th);
    return k;
}

typedef struct {
    uint64_t seed, skip, count;
    const uint8_t* alphabet;
    uint32_t k;
    uint8_t* out;
} ro_fill_job;

static void* ro_fill_run(void* arg) {
    ro_fill_job* j = (ro_fill_job*)arg;
    ro_splitmix64_fill(j->seed, j->skip, j->count, j->alphabet, j->k, j->out);
    return NULL;
}

/* ro_splitmix64_fill split over `threads` pthreads (counter-based: byte i depends only
 * on skip + i). */
void ro_fill_mt(uint64_t seed, uint64_t skip, uint64_t count, const uint8_t* alphabet, uint32_t k,
                uint8_t* out, int threads) {
    if (threads < 1) threads = 1;
    const uint64_t chunk = (count + (uint64_t)threads - 1) / (uint64_t)threads;
    ro_fill_job* jobs = (ro_fill_job*)calloc((size_t)threads, sizeof(ro_fill_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    int nj = 0;
    for (int w = 0; w < threads; ++w) {
        uint64_t s = (uint64_t)w * chunk, e = s + chunk;
        if (e > count) e = count;
        if (s >= e) break;
        ro_fill_job* j = &jobs[nj++];
        j->seed = seed; j->skip = skip + s; j->count = e - s; j->alphabet = alphabet; j->k = k;
        j->out = out + s;
    }
    for (int i = 0; i < nj; ++i) pthread_create(&th[i], NULL, ro_fill_run, &jobs[i]);
    for (int i = 0; i < nj; ++i) pthread_join(th[i], NULL);
    free(jobs);
    free(th);
}

/* matcher.py:139-153 for one equal-length group, over windows [start, stop), on pthreads:
 * each window's hash (rolled, as above) is looked up among the sorted pattern hashes
 * (the reference compares it with every indexed hash, :147-148 -- same hit set) and
 * every pattern carrying it is byte-compared (:149-153).  Output as ro_search_multi:
 * pairs grouped per pattern index, ascending offsets; counts[P] per-pattern totals. */
typedef struct {
    const uint8_t* text;
    const uint8_t* pats;
    const ro_key* keys;
    const uint8_t* filt; /* 2^16-bit presence filter over the low 16 hash bits */
    uint32_t P;
    uint64_t m, start, stop;
    int64_t* offs; /* interleaved (offset, index) pairs */
    uint64_t n, cap;
} ro_multi_job;

static void* ro_multi_run(void* arg) {
    ro_multi_job* j = (ro_multi_job*)arg;
    const uint8_t* t = j->text;
    const uint64_t m = j->m;
    const uint64_t top = m - 1 < 64 ? m - 1 : 64;
    uint64_t h = ro_hash_full(t + j->start, m);
    for (uint64_t x = j->start; x < j->stop; ++x) {
        const uint32_t lo = (uint32_t)(h & 0xffff);
        if (j->filt[lo >> 3] & (1u << (lo & 7))) {
            uint32_t a = 0, b = j->P;
            while (a < b) {
                uint32_t mid = (a + b) >> 1;
                if (j->keys[mid].h < h) a = mid + 1; else b = mid;
            }
            for (uint32_t q = a; q < j->P && j->keys[q].h == h; ++q) {
                const uint32_t i = j->keys[q].idx;
                if (memcmp(t + x, j->pats + (uint64_t)i * m, m) == 0) {
                    ro_push(&j->offs, &j->n, &j->cap, (int64_t)x);
                    ro_push(&j->offs, &j->n, &j->cap, (int64_t)i);
                }
            }
        }
        if (x + 1 < j->stop) {
            const uint64_t out = top < 64 ? ((uint64_t)t[x] << top) : 0;
            h = ((h - out) << 1) + (uint64_t)t[x + m];
        }
    }
    return NULL;
}

uint64_t ro_search_multi_mt(const uint8_t* text, uint64_t n, const uint8_t* pats,
                            const uint64_t* phash, uint32_t P, uint64_t m, int threads,
                            int64_t* out_off, uint32_t* out_idx, uint64_t cap, uint64_t* counts) {
    for (uint32_t i = 0; i < P; ++i) counts[i] = 0;
    if (m == 0 || m > n || P == 0) return 0;
    if (threads < 1) threads = 1;
    const uint64_t nw = n - m + 1;
    ro_key* keys = (ro_key*)malloc(sizeof(ro_key) * P);
    uint8_t* filt = (uint8_t*)calloc(1 << 13, 1);
    for (uint32_t i = 0; i < P; ++i) {
        keys[i].h = phash[i];
        keys[i].idx = i;
        const uint32_t lo = (uint32_t)(phash[i] & 0xffff);
        filt[lo >> 3] |= (uint8_t)(1u << (lo & 7));
    }
    qsort(keys, P, sizeof(ro_key), ro_key_cmp);
    const uint64_t chunk = (nw + (uint64_t)threads - 1) / (uint64_t)threads;
    ro_multi_job* jobs = (ro_multi_job*)calloc((size_t)threads, sizeof(ro_multi_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    int nj = 0;
    for (int w = 0; w < threads; ++w) {
        uint64_t s = (uint64_t)w * chunk, e = s + chunk;
        if (e > nw) e = nw;
        if (s >= e) break;
        ro_multi_job* j = &jobs[nj++];
        j->text = text; j->pats = pats; j->keys = keys; j->filt = filt; j->P = P; j->m = m;
        j->start = s; j->stop = e;
    }
    for (int i = 0; i < nj; ++i) pthread_create(&th[i], NULL, ro_multi_run, &jobs[i]);
    for (int i = 0; i < nj; ++i) pthread_join(th[i], NULL);
    for (int i = 0; i < nj; ++i)
        for (uint64_t q = 0; q < jobs[i].n; q += 2) counts[jobs[i].offs[q + 1]]++;
    uint64_t* base = (uint64_t*)calloc(P + 1, sizeof(uint64_t));
    for (uint32_t i = 0; i < P; ++i) base[i + 1] = base[i] + counts[i];
    /* ranges are ascending, so filling in range order keeps every pattern's offsets sorted */
    for (int i = 0; i < nj; ++i) {
        for (uint64_t q = 0; q < jobs[i].n; q += 2) {
            const uint32_t idx = (uint32_t)jobs[i].offs[q + 1];
            const uint64_t pos = base[idx]++;
            if (pos < cap) { out_off[pos] = jobs[i].offs[q]; out_idx[pos] = idx; }
        }
        free(jobs[i].offs);
    }
    uint64_t total = 0;
    for (uint32_t i = 0; i < P; ++i) total += counts[i];
    free(base);
    free(jobs);
    free(th);
    free(keys);
    free(filt);
    return total;
}
