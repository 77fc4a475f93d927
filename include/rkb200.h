/*
 * rkb200.h -- C ABI of the B200-native Rabin-Karp scan (librkb200.so).
 *
 * The drop-in seam is the reference's scan module, rkmatch._scan
 * (/root/reference/pkg/src/rkmatch/_scan.py), which the search API
 * (matcher.py, parallel.py) calls directly.  Every entry point below replaces one
 * reference function; the Python host layer (paper_1810_01051_b200/) binds them with
 * ctypes and keeps the reference's public signatures, validation order and exceptions.
 *
 * Conventions
 *   - Plain pointers and sizes only.  `d_` pointers are device memory of the context's
 *     device, `h_` pointers are host memory (pinned or pageable).
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - Every function returns 0 on success, RK_EINVAL for argument errors (the Python
 *     layer maps it to ValueError), RK_ECUDA for CUDA failures and RK_ENCCL for NCCL
 *     failures (RuntimeError).
 *     rk_last_error() returns the calling thread's last message.
 *   - A context owns per-device scratch (per-tile match counts and hit masks, counter
 *     sets, the pattern cache, staging buffers).  Calls on one context are serialised by
 *     its mutex, and the scratch is stream-ordered: a call on a different stream than the
 *     previous one first makes its stream wait for the work already queued on that one
 *     (so the previous call's stream must still exist at the next call).  For concurrent
 *     scans use one context per stream.
 *   - Hash: h = sum b_i * 2^(m-1-i) mod 2^64 (rkhash.py:21-28).  Window x covers text
 *     bytes [x, x+m).  Offsets are 0-based int64, strictly ascending.
 */
#ifndef RKB200_H
#define RKB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RK_OK 0
#define RK_EINVAL 1
#define RK_ECUDA 2
#define RK_ENCCL 3

typedef struct rk_ctx rk_ctx_t;

/* Library identification ("rkb200 <version> sm_100a"). */
const char* rk_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* rk_last_error(void);
/* Number of visible CUDA devices (0 when no driver/GPU). */
int rk_device_count(void);

/* Create / destroy a scan context bound to `device`. */
int rk_ctx_create(int device, rk_ctx_t** out);
int rk_ctx_destroy(rk_ctx_t* ctx);

/*
 * rk_scan -- replaces _scan_range (_scan.py:28-50) and scan (_scan.py:53-68).
 * Scans windows x in [start, stop) of the device text (n bytes) for the m-byte host
 * pattern whose 64-bit hash the caller passes as hx (the reference passes hx the same
 * way, hash_pattern_host parallel.py:104-108).  Writes the first min(matches, cap)
 * matching window starts, ascending, to d_out and returns the true totals:
 *   *matches    windows whose hash equals hx AND whose bytes equal the pattern
 *   *collisions windows whose hash equals hx but whose bytes differ
 *   *hash_hits  matches + collisions (ScanStats.hash_hits, matcher.py:45-55)
 * Requires stop + m - 1 <= n.  A caller seeing matches > cap fetches all of them with
 * rk_scan_fetch into a larger buffer (the reference rescans instead, _scan.py:64-67).
 * Blocks the host until the result is known.
 */
int rk_scan(rk_ctx_t* ctx, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern,
            uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t* d_out,
            uint64_t cap, uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits,
            void* stream);

/*
 * rk_scan_async -- rk_scan without the host synchronisation: enqueues the scan on
 * `stream`; `out_bias` is added to every written offset (shard / staging origin).
 * If d_counts (device, 3 x u64) is non-NULL, {matches, hash_hits, collisions} are
 * copied there on the stream; rk_scan_result() returns the totals of the last scan of
 * this context to the host.
 */
int rk_scan_async(rk_ctx_t* ctx, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern,
                  uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t* d_out,
                  uint64_t cap, int64_t out_bias, uint64_t* d_counts, void* stream);
int rk_scan_result(rk_ctx_t* ctx, uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits,
                   void* stream);

/*
 * rk_scan_fetch -- the overflow protocol of scan (_scan.py:61-67) without the rescan:
 * re-writes the ordered offsets of this context's last rk_scan / rk_scan_async (which
 * must have been its last call) into d_out, now with room for cap of them, from the
 * per-tile results the scan left on the device.  Asynchronous on `stream`; only the
 * ordered-emission kernel runs.  RK_EINVAL if the last call was not a device scan.
 */
int rk_scan_fetch(rk_ctx_t* ctx, int64_t* d_out, uint64_t cap, void* stream);

/*
 * rk_scan_bitmap -- MatchResult.to_bitmap (matcher.py:36-42) produced on the device:
 * d_bitmap (ceil((stop-start)/32) u32 words, caller-allocated) receives bit i (bit i%32
 * of word i/32) = 1 iff window start+i matches.  1 bit per window instead of 8 bytes
 * per match.  d_counts (device, 3 x u64, optional) receives
 * {matches, hash_hits, collisions}.  Asynchronous on `stream`.
 */
int rk_scan_bitmap(rk_ctx_t* ctx, const uint8_t* d_text, uint64_t n, const uint8_t* h_pattern,
                   uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, uint32_t* d_bitmap,
                   uint64_t* d_counts, void* stream);

/*
 * rk_scan_host -- the end-to-end path for a HOST text (search_sequential /
 * search_parallel called with bytes, matcher.py:101-122, parallel.py:124-177).  The text
 * is staged into HBM in chunks with cudaMemcpyAsync on a copy stream (through an
 * internal pinned ring when h_text is pageable), each chunk scanned as soon as it lands
 * while the next one is in flight, and the ordered offsets are copied into h_out
 * (first min(matches, cap)).  Synchronous.
 */
int rk_scan_host(rk_ctx_t* ctx, const uint8_t* h_text, uint64_t n, const uint8_t* h_pattern,
                 uint32_t m, uint64_t hx, uint64_t start, uint64_t stop, int64_t* h_out,
                 uint64_t cap, uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits);
/*
 * rk_scan_host_batch -- one HOST text, P patterns: search_sequential for each pattern
 * (matcher.py:101-122) -- the reference CLI's per-pattern loop over a pattern file
 * (cli.py:105-118) -- with the text crossing PCIe ONCE.  Pattern i is h_lengths[i] bytes
 * of h_patterns (back to back) with hash h_hashes[i]; its windows are [0, n - m_i + 1).
 * The text is staged chunk by chunk as in rk_scan_host and every pattern's windows ending
 * in a chunk are scanned as soon as it lands.  matches / collisions / hash_hits (P
 * entries each) receive every pattern's totals; h_out the first cap offsets of the
 * concatenation (pattern 0's ordered offsets, then pattern 1's, ...).  Synchronous.
 */
#define RK_BATCH_MAX_PATTERNS 64
int rk_scan_host_batch(rk_ctx_t* ctx, const uint8_t* h_text, uint64_t n,
                       const uint8_t* h_patterns, const uint32_t* h_lengths,
                       const uint64_t* h_hashes, uint32_t P, int64_t* h_out, uint64_t cap,
                       uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits);
/* Copies offsets [first, first+count) of the last rk_scan_host / rk_scan_host_batch of
 * this context (all of them are kept on the device, so a caller whose cap was too small
 * never rescans; for a batch, indices run over the per-pattern concatenation). */
int rk_scan_host_fetch(rk_ctx_t* ctx, int64_t* h_out, uint64_t first, uint64_t count);

/*
 * rk_multi_scan -- one equal-length group of search_multi (matcher.py:139-153).
 * h_patterns holds P deduplicated patterns of length m back to back (PatternSet order,
 * matcher.py:66-84), h_hashes their hash_full values.  Writes up to cap (offset, index)
 * pairs, ordered by (pattern index, offset) -- the reference's per-pattern ascending
 * lists -- and returns the number of pairs.  Requires 1 <= P <= RK_MULTI_MAX_PATTERNS.
 */
#define RK_MULTI_MAX_PATTERNS 4096
int rk_multi_scan(rk_ctx_t* ctx, const uint8_t* d_text, uint64_t n, const uint8_t* h_patterns,
                  uint32_t P, uint32_t m, const uint64_t* h_hashes, int64_t* d_off,
                  uint32_t* d_idx, uint64_t cap, uint64_t* pairs, void* stream);

/*
 * rk_multi_scan_mixed -- a whole PatternSet of mixed lengths (matcher.py:125-157).
 * h_patterns holds the P deduplicated patterns back to back, pattern i being
 * h_lengths[i] bytes; pair indices are positions in this list.  Lengths >= 7 share one
 * sweep over the text per 64 distinct lengths (the reference runs one pass per length,
 * matcher.py:139-153); the lengths 4..6 share one more sweep and 1..3 another (at most
 * two for all lengths < 7).  Patterns longer than the text
 * have no windows.  Output and ordering as rk_multi_scan.
 */
int rk_multi_scan_mixed(rk_ctx_t* ctx, const uint8_t* d_text, uint64_t n,
                        const uint8_t* h_patterns, const uint32_t* h_lengths, uint32_t P,
                        const uint64_t* h_hashes, int64_t* d_off, uint32_t* d_idx, uint64_t cap,
                        uint64_t* pairs, void* stream);

/*
 * rk_window_hashes -- _scan.py:71-91: d_out[x - start] = hash of window x for
 * x in [start, stop).  Requires stop - 1 + m <= n.
 */
int rk_window_hashes(rk_ctx_t* ctx, const uint8_t* d_text, uint64_t n, uint32_t m,
                     uint64_t start, uint64_t stop, uint64_t* d_out, void* stream);

/*
 * rk_generate -- datagen.generate on device (datagen.py:68-77 with the counter form of
 * splitmix64_stream, datagen.py:37-48): d_out[i] = alphabet[z_{skip+i+1} mod k].
 */
int rk_generate(rk_ctx_t* ctx, uint8_t* d_out, uint64_t count, uint64_t seed, uint64_t skip,
                const uint8_t* h_alphabet, uint32_t k, void* stream);

/*
 * Multi-GPU (one process per GPU) -- the range partition and ordered merge of
 * search_parallel (parallel.py:155-172) across GPUs.  NCCL is loaded at run time
 * (libnccl.so.2, or $RKB200_NCCL_LIB); where it is absent these return RK_ENCCL.
 *
 * rk_comm_get_unique_id writes the 128-byte NCCL unique id (on one rank; the caller ships
 * it to the others, e.g. through torch.distributed's store).  rk_comm_init creates this
 * rank's communicator over the context's device (collective over all ranks).
 * $RKB200_COMM_LOG=1 logs each rank's init to stderr.
 */
#define RK_COMM_ID_BYTES 128
typedef struct rk_comm rk_comm_t;
int rk_comm_get_unique_id(uint8_t* id);
int rk_comm_init(rk_ctx_t* ctx, const uint8_t* id, int nranks, int rank, rk_comm_t** out);
int rk_comm_destroy(rk_comm_t* comm);
int rk_comm_info(rk_comm_t* comm, int* nranks, int* rank, int* nccl_version);

/*
 * rk_shard_range -- rank's part of the strong partition of an n-byte text for m-byte
 * windows (parallel.py:155-161: ceil(W / G) contiguous windows per rank, W = n - m + 1):
 * global windows [win_lo, win_hi) and the bytes [byte_lo, byte_hi) they read (the
 * shard plus its (m-1)-byte halo).
 */
int rk_shard_range(uint64_t n, uint32_t m, int nranks, int rank, uint64_t* win_lo,
                   uint64_t* win_hi, uint64_t* byte_lo, uint64_t* byte_hi);

/*
 * rk_scan_sharded -- collective over the communicator's ranks.  Each rank passes the bytes
 * it holds, text = global bytes [byte_lo, byte_lo + len) (device memory of the context's
 * device, or host memory: then staged into HBM chunk by chunk as in rk_scan_host), and
 * its global windows [win_lo, win_hi) (which must lie in those bytes).  Every rank scans
 * its own windows with no inter-GPU traffic; then the ranks' counters are all-gathered
 * and every rank's ordered offsets are broadcast into every rank's d_out at the rank's
 * prefix (an allgather-v: ranks in order = globally ascending).  d_out receives the first
 * min(total, cap) GLOBAL offsets (stream-ordered on `stream`); *matches / *collisions /
 * *hash_hits are the totals over all ranks, known to the host on return.
 */
int rk_scan_sharded(rk_comm_t* comm, const uint8_t* text, uint64_t len, uint64_t byte_lo,
                    const uint8_t* h_pattern, uint32_t m, uint64_t hx, uint64_t win_lo,
                    uint64_t win_hi, int64_t* d_out, uint64_t cap, uint64_t* matches,
                    uint64_t* collisions, uint64_t* hash_hits, void* stream);

/*
 * rk_scan_sharded_batch -- rk_scan_sharded for P patterns over the same device shard in
 * one collective: pattern i (h_lengths[i] bytes of h_patterns, hash h_hashes[i]) over its
 * global windows [win_lo[i], win_hi[i]); its global ordered offsets go to d_outs[i] (a
 * host array of P device pointers; the list is written only if it fits caps[i] -- else
 * call again with room) and matches / collisions / hash_hits[i] receive the totals over
 * all ranks.  The P local scans run back to back, then ONE all-gather of every rank's
 * counters, one host read and one NCCL group of broadcasts (rk_scan_sharded costs one
 * host round trip per pattern).  P <= RK_BATCH_MAX_PATTERNS; device texts only.
 */
int rk_scan_sharded_batch(rk_comm_t* comm, const uint8_t* d_text, uint64_t len, uint64_t byte_lo,
                          const uint8_t* h_patterns, const uint32_t* h_lengths,
                          const uint64_t* h_hashes, uint32_t P, const uint64_t* win_lo,
                          const uint64_t* win_hi, int64_t* const* d_outs, const uint64_t* caps,
                          uint64_t* matches, uint64_t* collisions, uint64_t* hash_hits,
                          void* stream);

/*
 * rk_scan_sharded_batch_async -- rk_scan_sharded_batch with no host round trip: each
 * pattern's local ordered offsets go into a fixed slab of `slab` offsets, ONE NCCL group
 * all-gathers every rank's counters and slabs, and a device kernel writes the global
 * ordered lists to d_outs[i] (up to caps[i]) and, per pattern, {matches, hash_hits,
 * collisions, overflow} to d_counts[4 i .. 4 i + 3] (device memory, the totals over all
 * ranks).  Everything is stream-ordered on `stream`; the call returns at once.  overflow
 * = 1: some rank found more than `slab` matches, the list is incomplete -- run
 * rk_scan_sharded_batch (or again with a larger slab).  The reference's ordered merge
 * of range results (parallel.py:168-172) without a host synchronisation per step.
 */
int rk_scan_sharded_batch_async(rk_comm_t* comm, const uint8_t* d_text, uint64_t len,
                                uint64_t byte_lo, const uint8_t* h_patterns,
                                const uint32_t* h_lengths, const uint64_t* h_hashes, uint32_t P,
                                const uint64_t* win_lo, const uint64_t* win_hi,
                                int64_t* const* d_outs, const uint64_t* caps, uint64_t slab,
                                uint64_t* d_counts, void* stream);

/*
 * rk_multi_scan_sharded -- search_multi (matcher.py:125-157) over a text sharded across the
 * communicator's ranks (collective).  Each rank passes the bytes it holds, d_text = global
 * bytes [byte_lo, byte_lo + len) in device memory, and the window starts it owns,
 * [start_lo, start_hi) (the held bytes must cover them plus the longest pattern's
 * (m - 1)-byte halo, unless the shard ends the text).  Every rank receives ALL ranks'
 * (offset, pattern index) pairs ordered by (index, offset) -- the reference's per-pattern
 * ascending lists -- the first min(total, cap) of them in d_off / d_idx; *pairs = total.
 * Patterns as rk_multi_scan_mixed; n_total = the whole text's length.
 */
int rk_multi_scan_sharded(rk_comm_t* comm, const uint8_t* d_text, uint64_t len, uint64_t byte_lo,
                          uint64_t n_total, const uint8_t* h_patterns, const uint32_t* h_lengths,
                          uint32_t P, const uint64_t* h_hashes, uint64_t start_lo,
                          uint64_t start_hi, int64_t* d_off, uint32_t* d_idx, uint64_t cap,
                          uint64_t* pairs, void* stream);

/* Copies offsets [first, first + count) of the last rk_scan_sharded on this communicator
 * whose total exceeded its cap (every rank keeps the whole gathered list, so a caller
 * whose cap was too small never rescans).  Stream-ordered on `stream`. */
int rk_comm_fetch(rk_comm_t* comm, int64_t* d_out, uint64_t first, uint64_t count, void* stream);

/* Number of kernel launches issued by this context so far (bench accounting). */
uint64_t rk_launch_count(rk_ctx_t* ctx);

#ifdef __cplusplus
}
#endif

#endif /* RKB200_H */
