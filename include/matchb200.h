/*
 * matchb200.h -- C ABI of the B200 exact string matching engine.
 *
 * Drop-in boundary for the reference's search path (arxiv/paper_1012_2547,
 * package `matchbench`).  The reference exposes the path as Python closures:
 *
 *   compile_X(p: bytes) -> run(hay) -> list[int]        (L1 searchers)
 *   AlgorithmDescriptor.compile / .search                (registry.py:27-44)
 *   search_X(pattern, text) / brute_force_search(...)    (core.py:139-161,
 *                                                         comparison.py:355-380,
 *                                                         bitparallel.py:425-458,
 *                                                         automata.py:144-149)
 *
 * This header is what a binding of that interface calls instead (the ctypes
 * binding lives in paper_1012_2547_b200/engine.py).  No
 * torch types cross it: plain pointers, sizes and a cudaStream_t passed as
 * void*.  Device pointers are marked d_, host pointers h_.
 *
 * Semantics (core.py:139-161): every 0-based start position of
 * the pattern in the text, overlapping occurrences included, strictly
 * ascending; m > n yields no positions; m == 0 is an error (core.py:56-57).
 *
 * Return codes: 0 on success, else one of MB_E*; mb_last_error() gives the
 * thread-local message.  Nothing falls back to the CPU.
 */
#ifndef MATCHB200_H
#define MATCHB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MB_OK 0
#define MB_EINVAL 1   /* bad argument (empty pattern, m too large, null ptr) */
#define MB_ENOMEM 2   /* device or host allocation failed */
#define MB_ECUDA 3    /* a CUDA runtime error (message in mb_last_error) */
#define MB_EOVERFLOW 4 /* output capacity too small; *count holds the need */

#define MB_MAX_M 8192 /* longest pattern a plan accepts (BASELINE.json configs use <= 1024) */

/* Kernel families. */
#define MB_FAM_AUTO 0
#define MB_FAM_SWAR 1    /* K1, m <= 3 or 5..8: SWAR xor/zero-byte packed compare, exact */
#define MB_FAM_WIN4 2    /* K1, 4 <= m <= 6: packed 32-bit window compare */
#define MB_FAM_ALIGNED 3 /* K1/K3, m >= 7: aligned-word q-gram anchor + smem verify */
#define MB_FAM_SHIFTOR 4 /* K2, m <= 64: per-thread bit-parallel Shift-And over 1-2 symbol bit planes (small alphabets; verified) */
#define MB_FAM_SAMPLED 5 /* K3, m >= 272: sampled q-gram hash filter, sublinear DRAM reads */
#define MB_FAM_GRAM 6    /* K1G, m >= 15: strided q-gram bloom filter over the staged tile (small alphabets) */

typedef struct mb_plan mb_plan;
typedef struct mb_ctx mb_ctx;

typedef struct {
  int family;            /* MB_FAM_* request (AUTO = engine choice) */
  int sigma_hint;        /* alphabet size if known (0 = unknown) */
  const int64_t* hist;   /* optional 256-entry text byte histogram for anchor choice */
  int anchor_words;      /* ALIGNED anchor words 1..3 (window 4w+3 bytes; 0 = engine choice) */
} mb_plan_opts;

typedef struct {
  int64_t m;
  int family;     /* chosen MB_FAM_* */
  int anchor;     /* pattern offset of the anchor window (ALIGNED, WIN4) / of K2's AND-step window */
  int delta;      /* bitmap index shift: bit b <-> position b - delta */
  int period;     /* smallest period of the pattern (== m if aperiodic) */
  int periodic;   /* 1 if verification uses the period/break-run test */
  int stride;     /* sampling stride S in bytes (K3 SAMPLED, K1G GRAM; else 0) */
  int gram;       /* gram length q in bytes (K3 SAMPLED, K1G GRAM; else 0) */
  int words;      /* ALIGNED anchor words (window 4 words + 3 bytes); K2 SHIFTOR: symbol bit planes (1 or 2); else 0 */
} mb_plan_info_t;

/* ---- plans: the compile_X(p) analogue (comparison.py:70-352 preprocessing) ---- */
int mb_plan_create(const uint8_t* h_pattern, int64_t m, const mb_plan_opts* opts, mb_plan** out);
void mb_plan_destroy(mb_plan* plan);
int mb_plan_info(const mb_plan* plan, mb_plan_info_t* info);

/* Host preprocessing tables (H1), identical to the reference functions:
 *   mb_plan_horspool  == comparison._horspool_table  (comparison.py:18-24)
 *   mb_plan_sunday    == comparison._sunday_table    (comparison.py:27-33)
 *   mb_plan_fwd_masks == bitparallel.forward_masks   (bitparallel.py:24-29),
 *                        256 x words little-endian 64-bit words per byte value
 *   mb_plan_kmp       == comparison.kmp_failure      (comparison.py:56-67), m+1 entries
 *   mb_plan_gram_hash == comparison._gram_hash of the pattern's q-grams (q in 3,5,8),
 *                        m-q+1 entries (comparison.py:227-231)                     */
int mb_plan_horspool(const mb_plan* plan, int64_t* h_out256);
int mb_plan_sunday(const mb_plan* plan, int64_t* h_out256);
int mb_plan_fwd_masks(const mb_plan* plan, uint64_t* h_out, int64_t words);
int mb_plan_kmp(const mb_plan* plan, int64_t* h_out);
int mb_plan_gram_hash(const mb_plan* plan, int q, uint32_t* h_out);

/* ---- contexts: per-thread workspace (tile flags, tickets) bound to a device.
 * Searches on one context may be issued on different streams: a search on
 * another stream than the previous one first waits for that one (the
 * context's tickets and scratch are shared). ---- */
int mb_ctx_create(int device, mb_ctx** out);
void mb_ctx_destroy(mb_ctx* ctx);

/* ---- device-resident search: the run(hay) analogue ----
 * Asynchronous on `stream`.  Writes min(count, cap) positions to d_out and the
 * full count to *d_count (device int64).  d_out may be NULL with cap 0 (count
 * only).  The text may have any alignment. */
int mb_find(mb_ctx* ctx, const mb_plan* plan, const uint8_t* d_text, int64_t n, int64_t* d_out,
            int64_t cap, int64_t* d_count, void* stream);

/* Batched: K plans against one text in one launch.  Output is CSR: pattern k's
 * positions are d_out[d_offsets[k] .. d_offsets[k+1]) (ascending), d_offsets
 * has K+1 device int64 entries; positions past cap are dropped but counted. */
int mb_find_batch(mb_ctx* ctx, const mb_plan* const* plans, int K, const uint8_t* d_text, int64_t n,
                  int64_t* d_out, int64_t cap, int64_t* d_offsets, void* stream);

/* Prepared batch (compile once, search many texts): holds the device params of
 * K plans and the tables of its batched pass (K5 aligned-word or K5b
 * byte-offset, chosen at creation).  The plans must outlive the batch. */
typedef struct mb_batch mb_batch;
int mb_batch_create(const mb_plan* const* plans, int K, mb_batch** out);
void mb_batch_destroy(mb_batch* batch);
int mb_find_batch_prepared(mb_ctx* ctx, const mb_batch* batch, const uint8_t* d_text, int64_t n, int64_t* d_out,
                           int64_t cap, int64_t* d_offsets, void* stream);

/* ---- host-buffer entry (the search_X(pattern, text) analogue, synchronous) ----
 * Copies the text host->device, scans, copies positions device->host.  Returns
 * MB_EOVERFLOW (with *h_count set) if cap is too small.  Compiled plans are
 * cached in the context by pattern bytes (up to 4096, freed with the context).
 * With cap <= 2^20 all cap entries of h_out may be written (those past the
 * count are unspecified). */
int mb_search_host(mb_ctx* ctx, const uint8_t* h_pattern, int64_t m, const uint8_t* h_text, int64_t n,
                   int64_t* h_out, int64_t cap, int64_t* h_count);
int mb_search_batch_host(mb_ctx* ctx, const uint8_t* const* h_patterns, const int64_t* ms, int K,
                         const uint8_t* h_text, int64_t n, int64_t* h_out, int64_t cap,
                         int64_t* h_offsets);

/* ---- K0: device byte histogram (Text.alphabet_size, core.py:42-44) ---- */
int mb_histogram(mb_ctx* ctx, const uint8_t* d_text, int64_t n, int64_t* d_hist256, void* stream);

/* Batched searches on this context that took a batched single pass (K5 / K5b). */
int64_t mb_ctx_mp_batches(const mb_ctx* ctx);

/* Number of this library's kernels launched so far in this process. */
int64_t mb_launch_count(void);
const char* mb_last_error(void);
const char* mb_version(void);

#ifdef __cplusplus
}
#endif
#endif
