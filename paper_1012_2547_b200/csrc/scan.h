// scan.h -- launch parameters of the sm_100a search pipeline.
//
// A search (or a batch of K patterns over one text) is three kernels -- or,
// for one pattern over at most one resident wave of tiles (~9 MiB), one:
// scan_kernel<Filter, FUSED> (a tile per CTA, match bits kept in registers,
// warp look-back over the tiles, positions written directly).
//
//  1. count kernel -- scan_kernel<Filter> (persistent, dynamic tile tickets,
//       no inter-CTA waits): TMA 1D bulk copy of tile + halo into a 2-3 stage
//       smem ring (mbarrier full/empty) -> filter: each lane tests 16 staged
//       bytes per round (packed-word compares) -> candidate bits -> verify
//       (only if a candidate exists and the filter is not exact): direct
//       window compare, warp-cooperative compare, or the period / break-run
//       test -> per-segment (2 KiB) count, matches stored as <= LIST_CAP
//       tile-relative uint16 offsets, else the segment's 256-byte bitmap.
//       Alternatives producing the same segment layout: sampled_kernel (K3,
//       long patterns), mp_scan_kernel (K5, one pass for a whole batch).
//  2. offsets_kernel -- exclusive scan of the segment counts (chunk totals +
//       one grid barrier when co-resident, else decoupled look-back) -> CSR
//       pattern ends; sparse sorted segments are expanded in place, the rest
//       queued (duplicate patterns of a batch read their representative's
//       segments)
//  3. expand_kernel -- warp per queued segment: list / bitmap -> ascending
//       int64 positions at out[offset ..]
//
// Bitmap coordinates: tile tau of a pattern covers bitmap indices
// b in [tau*TILE, (tau+1)*TILE); index b stands for start position
// s = b - delta - off, where off is the text pointer's misalignment below 16 B
// and delta the family's anchor shift.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "plan.h"

namespace mb {

#ifndef MB_NWARP
#define MB_NWARP 16
#endif
#ifndef MB_STAGES
#define MB_STAGES 3
#endif
constexpr int NWARP = MB_NWARP;   // consumer warps; warp NWARP is the TMA producer
constexpr int TILE = NWARP * 2048; // bitmap positions per tile (one TMA stage): 2 KiB per consumer warp
constexpr int NT = NWARP * 32;    // consumer threads
constexpr int SEG = TILE / NWARP; // positions per consumer-warp segment
constexpr int SEG_WORDS = SEG / 32;
constexpr int STAGES = MB_STAGES;  // TMA ring depth (max; scan_kernel may run with 2, see ScanParams.nstages)
constexpr int LIST_CAP = 32;      // sparse segments keep <= 32 uint16 tile offsets
// ticket counters (one uint64 each, zeroed between searches):
// count-kernel launches of one batch: one per family key (engine.cu
// family_key: SWAR m = 1,2,3,5..8 (7), WIN4 and WIN4E (2), ALIGNED 1/2/3 words
// and RUN1 (4), SAMPLED (1), K2 with one / two planes (2), GRAM (S, Q) (4) = NFAMILY_KEYS),
// twice with a batch pass (scans + overflow fallback)
constexpr int NFAMILY_KEYS = 20;
constexpr int MAX_GROUPS = 2 * NFAMILY_KEYS;  // slots 0..39
constexpr int TICKET_OFFSETS = MAX_GROUPS;    // offsets_kernel chunks (ticket order)
constexpr int MAX_MP_CHUNKS = 7;    // batch-pass table chunks (MP_CHUNK patterns each)
constexpr int TICKET_MP0 = TICKET_OFFSETS + 1;
constexpr int TICKET_DENSE = TICKET_MP0 + MAX_MP_CHUNKS;  // segments queued for expand_kernel (even epochs)
constexpr int TICKET_DONE = TICKET_DENSE + 1;       // offsets_kernel CTAs that finished (the last one zeroes the slots)
constexpr int TICKET_DENSE_ODD = TICKET_DONE + 1;   // expand queue of odd epochs
constexpr int TICKET_OFFBAR = TICKET_DENSE_ODD + 1; // offsets_kernel grid barrier (co-resident grid)
constexpr int TICKET_MPBAR = TICKET_OFFBAR + 1;     // batch pass: grid barrier after its prologue zeroes the counts
constexpr int NTICKETS = TICKET_MPBAR + 1;
constexpr int MP_CHUNK = 512;     // patterns per MP table (smem budget)
constexpr int32_t REP_COPY = 1 << 30;  // ScanParams.rep flag (see there)

struct StageHdr {
  int64_t tk;   // global tile ticket (-1: no more work)
  int64_t tau;  // tile index within the pattern
  int32_t k;    // pattern index
  int32_t pad;
};
// dynamic smem: [hdr x STAGES][full x STAGES][empty x STAGES] | stages | per-warp
// segment bitmaps | per-warp break / next-break arrays
constexpr int SM_HDR = 0;
constexpr int SM_FULL = SM_HDR + 32 * STAGES;
constexpr int SM_EMPTY = SM_FULL + 8 * STAGES;
constexpr int SM_STAGES = (SM_EMPTY + 8 * STAGES + 127) & ~127;  // stage s: [pattern pat_cap][text pre + TILE + post]

struct ScanParams {
  const uint8_t* text;  // 16-byte aligned base (text pointer rounded down)
  int64_t off;          // original pointer - base (0..15)
  int64_t n;            // text length
  int64_t nv16;         // round_up(off + n, 16): bytes readable from base
  int64_t ntiles;       // tiles per pattern
  int64_t total_tiles;  // K * ntiles
  const PatDev* pats;   // K entries
  int K;
  int pre, post;        // max margins over the batch
  int stage_bytes;
  int brk_words;        // per-warp break-bitmap words (multiple of 4; 0 if no periodic pattern)
  int pat_cap;          // pattern bytes reserved in smem (multiple of 16)
  int nstages;          // TMA ring depth of this launch (2..STAGES): 2 when 3 would cost a CTA per SM
  unsigned long long* ticket;  // [g]: tile tickets of family group g, [TICKET_OFFSETS]: scan chunks
  int ticket_slot;      // this launch's ticket counter
  const int32_t* plist; // family group -> batch pattern index (null: identity)
  int group_k;          // patterns in this launch's family group
  int64_t group_tiles;  // group_k * ntiles
  uint16_t* counts;     // per segment (tile * NWARP + warp); <= SEG
  uint16_t* lists;      // per segment LIST_CAP tile-relative offsets
  uint32_t* bitmaps;    // per segment SEG_WORDS words (dense segments only)
  int64_t* seglist;     // expand queue (length in ticket[dense_slot]): segment | count << 48
  int64_t* toff;        // per queue entry: exclusive output offset
  int64_t* qpos;        // per queue entry: position of the segment's bit 0
  const int32_t* rep;   // batch pattern -> representative whose segments hold its matches (null: itself);
                        // | REP_COPY: its output is copied from the representative's (replicate_kernel)
  uint64_t* state;      // look-back flags of offsets_kernel (per chunk)
  uint32_t epoch;
  int64_t* out;         // positions (may be null: count only)
  int64_t cap;
  int64_t* offsets_plus1;   // entry k <- inclusive prefix after pattern k
  int64_t* csr0;            // set to 0 by offsets_kernel when non-null (the CSR's leading entry)
  const int64_t* out_base;  // device: output index where this launch starts (null = 0)
  int unsorted_lists;       // lists were filled in arbitrary order (MP path): sort on expand
  const unsigned int* run_if;  // count kernels exit at once unless *run_if != 0 (batch-pass fallback)
  const unsigned int* need;    // per batch pattern: 0 = the batch pass covered it (skip its tiles), else scan
  int dense_slot;              // ticket slot counting this search's expand queue (alternates by epoch parity:
                               // expand_kernel zeroes every slot but this one once the offsets grid is
                               // complete; the next search, of the other parity, zeroes it)
  int offs_resident;           // offsets_kernel grid fits on the GPU at once: chunk = blockIdx.x
};

// Batched multi-pattern single pass (K5 "MP"): every anchor gram of every
// pattern of the batch in one smem table; one TMA pass over the text.
struct MPParams {
  const uint8_t* text;
  int64_t off, n, nv16;
  int64_t ntiles_text;  // tiles over the text (ticket range)
  int64_t ntiles;       // tiles per pattern in the segment layout (= ScanParams.ntiles)
  int pre, post, stage_bytes;
  int nstages;             // TMA ring depth (2..STAGES), as for ScanParams
  unsigned long long* ticket;
  const uint32_t* bloom;   // 65536 bits over gram * 0x9E3779B1 >> 16
  const uint32_t* bstart;  // (1 << B) + 1 bucket starts
  const uint2* ents;       // aligned pass: {gram, (batch index << 16) | (anchor + j)} sorted by bucket
  const uint4* ents4;      // byte-offset pass: {gram lo, gram hi, (batch index << 16) | a, 0} sorted by bucket
  int B, nents;
  int kbase;               // batch index of this chunk's first pattern
  int exact_local;         // exact pass whose patterns all have bitmap shift 0: a hit lands in the segment of the warp
                           // that found it -- counts and list slots per warp in smem (MP_CHUNK packed uint16), no global atomics
  int exact_m;             // byte-offset pass: every pattern has this length = the gram (0: verify); the entry's
                           // low 16 bits then hold the pattern's bitmap shift (delta) instead of an anchor
  const PatDev* pats;      // whole batch
  uint16_t* counts;        // segment layout, zeroed before the launch
  uint16_t* lists;
  unsigned int* overflow;  // any-flag: some pattern needs its per-pattern scan (run_if of the scans)
  unsigned int* need;      // per batch pattern: set when one of its segments exceeds LIST_CAP
  // prologue of the first pass launch of a search (zero_n > 0): zero the
  // counts (zero_n uint16, overflow word included), copy need_src -> need
  // (K flags, when need_src is set), then one grid barrier on *bar
  int64_t zero_n;
  const unsigned int* need_src;
  int need_k;
  unsigned long long* bar;
};

}  // namespace mb
