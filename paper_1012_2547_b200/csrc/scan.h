// scan.cuh -- the sm_100a scan kernel: (pattern(s), text) -> ordered positions.
//
// One persistent kernel family, templated on the filter (K1/K3 of SURVEY.md 2):
//
//   tile ticket (atomic, global order)                    [decoupled look-back order]
//     -> TMA 1D bulk copy of the tile + halo into a 4-stage smem ring (mbarrier)
//     -> filter phase: each lane scans 16 bytes/round from smem, packed-word
//        compare -> candidate bits (16 per lane) -> tile bitmap in smem
//     -> verify phase (only if any candidate and the filter is not exact):
//        candidate bits re-checked against the staged text in smem, either
//        directly or by the period/break-run test for periodic patterns
//     -> block popcount -> warp-parallel decoupled look-back -> exclusive offset
//     -> expansion: set bits -> int64 positions, ascending, at out[offset ..]
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

constexpr int TILE = 16384;       // bitmap positions per tile
constexpr int NT = 256;           // threads per CTA (8 warps)
constexpr int NWARP = NT / 32;
constexpr int STAGES = 4;         // TMA ring depth
constexpr int ROUNDS = TILE / (NWARP * 512);  // 512 positions per warp-round
constexpr int BM_WORDS = TILE / 32;
// shared-memory tail after the stage ring: [bars][tickets][bitmap][breaks]
// [next-break][reduction][pattern]; break/pattern sizes are per launch.
constexpr int SM_BARS = 0;
constexpr int SM_TK = SM_BARS + 8 * STAGES;
constexpr int SM_BM = SM_TK + 8 * STAGES;
constexpr int SM_BRK = SM_BM + 4 * BM_WORDS;

struct ScanParams {
  const uint8_t* text;  // 16-byte aligned base (text pointer rounded down)
  int64_t off;          // original pointer - base (0..15)
  int64_t n;            // text length
  int64_t nv16;         // round_up(off + n, 16): bytes readable from base
  int64_t ntiles;       // tiles per pattern
  int64_t total_tickets;
  const PatDev* pats;   // K entries
  int K;
  int pre, post;        // max margins over the batch
  int stage_bytes;
  int brk_words;        // break-bitmap words (multiple of 4)
  int pat_cap;          // pattern bytes reserved in smem (multiple of 16)
  uint64_t* state;      // look-back flags, >= total_tickets entries
  uint32_t epoch;
  unsigned long long* ticket;
  int64_t* out;         // positions (may be null: count only)
  int64_t cap;
  int64_t* offsets_plus1;  // entry k <- inclusive prefix after pattern k
  const int64_t* out_base; // device: output index where this launch starts (null = 0)
};

}  // namespace mb
