// plan.h -- shared plan structures (host preprocessing <-> device scan).
#pragma once
#include <stdint.h>
#ifndef __CUDACC__
#define __host__
#define __device__
#endif

#include <string>
#include <vector>

#include "../../include/matchb200.h"

namespace mb {

// Per-pattern scan parameters as the kernel reads them (one entry per pattern
// of a batch; a single search is a batch of one).
struct PatDev {
  const uint8_t* bytes;  // device copy of the pattern
  int64_t m;
  int32_t family;
  int32_t anchor;   // pattern offset of the anchor window
  int32_t delta;    // bitmap index b <-> start position s = b - delta - text_misalignment
  int32_t per;      // smallest period
  int32_t L;        // m - per when periodic (break-run length), else 0
  int32_t periodic; // verification by first period block + no break in [s, s+L)
  int32_t exact;    // filter alone decides (no verification)
  int32_t pre;      // staged bytes before the tile's first bit (multiple of 16)
  int32_t post;     // staged bytes after the tile's last bit (multiple of 16)
  uint32_t G[12];   // filter words (family specific); ALIGNED: G[4w + j] = p[a+j+4w .. +4);
                    // K2: per plane {byte-bit mask, gather multiplier, pattern plane bits 0..31, 32..63}
  // K3 sampled q-gram filter (family MB_FAM_SAMPLED); K1G (MB_FAM_GRAM) uses S, q
  int32_t S;        // sampling stride in bytes (K3: multiple of 16, >= 256; K1G: 8 or 16); K2: AND steps at pattern positions < 32
  int32_t q;        // gram bytes (K3: 4, 8, 16 or 32; K1G: 8 or 16); K2: AND steps at positions >= 32
  int32_t B;        // log2 of the bucket count
  int32_t nw;       // ALIGNED: anchor words (window 4 nw + 3 bytes), 1..3; K2: symbol bit planes (1 or 2)
  int32_t mpa;      // K5 batched pass: 7-byte anchor window offset (m >= 7), whatever the family
  uint32_t mpG[4];  // K5 grams p[mpa+j .. mpa+j+4), j = 0..3
  const uint32_t* bloom;   // K3: 65536-bit filter over gram hashes; K1G: GRAM_BLOOM_WORDS words; K2: step table (device)
  const uint16_t* bstart;  // (1 << B) + 1 bucket starts (device)
  const uint16_t* bent;    // S entries: pattern offsets j sorted by bucket (device)
};

// K3 sampled-kernel geometry shared with the planner: a warp unit covers
// K3_UNIT_SEGS 2 KiB segments and lists at most K3_LIST matches at a time --
// the unit's verified occurrences plus one round's unverified gram hits
// (<= 4 per sample, one sample per lane).  The planner takes only patterns
// whose smallest period keeps a unit's occurrences within that bound.
constexpr int K3_UNIT_SEGS = 128;
constexpr int K3_LIST = 1024;
constexpr int K3_BATCH_HITS = 4 * 32;
constexpr int64_t K3_MIN_PERIOD = (int64_t)K3_UNIT_SEGS * 2048 / (K3_LIST - K3_BATCH_HITS - 2) + 1;

// gram hash shared by host table build and device lookup (words little-endian)
__host__ __device__ inline uint32_t gram_mix(const uint32_t* w, int nw) {
  uint32_t h = 0x9E3779B9u;
  for (int i = 0; i < nw; i++) h = (h ^ w[i]) * 0x85EBCA6Bu + (h >> 15);
  return h ^ (h >> 13);
}

// K1G (MB_FAM_GRAM): strided q-gram bloom filter over the staged tile.  One
// sample per S bytes (S = 8 or 16, S-aligned virtual positions) hashed once:
// GRAM_BLOOM_WORDS words per warp in smem, 3 bits per gram inside one word
// (blocked bloom), filled with the grams p[j..j+Q), j in [0, S); followed by
// the S gram hashes (GRAM_TABLE_WORDS in all), which resolve a bloom hit to
// its candidate offsets j by hash equality (the slow path verifies them).
constexpr int GRAM_BLOOM_WORDS = 128;
constexpr int GRAM_TABLE_WORDS = GRAM_BLOOM_WORDS + 16;
__host__ __device__ inline uint32_t gram_bloom_hash(const uint32_t* g, int nw) {
  uint32_t h = g[0] * 0x9E3779B1u ^ g[1] * 0x85EBCA77u;
  if (nw == 4) h ^= g[2] * 0xC2B2AE3Du ^ g[3] * 0x27D4EB2Fu;
  return h;
}
__host__ __device__ inline uint32_t gram_bloom_bits(uint32_t h) {
  return (1u << ((h >> 20) & 31)) | (1u << ((h >> 15) & 31)) | (1u << ((h >> 10) & 31));
}

// K2 (MB_FAM_SHIFTOR, bit-plane Shift-And) geometry shared with the planner
constexpr int SO_PLANE_WORDS = 68;  // per plane: 64 segment words + 2 halo words (m - 1 <= 63 bits), padded
constexpr int SO_MAX_STEPS = 24;    // AND steps per start; table entries {shift, plane-A xor mask, plane-B xor mask, 0}
constexpr int SO_WARP_WORDS = 2 * SO_PLANE_WORDS + 4 * SO_MAX_STEPS;  // per-warp smem: planes + step table

struct PlanHost {
  int64_t m = 0;
  std::vector<uint8_t> pat;
  int64_t hor[256];
  int64_t sun[256];
  std::vector<int64_t> kmp;
  int period = 0;
  int family = 0;
  int anchor = 0;
  PatDev dev;
  // K3 tables (host copies; uploaded with the pattern)
  std::vector<uint32_t> bloom;
  std::vector<uint16_t> bstart, bent;
  double entropy = 0;              // bits per byte of the pattern's byte distribution
};

void horspool_table(const uint8_t* p, int64_t m, int64_t* tbl);
void sunday_table(const uint8_t* p, int64_t m, int64_t* tbl);
void kmp_failure(const uint8_t* p, int64_t m, int64_t* fail);
void forward_masks(const uint8_t* p, int64_t m, uint64_t* out, int64_t words);
uint32_t gram_hash(const uint8_t* s, int64_t start, int q);
int build_plan(const uint8_t* pat, int64_t m, const mb_plan_opts* opts, PlanHost* ph, std::string* err);

}  // namespace mb
