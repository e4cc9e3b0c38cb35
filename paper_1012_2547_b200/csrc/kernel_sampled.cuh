// kernel_sampled.cuh -- sampled_kernel: K3 sampled q-gram filter (one 128-byte line per S text bytes)
// (part of libmatchb200; included by engine.cu)
#pragma once

namespace mb {

// ------------------------------------------------ kernel 1b: sampled q-gram scan (K3)
// For long, non-periodic patterns: only the q-gram at every
// S-th text position is read (one 128-byte DRAM line per sample instead of S
// bytes); a bloom filter + bucketed offset lists in smem map a gram to the
// pattern offsets j where it occurs, each giving a candidate start s = x - j
// that is verified against the text in global memory.  A warp owns SMP_SEGS
// consecutive segments (16 tiles) and reads every sample whose bit range
// [S*i, S*i + S) meets them, 5 independent 16-byte loads per lane in flight
// (a 128-segment unit has ~260 samples at S = 1008: two batches of 160).
// Output (segment counts, uint16 tile-relative lists) is the scan kernel's, so
// offsets/expand are shared.
constexpr int SMP_SEGS = K3_UNIT_SEGS;  // segments per warp unit (128 = 16 tiles, 256 KiB)
constexpr int SMP_LIST = K3_LIST;       // per-warp match capacity (plan.h: the planner's period bound)
#ifndef MB_SMP_ILP
#define MB_SMP_ILP 5
#endif
#ifndef MB_SMP_WARPS
#define MB_SMP_WARPS 8
#endif
constexpr int SMP_ILP = MB_SMP_ILP;     // samples per lane per batch
static_assert(4 * 32 <= K3_BATCH_HITS, "a round's gram hits must fit the planner's list headroom");
constexpr int SMP_WARPS = MB_SMP_WARPS; // warps per sampled_kernel CTA (independent of the scan tiling)
constexpr int SMP_NT = SMP_WARPS * 32;
__device__ __forceinline__ int sampled_probe(const ScanParams& P, const PatDev& pd, const uint32_t* bloom,
                                             const uint16_t* bstart, const uint16_t* bent, const uint8_t* spat,
                                             const uint32_t* w, int64_t x, int64_t ulo, int64_t uhi, int64_t blo,
                                             int64_t bhi, uint32_t* found) {
  const uint32_t h = gram_mix(w, pd.q >> 2);
  if (!((bloom[h >> 21] >> ((h >> 16) & 31)) & 1u)) return 0;
  int nf = 0;
  const uint32_t bk = h >> (32 - pd.B);
  for (int e = bstart[bk]; e < bstart[bk + 1] && nf < 4; e++) {
    const int j = bent[e];
    bool eq = true;
    for (int c = 0; c < pd.q && eq; c++) eq = spat[j + c] == (uint8_t)(w[c >> 2] >> (8 * (c & 3)));
    if (!eq) continue;
    const int64_t sv = x - j;           // virtual start
    const int64_t bit = sv + pd.delta;  // = x - j + S - 1, inside [x, x + S)
    if (bit < ulo || bit >= uhi || bit < blo || bit > bhi) continue;
    MB_CHECK(sv >= P.off && sv + pd.m <= P.off + P.n);
    found[nf++] = (uint32_t)(bit - ulo);  // gram match: verified by the whole warp (sampled_verify)
  }
  return nf;
}

// Warp-cooperative verification of the gram matches appended to a warp's list
// wl[from, n) (ascending): one candidate at a time, lane l comparing text
// bytes l, l + 32, ... (independent coalesced loads; one lane looping over m
// bytes alone took ~100 cycles per byte, 63 us for a 1024-byte occurrence).
// Failures are dropped in place (order kept); returns the new list length.
// Run outside the sample loop, so that loop's registers do not carry it.
__device__ __forceinline__ uint32_t sampled_verify(const ScanParams& P, const PatDev& pd, const uint8_t* spat,
                                                   int64_t ulo, uint32_t* wl, uint32_t from, uint32_t n, int lane) {
  uint32_t keep = from;
  for (uint32_t e = from; e < n; e++) {
    const uint32_t rel = wl[e];
    const uint8_t* tp = P.text + (ulo + rel - pd.delta);
    bool bad = false;
    for (int c = lane; c < pd.m; c += 32) bad |= __ldg(tp + c) != spat[c];
    const bool ok = !__any_sync(0xffffffffu, bad);
    if (ok && lane == 0) wl[keep] = rel;  // keep <= e: in place
    keep += ok ? 1u : 0u;
    __syncwarp();
  }
  return keep;
}

#ifndef MB_SMP_MINB
#define MB_SMP_MINB 3
#endif
__global__ void __launch_bounds__(SMP_NT, MB_SMP_MINB) sampled_kernel(const ScanParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* bloom = reinterpret_cast<uint32_t*>(smem);                 // 2048 words
  uint16_t* bstart = reinterpret_cast<uint16_t*>(smem + 8192);         // <= 1025
  uint16_t* bent = reinterpret_cast<uint16_t*>(smem + 8192 + 2064);    // <= 4096
  uint32_t* lists = reinterpret_cast<uint32_t*>(smem + 8192 + 2064 + 8192);  // [SMP_WARPS][SMP_LIST]
  int64_t* s_ticket = reinterpret_cast<int64_t*>(lists + SMP_WARPS * SMP_LIST);
  pdl_trigger();  // the next grid may be scheduled as SMs drain
  pdl_wait();     // (see scan_kernel: count kernels are programmatic dependent launches)
  if (P.run_if && *P.run_if == 0u) return;  // conditional fallback launch (MP did not overflow)
  uint8_t* spat = reinterpret_cast<uint8_t*>(s_ticket + 2);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t segs = P.ntiles * NWARP;                                   // segments per pattern
  const int64_t wunits = (segs + SMP_SEGS - 1) / SMP_SEGS;                 // warp units per pattern
  const int64_t units = (wunits + SMP_WARPS - 1) / SMP_WARPS;              // CTA units per pattern
  const int64_t total = units * P.group_k;
  int cur_k = -1;
  PatDev pd;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_ticket[0] = (int64_t)atomicAdd(&P.ticket[P.ticket_slot], 1ULL);
    __syncthreads();
    const int64_t t = s_ticket[0];
    if (t >= total) break;
    const int kg = (int)(t / units);
    const int k = P.plist ? P.plist[kg] : kg;  // family group -> batch index
    if (P.need && !P.need[k]) {  // covered by the batch pass: jump to the next pattern's units
      if (tid == 0) atomicMax(&P.ticket[P.ticket_slot], (unsigned long long)(kg + 1) * (unsigned long long)units);
      continue;
    }
    const int64_t u = t - (int64_t)kg * units;
    if (k != cur_k) {  // load this pattern's tables (uniform across the CTA)
      pd = P.pats[k];
      const int nb = (1 << pd.B) + 1;
      for (int i = tid; i < 2048; i += SMP_NT) bloom[i] = pd.bloom[i];
      for (int i = tid; i < nb; i += SMP_NT) bstart[i] = pd.bstart[i];
      for (int i = tid; i < pd.S; i += SMP_NT) bent[i] = pd.bent[i];
      for (int i = tid; i < pd.m; i += SMP_NT) spat[i] = pd.bytes[i];
      cur_k = k;
      __syncthreads();
    }
    const int64_t wu = u * SMP_WARPS + warp;
    if (wu >= wunits) continue;
    const int64_t seg0 = wu * SMP_SEGS;
    const int nsegs = (int)(segs - seg0 < SMP_SEGS ? segs - seg0 : SMP_SEGS);
    const int64_t ulo = seg0 * SEG, uhi = ulo + (int64_t)nsegs * SEG;  // bits of this unit
    const int64_t blo = P.off + pd.delta, bhi = P.off + pd.delta + P.n - pd.m;
    const int64_t S = pd.S;
    const int q = pd.q;
    const int64_t tlimit = P.off + P.n;  // virtual end of the text
    const int64_t i0 = ulo / S, i1 = (uhi - 1) / S;
    uint32_t* wl = lists + warp * SMP_LIST;
    uint32_t nmatch = 0, nver = 0;  // wl[0, nver) verified, wl[nver, nmatch) gram matches
    for (int64_t ib = i0; ib <= i1; ib += 32 * SMP_ILP) {
      uint4 g[SMP_ILP], g2[SMP_ILP];
#pragma unroll
      for (int r = 0; r < SMP_ILP; r++) {  // issue every load of the batch first
        const int64_t i = ib + r * 32 + lane;
        const int64_t x = S * i;
        if (i <= i1 && x + q <= tlimit) {
          MB_CHECK(x >= 0 && x + 16 * (q == 32 ? 2 : 1) <= P.nv16 && (x & 15) == 0);
          g[r] = __ldcs(reinterpret_cast<const uint4*>(P.text + x));
          if (q == 32) g2[r] = __ldcs(reinterpret_cast<const uint4*>(P.text + x + 16));
        }
      }
#pragma unroll
      for (int r = 0; r < SMP_ILP; r++) {
        const int64_t i = ib + r * 32 + lane;
        const int64_t x = S * i;
        uint32_t found[4];
        int nf = 0;
        if (i <= i1 && x + q <= tlimit) {
          const uint32_t w[8] = {g[r].x, g[r].y, g[r].z, g[r].w, g2[r].x, g2[r].y, g2[r].z, g2[r].w};
          nf = sampled_probe(P, pd, bloom, bstart, bent, spat, w, x, ulo, uhi, blo, bhi, found);
        }
        // ascending: lanes own disjoint increasing bit ranges; bucket entries are in ascending start order
        const uint32_t any = __ballot_sync(0xffffffffu, nf != 0);
        if (any) {
          if (nmatch + 4 * 32 > SMP_LIST) {  // room for this round's gram matches (<= 4 per lane)
            __syncwarp();
            nmatch = nver = sampled_verify(P, pd, spat, ulo, wl, nver, nmatch, lane);
          }
          uint32_t inc = nf;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
          }
          const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
          const uint32_t pos = nmatch + inc - nf;
          for (int f = 0; f < nf; f++)
            if (pos + f < SMP_LIST) wl[pos + f] = found[f];
          nmatch += tot;
        }
      }
    }
    __syncwarp();
    if (nmatch > nver) nmatch = sampled_verify(P, pd, spat, ulo, wl, nver, nmatch, lane);
    if (nmatch > SMP_LIST) __trap();  // impossible: verified before the list could overflow
    __syncwarp();
    // per-segment counts and uint16 tile-relative lists, as scan_kernel writes them
    for (int sl = lane; sl < nsegs; sl += 32) {
      const uint32_t lo = sl * SEG, hi = lo + SEG;
      uint32_t c = 0, first = 0;
      for (uint32_t e = 0; e < nmatch; e++) {
        const uint32_t v = wl[e];
        if (v < lo) first = e + 1;
        else if (v < hi) c++;
      }
      const int64_t g = (int64_t)k * segs + seg0 + sl;
      P.counts[g] = (uint16_t)c;
      const uint32_t tile_rel = (uint32_t)(((seg0 + sl) % NWARP) * SEG);  // segment start within its tile
      if (c <= LIST_CAP) {
        for (uint32_t e = 0; e < c; e++) P.lists[g * LIST_CAP + e] = (uint16_t)(wl[first + e] - lo + tile_rel);
      } else {
        uint32_t* bmw = P.bitmaps + g * SEG_WORDS;
        for (int q2 = 0; q2 < SEG_WORDS; q2++) bmw[q2] = 0;
        for (uint32_t e = 0; e < c; e++) {
          const uint32_t r = wl[first + e] - lo;
          bmw[r >> 5] |= 1u << (r & 31);
        }
      }
    }
  }
}


}  // namespace mb
