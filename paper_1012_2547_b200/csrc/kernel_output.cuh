// kernel_output.cuh -- offsets_kernel (segment-count scan + fused sparse expansion) and expand_kernel (dense / MP segments)
// (part of libmatchb200; included by engine.cu)
#pragma once

namespace mb {

// ------------------------------------------------ kernel 2: segment offsets (scan)
// Exclusive scan of per-segment counts in SCAN_CHUNK pieces; chunk order =
// ticket order taken at CTA start (no prefetch), so each chunk only waits on
// chunks already running -- the decoupled look-back never stalls on a queued
// predecessor.
template <int PER>  // counts per thread: chunk = NT * PER (host picks PER for >= 2 chunks per SM)
__global__ void __launch_bounds__(NT, 2) offsets_kernel(const ScanParams P) {
  __shared__ int64_t wsum[NWARP];
  __shared__ uint32_t s_cnt[PER / 2 * NT];
  __shared__ int64_t s_excl;
  __shared__ int64_t s_chunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();  // counts / lists / bitmaps of the count kernel(s)
  if (tid == 0) s_chunk = (int64_t)atomicAdd(&P.ticket[TICKET_OFFSETS], 1ULL);
  __syncthreads();
  const int64_t ch = s_chunk;
  const int64_t nseg = P.total_tiles * NWARP;
  const int64_t base = ch * (int64_t)(NT * PER);
  static_assert(PER % 8 == 0, "vector loads of 8 uint16 counts");
  // PER uint16 counts kept packed two per register (2 CTAs per SM fit)
  uint32_t v2[PER / 2];
  uint32_t tsum32 = 0;
  const uint4* cv = reinterpret_cast<const uint4*>(P.counts + base + (int64_t)tid * PER);
#pragma unroll
  for (int q8 = 0; q8 < PER / 8; q8++) {
    const uint4 x = cv[q8];  // counts are allocated to a whole number of chunks
    v2[4 * q8] = x.x, v2[4 * q8 + 1] = x.y, v2[4 * q8 + 2] = x.z, v2[4 * q8 + 3] = x.w;
  }
  if (base + (int64_t)NT * PER > nseg) {  // last chunk: zero the slots past the last segment
#pragma unroll
    for (int q = 0; q < PER; q++)
      if (base + (int64_t)tid * PER + q >= nseg) v2[q >> 1] &= (q & 1) ? 0x0000FFFFu : 0xFFFF0000u;
  }
#pragma unroll
  for (int h = 0; h < PER / 2; h++) tsum32 += (v2[h] & 0xFFFFu) + (v2[h] >> 16);
  const int64_t tsum = tsum32;
  int64_t inc = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int64_t chunk_total = 0, wbefore = 0;
  for (int q = 0; q < NWARP; q++) {
    chunk_total += wsum[q];
    wbefore += q < warp ? wsum[q] : 0;
  }
  // block-wide decoupled look-back: the whole CTA reads NT predecessors per
  // round trip (a 16 GiB single-pattern search has 512 chunks: one round trip)
  __shared__ int s_incl_min;
  __shared__ unsigned long long s_sum;
  if (tid == 0) {
    st_relaxed(&P.state[ch], pack_state(P.epoch, ch == 0 ? ST_INCL : ST_AGG, (uint64_t)chunk_total));
    s_excl = 0;
  }
  int64_t j = ch - 1;  // newest predecessor of this window
  while (j >= 0) {     // uniform across the CTA (j, s_incl_min read after barriers)
    if (tid == 0) {
      s_incl_min = 0x7fffffff;
      s_sum = 0;
    }
    __syncthreads();
    const int64_t idx = j - tid;
    uint64_t sv = 0;
    if (idx >= 0) {
      while (true) {
        sv = ld_relaxed(&P.state[idx]);
        if ((uint32_t)(sv >> 40) == P.epoch && ((sv >> 38) & 3)) break;
        __nanosleep(20);
      }
      if (((sv >> 38) & 3) == ST_INCL) atomicMin(&s_incl_min, tid);
    }
    __syncthreads();
    const int first = s_incl_min;  // nearest predecessor holding an inclusive prefix
    if (idx >= 0 && tid <= first) atomicAdd(&s_sum, (unsigned long long)(sv & ((1ULL << 38) - 1)));
    __syncthreads();
    if (tid == 0) s_excl += (int64_t)s_sum;
    if (first != 0x7fffffff || j - NT < 0) break;
    j -= NT;
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    if (ch > 0) st_relaxed(&P.state[ch], pack_state(P.epoch, ST_INCL, (uint64_t)(s_excl + chunk_total)));
    s_excl += P.out_base ? *P.out_base : 0;
  }
  __syncthreads();
  int64_t run = s_excl + wbefore + inc - tsum;
  const int64_t seg_per_pat = P.ntiles * NWARP;
  // Sorted sparse segments (<= LIST_CAP uint16 offsets) are expanded right here;
  // dense or unsorted (MP) segments are queued for expand_kernel with their offset.
  const bool fuse = P.out && !P.unsorted_lists;
  int cur_k = -1;
  int64_t shift = 0;
  // pattern of this thread's first segment and the segment's rank within it
  // (one division per thread; the CSR end is written at rank seg_per_pat - 1)
  int64_t kq = (base + (int64_t)tid * PER) / seg_per_pat;
  int64_t rem = base + (int64_t)tid * PER - kq * seg_per_pat;
  // the counts go through shared memory (transposed: conflict-free) so the
  // output loop below is not unrolled and the kernel stays at 2 CTAs per SM
#pragma unroll
  for (int h = 0; h < PER / 2; h++) s_cnt[h * NT + tid] = v2[h];
  // nothing to emit and no pattern ends in this thread's range: done
  if (tsum == 0 && rem + PER < seg_per_pat) return;
#pragma unroll 1
  for (int q = 0; q < PER; q++) {
    const int64_t t = base + (int64_t)tid * PER + q;
    const uint32_t vq = (s_cnt[(q >> 1) * NT + tid] >> (16 * (q & 1))) & 0xFFFFu;
    if (t < nseg) {
      if (vq && P.out) {
        if (fuse && vq <= (uint32_t)LIST_CAP) {
          const int64_t tile = t / NWARP;
          const int k = (int)(tile / P.ntiles);
          if (k != cur_k) {
            shift = P.pats[k].delta + P.off;
            cur_k = k;
          }
          const int64_t pos0 = (tile % P.ntiles) * TILE - shift;
          const uint16_t* L = P.lists + t * LIST_CAP;
          for (uint32_t e = 0; e < vq; e++)
            if (run + e < P.cap) P.out[run + e] = pos0 + L[e];
        } else {
          P.toff[t] = run;
          const unsigned long long slot = atomicAdd(&P.ticket[TICKET_DENSE], 1ULL);
          P.seglist[slot] = t;
        }
      }
      if (rem == seg_per_pat - 1) P.offsets_plus1[kq] = run + vq;
    }
    run += vq;
    if (++rem == seg_per_pat) rem = 0, kq++;
  }
}

// ------------------------------------------------ kernel 3: expansion
// The segments offsets_kernel queued (dense, or MP's unsorted lists), a warp
// per segment: unsorted lists get a 32-lane bitonic sort, dense segments
// expand their 64-word bitmap 32 words at a time through a per-warp smem
// staging buffer so every global store is a coalesced run.
constexpr int EXP_WARPS = 4;
__global__ void __launch_bounds__(EXP_WARPS * 32) expand_kernel(const ScanParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();  // queue and offsets of offsets_kernel
  const int64_t nq = (int64_t)P.ticket[TICKET_DENSE];
  int cur_k = -1;
  int64_t shift = 0;
  for (int64_t qi = (int64_t)blockIdx.x * EXP_WARPS + warp; qi < nq; qi += (int64_t)gridDim.x * EXP_WARPS) {
    {
      const int64_t g = P.seglist[qi];
      const uint32_t c = P.counts[g];
      const int64_t tile = g / NWARP;
      const int k = (int)(tile / P.ntiles);
      if (k != cur_k) {
        shift = P.pats[k].delta + P.off;
        cur_k = k;
      }
      const int64_t pos0 = (tile % P.ntiles) * TILE - shift;  // tile-relative offsets below
      const int64_t o = P.toff[g];
      if (o >= P.cap) continue;
      if (c <= LIST_CAP) {
        uint32_t v = lane < (int)c ? (uint32_t)P.lists[g * LIST_CAP + lane] : 0xFFFFFFFFu;
        if (P.unsorted_lists) {  // MP fills list slots atomically: warp bitonic sort of <= 32 offsets
#pragma unroll
          for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
              const uint32_t o2 = __shfl_xor_sync(0xffffffffu, v, jj);
              const bool up = ((lane & kk) == 0);
              const bool lower = ((lane & jj) == 0);
              v = (lower == up) ? min(v, o2) : max(v, o2);
            }
        }
        if (lane < (int)c && o + lane < P.cap) P.out[o + lane] = pos0 + v;
        continue;
      }
      // dense: the 64 bitmap words (2 per lane), exclusive popcount prefix, then
      // one word per step broadcast to the warp -- lane i writes bit i's
      // position at its rank, so a full word is one coalesced 256-byte store
      const uint32_t* bmw = P.bitmaps + g * SEG_WORDS;
      const int64_t segpos = pos0 + (g % NWARP) * SEG;
      const uint32_t xa = bmw[lane], xb = bmw[32 + lane];
      const uint32_t pa = __popc(xa), pb = __popc(xb);
      uint32_t ia = pa, ib = pb;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t va = __shfl_up_sync(0xffffffffu, ia, d);
        const uint32_t vb = __shfl_up_sync(0xffffffffu, ib, d);
        if (lane >= d) ia += va, ib += vb;
      }
      const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31);
      const uint32_t ea = ia - pa, eb = ta + ib - pb;
      const uint32_t below = (1u << lane) - 1u;
      // 32-bit ranks against the room left in the output (o < cap checked above)
      const uint32_t lim = (uint32_t)(P.cap - o < (int64_t)SEG ? P.cap - o : (int64_t)SEG);
      int64_t* const dst = P.out + o;
      const int64_t v0 = segpos + lane;
#pragma unroll 8
      for (int w = 0; w < 32; w++) {
        const uint32_t x = __shfl_sync(0xffffffffu, xa, w);
        const uint32_t r = __shfl_sync(0xffffffffu, ea, w) + __popc(x & below);
        st_if((((x >> lane) & 1u) != 0) & (r < lim), dst + r, v0 + 32 * w);
      }
#pragma unroll 8
      for (int w = 0; w < 32; w++) {
        const uint32_t x = __shfl_sync(0xffffffffu, xb, w);
        const uint32_t r = __shfl_sync(0xffffffffu, eb, w) + __popc(x & below);
        st_if((((x >> lane) & 1u) != 0) & (r < lim), dst + r, v0 + 32 * (32 + w));
      }
    }
  }
}


}  // namespace mb
