// kernel_output.cuh -- offsets_kernel (segment-count scan + fused sparse expansion) and expand_kernel (dense / MP segments)
// (part of libmatchb200; included by engine.cu)
#pragma once

namespace mb {

// ------------------------------------------------ kernel 2: segment offsets (scan)
// Exclusive scan of per-segment counts in OT * PER-count chunks, one per CTA.
// Co-resident grids (every realistic single search, 16 GiB included): each
// CTA publishes its chunk total, passes one grid barrier and sums its
// predecessors' totals.  Otherwise chunk order = ticket order taken at CTA
// start (no prefetch), so each chunk only waits on chunks already running --
// the decoupled look-back never stalls on a queued predecessor.
#ifndef MB_FUSE_MAX
#define MB_FUSE_MAX 16
#endif
constexpr int FUSE_MAX = MB_FUSE_MAX;  // sorted lists; unsorted ones at most 8 (the sort network's width)
static_assert(FUSE_MAX <= 16, "fused lists are read as two 16-byte vectors");

// 8-input sorting network (19 compare-exchanges)
__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}
__device__ __forceinline__ void sort8(uint32_t* v) {
  cswap(v[0], v[2]); cswap(v[1], v[3]); cswap(v[4], v[6]); cswap(v[5], v[7]);
  cswap(v[0], v[4]); cswap(v[1], v[5]); cswap(v[2], v[6]); cswap(v[3], v[7]);
  cswap(v[0], v[1]); cswap(v[2], v[3]); cswap(v[4], v[5]); cswap(v[6], v[7]);
  cswap(v[2], v[4]); cswap(v[3], v[5]);
  cswap(v[1], v[4]); cswap(v[3], v[6]);
  cswap(v[1], v[2]); cswap(v[3], v[4]); cswap(v[5], v[6]);
}

// PER counts per thread, OT threads per CTA: chunk = OT * PER (host picks the
// largest chunk that still gives >= 2 chunks per SM; 16 GiB texts take
// 256-thread CTAs x 64 counts so the 512 chunks stay co-resident at 4 CTAs/SM)
template <int PER, int OT>
__global__ void __launch_bounds__(OT, 1024 / OT) offsets_kernel(const ScanParams P) {
  constexpr int OW = OT / 32;  // warps of this CTA
  __shared__ int64_t wsum[OW];
  __shared__ uint32_t s_cnt[PER / 2 * OT];
  __shared__ int64_t s_excl;
  __shared__ int64_t s_chunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  MB_TRACE_MARK(2);
  pdl_trigger();  // expand_kernel's CTAs get resident now and wait for this grid in pdl_wait
  // chunk id: CTA index when the whole grid is co-resident (any order is
  // then safe), else a ticket in CTA start order.  Everything that does not
  // depend on the count kernel's results is set up before pdl_wait, while
  // its tail drains: chunk id, this thread's first pattern and its shift.
  if (tid == 0) s_chunk = P.offs_resident ? (int64_t)blockIdx.x : (int64_t)atomicAdd(&P.ticket[TICKET_OFFSETS], 1ULL);
  __syncthreads();
  const int64_t ch = s_chunk;
  const int64_t nseg = P.total_tiles * NWARP;
  const int64_t base = ch * (int64_t)(OT * PER);
  const int64_t seg_per_pat = P.ntiles * NWARP;
  // pattern of this thread's first segment and the segment's rank within it
  // (one division per thread; the CSR end is written at rank seg_per_pat - 1)
  int64_t kq = (base + (int64_t)tid * PER) / seg_per_pat;
  int64_t rem = base + (int64_t)tid * PER - kq * seg_per_pat;
  int cur_k = (int)kq;
  int64_t shift = kq < P.K ? P.pats[kq].delta + P.off : 0;
  // representatives (duplicate patterns read their representative's
  // segments): segment rank r of pattern k lives at rep[k] * seg_per_pat + r.
  // A thread's PER <= 32 segments span at most patterns kq and kq + 1
  // (seg_per_pat >= 16)
  int64_t rb0 = kq * seg_per_pat, rb1 = (kq + 1) * seg_per_pat;  // data bases of kq, kq + 1
  bool cp0 = false, cp1 = false;  // kq, kq + 1 filled by replicate_kernel
  if (P.rep) {
    if (kq < P.K) rb0 = (int64_t)(P.rep[kq] & ~REP_COPY) * seg_per_pat, cp0 = (P.rep[kq] & REP_COPY) != 0;
    if (kq + 1 < P.K) rb1 = (int64_t)(P.rep[kq + 1] & ~REP_COPY) * seg_per_pat, cp1 = (P.rep[kq + 1] & REP_COPY) != 0;
  }
  int64_t rbase = rb0;  // data base of cur_k
  bool rcopy = cp0;     // cur_k is filled by replicate_kernel
  if (P.csr0 && blockIdx.x == 0 && tid == 0) *P.csr0 = 0;
  pdl_wait();     // counts / lists / bitmaps of the count kernel(s)
  MB_TRACE_MARK(4);
  MB_TRACE_MARK(5);
  static_assert(PER % 8 == 0, "vector loads of 8 uint16 counts");
  // PER uint16 counts kept packed two per register (2 CTAs per SM fit)
  uint32_t v2[PER / 2];
  uint32_t tsum32 = 0;
  // data index of this thread's segment q (8-count groups never straddle a
  // pattern: seg_per_pat is a multiple of 16)
  auto dseg = [&](int q) -> int64_t {
    const int64_t r = rem + q;
    return r < seg_per_pat ? rb0 + r : rb1 + (r - seg_per_pat);
  };
  if (!P.rep) {
    // no duplicates: the chunk's counts are one contiguous run -- read it with
    // coalesced 16-byte loads (granule g = q8 * OT + tid; a thread reading its
    // own PER counts touches 32 lines per load, half of every sector unused:
    // 30 us per pass over config 3's 16.4 M counts) and hand every granule to
    // its owner thread through s_cnt, in the layout the counts keep below
    constexpr int GPT = PER / 8;  // granules per thread
    const uint4* c16 = reinterpret_cast<const uint4*>(P.counts + base);
#pragma unroll
    for (int q8 = 0; q8 < GPT; q8++) {
      const int g = q8 * OT + tid;
      const uint4 x = c16[g];  // (counts are allocated to a whole number of chunks)
      const int o = g / GPT, q = g % GPT;
      s_cnt[(4 * q + 0) * OT + o] = x.x;
      s_cnt[(4 * q + 1) * OT + o] = x.y;
      s_cnt[(4 * q + 2) * OT + o] = x.z;
      s_cnt[(4 * q + 3) * OT + o] = x.w;
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < PER / 2; h++) v2[h] = s_cnt[h * OT + tid];
    __syncthreads();  // the rows are rewritten (last chunk: zeroed tail) below
  } else {
#pragma unroll
    for (int q8 = 0; q8 < PER / 8; q8++) {
      // counts are allocated to a whole number of chunks; past the last pattern
      // the slots are read unmapped and zeroed below
      const int64_t t0 = base + (int64_t)tid * PER + 8 * q8;
      const uint4 x = *reinterpret_cast<const uint4*>(P.counts + (t0 < nseg ? dseg(8 * q8) : t0));
      v2[4 * q8] = x.x, v2[4 * q8 + 1] = x.y, v2[4 * q8 + 2] = x.z, v2[4 * q8 + 3] = x.w;
    }
  }
  if (base + (int64_t)OT * PER > nseg) {  // last chunk: zero the slots past the last segment
#pragma unroll
    for (int q = 0; q < PER; q++)
      if (base + (int64_t)tid * PER + q >= nseg) v2[q >> 1] &= (q & 1) ? 0x0000FFFFu : 0xFFFF0000u;
  }
  {
    // both 16-bit halves of every word summed at once, in 4 independent
    // accumulators (<= 16 counts of <= 2048 each: no carry between the halves)
    uint32_t a4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int h = 0; h < PER / 2; h++) a4[h & 3] += v2[h];
#pragma unroll
    for (int i = 0; i < 4; i++) tsum32 += (a4[i] & 0xFFFFu) + (a4[i] >> 16);
  }
  static_assert(PER / 2 / 4 * 2048 <= 65535, "packed count sums must not carry");
  const int64_t tsum = tsum32;
  // the first 8 list entries of this thread's first non-empty segment are
  // fetched now, so they arrive during the exclusive-offset computation
  // (threads without matches -- nearly all of a sparse batch -- skip the search)
  int fq = -1;
  if (tsum32) {
#pragma unroll
    for (int h = PER / 2 - 1; h >= 0; h--)
      if (v2[h]) fq = 2 * h + ((v2[h] & 0xFFFFu) ? 0 : 1);
  }
  uint4 pre = make_uint4(0, 0, 0, 0);
  if (fq >= 0 && P.out) pre = *reinterpret_cast<const uint4*>(P.lists + dseg(fq) * LIST_CAP);
  // the counts go through shared memory (transposed: conflict-free) so the
  // output loop below is not unrolled, and they stop occupying registers
  // across the prefix computation (the 64-count variant would spill); the
  // coalesced path has them there already (unless the last chunk zeroed a tail)
  if (P.rep || base + (int64_t)OT * PER > nseg) {
#pragma unroll
    for (int h = 0; h < PER / 2; h++) s_cnt[h * OT + tid] = v2[h];
  }
  int64_t inc = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int64_t chunk_total = 0, wbefore = 0;
  for (int q = 0; q < OW; q++) {
    chunk_total += wsum[q];
    wbefore += q < warp ? wsum[q] : 0;
  }
  __shared__ int s_first[OW];
  __shared__ unsigned long long s_part[OW];
  if (tid == 0) {
    st_relaxed(&P.state[ch], pack_state(P.epoch, ch == 0 ? ST_INCL : ST_AGG, (uint64_t)chunk_total));
    s_excl = 0;
  }
  MB_TRACE_MARK(24);
  MB_TRACE_MARK(25);
  int64_t j = ch - 1;  // newest predecessor of this window
  if (P.offs_resident) {
    // every chunk is resident: one grid barrier once all chunk totals are
    // published, then each CTA sums its predecessors' totals directly (no
    // polling of not-yet-published flags by every thread of every CTA)
    if (tid == 0) {
      __threadfence();
      atomicAdd(&P.ticket[TICKET_OFFBAR], 1ULL);
      while (ld_acquire(&P.ticket[TICKET_OFFBAR]) < (unsigned long long)gridDim.x) __nanosleep(32);
    }
    __syncthreads();
    unsigned long long v = 0;
    for (int64_t i = tid; i < ch; i += OT) v += ld_relaxed(&P.state[i]) & ((1ULL << 38) - 1);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    if (lane == 0) s_part[warp] = v;
    __syncthreads();
    if (tid == 0) {
      unsigned long long sum = 0;
#pragma unroll
      for (int w = 0; w < OW; w++) sum += s_part[w];
      s_excl = (int64_t)sum;
    }
    j = -1;
  }
  // otherwise block-wide decoupled look-back: the whole CTA reads OT
  // predecessors per round trip; the nearest inclusive predecessor and the sum
  // up to it are found with warp ballots / shuffles and one word per warp in
  // smem (no smem atomics)
  while (j >= 0) {     // uniform across the CTA (j, first read after barriers)
    const int64_t idx = j - tid;
    uint64_t sv = 0;
    bool incl = false;
    if (idx >= 0) {
      while (true) {
        sv = ld_relaxed(&P.state[idx]);
        if ((uint32_t)(sv >> 40) == P.epoch && ((sv >> 38) & 3)) break;
        __nanosleep(20);
      }
      incl = ((sv >> 38) & 3) == ST_INCL;
    }
    const uint32_t bi = __ballot_sync(0xffffffffu, incl);
    if (lane == 0) s_first[warp] = bi ? warp * 32 + __ffs(bi) - 1 : 0x7fffffff;
    __syncthreads();
    int first = 0x7fffffff;  // nearest predecessor holding an inclusive prefix
#pragma unroll
    for (int w = 0; w < OW; w++) first = min(first, s_first[w]);
    unsigned long long v = (idx >= 0 && tid <= first) ? (sv & ((1ULL << 38) - 1)) : 0ULL;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    if (lane == 0) s_part[warp] = v;
    __syncthreads();
    if (tid == 0) {
      unsigned long long sum = 0;
#pragma unroll
      for (int w = 0; w < OW; w++) sum += s_part[w];
      s_excl += (int64_t)sum;
    }
    if (first != 0x7fffffff || j - OT < 0) break;
    j -= OT;
    __syncthreads();  // s_first / s_part are rewritten next round
  }
  __syncthreads();
  MB_TRACE_MARK(7);
  if (tid == 0) {
    // look-back mode only: in barrier mode other CTAs may still be summing
    // this chunk's published total
    if (ch > 0 && !P.offs_resident) st_relaxed(&P.state[ch], pack_state(P.epoch, ST_INCL, (uint64_t)(s_excl + chunk_total)));
    s_excl += P.out_base ? *P.out_base : 0;
  }
  __syncthreads();
  int64_t run = s_excl + wbefore + inc - tsum;
  // Sorted sparse segments (<= LIST_CAP uint16 offsets) are expanded right here;
  // dense or unsorted (MP) segments are queued for expand_kernel with their offset.
  // lists of up to FUSE_MAX entries are expanded right here by their thread
  // (unsorted batch-pass lists sorted in registers by a 19-comparator
  // network); longer ones go to expand_kernel, whose warp per segment writes
  // them coalesced (a thread looping over 32 scattered stores is slower)
  const uint32_t fuse_max = !P.out ? 0u : P.unsorted_lists ? (uint32_t)min(FUSE_MAX, 8) : (uint32_t)FUSE_MAX;
  // expand-queue slots: a thread's queued segments take consecutive slots in
  // segment order and a warp's threads consecutive ranges (one atomic per
  // warp), so expand_kernel's neighbouring warps write neighbouring output
  // regions (a dense text queues every segment)
  unsigned long long qslot = 0;
  {
    uint32_t nqd = 0;
    if (P.out && tsum32 > fuse_max)  // (a thread whose counts sum to <= fuse_max queues nothing)
#pragma unroll 1
      for (int q = 0; q < PER; q++) {
        const uint32_t vq = (s_cnt[(q >> 1) * OT + tid] >> (16 * (q & 1))) & 0xFFFFu;
        const bool cp = rem + q < seg_per_pat ? cp0 : cp1;
        nqd += (base + (int64_t)tid * PER + q < nseg && vq > fuse_max && !cp) ? 1u : 0u;
      }
    if (__any_sync(0xffffffffu, nqd != 0)) {
      uint32_t qinc = nqd;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, qinc, d);
        if (lane >= d) qinc += v;
      }
      const uint32_t wtotal = __shfl_sync(0xffffffffu, qinc, 31);
      unsigned long long wbase = 0;
      if (lane == 0) wbase = atomicAdd(&P.ticket[P.dense_slot], (unsigned long long)wtotal);
      qslot = __shfl_sync(0xffffffffu, wbase, 0) + (qinc - nqd);
    }
  }
  // nothing to emit and no pattern ends in this thread's range: done
  const bool idle = tsum == 0 && rem + PER < seg_per_pat;
#pragma unroll 1
  for (int q = 0; q < (idle ? 0 : PER); q++) {
    const int64_t t = base + (int64_t)tid * PER + q;
    const uint32_t vq = (s_cnt[(q >> 1) * OT + tid] >> (16 * (q & 1))) & 0xFFFFu;
    if (t < nseg) {
      if (vq && P.out) {
        if (kq != cur_k) {  // (kq, rem) = (pattern, rank) of segment t
          shift = P.pats[kq].delta + P.off;
          cur_k = (int)kq;
          rbase = rb1;  // a thread's range reaches at most pattern kq + 1
          rcopy = cp1;
        }
        // a REP_COPY duplicate's positions are copied from its representative's
        // range afterwards (replicate_kernel): no list or queue work here
        if (!rcopy) {
          const int64_t ds = rbase + rem;  // data segment (the representative's for a duplicate)
          if (vq <= fuse_max) {
            const int64_t pos0 = (rem / NWARP) * TILE - shift;  // position of tile offset 0
            const uint16_t* L = P.lists + ds * LIST_CAP;
            if (!P.unsorted_lists) {
              // the list's (<= FUSE_MAX = 16) entries as two 16-byte loads
              // issued together (the first 8 prefetched for the first list)
              const uint4* L4 = reinterpret_cast<const uint4*>(L);  // 64-byte aligned list
              const uint4 la = q == fq ? pre : L4[0];
              const uint4 lb = vq > 8 ? L4[1] : make_uint4(0, 0, 0, 0);
              for (uint32_t e = 0; e < vq; e++) {
                const uint4 lq = e < 8 ? la : lb;
                const uint32_t i = e & 7;
                const uint32_t w = (i >> 1) == 0 ? lq.x : (i >> 1) == 1 ? lq.y : (i >> 1) == 2 ? lq.z : lq.w;
                if (run + e < P.cap) P.out[run + e] = pos0 + ((w >> (16 * (i & 1))) & 0xFFFFu);
              }
            } else {
              const uint4 raw = q == fq ? pre : *reinterpret_cast<const uint4*>(L);  // 8 slots (64-byte aligned list)
              uint32_t v[8] = {raw.x & 0xFFFFu, raw.x >> 16, raw.y & 0xFFFFu, raw.y >> 16,
                               raw.z & 0xFFFFu, raw.z >> 16, raw.w & 0xFFFFu, raw.w >> 16};
  #pragma unroll
              for (int e = 0; e < 8; e++)
                if ((uint32_t)e >= vq) v[e] = 0xFFFFFFFFu;
              sort8(v);
  #pragma unroll
              for (int e = 0; e < 8; e++)
                if ((uint32_t)e < vq && run + e < P.cap) P.out[run + e] = pos0 + v[e];
            }
          } else {
            // queue entry: segment | count << 48, output offset, position of bit 0
            const unsigned long long slot = qslot++;
            P.seglist[slot] = ds | ((int64_t)vq << 48);
            P.toff[slot] = run;
            P.qpos[slot] = rem * SEG - shift;
          }
        }
      }
      if (rem == seg_per_pat - 1) P.offsets_plus1[kq] = run + vq;
    }
    run += vq;
    if (++rem == seg_per_pat) rem = 0, kq++;
  }
  MB_TRACE_SYNC_MARK(9);
  // ticket reset for the next search: expand_kernel does it when it follows
  if (!P.out || P.cap <= 0) reset_tickets_if_last(P.ticket, NTICKETS, TICKET_DONE, -1);
}

// ------------------------------------------------ kernel 3: expansion
// The segments offsets_kernel queued (dense, or MP's unsorted lists), a warp
// per queue entry, software-pipelined: the entry two steps ahead and the list
// / bitmap words one step ahead are in flight while the current segment is
// written.  An entry carries everything but the match bits (segment | count,
// output offset, position of bit 0), so no pattern lookup or division sits on
// the path.  Unsorted (MP) lists get a 32-lane bitonic sort.  Dense segments
// (bitmaps; each lane holds 64 consecutive bits) are written in 256-byte rows
// ALIGNED to the output's 256-byte lines (first and last row partial), from
//  * a table of its runs of ones when there are at most EXP_RUNS of them,
//    32 matches long on average (c^m over a text of mostly c): position =
//    row index + a per-run offset;
//  * else a per-warp smem run of uint16 offsets, the set bits extracted one
//    by one (brev + clz, a running pointer; >= 50% set: a predicated pass).
// tools/probe_expand_pattern.cu (B200): rows starting at the segment's own
// offset straddle two lines each and write at 4.0-4.6 TB/s (16 KB regions, a
// warp each); line-aligned rows at 5.5-6.0.
#ifndef MB_EXP_WARPS
#define MB_EXP_WARPS 8
#endif
constexpr int EXP_WARPS = MB_EXP_WARPS;
constexpr int EXP_RUNS = 32;  // run table entries per warp (one per lane)

struct ExpSeg {  // one queued segment as a lane holds it
  int64_t g, o, sp;
  uint32_t c, lv, xa, xb;
};
__device__ __forceinline__ void exp_head(const ScanParams& P, int64_t qi, int64_t* ent, int64_t* o, int64_t* sp) {
  *ent = P.seglist[qi];
  *o = P.toff[qi];
  *sp = P.qpos[qi];
}
__device__ __forceinline__ ExpSeg exp_load(const ScanParams& P, int64_t ent, int64_t o, int64_t sp, int lane) {
  ExpSeg e;
  e.g = ent & ((1LL << 48) - 1);
  e.c = (uint32_t)(ent >> 48);
  e.o = o;
  e.sp = sp;
  e.lv = e.xa = e.xb = 0;
  if (e.c <= LIST_CAP) {
    e.lv = P.lists[e.g * LIST_CAP + lane];
  } else {  // bits [64 lane, 64 lane + 64) of the segment
    const uint2 x = reinterpret_cast<const uint2*>(P.bitmaps + e.g * SEG_WORDS)[lane];
    e.xa = x.x, e.xb = x.y;
  }
  return e;
}

// out[i] = sp + v: the 64-bit add done once per segment when the low word cannot carry
__device__ __forceinline__ void exp_store(int64_t* d, int64_t sp, uint32_t v, bool nocarry) {
  if (nocarry) {
    const uint2 r = make_uint2((uint32_t)sp + v, (uint32_t)((uint64_t)sp >> 32));
    *reinterpret_cast<uint2*>(d) = r;
  } else {
    *d = sp + v;
  }
}

__global__ void __launch_bounds__(EXP_WARPS * 32) expand_kernel(const ScanParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint16_t s_run[EXP_WARPS][SEG];  // dense segments: staged offsets per warp
  __shared__ uint32_t s_tab[EXP_WARPS][2 * EXP_RUNS + 2];  // run table: first position, output rank
  uint16_t* const sb = s_run[warp];
  uint32_t* const tab_s = s_tab[warp];
  uint32_t* const tab_o = s_tab[warp] + EXP_RUNS + 1;
  MB_TRACE_MARK(10);
  pdl_wait();  // queue and offsets of offsets_kernel
  MB_TRACE_MARK(12);
  // the count and offsets grids are complete: zero every ticket but this
  // search's queue count (read below; the next search, of the other epoch
  // parity, zeroes it), so the next search needs no memset
  if (blockIdx.x == 0 && threadIdx.x < NTICKETS && threadIdx.x != P.dense_slot) P.ticket[threadIdx.x] = 0ULL;
  const int64_t nq = (int64_t)P.ticket[P.dense_slot];
  const int64_t stride = (int64_t)gridDim.x * EXP_WARPS;
  // element misalignment of the output against its 256-byte lines
  const uint32_t omis = (uint32_t)(((uintptr_t)P.out >> 3) & 31u);
  int64_t qi = (int64_t)blockIdx.x * EXP_WARPS + warp;
  ExpSeg cur;
  int64_t h_ent = 0, h_o = 0, h_sp = 0;  // entry qi + stride
  bool have_nxt = false;
  if (qi < nq) {
    int64_t ent, o, sp;
    exp_head(P, qi, &ent, &o, &sp);
    cur = exp_load(P, ent, o, sp, lane);
    if (qi + stride < nq) exp_head(P, qi + stride, &h_ent, &h_o, &h_sp), have_nxt = true;
  }
  while (qi < nq) {
    ExpSeg nxt;
    int64_t n_ent = 0, n_o = 0, n_sp = 0;
    bool have_nn = false;
    if (have_nxt) {  // prefetch: issued before the current segment's work
      nxt = exp_load(P, h_ent, h_o, h_sp, lane);
      if (qi + 2 * stride < nq) exp_head(P, qi + 2 * stride, &n_ent, &n_o, &n_sp), have_nn = true;
    }
    const uint32_t c = cur.c;
    const int64_t o = cur.o;
    if (o < P.cap) {
      if (c <= LIST_CAP) {
        // lists hold tile-relative offsets: position = tile origin + entry
        const int64_t pos0 = cur.sp - (cur.g & (NWARP - 1)) * SEG;
        uint32_t v = lane < (int)c ? (cur.lv & 0xFFFFu) : 0xFFFFFFFFu;
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
      } else {
        // dense: the lane's 64 bits, exclusive prefix e of the ones before them
        const uint32_t xa = cur.xa, xb = cur.xb;
        const uint32_t pc = __popc(xa) + __popc(xb);
        // starts of runs of ones (bit b set, bit b - 1 clear; the previous lane's top bit carries in)
        const bool try_runs = c >= 32u * 16u;  // (a run table pays from 32 matches per run: not below 512)
        uint32_t sa = 0, sb2 = 0;
        if (try_runs) {
          const uint32_t prev_top = __shfl_up_sync(0xffffffffu, xb, 1) >> 31;
          sa = xa & ~((xa << 1) | (lane ? prev_top : 0u));
          sb2 = xb & ~((xb << 1) | (xa >> 31));
        }
        const uint32_t nr = __popc(sa) + __popc(sb2);
        uint32_t inc = pc | (nr << 16);  // both prefixes in one scan (sum pc <= 2048, sum nr <= 1024)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += v;
        }
        const uint32_t R = __shfl_sync(0xffffffffu, inc, 31) >> 16;
        const uint32_t e = (inc & 0xFFFFu) - pc;
        const uint32_t lim = (uint32_t)(P.cap - o < (int64_t)c ? P.cap - o : (int64_t)c);
        const int64_t sp = cur.sp;
        const bool nocarry = (uint32_t)sp <= 0xFFFF0000u;
        int64_t* const d0 = P.out + o;
        // rows on 256-byte lines: element i of the segment sits at line offset
        // (o + omis + i) & 31; aligned index j = i + head
        const uint32_t head = (uint32_t)((o + omis) & 31);
        const uint32_t iend = head + lim;
        if (try_runs && R <= (uint32_t)EXP_RUNS && c >= 32u * R) {  // few LONG runs (a row per run at least): c^m with short m
                                                          // over random text has dozens of 1-2 match runs -- staged below
          // ---- run-structured (c^m over a text of mostly c, config 5): a table of
          // (first position, output rank) per run; a row inside one run is
          // position = i + one warp-uniform offset -- no staging of positions
          uint32_t ri = (inc >> 16) - nr;
          uint32_t x = sa;
          while (x) {
            const uint32_t bq = __ffs(x) - 1;
            x &= x - 1;
            tab_s[ri] = 64u * lane + bq;
            tab_o[ri] = e + __popc(xa & ((1u << bq) - 1u));
            ri++;
          }
          x = sb2;
          while (x) {
            const uint32_t bq = __ffs(x) - 1;
            x &= x - 1;
            tab_s[ri] = 64u * lane + 32u + bq;
            tab_o[ri] = e + __popc(xa) + __popc(xb & ((1u << bq) - 1u));
            ri++;
          }
          if (lane == 0) tab_o[R] = 0xFFFFFFFFu;  // sentinel: no run starts at or after rank c
          __syncwarp();
          // run by run (warp-uniform bounds): the rows of run r cover the aligned
          // indices [O_r + head, O_{r+1} + head); a row shared by two runs is
          // written by both, each its own lanes
          // (the low-word add and the row pointer are strength-reduced by hand: 3-4
          // instructions per 256-byte row, so a few warps per SM keep the stores flowing)
          const uint32_t splo = (uint32_t)sp, sphi = (uint32_t)((uint64_t)sp >> 32);
          for (uint32_t r = 0; r < R; r++) {
            const uint32_t O = tab_o[r];
            if (O >= lim) break;
            const uint32_t On = min(tab_o[r + 1], lim);
            const uint32_t dl = tab_s[r] - O;  // position - rank inside this run
            const uint32_t jlo = O + head, jhi = On + head;
            uint32_t j = (jlo & ~31u) + lane;
            if (nocarry) {
              uint2* p = reinterpret_cast<uint2*>(d0 + ((int64_t)j - (int64_t)head));
              uint32_t v = splo + (j - head + dl);
              if (j >= jlo && j < jhi) *p = make_uint2(v, sphi);
              j += 32, p += 32, v += 32;
#pragma unroll 1
              for (; j + 96 < jhi; j += 128, p += 128, v += 128) {
                p[0] = make_uint2(v, sphi);
                p[32] = make_uint2(v + 32, sphi);
                p[64] = make_uint2(v + 64, sphi);
                p[96] = make_uint2(v + 96, sphi);
              }
              for (; j < jhi; j += 32, p += 32, v += 32) *p = make_uint2(v, sphi);
            } else {
              if (j >= jlo && j < jhi) d0[j - head] = sp + (j - head + dl);
              for (j += 32; j < jhi; j += 32) d0[j - head] = sp + (j - head + dl);
            }
          }
        } else {
          // ---- general: set bits -> uint16 offsets in the warp's smem run
          uint16_t* w = sb + e;
          const uint32_t ba = 64u * lane;
          if (c >= SEG / 2) {  // >= 50% set: every bit position once, predicated
#pragma unroll
            for (int bq = 0; bq < 32; bq++)
              if ((xa >> bq) & 1u) *w++ = (uint16_t)(ba + bq);
#pragma unroll
            for (int bq = 0; bq < 32; bq++)
              if ((xb >> bq) & 1u) *w++ = (uint16_t)(ba + 32u + bq);
          } else {
            uint32_t y = __brev(xa);
            while (y) {
              const uint32_t bq = __clz(y);
              y ^= 0x80000000u >> bq;
              *w++ = (uint16_t)(ba + bq);
            }
            y = __brev(xb);
            while (y) {
              const uint32_t bq = __clz(y);
              y ^= 0x80000000u >> bq;
              *w++ = (uint16_t)(ba + 32u + bq);
            }
          }
          __syncwarp();
          if (nocarry) {  // (decided once per segment; pointers advanced by hand)
            const uint32_t splo = (uint32_t)sp, sphi = (uint32_t)((uint64_t)sp >> 32);
            uint32_t j = lane;
            if (j >= head && j < iend) *reinterpret_cast<uint2*>(d0 + (j - head)) = make_uint2(splo + sb[j - head], sphi);
            j += 32;
            uint2* p = reinterpret_cast<uint2*>(d0 + ((int64_t)j - (int64_t)head));
            const uint16_t* q = sb + ((int32_t)j - (int32_t)head);
#pragma unroll 4
            for (; j < iend; j += 32, p += 32, q += 32) *p = make_uint2(splo + *q, sphi);
          } else {
            for (uint32_t j = lane; j < iend; j += 32) {
              const uint32_t i = j - head;  // wraps below 0 for the first row's leading lanes
              if (i < lim) d0[i] = sp + sb[i];
            }
          }
        }
        __syncwarp();  // the next segment overwrites sb / the run table
      }
    }
    if (!have_nxt) break;
    qi += stride;
    cur = nxt;
    have_nxt = have_nn;
    h_ent = n_ent, h_o = n_o, h_sp = n_sp;
  }
  MB_TRACE_SYNC_MARK(13);
}


// ------------------------------------------------ kernel 4: duplicate patterns
// A batch pattern identical to an earlier one (its representative) gets the
// representative's positions copied into its own CSR range, once expand_kernel
// has written them.  Batches of up to REPL_MAXK patterns: every CTA ranks the
// duplicates and prefixes their (capacity-capped) sizes in smem, then the
// warps copy 256-position chunks of the concatenated duplicate ranges
// grid-stride, so the whole grid writes one advancing window (a grid-stride
// write stream; CTA-per-duplicate regions wrote at ~2.5-4.7 TB/s).  Larger
// batches: a CTA per duplicate.  8-byte copies (source and destination
// parities may differ); sources are usually L2-resident.
constexpr int REPL_MAXK = 2048;
__global__ void __launch_bounds__(512) replicate_kernel(const ScanParams P) {
  __shared__ int64_t s_pref[REPL_MAXK + 1];  // exclusive prefix of duplicate sizes, by duplicate rank
  __shared__ int32_t s_dup[REPL_MAXK];       // pattern index of each duplicate rank
  __shared__ int64_t s_wsum[16];
  __shared__ int s_wcnt[16];
  pdl_wait();  // the representatives' positions (expand_kernel)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base0 = P.out_base ? *P.out_base : 0;
  auto start = [&](int k) -> int64_t { return k ? P.offsets_plus1[k - 1] : base0; };
  if (P.K > REPL_MAXK) {
    for (int k = blockIdx.x; k < P.K; k += gridDim.x) {
      if (!(P.rep[k] & REP_COPY)) continue;
      const int r = P.rep[k] & ~REP_COPY;
      const int64_t d0 = start(k), lim = min(P.offsets_plus1[k], P.cap) - d0;
      const int64_t* src = P.out + start(r);
      int64_t* dst = P.out + d0;
      for (int64_t i = tid; i < lim; i += 512) dst[i] = src[i];
    }
    return;
  }
  // 1. rank the duplicates (4 patterns per thread) and prefix their sizes
  int64_t sz[4];
  int nd_t = 0;
  int64_t sum_t = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int k = 4 * tid + q;
    sz[q] = -1;
    if (k < P.K && (P.rep[k] & REP_COPY)) {
      const int64_t d0 = start(k);
      sz[q] = max(min(P.offsets_plus1[k], P.cap) - d0, (int64_t)0);
      nd_t++;
      sum_t += sz[q];
    }
  }
  int nd_inc = nd_t;
  int64_t sum_inc = sum_t;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int on = __shfl_up_sync(0xffffffffu, nd_inc, d);
    const int64_t os = __shfl_up_sync(0xffffffffu, sum_inc, d);
    if (lane >= d) nd_inc += on, sum_inc += os;
  }
  if (lane == 31) s_wcnt[warp] = nd_inc, s_wsum[warp] = sum_inc;
  __syncthreads();
  int nd_before = 0, nd_all = 0;
  int64_t sum_before = 0, sum_all = 0;
  for (int w = 0; w < 16; w++) {
    nd_all += s_wcnt[w], sum_all += s_wsum[w];
    if (w < warp) nd_before += s_wcnt[w], sum_before += s_wsum[w];
  }
  int rank = nd_before + nd_inc - nd_t;
  int64_t pref = sum_before + sum_inc - sum_t;
#pragma unroll
  for (int q = 0; q < 4; q++)
    if (sz[q] >= 0) s_pref[rank] = pref, s_dup[rank] = 4 * tid + q, pref += sz[q], rank++;
  if (tid == 0) s_pref[nd_all] = sum_all;
  __syncthreads();
  // 2. 1024-position chunks of the concatenated ranges, grid-stride by warp
  // (one smem search per chunk), copied in pieces of 8 rows of 32 positions
  // aligned to the destination's 256-byte lines
  const uint32_t omis = (uint32_t)(((uintptr_t)P.out >> 3) & 31u);
  const int64_t nchunks = (sum_all + 1023) / 1024;
  for (int64_t c = (int64_t)blockIdx.x * 16 + warp; c < nchunks; c += (int64_t)gridDim.x * 16) {
    int64_t e = c * 1024;
    const int64_t e_end = min(e + 1024, sum_all);
    int lo = 0, hi = nd_all - 1;  // last duplicate whose range starts at or before e
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pref[mid] <= e) lo = mid; else hi = mid - 1;
    }
    for (int d = lo; e < e_end; d++) {
      const int k = s_dup[d];
      const int r = P.rep[k] & ~REP_COPY;
      const int64_t run_end = min(e_end, s_pref[d + 1]);
      const int64_t doff = start(k) - s_pref[d];  // destination index of concatenated index 0 of this run
      const int64_t* src = P.out + start(r) - s_pref[d];
      int64_t* dst = P.out + doff;
      while (e < run_end) {
        // rows start on a destination line: back up to it, mask the lanes before e
        const int64_t e0 = e - (int64_t)((uint32_t)(e + doff + omis) & 31u);
        const int64_t piece_end = min(run_end, e0 + 256);
        // all of a lane's loads first (src and dst share P.out, so the compiler
        // would otherwise keep each load behind the previous store)
        int64_t v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int64_t i = e0 + lane + 32 * j;
          if (i >= e && i < piece_end) v[j] = src[i];
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int64_t i = e0 + lane + 32 * j;
          if (i >= e && i < piece_end) __stcs(dst + i, v[j]);
        }
        e = piece_end;
      }
    }
  }
}

}  // namespace mb
