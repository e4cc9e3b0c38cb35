// kernel_mp.cuh -- mp_scan_kernel: K5 batched multi-pattern single pass; hist_kernel: K0 byte histogram
// (part of libmatchb200; included by engine.cu)
#pragma once

namespace mb {

// ------------------------------------------------ kernel 1c: batched multi-pattern pass (K5 "MP")
// One TMA pass over the text serves a whole batch: each 4-aligned text word X
// is hashed once; a bloom bit test in smem rejects almost every word, and a
// hit walks the bucket of {gram, pattern, mpa+j} entries (every plan with
// m >= 7 carries one-word anchor grams mpG for this pass, whatever its own
// family).  A verified occurrence (k, s) is recorded at pattern k's own bitmap
// bit b = s + off + delta_k -- the bit its family's scan would set -- in the
// segment holding b (usually this warp's; a far delta puts it in another
// segment or tile): one 16-bit atomic count and an (unordered) list slot;
// offsets/expand are shared (expand sorts MP lists).  Segments above LIST_CAP
// set `overflow` and the per-pattern scans re-run the batch on the device.
// A verified occurrence of batch pattern k whose family scan would set bit b
// (virtual start + delta): one 16-bit atomic count and an unordered list slot
// in the segment holding b (segment layout of ScanParams); overflow past
// LIST_CAP hands the pattern to its per-pattern scan (need[k], any-flag).
__device__ __forceinline__ void mp_record(const MPParams& P, int k, int64_t b) {
  const int64_t tb = b / TILE;
  MB_CHECK(b >= 0 && tb < P.ntiles);
  const int64_t g = ((int64_t)k * P.ntiles + tb) * NWARP + (b - tb * TILE) / SEG;
  unsigned int* wptr = reinterpret_cast<unsigned int*>(P.counts) + (g >> 1);
  const unsigned int sh = 16u * (unsigned)(g & 1);
  const unsigned int old = (atomicAdd(wptr, 1u << sh) >> sh) & 0xFFFFu;
  if (old < (unsigned)LIST_CAP) {
    P.lists[g * LIST_CAP + old] = (uint16_t)(b - tb * TILE);
  } else {  // this pattern falls back to its own family scan
    P.need[k] = 1u;
    atomicExch(P.overflow, 1u);
  }
}

// Batched-pass verification of a gram hit: candidate start sv of batch-chunk
// pattern kl against the staged tile.  The first min(m, 16) bytes are compared
// word-wise by the lane; a short pattern is recorded right away, a longer
// survivor is queued (up to 4 per lane and round, else verified word-wise by
// the lane) for mp_verify_queued, where the whole warp compares it.
struct MPCand {
  int n;
  int64_t sv[4];
  int kl[4];
};
__device__ __forceinline__ bool mp_head_ok(const uint8_t* tp, const uint8_t* pp, int64_t m) {
  const int hb = m < 16 ? (int)m : 16;
  int k = 0;
  for (; k + 4 <= hb; k += 4)
    if (lds32u(tp + k) != __ldg(reinterpret_cast<const uint32_t*>(pp + k))) return false;
  if (k < hb) {
    const uint32_t mask = (1u << (8 * (hb - k))) - 1u;
    if ((lds32u(tp + k) ^ __ldg(reinterpret_cast<const uint32_t*>(pp + k))) & mask) return false;
  }
  return true;
}
__device__ __forceinline__ bool mp_tail_ok(const uint8_t* tp, const uint8_t* pp, int64_t m, int k0, int step) {
  bool bad = false;
  for (int64_t k = k0; k < m; k += step) {
    uint32_t diff = lds32u(tp + k) ^ __ldg(reinterpret_cast<const uint32_t*>(pp + k));
    if (m - k < 4) diff &= (1u << (8 * (m - k))) - 1u;
    bad |= diff != 0;
  }
  return !bad;
}
__device__ __forceinline__ void mp_candidate(const MPParams& P, MPCand& q, const uint8_t* tp, int64_t sv, int kl) {
  const PatDev* pd = P.pats + P.kbase + kl;
  const int64_t m = pd->m;
  if (!mp_head_ok(tp, pd->bytes, m)) return;
  if (m <= 16) {
    mp_record(P, P.kbase + kl, sv + pd->delta);
  } else if (q.n < 4) {
    q.sv[q.n] = sv, q.kl[q.n] = kl, q.n++;
  } else if (mp_tail_ok(tp, pd->bytes, m, 16, 4)) {
    mp_record(P, P.kbase + kl, sv + pd->delta);
  }
}
// the lanes' queued long candidates, one at a time by the whole warp (lane l
// compares words 16 + 4 l, + 128, ...); call from all lanes
__device__ __forceinline__ void mp_verify_queued(const MPParams& P, const MPCand& q, const uint8_t* S, int64_t B0,
                                                 int lane) {
  uint32_t pend = __ballot_sync(0xffffffffu, q.n > 0);
  while (pend) {
    const int src = __ffs(pend) - 1;
    pend &= pend - 1;
    const int ns = __shfl_sync(0xffffffffu, q.n, src);
#pragma unroll
    for (int f = 0; f < 4; f++) {
      if (f >= ns) break;
      const int64_t sv = __shfl_sync(0xffffffffu, (long long)q.sv[f], src);
      const int kl = __shfl_sync(0xffffffffu, q.kl[f], src);
      const PatDev* pd = P.pats + P.kbase + kl;
      const bool ok = mp_tail_ok(S + (sv - B0), pd->bytes, pd->m, 16 + 4 * lane, 128);
      if (__all_sync(0xffffffffu, ok) && lane == src) mp_record(P, P.kbase + kl, sv + pd->delta);
    }
  }
}

// Prologue of a search's first batch-pass launch (grid co-resident): zero the
// segment counts (the pass counts with atomics), fill the per-pattern scan
// flags from their immutable source, one grid barrier -- instead of two
// separate memset / copy operations ahead of the launch.  The NT consumer
// threads of every CTA (the producer warp is loading tiles meanwhile).
__device__ __forceinline__ void mp_prologue(const MPParams& P) {
  if (!P.zero_n) return;
  const int64_t nth = (int64_t)gridDim.x * NT;
  const int64_t gid = (int64_t)blockIdx.x * NT + threadIdx.x;
  const int64_t n8 = P.zero_n / 8;  // uint4 = 8 counts (the counts array is 16-byte aligned)
  for (int64_t i = gid; i < n8; i += nth) reinterpret_cast<uint4*>(P.counts)[i] = make_uint4(0, 0, 0, 0);
  for (int64_t i = 8 * n8 + gid; i < P.zero_n; i += nth) P.counts[i] = 0;
  if (P.need_src)
    for (int64_t i = gid; i < P.need_k; i += nth) P.need[i] = P.need_src[i];
  consumer_sync();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(P.bar, 1ULL);
    while (ld_acquire(P.bar) < (unsigned long long)gridDim.x) __nanosleep(32);
  }
}

// TMA producer of the batched passes: text tiles (+ halo) into the ring.
__device__ __forceinline__ void mp_produce(const MPParams& P, StageHdr* hdr, uint64_t* full, uint64_t* empty,
                                           uint8_t* stages) {
  const int NS = P.nstages;
  int s = 0;
  uint32_t ph = 0;
  for (int it = 0;; it++, s = (s + 1 == NS) ? (ph ^= 1u, 0) : s + 1) {
    if (it >= NS) mbar_wait(&empty[s], ph ^ 1u);
    const unsigned long long tk = atomicAdd(P.ticket, 1ULL);
    if ((int64_t)tk >= P.ntiles_text) {
      hdr[s].tk = -1;
      mbar_arrive(&full[s]);
      break;
    }
    hdr[s].tk = (int64_t)tk;
    hdr[s].tau = (int64_t)tk;
    const int64_t start = (int64_t)tk * TILE - P.pre;
    const int64_t end = (int64_t)tk * TILE + TILE + P.post;
    const int64_t cs = start < 0 ? 0 : start;
    const int64_t ce = end > P.nv16 ? P.nv16 : end;
    const uint32_t tb = ce > cs ? (uint32_t)(ce - cs) : 0u;
    uint8_t* st = stages + s * P.stage_bytes;
    mbar_expect_tx(&full[s], tb);
    if (tb) bulk_g2s(st + (cs - start), P.text + cs, tb, &full[s]);
  }
}

__global__ void __launch_bounds__(NT + 32) mp_scan_kernel(const MPParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + SM_HDR);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM_FULL);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + SM_EMPTY);
  uint8_t* stages = smem + SM_STAGES;
  uint32_t* bloom = reinterpret_cast<uint32_t*>(stages + P.nstages * P.stage_bytes);
  uint32_t* bstart = bloom + 2048;
  uint2* ents = reinterpret_cast<uint2*>(bstart + (((1 << P.B) + 1 + 3) & ~3));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // barriers first: the producer starts the tile loads while the consumers
  // stage the tables (and run the search's prologue)
  if (tid == 0) {
    for (int s = 0; s < P.nstages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp < NWARP) {
    for (int i = tid; i < 2048; i += NT) bloom[i] = P.bloom[i];
    for (int i = tid; i <= (1 << P.B); i += NT) bstart[i] = P.bstart[i];
    for (int i = tid; i < P.nents; i += NT) ents[i] = P.ents[i];
    mp_prologue(P);
    consumer_sync();
  }

  if (warp == NWARP) {  // ---------------- producer: text tiles only
    if (lane == 0) mp_produce(P, hdr, full, empty, stages);
    return;
  }

  const int c0 = warp * SEG;
  const int NS = P.nstages;
  int s = 0;
  uint32_t ph = 0;
  for (;; s = (s + 1 == NS) ? (ph ^= 1u, 0) : s + 1) {
    mbar_wait(&full[s], ph);
    const int64_t tau = hdr[s].tk;
    if (tau < 0) break;
    const int64_t B0 = tau * TILE;
    const uint8_t* S = stages + s * P.stage_bytes + P.pre;  // S[c] = virtual byte B0 + c
#pragma unroll 1
    for (int r = 0; r < SEG / 512; r++) {
      const int c = c0 + r * 512 + lane * 16;
      const uint4 X4 = *reinterpret_cast<const uint4*>(S + c);
      const uint32_t w[4] = {X4.x, X4.y, X4.z, X4.w};
      uint32_t hits = 0;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint32_t h = w[q] * 0x9E3779B1u;
        hits |= ((bloom[h >> 21] >> ((h >> 16) & 31)) & 1u) << q;
      }
      MPCand cq;
      cq.n = 0;
      while (hits) {  // rare: bucket walk + verification
        const int q = __ffs(hits) - 1;
        hits &= hits - 1;
        const uint32_t X = w[q];
        const uint32_t h = X * 0x9E3779B1u;
        const uint32_t bk = h >> (32 - P.B);
        const int64_t x = B0 + c + 4 * q;  // virtual position of the word
        for (uint32_t e = bstart[bk]; e < bstart[bk + 1]; e++) {
          const uint2 en = ents[e];
          if (en.x != X) continue;
          const int kl = (int)(en.y >> 16);  // pattern within this chunk
          const int aj = (int)(en.y & 0xFFFFu);
          const int64_t sv = x - aj;  // virtual start
          const int64_t spos = sv - P.off;
          const int64_t m = P.pats[P.kbase + kl].m;
          if (spos < 0 || spos + m > P.n) continue;
          const uint8_t* tp = S + (sv - B0);
          MB_CHECK(tp >= stages + s * P.stage_bytes && tp + m + 4 <= stages + (s + 1) * P.stage_bytes);
          mp_candidate(P, cq, tp, sv, kl);
        }
      }
      mp_verify_queued(P, cq, S, B0, lane);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// ------------------------------------------------ kernel 1d: batched pass over every byte offset (K5b "MPB")
// For batches the aligned-word pass cannot take (patterns shorter than 7,
// small alphabets): each pattern contributes one q-byte gram (its rarest, at
// offset a_k; q in {2, 3, 4, 8} for the whole batch) and every text position's
// q-byte window is hashed once: bloom bit in smem, then a bucket of
// {gram, pattern, a_k} entries, the full pattern verified in the staged tile,
// the occurrence recorded as in the aligned pass.  Q = q.  Q = 16 (small
// alphabets: sigma = 2 has 8 bits per 8-byte gram): the entry keeps gram words
// 0-1 and a fingerprint of words 2-3, the hash covers all four.
template <int Q>
__global__ void __launch_bounds__(NT + 32) mpb_scan_kernel(const MPParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + SM_HDR);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM_FULL);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + SM_EMPTY);
  uint8_t* stages = smem + SM_STAGES;
  uint32_t* bloom = reinterpret_cast<uint32_t*>(stages + P.nstages * P.stage_bytes);
  uint32_t* bstart = bloom + 2048;
  uint4* ents = reinterpret_cast<uint4*>(bstart + (((1 << P.B) + 1 + 3) & ~3));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // exact_local: this warp's per-pattern match counts of its current segment (packed uint16 pairs)
  uint32_t* wc = reinterpret_cast<uint32_t*>(ents + P.nents) + (warp < NWARP ? warp : 0) * (MP_CHUNK / 2);
  // barriers first: the producer starts the tile loads while the consumers
  // stage the tables (and run the search's prologue)
  if (tid == 0) {
    for (int s = 0; s < P.nstages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp < NWARP) {
    for (int i = tid; i < 2048; i += NT) bloom[i] = P.bloom[i];
    for (int i = tid; i <= (1 << P.B); i += NT) bstart[i] = P.bstart[i];
    for (int i = tid; i < P.nents; i += NT) ents[i] = P.ents4[i];
    if (P.exact_local)
      for (int i = lane; i < MP_CHUNK / 2; i += 32) wc[i] = 0u;
    mp_prologue(P);
    consumer_sync();
  }
  if (warp == NWARP) {
    if (lane == 0) mp_produce(P, hdr, full, empty, stages);
    return;
  }
  constexpr uint32_t QMASK = Q >= 4 ? 0xFFFFFFFFu : ((1u << (8 * Q)) - 1u);
  const int c0 = warp * SEG;
  const int NS = P.nstages;
  int s = 0;
  uint32_t ph = 0;
  for (;; s = (s + 1 == NS) ? (ph ^= 1u, 0) : s + 1) {
    mbar_wait(&full[s], ph);
    const int64_t tau = hdr[s].tk;
    if (tau < 0) break;
    const int64_t B0 = tau * TILE;
    const uint8_t* S = stages + s * P.stage_bytes + P.pre;  // S[c] = virtual byte B0 + c
#pragma unroll 1
    for (int r = 0; r < SEG / 512; r++) {
      const int c = c0 + r * 512 + lane * 16;
      MB_CHECK(S + c + 36 <= stages + (s + 1) * P.stage_bytes);
      const uint4 X = *reinterpret_cast<const uint4*>(S + c);
      const uint4 Y = *reinterpret_cast<const uint4*>(S + c + 16);  // words 4-5 (Q = 16: 4-7, 8)
      const uint32_t Z = Q == 16 ? *reinterpret_cast<const uint32_t*>(S + c + 32) : 0u;
      const uint32_t w[9] = {X.x, X.y, X.z, X.w, Y.x, Y.y, Y.z, Y.w, Z};
      uint32_t hits = 0;
      MPCand cq;
      cq.n = 0;
      auto gram = [&](int p, uint32_t* lo, uint32_t* hi, uint32_t* fp) -> uint32_t {  // hash of window p
        const int i = p >> 2, sh = 8 * (p & 3);
        *lo = __funnelshift_r(w[i], w[i + 1], sh) & QMASK;
        *hi = Q >= 8 ? __funnelshift_r(w[i + 1], w[i + 2], sh) : 0u;
        if (Q == 16) {
          const uint32_t w2 = __funnelshift_r(w[i + 2], w[i + 3], sh), w3 = __funnelshift_r(w[i + 3], w[i + 4], sh);
          *fp = w2 ^ (w3 * 0x9E3779B1u);
          return *lo * 0x9E3779B1u ^ *hi * 0x85EBCA77u ^ w2 * 0xC2B2AE3Du ^ w3 * 0x27D4EB2Fu;
        }
        *fp = 0u;
        return *lo * 0x9E3779B1u ^ *hi * 0x85EBCA77u;
      };
#pragma unroll
      for (int p = 0; p < 16; p++) {
        uint32_t lo, hi, fp;
        const uint32_t h = gram(p, &lo, &hi, &fp);
        hits |= ((bloom[h >> 21] >> ((h >> 16) & 31)) & 1u) << p;
      }
      while (hits) {  // bucket walk + verification
        const int p = __ffs(hits) - 1;
        hits &= hits - 1;
        uint32_t lo, hi, fp;
        const uint32_t h = gram(p, &lo, &hi, &fp);
        const uint32_t bk = h >> (32 - P.B);
        const int64_t x = B0 + c + p;  // virtual position of the window
        for (uint32_t e = bstart[bk]; e < bstart[bk + 1]; e++) {
          const uint4 en = ents[e];
          if (en.x != lo || en.y != hi || en.w != fp) continue;
          const int kl = (int)(en.z >> 16);
          if (P.exact_m) {  // the gram is the whole pattern: an occurrence, recorded at its family's bit
            const int64_t sp0 = x - P.off;
            if (sp0 >= 0 && sp0 + P.exact_m <= P.n) {
              if (P.exact_local) {
                // bit = position: this warp's own segment of pattern kl -- the slot from
                // the warp's smem counter (flushed to the global counts after the segment)
                const unsigned int sh = 16u * (unsigned)(kl & 1);
                const unsigned int old = (atomicAdd(&wc[kl >> 1], 1u << sh) >> sh) & 0xFFFFu;
                if (old < (unsigned)LIST_CAP) {
                  const int64_t g = ((int64_t)(P.kbase + kl) * P.ntiles + tau) * NWARP + warp;
                  P.lists[g * LIST_CAP + old] = (uint16_t)(c + p);
                } else {
                  P.need[P.kbase + kl] = 1u;
                  atomicExch(P.overflow, 1u);
                }
              } else {
                mp_record(P, P.kbase + kl, x + (int64_t)(en.z & 0xFFFFu));
              }
            }
            continue;
          }
          const int a = (int)(en.z & 0xFFFFu);
          const int64_t sv = x - a;  // virtual start
          const int64_t spos = sv - P.off;
          const int64_t m = P.pats[P.kbase + kl].m;
          if (spos < 0 || spos + m > P.n) continue;
          const uint8_t* tp = S + (sv - B0);
          MB_CHECK(tp >= stages + s * P.stage_bytes && tp + m + 4 <= stages + (s + 1) * P.stage_bytes);
          mp_candidate(P, cq, tp, sv, kl);
        }
      }
      mp_verify_queued(P, cq, S, B0, lane);
    }
    __syncwarp();
    if (P.exact_local) {  // the segment's counts: plain stores (this warp is their only writer), counters cleared
      for (int i = lane; i < MP_CHUNK / 2; i += 32) {
        const uint32_t v = wc[i];
        if (v) {
          wc[i] = 0u;
          if (v & 0xFFFFu) P.counts[((int64_t)(P.kbase + 2 * i) * P.ntiles + tau) * NWARP + warp] = (uint16_t)(v & 0xFFFFu);
          if (v >> 16) P.counts[((int64_t)(P.kbase + 2 * i + 1) * P.ntiles + tau) * NWARP + warp] = (uint16_t)(v >> 16);
        }
      }
      __syncwarp();
    }
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// dst[i] = *src for i < n (CSR ends of patterns that cannot match, chained batches)
__global__ void fill_kernel(int64_t* dst, const int64_t* src, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = *src;
}

// K0: byte histogram (Text.alphabet_size, core.py:42-44).  16-byte coalesced
// loads (4 in flight per thread), one private 256-bin histogram per warp in
// smem (a byte-per-load loop with one CTA-wide histogram ran at 2.0 TB/s,
// bound by its load instructions), merged per CTA and added to the result.
constexpr int HIST_WARPS = 8;
__global__ void __launch_bounds__(HIST_WARPS * 32) hist_kernel(const uint8_t* t, int64_t n, unsigned long long* hist) {
  __shared__ unsigned int h[HIST_WARPS][256];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < HIST_WARPS * 256; i += HIST_WARPS * 32) (&h[0][0])[i] = 0;
  __syncthreads();
  unsigned int* hw = h[warp];
  auto add4 = [&](uint32_t w) {
    atomicAdd(&hw[w & 0xFFu], 1u);
    atomicAdd(&hw[(w >> 8) & 0xFFu], 1u);
    atomicAdd(&hw[(w >> 16) & 0xFFu], 1u);
    atomicAdd(&hw[w >> 24], 1u);
  };
  // head bytes up to the first 16-byte boundary, 16-byte body, tail bytes
  const int64_t mis = (int64_t)((16 - ((uintptr_t)t & 15)) & 15);
  const int64_t head = n < mis ? n : mis;
  const uint4* body = reinterpret_cast<const uint4*>(t + head);
  const int64_t nv = (n - head) / 16;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid, stride = (int64_t)gridDim.x * blockDim.x;
  if (gtid < head) atomicAdd(&hw[t[gtid]], 1u);
  for (int64_t i = head + 16 * nv + gtid; i < n; i += stride) atomicAdd(&hw[t[i]], 1u);
  int64_t i = gtid;
  for (; i + 3 * stride < nv; i += 4 * stride) {
    const uint4 a = body[i], b = body[i + stride], c = body[i + 2 * stride], d = body[i + 3 * stride];
    add4(a.x), add4(a.y), add4(a.z), add4(a.w);
    add4(b.x), add4(b.y), add4(b.z), add4(b.w);
    add4(c.x), add4(c.y), add4(c.z), add4(c.w);
    add4(d.x), add4(d.y), add4(d.z), add4(d.w);
  }
  for (; i < nv; i += stride) {
    const uint4 a = body[i];
    add4(a.x), add4(a.y), add4(a.z), add4(a.w);
  }
  __syncthreads();
  for (int bin = tid; bin < 256; bin += HIST_WARPS * 32) {
    unsigned int v = 0;
#pragma unroll
    for (int w = 0; w < HIST_WARPS; w++) v += h[w][bin];
    if (v) atomicAdd(&hist[bin], (unsigned long long)v);
  }
}


}  // namespace mb
