// engine.cu -- sm_100a kernels and the C ABI of the B200 exact matcher.
//
// See scan.h for the kernel pipeline and DESIGN.md for the data layout,
// roofline and per-family byte budgets.  Reference semantics:
// pkg/src/matchbench/core.py:139-161 (all start positions, overlapping,
// ascending; m > n -> none).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "plan.h"
#include "scan.h"

namespace mb {

// Bounds assertions for the debug build (make debug -> libmatchb200_dbg.so):
// every shared-memory window a kernel reads is checked against its stage and
// every global read against the text; a violation traps.  compute-sanitizer is
// closed on this GPU pool, so this build stands in for memcheck
// (tests/test_gpu_bounds.py).  Compiled out of the product library.
#ifdef MB_BOUNDS_CHECK
#define MB_CHECK(cond)                                                  \
  do {                                                                  \
    if (!(cond)) {                                                      \
      printf("MB_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
      __trap();                                                         \
    }                                                                   \
  } while (0)
#else
#define MB_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// TMA 1D bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// look-back flag word: [epoch:24][status:2][value:38]
constexpr uint64_t ST_AGG = 1, ST_INCL = 2;
__device__ __forceinline__ uint64_t pack_state(uint32_t epoch, uint64_t st, uint64_t val) {
  return ((uint64_t)epoch << 40) | (st << 38) | (val & ((1ULL << 38) - 1));
}

// ----------------------------------------------------------- SWAR primitives
// exact per-byte zero flags (0x80 in each zero byte) -> 4-bit mask
__device__ __forceinline__ uint32_t zero_bytes4(uint32_t x) {
  uint32_t y = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);
  return ((y >> 7) * 0x01020408u) >> 24 & 0xFu;
}
__device__ __forceinline__ uint32_t shr8(uint32_t lo, uint32_t hi, int k) {
  return __funnelshift_r(lo, hi, 8 * k);
}

// -------------------------------------------------------------- filters
// Each filter looks at the 16 staged bytes of one lane (w[0..3]) plus the
// next word (w[4]) and returns the candidate mask over the lane's 16 bitmap
// positions: a cheap existence test first, the exact bit set only on a hit.

// K1 / m <= 3: byte d of x_k is zero iff t[v..v+m) == p (v = 4k + d).
template <int M>
struct FiltSWAR {
  __device__ static __forceinline__ uint32_t run(const uint32_t* w, const PatDev& P) {
    uint32_t x[4], acc = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t v = w[k] ^ P.G[0];
      if (M >= 2) v |= shr8(w[k], w[k + 1], 1) ^ P.G[1];
      if (M >= 3) v |= shr8(w[k], w[k + 1], 2) ^ P.G[2];
      x[k] = v;
      acc |= (v - 0x01010101u) & ~v;
    }
    if (!(acc & 0x80808080u)) return 0;
    uint32_t mk = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) mk |= zero_bytes4(x[k]) << (4 * k);
    return mk;
  }
};

// K1 / 4 <= m <= 6: 32-bit window at every byte offset vs the anchor word.
struct FiltWIN4 {
  __device__ static __forceinline__ uint32_t run(const uint32_t* w, const PatDev& P) {
    const uint32_t g = P.G[0];
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      hit |= (w[k] == g) | (shr8(w[k], w[k + 1], 1) == g) | (shr8(w[k], w[k + 1], 2) == g) |
             (shr8(w[k], w[k + 1], 3) == g);
    }
    if (!hit) return 0;
    uint32_t mk = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int d = 0; d < 4; d++)
        if (shr8(w[k], w[k + 1], d) == g) mk |= 1u << (4 * k + d);
    return mk;
  }
};

// K1/K3 / m >= 7: every occurrence contains one 4-aligned text word inside its
// 7-byte anchor window [a, a+7); that word equals p[a+j .. a+j+4) for exactly
// one j in 0..3.  Word k matching G_j marks bitmap position 4k + 3 - j.
struct FiltALIGNED {
  __device__ static __forceinline__ uint32_t run(const uint32_t* w, const PatDev& P) {
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 4; k++)
      hit |= (w[k] == P.G[0]) | (w[k] == P.G[1]) | (w[k] == P.G[2]) | (w[k] == P.G[3]);
    if (!hit) return 0;
    uint32_t mk = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int j = 0; j < 4; j++)
        if (w[k] == P.G[j]) mk |= 1u << (4 * k + 3 - j);
    return mk;
  }
};

// K2 / 7 <= m <= 64, small alphabets (bitparallel.py:41-63 compile_so): per-lane
// bit-parallel Shift-Or over a 64-position run of the segment (+ m-1 bytes of
// look-ahead).  Exact, no verification.  W = 32 or 64 bits of state.
template <int W>
struct FiltSO {
  static constexpr bool kShiftOr = true;
  static constexpr int kW = W;
};
template <class F, class = void>
struct is_shiftor : std::false_type {};
template <class F>
struct is_shiftor<F, std::void_t<decltype(F::kShiftOr)>> : std::true_type {};

template <int W>
__device__ __forceinline__ void shiftor_lane(const uint8_t* q, int m, const uint64_t* masks, uint32_t& w0,
                                             uint32_t& w1) {
  using T = typename std::conditional<W == 32, uint32_t, uint64_t>::type;
  T D = ~T(0);
  uint64_t acc = 0;  // shift register of match bits; after 64 + m - 1 bytes holds positions 0..63
  const int total = 64 + m - 1;
  const int hb = m - 1;
  int y = 0;
  for (; y + 4 <= total; y += 4) {
    const uint32_t word = *reinterpret_cast<const uint32_t*>(q + y);
#pragma unroll
    for (int b = 0; b < 4; b++) {
      D = (D << 1) | (T)masks[(word >> (8 * b)) & 0xFFu];
      acc = (acc >> 1) | ((uint64_t)((~D >> hb) & 1u) << 63);
    }
  }
  for (; y < total; y++) {
    D = (D << 1) | (T)masks[q[y]];
    acc = (acc >> 1) | ((uint64_t)((~D >> hb) & 1u) << 63);
  }
  w0 = (uint32_t)acc;
  w1 = (uint32_t)(acc >> 32);
}

// ------------------------------------------------------------ verification
// Direct window compare in shared memory (core.py:131-136 match_at).
__device__ __forceinline__ bool verify_direct(const uint8_t* s, const uint8_t* pat, int m) {
  for (int k = 0; k < m; k++)
    if (s[k] != pat[k]) return false;
  return true;
}

// Per-warp break bitmap of a segment: bit q of word i set iff
// t[y] != t[y + per] for y = y0 + 32 i + q (y relative to the segment's first
// start position).  nbw[i] = first break at or after word i (relative to y0).
__device__ __forceinline__ uint32_t lds32u(const uint8_t* p) {  // unaligned 4-byte smem read
  const uintptr_t a = (uintptr_t)p;
  const uint32_t* b = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  return __funnelshift_r(b[0], b[1], 8 * (uint32_t)(a & 3));
}

__device__ void warp_breaks(const uint8_t* Yseg, int per, int nwords, uint32_t* brk, int32_t* nbw) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < nwords; i += 32) {  // SWAR: 4 byte pairs per compare
    const uint8_t* q = Yseg + 32 * i;
    uint32_t bits = 0;
#pragma unroll
    for (int b = 0; b < 32; b += 4) bits |= ((~zero_bytes4(lds32u(q + b) ^ lds32u(q + b + per))) & 0xFu) << b;
    brk[i] = bits;
  }
  __syncwarp();
  const int seg = (nwords + 31) / 32;
  const int lo = lane * seg, hi = min(nwords, lo + seg);
  int first = 0x7fffffff;
  for (int i = hi - 1; i >= lo; i--)
    if (brk[i]) first = 32 * i + __ffs(brk[i]) - 1;
  int suf = first;  // inclusive suffix-min over lanes
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int o = __shfl_down_sync(0xffffffffu, suf, d);
    if (lane + d < 32) suf = min(suf, o);
  }
  int cur = __shfl_down_sync(0xffffffffu, suf, 1);
  if (lane == 31) cur = 0x7fffffff;
  for (int i = hi - 1; i >= lo; i--) {
    if (brk[i]) cur = 32 * i + __ffs(brk[i]) - 1;
    nbw[i] = cur;
  }
  if (lane == 0) nbw[nwords] = 0x7fffffff;
  __syncwarp();
}

// ---------------------------------------------------------------- kernel 1: scan
// Warp-specialised: warp NWARP is the TMA producer (ticket -> bulk copies of
// the tile+halo and of the pattern into a free stage), warps 0..NWARP-1 are
// consumers that each own one SEG-position segment of every tile.  Stages are
// handed over through full/empty mbarriers; there is no block-wide barrier in
// the loop, so warps drift independently within the ring.
template <class Filt>
__global__ void __launch_bounds__(NT + 32) scan_kernel(const ScanParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + SM_HDR);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM_FULL);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + SM_EMPTY);
  uint8_t* stages = smem + SM_STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (P.run_if && *P.run_if == 0u) return;  // conditional fallback launch (MP did not overflow)
  uint32_t* bm = reinterpret_cast<uint32_t*>(stages + STAGES * P.stage_bytes) + warp * SEG_WORDS;
  uint32_t* brk = reinterpret_cast<uint32_t*>(stages + STAGES * P.stage_bytes + NWARP * SEG_WORDS * 4) +
                  warp * 2 * (P.brk_words + 4);
  int32_t* nbw = reinterpret_cast<int32_t*>(brk + P.brk_words + 4);
  uint64_t* so_s = reinterpret_cast<uint64_t*>(stages + STAGES * P.stage_bytes + NWARP * SEG_WORDS * 4 +
                                               NWARP * 2 * (P.brk_words + 4) * 4) +
                   warp * 256;  // K2 only: per-warp shift-or masks

  if (tid == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NWARP) {  // ---------------- producer
    if (lane == 0) {
      for (int it = 0;; it++) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(it / STAGES - 1) & 1u);
        const unsigned long long tk = atomicAdd(&P.ticket[P.ticket_slot], 1ULL);
        if ((int64_t)tk >= P.group_tiles) {
          hdr[s].tk = -1;
          mbar_arrive(&full[s]);
          break;
        }
        const int kg = (int)((int64_t)tk / P.ntiles);
        const int k = P.plist ? P.plist[kg] : kg;  // this launch's family group -> batch index
        const int64_t tau = (int64_t)tk - (int64_t)kg * P.ntiles;
        hdr[s].tk = (int64_t)k * P.ntiles + tau;   // global tile id (segment index base)
        hdr[s].k = k;
        hdr[s].tau = tau;
        const int64_t start = tau * TILE - P.pre;
        const int64_t end = tau * TILE + TILE + P.post;
        const int64_t cs = start < 0 ? 0 : start;
        const int64_t ce = end > P.nv16 ? P.nv16 : end;
        const uint32_t tb = ce > cs ? (uint32_t)(ce - cs) : 0u;
        const PatDev* pd = P.pats + k;
        const uint32_t pb = (uint32_t)((pd->m + 15) & ~15LL);
        uint8_t* st = stages + s * P.stage_bytes;
        mbar_expect_tx(&full[s], tb + pb);
        bulk_g2s(st, pd->bytes, pb, &full[s]);
        if (tb) bulk_g2s(st + P.pat_cap + (cs - start), P.text + cs, tb, &full[s]);
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int c0 = warp * SEG;  // this warp's segment of every tile
  int cur_k = -1;
  PatDev pd;
  int64_t blo = 0, bhi = -1;
  for (int it = 0;; it++) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (uint32_t)(it / STAGES) & 1u);
    const int64_t tk = hdr[s].tk;
    if (tk < 0) break;
    const int k = hdr[s].k;
    if (k != cur_k) {  // per-pattern parameters stay in registers across tiles
      pd = P.pats[k];
      blo = P.off + pd.delta;               // valid bits: s = b - delta - off in [0, n-m]
      bhi = P.off + pd.delta + P.n - pd.m;  // inclusive (may be < blo)
      cur_k = k;
      if constexpr (is_shiftor<Filt>::value) {  // this warp's copy of the 256 shift-or masks
        for (int i = lane; i < 256; i += 32) so_s[i] = pd.so_masks[i];
        __syncwarp();
      }
    }
    const int64_t B0 = hdr[s].tau * TILE;
    const uint8_t* spat = stages + s * P.stage_bytes;
    const uint8_t* S = spat + P.pat_cap + P.pre;  // S[c] = virtual text byte B0 + c
    const uint8_t* const sbeg = spat + P.pat_cap;  // staged text window [sbeg, send)
    const uint8_t* const send = spat + P.stage_bytes;
    (void)sbeg, (void)send;
    MB_CHECK(S + c0 + SEG + 4 <= send);
    const int64_t segb = B0 + c0;
    const bool interior = segb >= blo && segb + SEG - 1 <= bhi;

    // this lane's 64 positions of the segment: linear bitmap words 2*lane, 2*lane+1
    uint32_t w0 = 0, w1 = 0;
    bool have;
    if constexpr (is_shiftor<Filt>::value) {
      // ---- K2: exact per-lane shift-or over positions [c0 + 64 lane, +64)
      MB_CHECK(S + c0 + 64 * lane + 64 + pd.m + 3 <= send);
      shiftor_lane<Filt::kW>(S + c0 + 64 * lane, (int)pd.m, so_s, w0, w1);
      if (!interior) {
        const int64_t b = segb + 64 * lane;
        uint64_t vm = 0;
        for (int i = 0; i < 64; i++)
          if (b + i >= blo && b + i <= bhi) vm |= 1ULL << i;
        w0 &= (uint32_t)vm;
        w1 &= (uint32_t)(vm >> 32);
      }
      have = __any_sync(0xffffffffu, (w0 | w1) != 0);
    } else {
      // ---- filter (fast path): 4 rounds of 512 positions, 16 per lane, masks kept in registers
      uint32_t mk[SEG / 512];
      bool anyc = false;
#pragma unroll
      for (int r = 0; r < SEG / 512; r++) {
        const int c = c0 + r * 512 + lane * 16;
        const uint4 X = *reinterpret_cast<const uint4*>(S + c);
        const uint32_t w[5] = {X.x, X.y, X.z, X.w, *reinterpret_cast<const uint32_t*>(S + c + 16)};
        mk[r] = Filt::run(w, pd);
        anyc |= (mk[r] != 0);
      }
      have = __any_sync(0xffffffffu, anyc);
      if (have) {
        // ---- slow path: validity mask at text edges, linear segment bitmap
#pragma unroll
        for (int r = 0; r < SEG / 512; r++) {
          uint32_t m = mk[r];
          if (!interior) {
            const int64_t b = segb + r * 512 + lane * 16;
            uint32_t vm = 0;
            for (int i = 0; i < 16; i++)
              if (b + i >= blo && b + i <= bhi) vm |= 1u << i;
            m &= vm;
          }
          const uint32_t other = __shfl_down_sync(0xffffffffu, m, 1);
          if (!(lane & 1)) bm[r * 16 + (lane >> 1)] = m | (other << 16);
        }
        __syncwarp();
        w0 = bm[2 * lane];
        w1 = bm[2 * lane + 1];
      }
    }
    uint32_t cnt = 0;
    if (have) {
      // ---- verify (exact filters skip this)
      if (!pd.exact && __any_sync(0xffffffffu, (w0 | w1) != 0)) {
        const uint8_t* Y0 = S - pd.delta;  // Y0[rel] = text byte at the start position of tile bit rel
        if (pd.periodic) {
          // s matches <=> t[s..s+per) = p[0..per) and no break t[y] != t[y+per] for
          // y in [s, s+L).  A break y kills starts [y-L+1, y]: walk the few breaks
          // that reach this lane's 64 starts, mask them out in bulk.
          const int nwords = (SEG + pd.L + 31) / 32;
          MB_CHECK(Y0 + c0 >= sbeg && Y0 + c0 + 32 * nwords + pd.per + 8 <= send);
          warp_breaks(Y0 + c0, pd.per, nwords, brk, nbw);
          uint64_t cand = ((uint64_t)w1 << 32) | w0;
          if (cand) {
            auto nb = [&](int y) -> int {
              if (y >= 32 * nwords) return 0x7fffffff;
              const uint32_t x = brk[y >> 5] >> (y & 31);
              return x ? y + __ffs(x) - 1 : nbw[(y >> 5) + 1];
            };
            const int q0 = 64 * lane, q1 = q0 + 63;
            uint64_t killed = 0;
            for (int y = nb(q0); y != 0x7fffffff && y - pd.L + 1 <= q1; y = nb(y + 1)) {
              const int lo = max(q0, y - pd.L + 1) - q0, hi = min(q1, y) - q0;
              if (lo <= hi) killed |= (hi - lo == 63) ? ~0ULL : (((1ULL << (hi - lo + 1)) - 1) << lo);
              if (y >= q1) break;
            }
            cand &= ~killed;
            if (pd.per > 4) {  // the 4 anchor bytes do not cover a full period: check one block
              uint64_t cc = cand;
              while (cc) {
                const int i = __ffsll((long long)cc) - 1;
                cc &= cc - 1;
                MB_CHECK(Y0 + c0 + q0 + i >= sbeg && Y0 + c0 + q0 + i + pd.per <= send);
                if (!verify_direct(Y0 + c0 + q0 + i, spat, pd.per)) cand &= ~(1ULL << i);
              }
            }
          }
          w0 = (uint32_t)cand;
          w1 = (uint32_t)(cand >> 32);
        } else if (pd.m >= 64) {
          // long windows: the whole warp verifies one candidate at a time,
          // lane l comparing 4-byte words l, l+32, ... (smem text vs pattern)
          const uint64_t mine = ((uint64_t)w1 << 32) | w0;
          uint64_t keep = 0;
          uint32_t active = __ballot_sync(0xffffffffu, mine != 0);
          while (active) {
            const int src = __ffs(active) - 1;
            active &= active - 1;
            uint64_t cm = ((uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(mine >> 32), src) << 32) |
                          __shfl_sync(0xffffffffu, (uint32_t)mine, src);
            while (cm) {
              const int i = __ffsll((long long)cm) - 1;
              cm &= cm - 1;
              const uint8_t* tw = Y0 + c0 + 64 * src + i;
              MB_CHECK(tw >= sbeg && tw + pd.m + 8 <= send);
              bool bad = false;
              for (int k = 4 * lane; k < pd.m; k += 128) {
                const uint32_t pw = *reinterpret_cast<const uint32_t*>(spat + k);
                uint32_t diff = lds32u(tw + k) ^ pw;
                if (pd.m - k < 4) diff &= (1u << (8 * (pd.m - k))) - 1u;
                bad |= diff != 0;
              }
              if (!__any_sync(0xffffffffu, bad) && lane == src) keep |= 1ULL << i;
            }
          }
          w0 = (uint32_t)keep;
          w1 = (uint32_t)(keep >> 32);
        } else {
          uint32_t ws[2] = {w0, w1};
#pragma unroll
          for (int h = 0; h < 2; h++) {
            uint32_t cw = ws[h], mw = 0;
            while (cw) {
              const int i = __ffs(cw) - 1;
              cw &= cw - 1;
              MB_CHECK(Y0 + c0 + 32 * (2 * lane + h) + i >= sbeg && Y0 + c0 + 32 * (2 * lane + h) + i + pd.m <= send);
              if (verify_direct(Y0 + c0 + 32 * (2 * lane + h) + i, spat, (int)pd.m)) mw |= 1u << i;
            }
            ws[h] = mw;
          }
          w0 = ws[0];
          w1 = ws[1];
        }
      }
      // ---- count + compact store (segment g = tile * NWARP + warp)
      const uint32_t c2 = __popc(w0) + __popc(w1);
      uint32_t inc = c2;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
      }
      cnt = __shfl_sync(0xffffffffu, inc, 31);
      const int64_t g = tk * NWARP + warp;
      if (cnt <= LIST_CAP) {
        uint32_t j = inc - c2;
        uint16_t* L = P.lists + g * LIST_CAP;
        uint64_t bits = ((uint64_t)w1 << 32) | w0;
        while (bits) {
          const int i = __ffsll((long long)bits) - 1;
          bits &= bits - 1;
          L[j++] = (uint16_t)(c0 + 64 * lane + i);
        }
      } else {
        reinterpret_cast<uint2*>(P.bitmaps + g * SEG_WORDS)[lane] = make_uint2(w0, w1);
      }
      __syncwarp();
    }
    if (lane == 0) {
      P.counts[tk * NWARP + warp] = (uint16_t)cnt;
      mbar_arrive(&empty[s]);
    }
  }
}

// ------------------------------------------------ kernel 1b: sampled q-gram scan (K3)
// For long, non-periodic patterns: only the q-gram at every
// S-th text position is read (one 128-byte DRAM line per sample instead of S
// bytes); a bloom filter + bucketed offset lists in smem map a gram to the
// pattern offsets j where it occurs, each giving a candidate start s = x - j
// that is verified against the text in global memory.  A warp owns SMP_SEGS
// consecutive segments (8 tiles) and reads every sample whose bit range
// [S*i, S*i + S) meets them, 4 independent 16-byte loads per lane in flight.
// Output (segment counts, uint16 tile-relative lists) is the scan kernel's, so
// offsets/expand are shared.
constexpr int SMP_SEGS = 64;     // segments per warp unit (= 8 tiles)
constexpr int SMP_LIST = 1024;   // per-warp match capacity per unit (bound: 131072/per + 2 < 1024)
#ifndef MB_SMP_ILP
#define MB_SMP_ILP 4
#endif
#ifndef MB_SMP_WARPS
#define MB_SMP_WARPS 16
#endif
constexpr int SMP_ILP = MB_SMP_ILP;     // samples per lane per batch
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
    const uint8_t* tp = P.text + sv;
    MB_CHECK(sv >= P.off && sv + pd.m <= P.off + P.n);
    bool ok = true;
    for (int c = 0; c < pd.m && ok; c++) ok = __ldg(tp + c) == spat[c];
    if (ok) found[nf++] = (uint32_t)(bit - ulo);
  }
  return nf;
}

__global__ void __launch_bounds__(SMP_NT) sampled_kernel(const ScanParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* bloom = reinterpret_cast<uint32_t*>(smem);                 // 2048 words
  uint16_t* bstart = reinterpret_cast<uint16_t*>(smem + 8192);         // <= 1025
  uint16_t* bent = reinterpret_cast<uint16_t*>(smem + 8192 + 2064);    // <= 4096
  uint32_t* lists = reinterpret_cast<uint32_t*>(smem + 8192 + 2064 + 8192);  // [SMP_WARPS][SMP_LIST]
  int64_t* s_ticket = reinterpret_cast<int64_t*>(lists + SMP_WARPS * SMP_LIST);
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
    uint32_t nmatch = 0;
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
    if (nmatch > SMP_LIST) __trap();  // impossible for the plans that choose K3 (see plan.cpp)
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

// ------------------------------------------------ kernel 2: segment offsets (scan)
// Exclusive scan of per-segment counts in SCAN_CHUNK pieces; chunk order =
// ticket order taken at CTA start (no prefetch), so each chunk only waits on
// chunks already running -- the decoupled look-back never stalls on a queued
// predecessor.
__global__ void __launch_bounds__(NT) offsets_kernel(const ScanParams P) {
  __shared__ int64_t wsum[NWARP];
  __shared__ int64_t s_excl;
  __shared__ int64_t s_chunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_chunk = (int64_t)atomicAdd(&P.ticket[TICKET_OFFSETS], 1ULL);
  __syncthreads();
  const int64_t ch = s_chunk;
  const int64_t nseg = P.total_tiles * NWARP;
  const int64_t base = ch * SCAN_CHUNK;
  constexpr int PER = SCAN_CHUNK / NT;  // 32 counts per thread, read as 16-byte vectors
  static_assert(PER % 8 == 0, "vector loads of 8 uint16 counts");
  uint32_t v[PER];
  int64_t tsum = 0;
  const uint4* cv = reinterpret_cast<const uint4*>(P.counts + base + (int64_t)tid * PER);
#pragma unroll
  for (int q8 = 0; q8 < PER / 8; q8++) {
    const uint4 x = cv[q8];  // counts are allocated to a whole number of chunks
    const uint32_t wds[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int h = 0; h < 8; h++) {
      const int q = 8 * q8 + h;
      const int64_t t = base + (int64_t)tid * PER + q;
      v[q] = t < nseg ? ((wds[h >> 1] >> (16 * (h & 1))) & 0xFFFFu) : 0u;
      tsum += v[q];
    }
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
  for (int q = 0; q < NWARP; q++) {
    chunk_total += wsum[q];
    wbefore += q < warp ? wsum[q] : 0;
  }
  if (warp == 0) {
    int64_t excl = 0;
    if (ch == 0) {
      if (lane == 0) st_relaxed(&P.state[0], pack_state(P.epoch, ST_INCL, (uint64_t)chunk_total));
    } else {
      if (lane == 0) st_relaxed(&P.state[ch], pack_state(P.epoch, ST_AGG, (uint64_t)chunk_total));
      int64_t j = ch - 1;
      while (true) {
        const int64_t idx = j - lane;
        uint64_t sv;
        if (idx < 0) {
          sv = pack_state(P.epoch, ST_INCL, 0);
        } else {
          while (true) {
            sv = ld_relaxed(&P.state[idx]);
            if ((uint32_t)(sv >> 40) == P.epoch && ((sv >> 38) & 3)) break;
            __nanosleep(20);
          }
        }
        const uint64_t st = (sv >> 38) & 3;
        const int64_t val = (int64_t)(sv & ((1ULL << 38) - 1));
        const uint32_t incl = __ballot_sync(0xffffffffu, st == ST_INCL);
        int64_t contrib = val;
        if (incl) contrib = lane <= __ffs(incl) - 1 ? val : 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, d);
        excl += contrib;
        if (incl) break;
        j -= 32;
      }
      if (lane == 0) st_relaxed(&P.state[ch], pack_state(P.epoch, ST_INCL, (uint64_t)(excl + chunk_total)));
    }
    if (lane == 0) s_excl = excl + (P.out_base ? *P.out_base : 0);
  }
  __syncthreads();
  int64_t run = s_excl + wbefore + inc - tsum;
  const int64_t seg_per_pat = P.ntiles * NWARP;
  // Sorted sparse segments (<= LIST_CAP uint16 offsets) are expanded right here,
  // their offsets never leave registers; dense or unsorted (MP) segments are
  // queued for expand_kernel with their offset.
  const bool fuse = P.out && !P.unsorted_lists;
  int cur_k = -1;
  int64_t shift = 0;
#pragma unroll
  for (int q = 0; q < PER; q++) {
    const int64_t t = base + (int64_t)tid * PER + q;
    if (t < nseg) {
      if (v[q] && P.out) {
        if (fuse && v[q] <= (uint32_t)LIST_CAP) {
          const int64_t tile = t / NWARP;
          const int k = (int)(tile / P.ntiles);
          if (k != cur_k) {
            shift = P.pats[k].delta + P.off;
            cur_k = k;
          }
          const int64_t pos0 = (tile % P.ntiles) * TILE - shift;
          const uint16_t* L = P.lists + t * LIST_CAP;
          for (uint32_t e = 0; e < v[q]; e++)
            if (run + e < P.cap) P.out[run + e] = pos0 + L[e];
        } else {
          P.toff[t] = run;
          const unsigned long long slot = atomicAdd(&P.ticket[TICKET_DENSE], 1ULL);
          P.seglist[slot] = t;
        }
      }
      if (t % seg_per_pat == seg_per_pat - 1) P.offsets_plus1[t / seg_per_pat] = run + v[q];
    }
    run += v[q];
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
#pragma unroll 4
      for (int w = 0; w < 32; w++) {
        const uint32_t x = __shfl_sync(0xffffffffu, xa, w);
        const uint32_t e = __shfl_sync(0xffffffffu, ea, w);
        if ((x >> lane) & 1u) {
          const int64_t idx = o + e + __popc(x & below);
          if (idx < P.cap) P.out[idx] = segpos + 32 * w + lane;
        }
      }
#pragma unroll 4
      for (int w = 0; w < 32; w++) {
        const uint32_t x = __shfl_sync(0xffffffffu, xb, w);
        const uint32_t e = __shfl_sync(0xffffffffu, eb, w);
        if ((x >> lane) & 1u) {
          const int64_t idx = o + e + __popc(x & below);
          if (idx < P.cap) P.out[idx] = segpos + 32 * (32 + w) + lane;
        }
      }
    }
  }
}

// ------------------------------------------------ kernel 1c: batched multi-pattern pass (K5 "MP")
// One TMA pass over the text serves a whole batch of anchor-filter (K1
// ALIGNED) patterns: each 4-aligned text word X is hashed once; a bloom bit
// test in smem rejects almost every word, and a hit walks the bucket of
// {gram, pattern, anchor+j} entries.  A verified occurrence (k, s) maps to the
// same bitmap bit b = s + off + a_k + 3 as the single-pattern ALIGNED plan, so
// it lands in the consumer's own segment of pattern k's segment layout: one
// 16-bit atomic count and an (unordered) list slot; offsets/expand are shared
// (expand sorts MP lists).  Segments above LIST_CAP set `overflow` and the
// host re-runs the batch through the per-pattern path.
__global__ void __launch_bounds__(NT + 32) mp_scan_kernel(const MPParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + SM_HDR);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM_FULL);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + SM_EMPTY);
  uint8_t* stages = smem + SM_STAGES;
  uint32_t* bloom = reinterpret_cast<uint32_t*>(stages + STAGES * P.stage_bytes);
  uint32_t* bstart = bloom + 2048;
  uint2* ents = reinterpret_cast<uint2*>(bstart + (((1 << P.B) + 1 + 3) & ~3));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 2048; i += NT + 32) bloom[i] = P.bloom[i];
  for (int i = tid; i <= (1 << P.B); i += NT + 32) bstart[i] = P.bstart[i];
  for (int i = tid; i < P.nents; i += NT + 32) ents[i] = P.ents[i];
  if (tid == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NWARP) {  // ---------------- producer: text tiles only
    if (lane == 0) {
      for (int it = 0;; it++) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(it / STAGES - 1) & 1u);
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
    return;
  }

  const int c0 = warp * SEG;
  for (int it = 0;; it++) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (uint32_t)(it / STAGES) & 1u);
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
          const PatDev* pd = P.pats + P.kbase + kl;
          const int64_t m = pd->m;
          if (spos < 0 || spos + m > P.n) continue;
          const uint8_t* tp = S + (sv - B0);
          MB_CHECK(tp >= stages + s * P.stage_bytes && tp + m <= stages + (s + 1) * P.stage_bytes);
          const uint8_t* pp = pd->bytes;
          bool ok = true;
          for (int64_t t = 0; t < m && ok; t++) ok = tp[t] == __ldg(pp + t);
          if (!ok) continue;
          // same bit as the single-pattern ALIGNED plan: b = sv + a + 3 -> this lane's chunk
          const int64_t b = sv + pd->delta;
          const int64_t g = ((int64_t)(P.kbase + kl) * P.ntiles + tau) * NWARP + warp;
          unsigned int* wptr = reinterpret_cast<unsigned int*>(P.counts) + (g >> 1);
          const unsigned int sh = 16u * (unsigned)(g & 1);
          const unsigned int old = (atomicAdd(wptr, 1u << sh) >> sh) & 0xFFFFu;
          if (old < (unsigned)LIST_CAP)
            P.lists[g * LIST_CAP + old] = (uint16_t)(b - B0);
          else
            atomicExch(P.overflow, 1u);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// K0: byte histogram (Text.alphabet_size, core.py:42-44)
__global__ void hist_kernel(const uint8_t* t, int64_t n, unsigned long long* hist) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) atomicAdd(&h[t[i]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

}  // namespace mb

// ===================================================================== C ABI
using namespace mb;

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
  return fail(MB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CUDA_TRY(x)                               \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)

struct mb_plan {
  PlanHost h;
  // device copy, uploaded on first use (plans are creatable without a GPU so
  // the host tables can be inspected anywhere); guarded for shared use
  mutable std::mutex mu;
  mutable uint8_t* d_buf = nullptr;  // [pattern | bloom | bucket starts | bucket entries]
  mutable PatDev* d_dev = nullptr;
  mutable PatDev dview;              // PatDev with device pointers (host copy)
  mutable int device = -1;
};

// Upload the plan to the current device once; returns the device PatDev.
static int plan_device(const mb_plan* p, const PatDev** out) {
  std::lock_guard<std::mutex> g(p->mu);
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (p->d_dev && p->device == dev) {
    *out = p->d_dev;
    return MB_OK;
  }
  if (p->d_dev) {  // used from another device: re-upload there
    cudaFree(p->d_buf);
    cudaFree(p->d_dev);
    p->d_buf = nullptr;
    p->d_dev = nullptr;
  }
  const PlanHost& h = p->h;
  const size_t pat_bytes = (size_t)((h.m + 16 + 15) & ~15LL);
  const size_t bloom_bytes = h.bloom.size() * 4;
  const size_t bs_bytes = (h.bstart.size() * 2 + 15) & ~(size_t)15;
  const size_t be_bytes = (h.bent.size() * 2 + 15) & ~(size_t)15;
  const size_t so_bytes = h.so_masks.size() * 8;
  const size_t total = pat_bytes + bloom_bytes + bs_bytes + be_bytes + so_bytes;
  if (cudaMalloc(&p->d_buf, total) != cudaSuccess) return fail(MB_ENOMEM, "plan upload alloc");
  if (cudaMalloc(&p->d_dev, sizeof(PatDev)) != cudaSuccess) {
    cudaFree(p->d_buf);
    p->d_buf = nullptr;
    return fail(MB_ENOMEM, "plan params alloc");
  }
  std::vector<uint8_t> img(total, 0);
  memcpy(img.data(), h.pat.data(), h.m);
  if (bloom_bytes) memcpy(img.data() + pat_bytes, h.bloom.data(), bloom_bytes);
  if (!h.bstart.empty()) memcpy(img.data() + pat_bytes + bloom_bytes, h.bstart.data(), h.bstart.size() * 2);
  if (!h.bent.empty()) memcpy(img.data() + pat_bytes + bloom_bytes + bs_bytes, h.bent.data(), h.bent.size() * 2);
  if (so_bytes) memcpy(img.data() + pat_bytes + bloom_bytes + bs_bytes + be_bytes, h.so_masks.data(), so_bytes);
  CUDA_TRY(cudaMemcpy(p->d_buf, img.data(), total, cudaMemcpyHostToDevice));
  PatDev d = h.dev;
  d.bytes = p->d_buf;
  d.bloom = bloom_bytes ? reinterpret_cast<const uint32_t*>(p->d_buf + pat_bytes) : nullptr;
  d.bstart = bloom_bytes ? reinterpret_cast<const uint16_t*>(p->d_buf + pat_bytes + bloom_bytes) : nullptr;
  d.bent = bloom_bytes ? reinterpret_cast<const uint16_t*>(p->d_buf + pat_bytes + bloom_bytes + bs_bytes) : nullptr;
  d.so_masks = so_bytes ? reinterpret_cast<const uint64_t*>(p->d_buf + pat_bytes + bloom_bytes + bs_bytes + be_bytes)
                        : nullptr;
  CUDA_TRY(cudaMemcpy(p->d_dev, &d, sizeof(PatDev), cudaMemcpyHostToDevice));
  p->dview = d;
  p->device = dev;
  *out = p->d_dev;
  return MB_OK;
}

struct mb_ctx {
  int device = 0;
  int nsm = 0;
  uint64_t* state = nullptr;
  int64_t state_cap = 0;
  uint16_t* counts = nullptr;
  int64_t counts_cap = 0;
  uint16_t* lists = nullptr;
  int64_t lists_cap = 0;
  uint32_t* bitmaps = nullptr;
  int64_t bitmaps_cap = 0;
  int64_t* toff = nullptr;
  int64_t toff_cap = 0;
  int64_t* seglist = nullptr;
  int64_t seglist_cap = 0;
  int32_t* plist = nullptr;
  int64_t plist_cap = 0;
  std::vector<int32_t> h_plist;
  uint32_t* mp_tab = nullptr;  // MP tables (bloom, bucket starts, entries) per chunk
  int64_t mp_tab_cap = 0;
  std::vector<uint32_t> h_mp;
  std::vector<double> h_ent;
  uint32_t epoch = 0;
  unsigned long long* ticket = nullptr;
  PatDev* d_pats = nullptr;
  int64_t pats_cap = 0;
  std::vector<PatDev> h_pats;
  // host-entry buffers
  uint8_t* d_text = nullptr;
  int64_t text_cap = 0;
  int64_t* d_out = nullptr;
  int64_t out_cap = 0;
  int64_t* d_offs = nullptr;
  int64_t offs_cap = 0;
  std::vector<mb_plan*> tmp_plans;
  cudaStream_t stream = nullptr;
};

extern "C" {

const char* mb_last_error(void) { return g_err.c_str(); }
const char* mb_version(void) { return "matchb200 0.1.0 (sm_100a)"; }
int64_t mb_launch_count(void) { return g_launches.load(); }

int mb_plan_create(const uint8_t* h_pattern, int64_t m, const mb_plan_opts* opts, mb_plan** out) {
  if (!out) return fail(MB_EINVAL, "null out");
  *out = nullptr;
  if (m < 1) return fail(MB_EINVAL, "pattern must have length >= 1");
  if (!h_pattern) return fail(MB_EINVAL, "null pattern");
  mb_plan* p = new mb_plan();
  std::string err;
  int rc = build_plan(h_pattern, m, opts, &p->h, &err);
  if (rc) {
    delete p;
    return fail(rc, err);
  }
  *out = p;
  return MB_OK;
}

void mb_plan_destroy(mb_plan* p) {
  if (!p) return;
  cudaFree(p->d_buf);
  cudaFree(p->d_dev);
  delete p;
}

int mb_plan_info(const mb_plan* p, mb_plan_info_t* info) {
  if (!p || !info) return fail(MB_EINVAL, "null argument");
  info->m = p->h.m;
  info->family = p->h.family;
  info->anchor = p->h.anchor;
  info->delta = p->h.dev.delta;
  info->period = p->h.period;
  info->periodic = p->h.dev.periodic;
  info->stride = p->h.family == MB_FAM_SAMPLED ? p->h.dev.S : 0;
  info->gram = p->h.family == MB_FAM_SAMPLED ? p->h.dev.q : 0;
  return MB_OK;
}

int mb_plan_horspool(const mb_plan* p, int64_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  memcpy(o, p->h.hor, sizeof(p->h.hor));
  return MB_OK;
}
int mb_plan_sunday(const mb_plan* p, int64_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  memcpy(o, p->h.sun, sizeof(p->h.sun));
  return MB_OK;
}
int mb_plan_fwd_masks(const mb_plan* p, uint64_t* o, int64_t words) {
  if (!p || !o || words < 1) return fail(MB_EINVAL, "bad argument");
  forward_masks(p->h.pat.data(), p->h.m, o, words);
  return MB_OK;
}
int mb_plan_kmp(const mb_plan* p, int64_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  memcpy(o, p->h.kmp.data(), sizeof(int64_t) * (p->h.m + 1));
  return MB_OK;
}
int mb_plan_gram_hash(const mb_plan* p, int q, uint32_t* o) {
  if (!p || !o) return fail(MB_EINVAL, "null argument");
  if (q != 3 && q != 5 && q != 8) return fail(MB_EINVAL, "q must be one of (3, 5, 8)");
  if (p->h.m < q) return fail(MB_EINVAL, "m < q");
  for (int64_t i = 0; i + q <= p->h.m; i++) o[i] = gram_hash(p->h.pat.data(), i, q);
  return MB_OK;
}

int mb_ctx_create(int device, mb_ctx** out) {
  if (!out) return fail(MB_EINVAL, "null out");
  *out = nullptr;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(MB_EINVAL, "bad device index");
  CUDA_TRY(cudaSetDevice(device));
  mb_ctx* c = new mb_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&c->ticket, 16 * sizeof(unsigned long long)) != cudaSuccess) {
    delete c;
    return fail(MB_ENOMEM, "ticket alloc");
  }
  *out = c;
  return MB_OK;
}

void mb_ctx_destroy(mb_ctx* c) {
  if (!c) return;
  cudaFree(c->state);
  cudaFree(c->counts);
  cudaFree(c->lists);
  cudaFree(c->bitmaps);
  cudaFree(c->toff);
  cudaFree(c->seglist);
  cudaFree(c->plist);
  cudaFree(c->mp_tab);
  cudaFree(c->ticket);
  cudaFree(c->d_pats);
  cudaFree(c->d_text);
  cudaFree(c->d_out);
  cudaFree(c->d_offs);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"

// grow-only device scratch
template <class T>
static int grow(T** p, int64_t* cap, int64_t need, const char* what) {
  if (need <= *cap) return MB_OK;
  cudaFree(*p);
  *p = nullptr;
  int64_t ncap = std::max<int64_t>(need, 1024);
  if (cudaMalloc(p, sizeof(T) * ncap) != cudaSuccess) {
    *cap = 0;
    return fail(MB_ENOMEM, std::string("scratch alloc: ") + what);
  }
  *cap = ncap;
  return MB_OK;
}

struct SampledTag {};

// Launch the count-producing kernel of one family group: patterns
// plist[0..gk) of the batch (indices into P.pats), ticket counter `slot`.
template <class F>
static int launch_group(mb_ctx* c, ScanParams P, const PatDev* h_pats, const int32_t* h_idx, const int32_t* d_idx,
                        int gk, int slot, cudaStream_t st) {
  int pre = 0, post = 0, maxL = 0;
  int64_t maxm = 1;
  bool any_periodic = false;
  for (int i = 0; i < gk; i++) {
    const PatDev& d = h_pats[h_idx[i]];
    maxm = std::max<int64_t>(maxm, d.m);
    if (d.periodic) maxL = std::max(maxL, d.L), any_periodic = true;
    pre = std::max(pre, d.pre);
    post = std::max(post, d.post);
  }
  P.plist = d_idx;
  P.group_k = gk;
  P.group_tiles = P.ntiles * gk;
  P.ticket_slot = slot;
  P.pre = pre;
  P.post = post;
  P.pat_cap = (int)((maxm + 15) & ~15);
  P.stage_bytes = (P.pat_cap + pre + TILE + post + 127) & ~127;
  P.brk_words = any_periodic ? ((((SEG + maxL + 31) / 32) + 1 + 3) & ~3) : 0;
  if constexpr (std::is_same<F, SampledTag>::value) {
    const size_t smem_s = 8192 + 2064 + 8192 + SMP_WARPS * SMP_LIST * 4 + 16 + P.pat_cap + 16;
    static std::mutex mu_s;
    static bool attr_s = false;
    static size_t occ_smem_s = 0;
    static int occ_s = 0;
    int per_sm_s = 0;
    {
      std::lock_guard<std::mutex> g(mu_s);
      if (!attr_s) {
        CUDA_TRY(cudaFuncSetAttribute(sampled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_s = true;
      }
      if (occ_smem_s != smem_s) {
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, sampled_kernel, SMP_NT, smem_s));
        occ_smem_s = smem_s;
      }
      per_sm_s = occ_s;
    }
    if (per_sm_s < 1) return fail(MB_ECUDA, "sampled kernel does not fit on an SM");
    const int64_t wunits = (P.ntiles * NWARP + SMP_SEGS - 1) / SMP_SEGS;
    const int64_t units = ((wunits + SMP_WARPS - 1) / SMP_WARPS) * gk;
    const int64_t grid_s = std::min<int64_t>(units, (int64_t)c->nsm * per_sm_s);
    sampled_kernel<<<(int)grid_s, SMP_NT, smem_s, st>>>(P);
  } else {
    const size_t smem = (size_t)SM_STAGES + (size_t)STAGES * P.stage_bytes + NWARP * SEG_WORDS * 4 +
                        (size_t)NWARP * 2 * (P.brk_words + 4) * 4 + (is_shiftor<F>::value ? NWARP * 256 * 8 : 0);
    static std::mutex mu;
    static bool attr_done = false;
    static size_t occ_smem = 0;
    static int occ_val = 0;
    int per_sm = 0;
    {
      std::lock_guard<std::mutex> g(mu);
      if (!attr_done) {
        CUDA_TRY(cudaFuncSetAttribute(scan_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_done = true;
      }
      if (occ_smem != smem) {
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_val, scan_kernel<F>, NT + 32, smem));
        occ_smem = smem;
      }
      per_sm = occ_val;
    }
    if (per_sm < 1) return fail(MB_ECUDA, "scan kernel does not fit on an SM");
    const int64_t grid = std::min<int64_t>(P.group_tiles, (int64_t)c->nsm * per_sm);
    scan_kernel<F><<<(int)grid, NT + 32, smem, st>>>(P);
  }
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

// family key: patterns sharing a key share one count-kernel launch
static int family_key(const PatDev& d) {
  if (d.family == MB_FAM_SWAR) return (int)(10 + d.m);
  if (d.family == MB_FAM_SHIFTOR) return d.m <= 32 ? 20 : 21;
  return d.family;
}

static int launch_family(mb_ctx* c, const ScanParams& P, const PatDev* h_pats, const int32_t* h_idx,
                         const int32_t* d_idx, int gk, int slot, cudaStream_t st) {
  const PatDev& d = h_pats[h_idx[0]];
  switch (d.family) {
    case MB_FAM_SWAR:
      if (d.m == 1) return launch_group<FiltSWAR<1>>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
      if (d.m == 2) return launch_group<FiltSWAR<2>>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
      return launch_group<FiltSWAR<3>>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
    case MB_FAM_WIN4: return launch_group<FiltWIN4>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
    case MB_FAM_ALIGNED: return launch_group<FiltALIGNED>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
    case MB_FAM_SAMPLED: return launch_group<SampledTag>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
    case MB_FAM_SHIFTOR: {
      int64_t maxm = 0;
      for (int i = 0; i < gk; i++) maxm = std::max<int64_t>(maxm, h_pats[h_idx[i]].m);
      if (maxm <= 32) return launch_group<FiltSO<32>>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
      return launch_group<FiltSO<64>>(c, P, h_pats, h_idx, d_idx, gk, slot, st);
    }
  }
  return fail(MB_EINVAL, "unknown kernel family");
}

// MP eligibility (K5): a batch of >= 8 anchor-filter (ALIGNED) patterns whose
// pooled anchors stay selective.  `rate` is the expected number of gram hits
// per text word, sum over patterns k and j of prod_i p(G_kj[i]), with byte
// probabilities p estimated from all pattern bytes of the batch (patterns are
// drawn from the text); MP runs when rate <= 0.05.
static bool mp_eligible(const PatDev* h_pats, const double* rate, int K) {
  if (!rate || K < 8 || K > MP_CHUNK * MAX_GROUPS || *rate > 0.05) return false;
  for (int k = 0; k < K; k++)
    if (h_pats[k].family != MB_FAM_ALIGNED) return false;
  return true;
}

// Host-built MP tables for patterns [k0, k0 + kc): bloom, bucket starts, entries.
static void mp_tables(const PatDev* h_pats, int k0, int kc, int* Bout, std::vector<uint32_t>& img) {
  const int nent = 4 * kc;
  int B = 4;
  while ((1 << B) < nent) B++;
  const int nb = 1 << B;
  const int bs_words = (nb + 1 + 3) & ~3;
  img.assign(2048 + bs_words + 2 * nent, 0u);
  uint32_t* bloom = img.data();
  uint32_t* bstart = bloom + 2048;
  std::vector<uint32_t> cnt(nb, 0);
  for (int i = 0; i < kc; i++)
    for (int j = 0; j < 4; j++) {
      const uint32_t h = h_pats[k0 + i].G[j] * 0x9E3779B1u;
      bloom[h >> 21] |= 1u << ((h >> 16) & 31);
      cnt[h >> (32 - B)]++;
    }
  for (int b = 0; b < nb; b++) bstart[b + 1] = bstart[b] + cnt[b];
  std::vector<uint32_t> fill(bstart, bstart + nb);
  uint32_t* ents = bstart + bs_words;
  for (int i = 0; i < kc; i++)
    for (int j = 0; j < 4; j++) {
      const uint32_t g = h_pats[k0 + i].G[j];
      const uint32_t b = (g * 0x9E3779B1u) >> (32 - B);
      const uint32_t e = fill[b]++;
      ents[2 * e] = g;
      ents[2 * e + 1] = ((uint32_t)i << 16) | (uint32_t)(h_pats[k0 + i].anchor + j);
    }
  *Bout = B;
}

// One search (K = 1) or batch: per family group one count kernel (or, for a
// selective batch of anchor-filter patterns, one MP pass over the text), then
// one offsets and one expand launch over all K patterns' segments, so the
// output is CSR in the caller's pattern order whatever the family mix.
static int run_search(mb_ctx* c, const PatDev* d_pats, const PatDev* h_pats, int K, const uint8_t* d_text,
                      int64_t n, int64_t* d_out, int64_t cap, int64_t* offsets_plus1, cudaStream_t st,
                      const double* mp_rate = nullptr) {
  ScanParams P;
  memset(&P, 0, sizeof(P));
  const uintptr_t addr = (uintptr_t)d_text;
  P.text = (const uint8_t*)(addr & ~(uintptr_t)15);
  P.off = (int64_t)(addr & 15);
  P.n = n;
  P.nv16 = (P.off + n + 15) & ~(int64_t)15;
  int64_t nbits = 0;
  for (int k = 0; k < K; k++)
    if (h_pats[k].m <= n) nbits = std::max<int64_t>(nbits, P.off + h_pats[k].delta + n - h_pats[k].m + 1);
  if (nbits == 0) {  // every pattern longer than the text
    CUDA_TRY(cudaMemsetAsync(offsets_plus1, 0, sizeof(int64_t) * K, st));
    return MB_OK;
  }
  P.ntiles = (nbits + TILE - 1) / TILE;
  P.total_tiles = P.ntiles * K;
  P.pats = d_pats;
  P.K = K;
  const int64_t T = P.total_tiles * NWARP;  // segments
  const int64_t nchunks = (T + SCAN_CHUNK - 1) / SCAN_CHUNK;
  int rc;
  // whole chunks (offsets_kernel reads 16-byte vectors) + 2 slots for the MP overflow flag
  if ((rc = grow(&c->counts, &c->counts_cap, nchunks * SCAN_CHUNK + 8, "counts"))) return rc;
  if ((rc = grow(&c->lists, &c->lists_cap, T * LIST_CAP, "lists"))) return rc;
  if ((rc = grow(&c->bitmaps, &c->bitmaps_cap, T * SEG_WORDS, "bitmaps"))) return rc;
  if ((rc = grow(&c->toff, &c->toff_cap, T, "tile offsets"))) return rc;
  if ((rc = grow(&c->seglist, &c->seglist_cap, T, "expand queue"))) return rc;
  if (nchunks > c->state_cap || c->epoch >= (1u << 24) - 4) {
    if ((rc = grow(&c->state, &c->state_cap, nchunks, "look-back state"))) return rc;
    CUDA_TRY(cudaMemsetAsync(c->state, 0, sizeof(uint64_t) * c->state_cap, st));
    c->epoch = 0;
  }
  P.counts = c->counts;
  P.lists = c->lists;
  P.bitmaps = c->bitmaps;
  P.toff = c->toff;
  P.seglist = c->seglist;
  P.state = c->state;
  P.ticket = c->ticket;
  P.out = d_out;
  P.cap = d_out ? cap : 0;
  P.offsets_plus1 = offsets_plus1;
  P.out_base = nullptr;

  auto finish = [&](bool unsorted) -> int {
    P.epoch = ++c->epoch;
    P.unsorted_lists = unsorted ? 1 : 0;
    offsets_kernel<<<(int)nchunks, NT, 0, st>>>(P);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    if (d_out && cap > 0) {
      const int64_t eg = std::min<int64_t>((T + EXP_WARPS - 1) / EXP_WARPS, (int64_t)c->nsm * 16);
      expand_kernel<<<(int)eg, EXP_WARPS * 32, 0, st>>>(P);
      g_launches++;
      CUDA_TRY(cudaGetLastError());
    }
    return MB_OK;
  };

  bool mp_used = false;
  if (mp_eligible(h_pats, mp_rate, K)) {
    int pre = 0, post = 0;
    for (int k = 0; k < K; k++) pre = std::max(pre, h_pats[k].pre), post = std::max(post, h_pats[k].post);
    MPParams M;
    memset(&M, 0, sizeof(M));
    M.text = P.text;
    M.off = P.off;
    M.n = n;
    M.nv16 = P.nv16;
    M.ntiles_text = (P.nv16 + TILE - 1) / TILE;
    M.ntiles = P.ntiles;
    M.pre = pre;
    M.post = post;
    M.stage_bytes = (pre + TILE + post + 127) & ~127;
    M.pats = d_pats;
    M.counts = c->counts;
    M.lists = c->lists;
    if ((rc = grow(&c->mp_tab, &c->mp_tab_cap, (int64_t)(2048 + 4 * MP_CHUNK + 8 + 8 * MP_CHUNK) * MAX_GROUPS,
                   "MP tables")))
      return rc;
    M.overflow = reinterpret_cast<unsigned int*>(c->counts + T);  // 4 spare bytes after the counts
    CUDA_TRY(cudaMemsetAsync(c->counts, 0, sizeof(uint16_t) * (T + 2), st));
    CUDA_TRY(cudaMemsetAsync(c->ticket, 0, 16 * sizeof(unsigned long long), st));
    c->h_mp.clear();
    std::vector<std::pair<int64_t, int>> chunk_at;  // (table word offset, B) per chunk
    for (int k0 = 0, ci = 0; k0 < K; k0 += MP_CHUNK, ci++) {
      std::vector<uint32_t> img;
      int B = 0;
      mp_tables(h_pats, k0, std::min(MP_CHUNK, K - k0), &B, img);
      chunk_at.push_back({(int64_t)c->h_mp.size(), B});
      c->h_mp.insert(c->h_mp.end(), img.begin(), img.end());
      while (c->h_mp.size() % 4) c->h_mp.push_back(0);
    }
    CUDA_TRY(cudaMemcpyAsync(c->mp_tab, c->h_mp.data(), sizeof(uint32_t) * c->h_mp.size(), cudaMemcpyHostToDevice, st));
    static std::mutex mu_mp;
    static bool attr_mp = false;
    {
      std::lock_guard<std::mutex> g(mu_mp);
      if (!attr_mp) {
        CUDA_TRY(cudaFuncSetAttribute(mp_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_mp = true;
      }
    }
    for (int k0 = 0, ci = 0; k0 < K; k0 += MP_CHUNK, ci++) {
      const int kc = std::min(MP_CHUNK, K - k0);
      const int B = chunk_at[ci].second;
      const int bs_words = ((1 << B) + 1 + 3) & ~3;
      M.bloom = c->mp_tab + chunk_at[ci].first;
      M.bstart = M.bloom + 2048;
      M.ents = reinterpret_cast<const uint2*>(M.bstart + bs_words);
      M.B = B;
      M.nents = 4 * kc;
      M.kbase = k0;
      M.ticket = c->ticket + TICKET_MP0 + ci;
      const size_t smem = (size_t)SM_STAGES + (size_t)STAGES * M.stage_bytes + 8192 + 4 * bs_words + 8 * M.nents;
      int per_sm = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mp_scan_kernel, NT + 32, smem));
      if (per_sm < 1) return fail(MB_ECUDA, "MP kernel does not fit on an SM");
      const int64_t grid = std::min<int64_t>(M.ntiles_text, (int64_t)c->nsm * per_sm);
      mp_scan_kernel<<<(int)grid, NT + 32, smem, st>>>(M);
      g_launches++;
      CUDA_TRY(cudaGetLastError());
    }
    // fallback without a host round trip: the per-pattern scan below runs only if
    // a segment overflowed (kernels read the flag and exit otherwise); lists are
    // sorted on expand either way (harmless for the already-sorted fallback lists)
    P.run_if = M.overflow;
    mp_used = true;
  }
  if (!mp_used) CUDA_TRY(cudaMemsetAsync(c->ticket, 0, 16 * sizeof(unsigned long long), st));
  // group patterns by family key (stable); a single group needs no index list
  std::vector<int> keys;
  std::vector<std::vector<int32_t>> groups;
  for (int k = 0; k < K; k++) {
    const int key = family_key(h_pats[k]);
    size_t g = 0;
    while (g < keys.size() && keys[g] != key) g++;
    if (g == keys.size()) {
      keys.push_back(key);
      groups.emplace_back();
    }
    groups[g].push_back(k);
  }
  if ((int)groups.size() > MAX_GROUPS) return fail(MB_EINVAL, "too many kernel families in one batch");
  if (groups.size() == 1) {
    if ((rc = launch_family(c, P, h_pats, groups[0].data(), nullptr, K, 0, st))) return rc;
  } else {
    if ((rc = grow(&c->plist, &c->plist_cap, K, "family index lists"))) return rc;
    c->h_plist.clear();
    for (auto& g : groups) c->h_plist.insert(c->h_plist.end(), g.begin(), g.end());
    CUDA_TRY(cudaMemcpyAsync(c->plist, c->h_plist.data(), sizeof(int32_t) * K, cudaMemcpyHostToDevice, st));
    int base = 0;
    for (size_t g = 0; g < groups.size(); g++) {
      if ((rc = launch_family(c, P, h_pats, groups[g].data(), c->plist + base, (int)groups[g].size(), (int)g, st)))
        return rc;
      base += (int)groups[g].size();
    }
  }
  return finish(mp_used);
}

extern "C" {

int mb_find(mb_ctx* c, const mb_plan* p, const uint8_t* d_text, int64_t n, int64_t* d_out, int64_t cap,
            int64_t* d_count, void* stream) {
  if (!c || !p || !d_count) return fail(MB_EINVAL, "null argument");
  if (n < 0 || cap < 0) return fail(MB_EINVAL, "negative size");
  if (n > 0 && !d_text) return fail(MB_EINVAL, "null text");
  cudaStream_t st = (cudaStream_t)stream;
  if (p->h.m > n) {
    CUDA_TRY(cudaMemsetAsync(d_count, 0, sizeof(int64_t), st));
    return MB_OK;
  }
  const PatDev* dd = nullptr;
  int rc = plan_device(p, &dd);
  if (rc) return rc;
  return run_search(c, dd, &p->dview, 1, d_text, n, d_out, cap, d_count, st);
}

int mb_find_batch(mb_ctx* c, const mb_plan* const* plans, int K, const uint8_t* d_text, int64_t n,
                  int64_t* d_out, int64_t cap, int64_t* d_offsets, void* stream) {
  if (!c || !plans || K < 1 || !d_offsets) return fail(MB_EINVAL, "bad argument");
  if (n < 0 || cap < 0) return fail(MB_EINVAL, "negative size");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(d_offsets, 0, sizeof(int64_t), st));
  // group consecutive runs of the same family into one launch each; the
  // look-back ticket order makes each group's output CSR-contiguous, so the
  // groups chain through d_offsets.
  c->h_pats.resize(K);
  for (int k = 0; k < K; k++) {
    if (!plans[k]) return fail(MB_EINVAL, "null plan in batch");
    const PatDev* dd = nullptr;
    int rc = plan_device(plans[k], &dd);
    if (rc) return rc;
    c->h_pats[k] = plans[k]->dview;
  }
  if (K > c->pats_cap) {
    cudaFree(c->d_pats);
    c->d_pats = nullptr;
    if (cudaMalloc(&c->d_pats, sizeof(PatDev) * K) != cudaSuccess) {
      c->pats_cap = 0;
      return fail(MB_ENOMEM, "batch params alloc");
    }
    c->pats_cap = K;
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_pats, c->h_pats.data(), sizeof(PatDev) * K, cudaMemcpyHostToDevice, st));
  double rate = 1e30;
  bool all_aligned = K >= 8;
  for (int k = 0; k < K && all_aligned; k++) all_aligned = c->h_pats[k].family == MB_FAM_ALIGNED;
  if (all_aligned) {
    rate = 0;
    double hist[256] = {0}, tot = 0;
    for (int k = 0; k < K; k++) {
      const auto& pb = plans[k]->h.pat;
      const size_t lim = std::min<size_t>(pb.size(), 64);
      for (size_t i = 0; i < lim; i++) hist[pb[i]] += 1, tot += 1;
    }
    for (int k = 0; k < K; k++)
      if (c->h_pats[k].family == MB_FAM_ALIGNED)
        for (int j = 0; j < 4; j++) {
          double pr = 1;
          for (int i = 0; i < 4; i++) pr *= hist[(c->h_pats[k].G[j] >> (8 * i)) & 0xFF] / tot;
          rate += pr;
        }
  }
  return run_search(c, c->d_pats, c->h_pats.data(), K, d_text, n, d_out, cap, d_offsets + 1, st, &rate);
}

int mb_histogram(mb_ctx* c, const uint8_t* d_text, int64_t n, int64_t* d_hist, void* stream) {
  if (!c || !d_hist) return fail(MB_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(d_hist, 0, 256 * sizeof(int64_t), st));
  if (n <= 0) return MB_OK;
  int64_t blocks = std::min<int64_t>((n + 4095) / 4096, (int64_t)c->nsm * 8);
  hist_kernel<<<(int)blocks, 256, 0, st>>>(d_text, n, (unsigned long long*)d_hist);
  g_launches++;
  CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

static int ensure_host_bufs(mb_ctx* c, int64_t n, int64_t outcap, int64_t nofs) {
  if (!c->stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  if (n > c->text_cap) {
    cudaFree(c->d_text);
    c->d_text = nullptr;
    if (cudaMalloc(&c->d_text, n + 16) != cudaSuccess) {
      c->text_cap = 0;
      return fail(MB_ENOMEM, "text buffer alloc");
    }
    c->text_cap = n;
  }
  if (outcap > c->out_cap) {
    cudaFree(c->d_out);
    c->d_out = nullptr;
    if (cudaMalloc(&c->d_out, sizeof(int64_t) * outcap) != cudaSuccess) {
      c->out_cap = 0;
      return fail(MB_ENOMEM, "output buffer alloc");
    }
    c->out_cap = outcap;
  }
  if (nofs > c->offs_cap) {
    cudaFree(c->d_offs);
    c->d_offs = nullptr;
    if (cudaMalloc(&c->d_offs, sizeof(int64_t) * nofs) != cudaSuccess) {
      c->offs_cap = 0;
      return fail(MB_ENOMEM, "offsets alloc");
    }
    c->offs_cap = nofs;
  }
  return MB_OK;
}

int mb_search_batch_host(mb_ctx* c, const uint8_t* const* h_patterns, const int64_t* ms, int K,
                         const uint8_t* h_text, int64_t n, int64_t* h_out, int64_t cap, int64_t* h_offsets) {
  if (!c || !h_patterns || !ms || K < 1 || !h_offsets) return fail(MB_EINVAL, "bad argument");
  if (n < 0 || cap < 0 || (n > 0 && !h_text)) return fail(MB_EINVAL, "bad text");
  std::vector<mb_plan*> plans(K, nullptr);
  auto cleanup = [&]() {
    for (auto* p : plans) mb_plan_destroy(p);
  };
  for (int k = 0; k < K; k++) {
    int rc = mb_plan_create(h_patterns[k], ms[k], nullptr, &plans[k]);
    if (rc) {
      cleanup();
      return rc;
    }
  }
  int rc = ensure_host_bufs(c, n, std::max<int64_t>(cap, 1), K + 1);
  if (rc) {
    cleanup();
    return rc;
  }
  cudaStream_t st = c->stream;
  if (n > 0) cudaMemcpyAsync(c->d_text, h_text, n, cudaMemcpyHostToDevice, st);
  rc = mb_find_batch(c, plans.data(), K, c->d_text, n, c->d_out, cap, c->d_offs, st);
  if (!rc) {
    cudaMemcpyAsync(h_offsets, c->d_offs, sizeof(int64_t) * (K + 1), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "batch search");
  }
  if (!rc) {
    int64_t total = h_offsets[K];
    int64_t ncopy = std::min(total, cap);
    if (ncopy > 0) {
      cudaError_t e = cudaMemcpy(h_out, c->d_out, sizeof(int64_t) * ncopy, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) rc = cuda_fail(e, "position copy");
    }
    if (!rc && total > cap) rc = fail(MB_EOVERFLOW, "output capacity too small");
  }
  cleanup();
  return rc;
}

int mb_search_host(mb_ctx* c, const uint8_t* h_pattern, int64_t m, const uint8_t* h_text, int64_t n,
                   int64_t* h_out, int64_t cap, int64_t* h_count) {
  if (!h_count) return fail(MB_EINVAL, "null count");
  int64_t offs[2] = {0, 0};
  int rc = mb_search_batch_host(c, &h_pattern, &m, 1, h_text, n, h_out, cap, offs);
  *h_count = offs[1];
  return rc;
}

}  // extern "C"
