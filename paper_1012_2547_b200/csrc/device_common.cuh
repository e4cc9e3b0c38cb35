// device_common.cuh -- PTX helpers (TMA bulk copy, mbarrier), SWAR primitives, the K1/K2 filters, verification and break-run helpers, MB_CHECK bounds assertions
// (part of libmatchb200; included by engine.cu)
#pragma once

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

// Kernel-phase timestamps for the trace build (make trace -> libmatchb200_trace.so,
// tools/trace_phases.py): slot i keeps the min (even) / max (odd) %globaltimer
// any CTA recorded there.  Compiled out of the product library.
#ifdef MB_TRACE
__device__ unsigned long long g_trace[32];
__device__ __forceinline__ void trace_mark(int slot) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (slot & 1) atomicMax(&g_trace[slot], t); else atomicMin(&g_trace[slot], t);
  }
}
#define MB_TRACE_MARK(slot) trace_mark(slot)
#define MB_TRACE_SYNC_MARK(slot) (__syncthreads(), trace_mark(slot))
#else
#define MB_TRACE_MARK(slot) \
  do {                      \
  } while (0)
#define MB_TRACE_SYNC_MARK(slot) MB_TRACE_MARK(slot)
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
__device__ __forceinline__ uint64_t ld_acquire(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// programmatic dependent launch: wait for the preceding grid's results /
// let the next grid's CTAs be scheduled
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// (pattern, tile within the pattern) of a global tile index: 32-bit division
// while the index fits (every realistic batch), 64-bit otherwise
__device__ __forceinline__ void split_tile(int64_t tile, int64_t ntiles, int* k, int64_t* tau) {
  if ((uint64_t)tile < 0xFFFFFFFFull && (uint64_t)ntiles < 0xFFFFFFFFull) {
    const uint32_t q = (uint32_t)tile / (uint32_t)ntiles;
    *k = (int)q;
    *tau = (int64_t)((uint32_t)tile - q * (uint32_t)ntiles);
  } else {
    *k = (int)(tile / ntiles);
    *tau = tile - (int64_t)*k * ntiles;
  }
}

// End of a search's last kernel (offsets_kernel of a count-only search): the
// last CTA to finish zeroes every ticket but keep_slot (-1: none), so the next
// search needs no memset.  (expand_kernel zeroes them at its start instead.)
// Call from all threads of every CTA.
__device__ __forceinline__ void reset_tickets_if_last(unsigned long long* ticket, int ntickets, int done_slot,
                                                      int keep_slot) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ticket[done_slot], 1ULL) == (unsigned long long)(gridDim.x - 1)) {
      __threadfence();
      for (int i = 0; i < ntickets; i++)
        if (i != keep_slot) ticket[i] = 0ULL;
    }
  }
}

// look-back flag word: [epoch:24][status:2][value:38]
constexpr uint64_t ST_AGG = 1, ST_INCL = 2;
__device__ __forceinline__ uint64_t pack_state(uint32_t epoch, uint64_t st, uint64_t val) {
  return ((uint64_t)epoch << 40) | (st << 38) | (val & ((1ULL << 38) - 1));
}

// barrier over the NT consumer threads of a warp-specialised CTA (the producer
// warp has returned); id 1 (id 0 is __syncthreads)
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory"); }

// Decoupled look-back by one warp: publish `agg` for item idx, then sum the
// predecessors' published values 32 at a time back to the nearest inclusive
// one; publish the inclusive prefix and return the exclusive one (all lanes).
// Items must be numbered in start order of their (running) producers.
__device__ __forceinline__ int64_t warp_lookback(uint64_t* state, int64_t idx, uint64_t agg, uint32_t epoch,
                                                 int lane) {
  if (lane == 0) st_relaxed(&state[idx], pack_state(epoch, idx == 0 ? ST_INCL : ST_AGG, agg));
  int64_t excl = 0;
  for (int64_t j = idx - 1; j >= 0; j -= 32) {
    const int64_t q = j - lane;
    uint64_t sv = 0;
    bool incl = false;
    if (q >= 0) {
      while (true) {
        sv = ld_relaxed(&state[q]);
        if ((uint32_t)(sv >> 40) == epoch && ((sv >> 38) & 3)) break;
        __nanosleep(20);
      }
      incl = ((sv >> 38) & 3) == ST_INCL;
    }
    const uint32_t bi = __ballot_sync(0xffffffffu, incl);
    const int first = bi ? __ffs(bi) - 1 : 32;  // nearest predecessor holding an inclusive prefix
    unsigned long long v = (q >= 0 && lane <= first) ? (sv & ((1ULL << 38) - 1)) : 0ULL;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    excl += (int64_t)v;
    if (bi) break;
  }
  if (lane == 0 && idx > 0) st_relaxed(&state[idx], pack_state(epoch, ST_INCL, (uint64_t)excl + agg));
  return excl;
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
// zero-byte flags of four words -> 16 mask bits: per word the exact 0x80 flags
// (3 operations), one IMAD gathering them into the top nibble (the partial
// products of (2^21 + 2^14 + 2^7 + 1) never overlap) and one funnel shift
// appending it -- 4 ALU + 1 FMA-pipe operations per word instead of 9.
__device__ __forceinline__ uint32_t zero_flags16(const uint32_t* x) {
  uint32_t acc = 0;
#pragma unroll
  for (int k = 3; k >= 0; k--) {
    const uint32_t y = ~(((x[k] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x[k] | 0x7F7F7F7Fu);  // 0x80 in each zero byte
    acc = __funnelshift_l(y * 0x00204081u, acc, 4);
  }
  return acc;
}
template <int M>
struct FiltSWAR {
  static constexpr bool kAlwaysExact = true;  // no verification code in this instantiation
  __device__ static __forceinline__ uint32_t run(const uint32_t* w, const PatDev& P) {
    uint32_t x[4], acc = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t v = w[k] ^ P.G[0];
#pragma unroll
      for (int j = 1; j < M; j++) v |= shr8(w[k + (j >> 2)], w[k + (j >> 2) + 1], j & 3) ^ P.G[j];
      x[k] = v;
      acc |= (v - 0x01010101u) & ~v;
    }
    if (!(acc & 0x80808080u)) return 0;
    return zero_flags16(x);
  }
  // the mask alone (no early-out test): while the warp's previous segment had
  // matches (small alphabets: every segment has)
  __device__ static __forceinline__ uint32_t run_direct(const uint32_t* w, const PatDev& P) {
    uint32_t x[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t v = w[k] ^ P.G[0];
#pragma unroll
      for (int j = 1; j < M; j++) v |= shr8(w[k + (j >> 2)], w[k + (j >> 2) + 1], j & 3) ^ P.G[j];
      x[k] = v;
    }
    return zero_flags16(x);
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
    return run_direct(w, P);
  }
  // The mask alone (no early-out test): cheaper where most warps would take
  // the mask pass anyway (the scan kernel switches to it per warp while the
  // previous segment had candidates, e.g. m = 4 over a 4-letter alphabet).
  __device__ static __forceinline__ uint32_t run_direct(const uint32_t* w, const PatDev& P) {
    const uint32_t g = P.G[0];
    uint32_t mk = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int d = 0; d < 4; d++)
        if (shr8(w[k], w[k + 1], d) == g) mk |= 1u << (4 * k + d);
    return mk;
  }
};

// K1 / 5 <= m <= 6 (auto): every occurrence's 5-byte anchor window [a, a+5)
// holds a 4-byte text window at an even offset e, equal to G0 = p[a..a+4) (e =
// s + a) or G1 = p[a+1..a+5) (e = s + a + 1): two windows per text word (the
// word and its 16-bit funnel shift) instead of WIN4's four.  delta = a + 1:
// word k's bits 4k..4k+3 = {w == G1, w == G0, f == G1, f == G0}.
struct FiltWIN4E {
  __device__ static __forceinline__ uint32_t run(const uint32_t* w, const PatDev& P) {
    const uint32_t g0 = P.G[0], g1 = P.G[1];
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t f = __funnelshift_r(w[k], w[k + 1], 16);
      hit |= (w[k] == g0) | (w[k] == g1) | (f == g0) | (f == g1);
    }
    if (!hit) return 0;
    uint32_t mk = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t f = __funnelshift_r(w[k], w[k + 1], 16);
      mk |= ((w[k] == g1 ? 1u : 0u) | (w[k] == g0 ? 2u : 0u) | (f == g1 ? 4u : 0u) | (f == g0 ? 8u : 0u)) << (4 * k);
    }
    return mk;
  }
};

// K1/K3 / m >= 7: every occurrence contains one 4-aligned text word inside its
// 7-byte anchor window [a, a+7); that word equals p[a+j .. a+j+4) for exactly
// one j in 0..3.  Word k matching G_j marks bitmap position 4k + 3 - j.  With
// NW anchor words (window 4 NW + 3 bytes) words k .. k+NW-1 must all match
// (G[4w + j] = p[a+j+4w .. +4)): small alphabets need NW = 2, 3 to keep the
// candidate rate low.  w[] holds 4 + NW - 1 >= 5 words.
template <int NW>
struct FiltALIGNED {
  __device__ static __forceinline__ uint32_t run(const uint32_t* w, const PatDev& P) {
    if constexpr (NW == 1) {
      bool hit = false;
#pragma unroll
      for (int k = 0; k < 4; k++)
        hit |= (w[k] == P.G[0]) | (w[k] == P.G[1]) | (w[k] == P.G[2]) | (w[k] == P.G[3]);
      if (!hit) return 0;
    }
    return run_direct(w, P);
  }
  __device__ static __forceinline__ uint32_t run_direct(const uint32_t* w, const PatDev& P) {
    uint32_t mk = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        bool h = w[k] == P.G[j];
        if (NW >= 2) h &= w[k + 1] == P.G[4 + j];
        if (NW >= 3) h &= w[k + 2] == P.G[8 + j];
        if (h) mk |= 1u << (4 * k + 3 - j);
      }
    return mk;
  }
};

// Run patterns c^m (period 1, m >= 7): the filter IS the exact test.  Each
// lane turns its 16 staged bytes per round into 16 "byte != c" bits (nothing
// to do when all 16 are c, one existence test when none is), pairs of lanes
// store them as words of the segment's nz bitmap (+ the m - 1 byte halo), and
// run1_lane_matches reads every start's verdict off that bitmap: a start
// survives iff no nz bit lies in [s, s + m).  delta = 0, no verification.
struct FiltRUN1 {
  static constexpr bool kRun1 = true;
};
template <class F, class = void>
struct is_run1 : std::false_type {};
template <class F>
struct is_run1<F, std::void_t<decltype(F::kRun1)>> : std::true_type {};
// nz bits of 16 bytes; sets anyc when a byte equals c (a start may survive nearby)
__device__ __forceinline__ uint32_t run1_nz16(const uint4& X, uint32_t c4, bool& anyc) {
  const uint32_t a = X.x ^ c4, b = X.y ^ c4, c = X.z ^ c4, d = X.w ^ c4;
  if (!(a | b | c | d)) {
    anyc = true;
    return 0u;
  }
  const uint32_t k = 0x01010101u;
  const uint32_t hz = (((a - k) & ~a) | ((b - k) & ~b) | ((c - k) & ~c) | ((d - k) & ~d)) & 0x80808080u;
  if (!hz) return 0xFFFFu;  // no byte equals c
  anyc = true;
  return ((~zero_bytes4(a)) & 0xFu) | (((~zero_bytes4(b)) & 0xFu) << 4) | (((~zero_bytes4(c)) & 0xFu) << 8) |
         (((~zero_bytes4(d)) & 0xFu) << 12);
}

// K2 / m <= 64, small alphabets (bitparallel.py:66-84 compile_sa, Shift-And,
// turned sideways): instead of one state word per text position, the text is
// packed into NP bit planes -- plane bit i = one chosen bit of text byte i, the
// bits picked by the planner so that the pattern's symbols get distinct codes
// (NP = 1 separates 2 symbols, NP = 2 up to 4) -- and every lane runs the
// bit-parallel AND over its 64 start positions at once:
//   M = AND_j ~((T >> j) ^ a_j),  a_j = plane bit of p[j], j in [a, a + D)
// i.e. 2 funnel shifts + 2 LOP3 per pattern position, plane and 64 starts.
// The planner picks the D <= SO_MAX_STEPS consecutive pattern positions that
// bring the expected survivors below 2^-16 per start (sigma = 2: 16 steps);
// survivors are verified like any other filter's candidates (verify_direct),
// which also rejects text bytes outside the pattern's alphabet (they alias to
// one of its codes).
template <int NP>
struct FiltSO {
  static constexpr bool kShiftOr = true;
  static constexpr int kNP = NP;
  static_assert(NP == 1 || NP == 2, "one or two symbol bit planes");
};

// 16 staged bytes -> 16 plane bits (bit i = selected bit of byte i).  Per word:
// mask the chosen bit of every byte, one IMAD gathers the four flags into the
// top nibble (mult = (2^28 + 2^21 + 2^14 + 2^7) >> bit: the partial products
// never overlap), one funnel shift appends it.
__device__ __forceinline__ uint32_t so_pack16(const uint4& X, uint32_t mask, uint32_t mult) {
  uint32_t acc = ((X.w & mask) * mult) >> 28;
  acc = __funnelshift_l((X.z & mask) * mult, acc, 4);
  acc = __funnelshift_l((X.y & mask) * mult, acc, 4);
  acc = __funnelshift_l((X.x & mask) * mult, acc, 4);
  return acc;
}

// `steps` AND steps over the 96-bit plane windows (a0, a1, a2) [and (b0, b1,
// b2)] of a lane's 64 starts; tab[k] = {shift, plane-A xor mask, plane-B xor
// mask, -}, one broadcast LDS.128 per step.
template <int NP>
__device__ __forceinline__ void so_and_steps(const uint4* tab, int steps, uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t b0, uint32_t b1, uint32_t b2, uint32_t& M0, uint32_t& M1) {
#pragma unroll 4
  for (int k = 0; k < steps; k++) {
    const uint4 e = tab[k];
    M0 &= __funnelshift_r(a0, a1, e.x) ^ e.y;
    M1 &= __funnelshift_r(a1, a2, e.x) ^ e.y;
    if constexpr (NP == 2) {
      M0 &= __funnelshift_r(b0, b1, e.x) ^ e.z;
      M1 &= __funnelshift_r(b1, b2, e.x) ^ e.z;
    }
  }
}
__device__ __forceinline__ uint32_t lds32u(const uint8_t* p);
// K1G / m >= Q + S - 1, small alphabets (plan.cpp choose_gram): the Q-byte gram
// at every S-th staged position x (S-aligned, S = 8 or 16) is hashed once and
// tested against the warp's blocked bloom of the pattern grams p[j..j+Q),
// j in [0, S) (gram_bloom_hash, 2 bits in one smem word); a bloom hit compares
// the gram with the S pattern grams in the staged pattern and marks bit
// x + S - 1 - j (delta = S - 1) for each equal one.  ~10 instructions per 16
// text bytes for S = 16 against ALIGNED's 32-48 compares at 2-3 anchor words.
template <int S, int Q>
struct FiltGRAM {
  static constexpr bool kGram = true;
  static constexpr int kS = S, kQ = Q;
  static_assert((S == 8 || S == 16) && (Q == 8 || Q == 16), "K1G variants");
};
template <class F, class = void>
struct is_gram : std::false_type {};
template <class F>
struct is_gram<F, std::void_t<decltype(F::kGram)>> : std::true_type {};

// w[0..5]: the lane's 16 staged bytes at x0 and the next 8; tab: the warp's
// GRAM_TABLE_WORDS (smem): bloom, then the S pattern gram hashes.  A bloom hit
// marks the offsets j whose gram hash equals the sample's (verified later).
template <int S, int Q>
__device__ __forceinline__ uint32_t gram_mask(const uint32_t* w, const uint32_t* tab) {
  uint32_t mk = 0;
#pragma unroll
  for (int t = 0; t < 16 / S; t++) {
    const uint32_t* g = w + t * (S / 4);
    const uint32_t h = gram_bloom_hash(g, Q / 4);
    const uint32_t bits = gram_bloom_bits(h);
    if ((tab[h >> 25] & bits) == bits) {  // rare
#pragma unroll
      for (int j = 0; j < S; j++)
        if (tab[GRAM_BLOOM_WORDS + j] == h) mk |= 1u << (t * S + S - 1 - j);
    }
  }
  return mk;
}

template <class F, class = void>
struct always_exact : std::false_type {};
template <class F>
struct always_exact<F, std::void_t<decltype(F::kAlwaysExact)>> : std::true_type {};

// Filters with a run_direct (the mask without the early-out test), used per
// warp while the previous segment had candidates (kernel_scan.cuh `busy`).
template <class F, class = void>
struct has_direct : std::false_type {};
template <class F>
struct has_direct<F, std::void_t<decltype(&F::run_direct)>> : std::true_type {};

template <class F, class = void>
struct is_shiftor : std::false_type {};
template <class F>
struct is_shiftor<F, std::void_t<decltype(F::kShiftOr)>> : std::true_type {};

// ------------------------------------------------------------ verification
// Direct window compare in shared memory (core.py:131-136 match_at), 4 bytes
// at a time: text words unaligned (lds32u), pattern 16-byte aligned.  Reads up
// to s + m + 4.
__device__ __forceinline__ uint32_t lds32u(const uint8_t* p) {  // unaligned 4-byte smem read
  // pointer arithmetic (not an integer round trip) keeps the shared address
  // space visible to the compiler: LDS, not generic LD
  const uint32_t mis = (uint32_t)((uintptr_t)p & 3);
  const uint32_t* b = reinterpret_cast<const uint32_t*>(p - mis);
  return __funnelshift_r(b[0], b[1], 8 * mis);
}
__device__ __forceinline__ bool verify_direct(const uint8_t* s, const uint8_t* pat, int m) {
  int k = 0;
  for (; k + 4 <= m; k += 4)
    if (lds32u(s + k) != *reinterpret_cast<const uint32_t*>(pat + k)) return false;
  if (k < m) {
    const uint32_t mask = (1u << (8 * (m - k))) - 1u;
    if ((lds32u(s + k) ^ *reinterpret_cast<const uint32_t*>(pat + k)) & mask) return false;
  }
  return true;
}

// Per-warp break bitmap of a segment: bit q of word i set iff
// t[y] != t[y + per] for y = y0 + 32 i + q (y relative to the segment's first
// start position).  nbw[i] = first break at or after word i (relative to y0).
__device__ __forceinline__ void warp_breaks(const uint8_t* Yseg, int per, int nwords, uint32_t* brk, int32_t* nbw);
// nbw[i] = first set bit of brk[] at or after word i (0x7fffffff if none);
// nbw[nwords] = none.  Reads brk[0..nwords).
__device__ __forceinline__ void warp_next_set(int nwords, const uint32_t* brk, int32_t* nbw) {
  const int lane = threadIdx.x & 31;
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

__device__ __forceinline__ void warp_breaks(const uint8_t* Yseg, int per, int nwords, uint32_t* brk, int32_t* nbw) {
  const int lane = threadIdx.x & 31;
  // 128 bytes (4 break words) per step, lane l on bytes [4l, 4l+4): consecutive
  // lanes read consecutive smem words (no bank conflicts); the 4-bit SWAR
  // results of 8 lanes are OR-combined into one break word
  for (int j = 0; 4 * j < nwords; j++) {
    const bool ok = 4 * j + (lane >> 3) < nwords;
    const uint8_t* q = Yseg + 128 * j + 4 * lane;
    uint32_t nib = ok ? ((~zero_bytes4(lds32u(q) ^ lds32u(q + per))) & 0xFu) << (4 * (lane & 7)) : 0u;
    nib |= __shfl_xor_sync(0xffffffffu, nib, 1);
    nib |= __shfl_xor_sync(0xffffffffu, nib, 2);
    nib |= __shfl_xor_sync(0xffffffffu, nib, 4);
    if (ok && (lane & 7) == 0) brk[4 * j + (lane >> 3)] = nib;
  }
  __syncwarp();
  warp_next_set(nwords, brk, nbw);
}

// OR a run of nbits (<= 32) flag bits into the bitmap at bit position y
__device__ __forceinline__ void or_bits(uint32_t* bm, int y, uint32_t bits) {
  if (!bits) return;
  atomicOr(&bm[y >> 5], bits << (y & 31));
  if (y & 31) {
    const uint32_t hi = bits >> (32 - (y & 31));
    if (hi) atomicOr(&bm[(y >> 5) + 1], hi);
  }
}

// Run patterns c^m (period 1): the exact match bits of this lane's 64 starts
// [64 l, 64 l + 64) of a segment, from its nz bitmap brk (bit y = start byte y
// is not c, words 0 .. nwords-1 cover the segment and its m - 1 byte halo;
// warp_run_nz without next-break arrays).  A start i survives iff no nz byte
// lies in [i, i + m): inside the lane by a width-m sliding OR of its 64 bits
// (m >= 64: nothing at or above i), past it by the first nz byte after the
// lane -- a warp suffix-min of the lanes' first nz bytes, lane 31 taking the
// first nz of the halo.  Replaces the next-break arrays and per-lane break
// walk of the general periodic test.  Call from all lanes.
__device__ __forceinline__ uint64_t run1_lane_matches(const uint32_t* brk, int nwords, int m, int lane) {
  const uint64_t z = ((uint64_t)brk[2 * lane + 1] << 32) | brk[2 * lane];
  int hfirst = 0x7fffffff;  // first nz of the halo words [SEG / 32, nwords)
  for (int i = SEG / 32 + lane; i < nwords; i += 32)
    if (brk[i]) {
      hfirst = 32 * i + __ffs(brk[i]) - 1;
      break;
    }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) hfirst = min(hfirst, __shfl_xor_sync(0xffffffffu, hfirst, d));
  const int first = z ? 64 * lane + __ffsll((long long)z) - 1 : 0x7fffffff;
  int suf = first;  // inclusive suffix-min over lanes
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_down_sync(0xffffffffu, suf, d);
    if (lane + d < 32) suf = min(suf, o);
  }
  int after = __shfl_down_sync(0xffffffffu, suf, 1);
  if (lane == 31) after = 0x7fffffff;
  after = min(after, hfirst);
  // start i survives the bytes after the lane iff i <= after - 64 l - m
  const int64_t T = (int64_t)after - 64 * lane - m;
  const uint64_t w2 = T < 0 ? 0ull : T >= 63 ? ~0ull : ((2ull << T) - 1ull);
  uint64_t w1;
  if (m >= 64) {  // no nz byte at or above i inside the lane
    const int hb = z ? 63 - __clzll((long long)z) : -1;
    w1 = hb == 63 ? 0ull : ~0ull << (hb + 1);
  } else {  // sliding OR of width m
    uint64_t r = z;
    int w = 1;
    while (2 * w <= m) r |= r >> w, w *= 2;
    if (w < m) r |= r >> (m - w);
    w1 = ~r;
  }
  return w1 & w2;
}

// Run patterns c^m (period 1): nz bitmap of the bytes != c over Y positions
// [0, 32 nwords) of a segment (Y0 + c0 = position 0).  The bulk [delta,
// delta + SEG) is the segment's own staged bytes, read as the filter read
// them (16 per lane and round, one LDS.128) and compared with c as words, so a
// clean chunk costs four compares; only the edge ranges go byte-exact through
// a warp loop.  Then nbw = next nz at or after each word.
__device__ __forceinline__ void warp_run_nz(const uint8_t* Yseg, const uint8_t* Sseg, int delta, uint32_t c4,
                                            int nwords, uint32_t* brk, int32_t* nbw, bool next = true) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < nwords; i += 32) brk[i] = 0;
  __syncwarp();
#pragma unroll
  for (int r = 0; r < SEG / 512; r++) {
    const uint4 X = *reinterpret_cast<const uint4*>(Sseg + r * 512 + lane * 16);
    const uint32_t a = X.x ^ c4, b = X.y ^ c4, c = X.z ^ c4, d = X.w ^ c4;
    if (a | b | c | d) {
      const uint32_t nz = ((~zero_bytes4(a)) & 0xFu) | (((~zero_bytes4(b)) & 0xFu) << 4) |
                          (((~zero_bytes4(c)) & 0xFu) << 8) | (((~zero_bytes4(d)) & 0xFu) << 12);
      or_bits(brk, delta + r * 512 + lane * 16, nz);
    }
  }
  // edges: [0, delta) and [delta + SEG, 32 nwords), 4 bytes per lane and step
  const int e1 = delta + SEG, end = 32 * nwords;
  const int n0 = (delta + 3) / 4, n1 = (end - e1 + 3) / 4;
  for (int q = lane; q < n0 + n1; q += 32) {
    const int y = q < n0 ? 4 * q : e1 + 4 * (q - n0);
    const int lim = q < n0 ? delta : end;
    uint32_t nz = (~zero_bytes4(lds32u(Yseg + y) ^ c4)) & 0xFu;
    if (lim - y < 4) nz &= (1u << (lim - y)) - 1u;
    or_bits(brk, y, nz);
  }
  __syncwarp();
  if (next) warp_next_set(nwords, brk, nbw);
}


}  // namespace mb
