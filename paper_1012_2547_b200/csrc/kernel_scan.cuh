// kernel_scan.cuh -- scan_kernel<Filter>: warp-specialised TMA ring, one 2 KiB segment per consumer warp (K1 filters, K1G gram, RUN1, K2 bit-plane Shift-And)
// (part of libmatchb200; included by engine.cu)
#pragma once

namespace mb {

// ---------------------------------------------------------------- kernel 1: scan
// FUSED (single-wave search of one pattern, grid = tiles, all resident): every
// CTA takes ONE tile; its consumer warps keep their segment's match bits in
// registers, the CTA's count goes through a warp look-back over the tiles (in
// ticket order) and the positions are written straight to the output -- the
// whole search is this one launch (fused_emit).
__device__ __forceinline__ void fused_emit(const ScanParams& P, int64_t tk, uint32_t cnt, uint32_t ex, uint32_t w0,
                                           uint32_t w1, int64_t pos0, int warp, int lane) {
  __shared__ uint32_t s_wc[NWARP];
  __shared__ int64_t s_base;
  if (tk < 0) {  // no tile (cannot happen with grid = tiles): still count this CTA for the reset
    if (warp == 0 && lane == 0 && atomicAdd(&P.ticket[TICKET_DONE], 1ULL) == (unsigned long long)(gridDim.x - 1))
      for (int i = 0; i < NTICKETS; i++) P.ticket[i] = 0ULL;
    return;
  }
  if (lane == 0) s_wc[warp] = cnt;
  consumer_sync();
  uint32_t tot = 0, before = 0;
#pragma unroll
  for (int w = 0; w < NWARP; w++) {
    const uint32_t x = s_wc[w];
    tot += x;
    before += w < warp ? x : 0u;
  }
  if (warp == 0) {
    int64_t excl = warp_lookback(P.state, tk, tot, P.epoch, lane);
    if (lane == 0) {
      excl += P.out_base ? *P.out_base : 0;
      s_base = excl;
      if (tk == P.ntiles - 1) P.offsets_plus1[0] = excl + tot;
      if (tk == 0 && P.csr0) *P.csr0 = 0;
    }
  }
  consumer_sync();
  if (P.out) {
    int64_t o = s_base + before + ex;
    const int64_t p = pos0 + 64 * lane;
    uint64_t bits = ((uint64_t)w1 << 32) | w0;
    while (bits) {
      const int i = __ffsll((long long)bits) - 1;
      bits &= bits - 1;
      if (o < P.cap) P.out[o] = p + i;
      o++;
    }
  }
  // every CTA took its ticket before its tile arrived: the last one to get
  // here zeroes all slots (tile tickets, this counter, both expand slots)
  if (warp == 0 && lane == 0 && atomicAdd(&P.ticket[TICKET_DONE], 1ULL) == (unsigned long long)(gridDim.x - 1))
    for (int i = 0; i < NTICKETS; i++) P.ticket[i] = 0ULL;
}

// Warp-specialised: warp NWARP is the TMA producer (ticket -> bulk copies of
// the tile+halo and of the pattern into a free stage), warps 0..NWARP-1 are
// consumers that each own one SEG-position segment of every tile.  Stages are
// handed over through full/empty mbarriers; there is no block-wide barrier in
// the loop, so warps drift independently within the ring.
template <class Filt, bool FUSED>
__global__ void __launch_bounds__(NT + 32, is_shiftor<Filt>::value ? 2 : 0) scan_kernel(const ScanParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + SM_HDR);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM_FULL);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + SM_EMPTY);
  uint8_t* stages = smem + SM_STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  MB_TRACE_MARK(0);
  pdl_trigger();  // the next grid (another family's scan, offsets) may be scheduled as SMs drain
  // count kernels of a batch are programmatic dependent launches: each waits
  // here for its predecessor -- transitively for the batch pass, whose
  // prologue zeroes the counts and whose flags gate the fallback scans -- so
  // launches that exit at once (pass did not overflow) overlap instead of
  // costing ~2.5 us each (a no-op when launched without the attribute)
  pdl_wait();
  if (P.run_if && *P.run_if == 0u) return;  // conditional fallback launch (MP did not overflow)
  const int NS = P.nstages;
  uint32_t* bm = reinterpret_cast<uint32_t*>(stages + NS * P.stage_bytes) + warp * SEG_WORDS;
  uint32_t* brk = reinterpret_cast<uint32_t*>(stages + NS * P.stage_bytes + NWARP * SEG_WORDS * 4) +
                  warp * 2 * (P.brk_words + 4);
  int32_t* nbw = reinterpret_cast<int32_t*>(brk + P.brk_words + 4);
  uint32_t* so_s = reinterpret_cast<uint32_t*>(stages + NS * P.stage_bytes + NWARP * SEG_WORDS * 4 +
                                               NWARP * 2 * (P.brk_words + 4) * 4) +
                   warp * SO_WARP_WORDS;  // K2 only: per-warp symbol bit planes of the segment + AND-step table
  (void)so_s;
  uint32_t* gbl = reinterpret_cast<uint32_t*>(stages + NS * P.stage_bytes + NWARP * SEG_WORDS * 4 +
                                              NWARP * 2 * (P.brk_words + 4) * 4) +
                  warp * GRAM_TABLE_WORDS;  // K1G only: per-warp gram bloom + hashes (same region as K2's masks)
  (void)gbl;

  if (tid == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NWARP) {  // ---------------- producer
    if (lane == 0) {
      // ring position without divisions: stage s, its use count's parity ph
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0;; it++) {
        if (it >= NS) mbar_wait(&empty[s], ph ^ 1u);
        unsigned long long tk;
        int kg = 0, k = 0;
        for (;;) {
          tk = atomicAdd(&P.ticket[P.ticket_slot], 1ULL);
          if ((int64_t)tk >= P.group_tiles) break;
          int64_t tau_unused;
          split_tile((int64_t)tk, P.ntiles, &kg, &tau_unused);
          k = P.plist ? P.plist[kg] : kg;  // this launch's family group -> batch index
          if (!P.need || P.need[k]) break;
          // covered by the batch pass: jump the counter to the next pattern's tiles
          atomicMax(&P.ticket[P.ticket_slot], (unsigned long long)(kg + 1) * (unsigned long long)P.ntiles);
        }
        if ((int64_t)tk >= P.group_tiles) {
          hdr[s].tk = -1;
          mbar_arrive(&full[s]);
          break;
        }
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
        if (FUSED) break;  // one tile per CTA (the consumers stop after it)
        if (++s == NS) s = 0, ph ^= 1u;
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int c0 = warp * SEG;  // this warp's segment of every tile
  int cur_k = -1;
  PatDev pd;
  int64_t blo = 0, bhi = -1;
  int s = 0;
  uint32_t ph = 0;
  uint32_t f_w0 = 0, f_w1 = 0, f_ex = 0, f_cnt = 0;  // FUSED: the one tile's results
  int64_t f_tk = -1, f_pos0 = 0;
  bool busy = false;  // the previous segment had candidates (has_direct filters: masks without the early-out)
  for (;; s = (s + 1 == NS) ? (ph ^= 1u, 0) : s + 1) {
    mbar_wait(&full[s], ph);
    const int64_t tk = hdr[s].tk;
    if (tk < 0) break;
    const int k = hdr[s].k;
    if (k != cur_k) {  // per-pattern parameters stay in registers across tiles
      pd = P.pats[k];
      blo = P.off + pd.delta;               // valid bits: s = b - delta - off in [0, n-m]
      bhi = P.off + pd.delta + P.n - pd.m;  // inclusive (may be < blo)
      cur_k = k;
      if constexpr (is_shiftor<Filt>::value) {  // this warp's copy of the pattern's AND-step table
        __syncwarp();
        for (int i = lane; i < 4 * (pd.S + pd.q); i += 32) so_s[2 * SO_PLANE_WORDS + i] = pd.bloom[i];
        __syncwarp();
      }
      if constexpr (is_gram<Filt>::value) {  // this warp's copy of the pattern's gram bloom
        __syncwarp();
        for (int i = lane; i < GRAM_TABLE_WORDS; i += 32) gbl[i] = pd.bloom[i];
        __syncwarp();
      }
    }
    const int64_t B0 = hdr[s].tau * TILE;
    const uint8_t* spat = stages + s * P.stage_bytes;
    const uint8_t* S = spat + P.pat_cap + P.pre;  // S[c] = virtual text byte B0 + c
    const uint8_t* const sbeg = spat + P.pat_cap;  // staged text window [sbeg, send)
    const uint8_t* const send = spat + P.stage_bytes;
    (void)sbeg, (void)send;
    MB_CHECK(S + c0 + SEG + 8 <= send);
    const int64_t segb = B0 + c0;
    const bool interior = segb >= blo && segb + SEG - 1 <= bhi;

    // this lane's 64 positions of the segment: linear bitmap words 2*lane, 2*lane+1
    uint32_t w0 = 0, w1 = 0;
    bool have;
    if constexpr (is_run1<Filt>::value) {
      // ---- c^m: nz bitmap of the segment + halo straight from the staged bytes
      const uint32_t c4 = 0x01010101u * spat[0];
      const int hw = ((int)pd.m + 30) >> 5;  // halo words covering m - 1 bits
      MB_CHECK(S + c0 + SEG + 32 * hw <= send);
      bool anyc = false;
      __syncwarp();  // the previous segment's bitmap has been read
#pragma unroll
      for (int r = 0; r < SEG / 512; r++) {
        const uint4 X = *reinterpret_cast<const uint4*>(S + c0 + r * 512 + lane * 16);
        const uint32_t nz = run1_nz16(X, c4, anyc);
        const uint32_t o = __shfl_down_sync(0xffffffffu, nz, 1);
        if (!(lane & 1)) brk[r * 16 + (lane >> 1)] = nz | (o << 16);
      }
      for (int h = 0; h < 2 * hw; h += 32) {  // halo: 16 bytes per lane, 2 hw lanes (hw <= 32)
        const int l2 = h + lane;
        uint32_t nz = 0xFFFFu;
        if (l2 < 2 * hw) {
          bool dummy = false;  // a c byte in the halo alone starts nothing in this segment
          nz = run1_nz16(*reinterpret_cast<const uint4*>(S + c0 + SEG + l2 * 16), c4, dummy);
        }
        const uint32_t o = __shfl_down_sync(0xffffffffu, nz, 1);
        if (!(lane & 1) && l2 < 2 * hw) brk[SEG / 32 + (l2 >> 1)] = nz | (o << 16);
      }
      have = __any_sync(0xffffffffu, anyc);
      if (have) {
        __syncwarp();
        const uint64_t mm = run1_lane_matches(brk, SEG / 32 + hw, (int)pd.m, lane);
        w0 = (uint32_t)mm;
        w1 = (uint32_t)(mm >> 32);
        if (!interior) {
          const int64_t b = segb + 64 * lane;
          uint64_t vm = 0;
          for (int i = 0; i < 64; i++)
            if (b + i >= blo && b + i <= bhi) vm |= 1ULL << i;
          w0 &= (uint32_t)vm;
          w1 &= (uint32_t)(vm >> 32);
        }
        have = __any_sync(0xffffffffu, (w0 | w1) != 0);
      }
    } else if constexpr (is_shiftor<Filt>::value) {
      // ---- K2: the segment's bytes packed into symbol bit planes (16 bytes
      // per lane and round, even lanes store a 32-bit plane word; lanes 0..3
      // add the 64-byte halo), then each lane ANDs the pattern's m shifted
      // plane words over its 64 starts [c0 + 64 lane, +64) (so_and_steps)
      constexpr int NP = Filt::kNP;
      MB_CHECK(S + c0 + SEG + 64 <= send);
      __syncwarp();  // the previous segment's plane words have been read
#pragma unroll
      for (int r = 0; r <= SEG / 512; r++) {
        if (r == SEG / 512 && lane >= 4) break;
        const uint4 X = *reinterpret_cast<const uint4*>(S + c0 + r * 512 + lane * 16);
#pragma unroll
        for (int pl = 0; pl < NP; pl++) {
          const uint32_t a = so_pack16(X, pd.G[4 * pl], pd.G[4 * pl + 1]);
          const uint32_t o = __shfl_down_sync(r == SEG / 512 ? 0xFu : 0xffffffffu, a, 1);
          if (!(lane & 1)) so_s[pl * SO_PLANE_WORDS + r * 16 + (lane >> 1)] = a | (o << 16);
        }
      }
      __syncwarp();
      w0 = w1 = 0xFFFFFFFFu;
      uint2 ta[2], tb[2];
#pragma unroll
      for (int pl = 0; pl < NP; pl++) {
        ta[pl] = *reinterpret_cast<const uint2*>(so_s + pl * SO_PLANE_WORDS + 2 * lane);
        tb[pl] = *reinterpret_cast<const uint2*>(so_s + pl * SO_PLANE_WORDS + 2 * lane + 2);
      }
      if constexpr (NP == 1) ta[1] = tb[1] = make_uint2(0u, 0u);
      // pd.S steps at pattern positions < 32 (window words 0..2), pd.q at >= 32 (words 1..3)
      const uint4* tab = reinterpret_cast<const uint4*>(so_s + 2 * SO_PLANE_WORDS);
      so_and_steps<NP>(tab, pd.S, ta[0].x, ta[0].y, tb[0].x, ta[1].x, ta[1].y, tb[1].x, w0, w1);
      if (pd.q) so_and_steps<NP>(tab + pd.S, pd.q, ta[0].y, tb[0].x, tb[0].y, ta[1].y, tb[1].x, tb[1].y, w0, w1);
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
        const uint2 Y = *reinterpret_cast<const uint2*>(S + c + 16);
        const uint32_t w[6] = {X.x, X.y, X.z, X.w, Y.x, Y.y};
        if constexpr (is_gram<Filt>::value)
          mk[r] = gram_mask<Filt::kS, Filt::kQ>(w, gbl);
        else if constexpr (has_direct<Filt>::value)
          mk[r] = busy ? Filt::run_direct(w, pd) : Filt::run(w, pd);
        else
          mk[r] = Filt::run(w, pd);
        anyc |= (mk[r] != 0);
      }
      have = __any_sync(0xffffffffu, anyc);
      busy = have;
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
      if (!always_exact<Filt>::value && !pd.exact &&
          __any_sync(0xffffffffu, (w0 | w1) != 0)) {
        const uint8_t* Y0 = S - pd.delta;  // Y0[rel] = text byte at the start position of tile bit rel
        if (pd.periodic) {
          // s matches <=> t[s..s+per) = p[0..per) and no break t[y] != t[y+per] for
          // y in [s, s+L).  A break y kills starts [y-L+1, y]: walk the few breaks
          // that reach this lane's 64 starts, mask them out in bulk.
          // Period 1 (c^m): the same test with "byte != c" for "break" and
          // m for L, built from word compares of the staged segment.
          const int Lk = pd.per == 1 ? (int)pd.m : pd.L;
          const int nwords = (SEG + Lk + 31) / 32;
          MB_CHECK(Y0 + c0 >= sbeg && Y0 + c0 + 32 * nwords + pd.per + 8 <= send);
          if (pd.per == 1)
            warp_run_nz(Y0 + c0, S + c0, pd.delta, 0x01010101u * spat[0], nwords, brk, nbw);
          else
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
            for (int y = nb(q0); y != 0x7fffffff && y - Lk + 1 <= q1; y = nb(y + 1)) {
              const int lo = max(q0, y - Lk + 1) - q0, hi = min(q1, y) - q0;
              if (lo <= hi) killed |= (hi - lo == 63) ? ~0ULL : (((1ULL << (hi - lo + 1)) - 1) << lo);
              if (y >= q1) break;
            }
            cand &= ~killed;
            if (pd.per > 4) {  // the 4 anchor bytes do not cover a full period: check one block
              uint64_t cc = cand;
              while (cc) {
                const int i = __ffsll((long long)cc) - 1;
                cc &= cc - 1;
                MB_CHECK(Y0 + c0 + q0 + i >= sbeg && Y0 + c0 + q0 + i + pd.per + 4 <= send);
                if (!verify_direct(Y0 + c0 + q0 + i, spat, pd.per)) cand &= ~(1ULL << i);
              }
            }
          }
          w0 = (uint32_t)cand;
          w1 = (uint32_t)(cand >> 32);
        } else if (pd.m >= 64) {
          // long windows: each lane rejects its candidates on the first 16
          // bytes; the survivors (rare unless the window really matches) are
          // verified by the whole warp one at a time, lane l comparing 4-byte
          // words l, l+32, ... -- long partial matches cost m/128 steps, not m/4
          uint64_t mine = ((uint64_t)w1 << 32) | w0, surv = 0;
          {
            const uint4 p16 = *reinterpret_cast<const uint4*>(spat);
            uint64_t cc = mine;
            while (cc) {
              const int i = __ffsll((long long)cc) - 1;
              cc &= cc - 1;
              const uint8_t* tw = Y0 + c0 + 64 * lane + i;
              MB_CHECK(tw >= sbeg && tw + 24 <= send);
              if (lds32u(tw) == p16.x && lds32u(tw + 4) == p16.y && lds32u(tw + 8) == p16.z &&
                  lds32u(tw + 12) == p16.w)
                surv |= 1ULL << i;
            }
          }
          mine = surv;
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
              MB_CHECK(tw >= sbeg && tw + pd.m + 8 <= send);  // lds32u reads up to tw + k + 8
              bool bad = false;
              for (int k = 16 + 4 * lane; k < pd.m; k += 128) {
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
              MB_CHECK(Y0 + c0 + 32 * (2 * lane + h) + i >= sbeg && Y0 + c0 + 32 * (2 * lane + h) + i + pd.m + 4 <= send);
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
      cnt = __reduce_add_sync(0xffffffffu, c2);  // one REDUX; the prefix scan only where offsets are needed
      auto prefix = [&]() -> uint32_t {  // exclusive prefix of c2 over the lanes
        uint32_t inc = c2;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += o;
        }
        return inc - c2;
      };
      if constexpr (FUSED) {
        f_w0 = w0, f_w1 = w1, f_ex = prefix();
      } else {
        const int64_t g = tk * NWARP + warp;
        if (cnt <= LIST_CAP) {
          uint32_t j = prefix();
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
    }
    if constexpr (FUSED) f_cnt = cnt, f_tk = tk, f_pos0 = B0 + c0 - P.off - pd.delta;
    if (lane == 0) {
      if constexpr (!FUSED) P.counts[tk * NWARP + warp] = (uint16_t)cnt;
      mbar_arrive(&empty[s]);
    }
    if constexpr (FUSED) break;
  }
  if constexpr (FUSED) fused_emit(P, f_tk, f_cnt, f_ex, f_w0, f_w1, f_pos0, warp, lane);
  MB_TRACE_MARK(1);
}


}  // namespace mb
