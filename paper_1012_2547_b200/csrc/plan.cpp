// plan.cpp -- host-side pattern preprocessing (H1) for the B200 engine.
//
// The compile_X(p) step of the reference (comparison.py:70-352,
// bitparallel.py:24-63) builds per-pattern tables once, outside the timed
// search.  Here a plan builds:
//   * the tables the reference defines, bit-identical to its functions
//     (Horspool / Quick-Search shifts, forward shift-and masks, KMP failure,
//     q-gram hashes) -- exposed through the C ABI and unit-tested against the
//     reference's own outputs (tests/golden/tables.json);
//   * the GPU scan parameters: kernel family, anchor window, bitmap shift,
//     smallest period, staged-tile margins.
#include "plan.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace mb {

// comparison.py:18-24 _horspool_table
void horspool_table(const uint8_t* p, int64_t m, int64_t* tbl) {
  for (int c = 0; c < 256; c++) tbl[c] = m;
  for (int64_t i = 0; i < m - 1; i++) tbl[p[i]] = m - 1 - i;
}

// comparison.py:27-33 _sunday_table
void sunday_table(const uint8_t* p, int64_t m, int64_t* tbl) {
  for (int c = 0; c < 256; c++) tbl[c] = m + 1;
  for (int64_t i = 0; i < m; i++) tbl[p[i]] = m - i;
}

// comparison.py:56-67 kmp_failure: fail[j] = longest proper border of p[:j]
void kmp_failure(const uint8_t* p, int64_t m, int64_t* fail) {
  for (int64_t j = 0; j <= m; j++) fail[j] = 0;
  int64_t k = 0;
  for (int64_t j = 1; j < m; j++) {
    while (k && p[j] != p[k]) k = fail[k];
    if (p[j] == p[k]) k++;
    fail[j + 1] = k;
  }
}

// bitparallel.py:24-29 forward_masks: bit j of table[c] set iff p[j] == c
void forward_masks(const uint8_t* p, int64_t m, uint64_t* out, int64_t words) {
  memset(out, 0, sizeof(uint64_t) * 256 * words);
  for (int64_t j = 0; j < m && j / 64 < words; j++) out[p[j] * words + j / 64] |= 1ULL << (j % 64);
}

// comparison.py:227-231 _gram_hash
uint32_t gram_hash(const uint8_t* s, int64_t start, int q) {
  uint32_t h = 0;
  for (int k = 0; k < q; k++) h = ((h << 1) + s[start + k]) & 0xFFFF;
  return h;
}

static inline uint32_t load_le32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// K2 (bit-plane Shift-And, device_common.cuh FiltSO): auto for small alphabets
// where the word filters are busy (see build_plan); costs ~0.75 operations per
// text byte and plane for the packing plus ~4.5 (one plane) / 8.5 (two) per
// pattern position and 64 starts, whatever the candidate density.
#ifndef MB_K2_LOG2_SURVIVORS
#define MB_K2_LOG2_SURVIVORS -16.0  // log2 of the expected survivors per start the AND steps aim for (one plane; two: +3)
#endif
#ifndef MB_K2_MAX_CAND
#define MB_K2_MAX_CAND (1.0 / 24)  // expected plane-code candidates per start above which verification dominates
#endif

// ALIGNED anchor-word thresholds (expected one-/two-word anchor hits per text
// word above which one more word is added); tuned on config 2.
#ifndef MB_SWAR_RATE
#define MB_SWAR_RATE 2e-2  // anchor hits per text word above which 5 <= m <= 8 take exact SWAR
#endif
#ifndef MB_SWAR_RATE4
#define MB_SWAR_RATE4 4e-3  // ... when the caller's text histogram shows at most 4 byte values (sigma <= 4: 1 GiB m = 5, 6 SWAR
                           // 0.29-0.31 ms vs WIN4 0.44; sigma = 8 keeps WIN4 / ALIGNED at 0.20-0.23)
#endif
#ifndef MB_ALIGNED2_RATE
#define MB_ALIGNED2_RATE 4e-3
#endif
#ifndef MB_ALIGNED3_RATE
#define MB_ALIGNED3_RATE 5e-2
#endif

static inline int round16(int64_t x) { return (int)((x + 15) & ~(int64_t)15); }


// K3 sampled q-gram filter: every occurrence of p contains the
// q-gram at exactly one text position x = S*i (S <= m - q + 1), at pattern offset
// j = x - s in [0, S).  The plan hashes the grams p[j..j+q), j in [0, S), into a
// 65536-bit bloom filter and bucketed offset lists.  Chosen only where sampling
// saves DRAM traffic (S >= 256: the fetch granule is a 128-byte line) and the
// filter stays selective: q * entropy(p) >= log2(S) + 12 bits and no gram occurs
// at more than 4 of the S offsets (periodic patterns keep the full scan).
static bool build_sampled(const uint8_t* pat, int64_t m, int64_t period, PlanHost* ph) {
  if (m < 272) return false;
  if (period < K3_MIN_PERIOD) return false;  // a unit's occurrences must fit the kernel's lists (plan.h)
  double cnt[256] = {0}, H = 0;
  for (int64_t i = 0; i < m; i++) cnt[pat[i]] += 1;
  for (int c = 0; c < 256; c++)
    if (cnt[c] > 0) H -= cnt[c] / m * std::log2(cnt[c] / m);
  for (int q : {4, 8, 16, 32}) {
    int64_t S = ((m - q + 1) / 16) * 16;
    if (S > 4096) S = 4096;
    if (S < 256) return false;
    if (q * H < std::log2((double)S) + 12) continue;
    const int nw = q / 4;
    int B = 1;
    while ((1 << B) < 2 * S && B < 10) B++;
    std::vector<uint32_t> hs(S);
    for (int64_t j = 0; j < S; j++) {
      uint32_t w[8];
      for (int k = 0; k < nw; k++) w[k] = load_le32(pat + j + 4 * k);
      hs[j] = gram_mix(w, nw);
    }
    // multiplicity of identical grams among the S offsets
    std::vector<int64_t> order(S);
    for (int64_t j = 0; j < S; j++) order[j] = j;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      int c = memcmp(pat + a, pat + b, q);
      return c < 0 || (c == 0 && a < b);
    });
    int maxmul = 1, run = 1;
    for (int64_t i = 1; i < S; i++) {
      run = memcmp(pat + order[i - 1], pat + order[i], q) == 0 ? run + 1 : 1;
      maxmul = std::max(maxmul, run);
    }
    if (maxmul > 4) continue;
    ph->bloom.assign(2048, 0u);
    ph->bstart.assign((1 << B) + 1, 0);
    ph->bent.assign(S, 0);
    std::vector<int> bc(1 << B, 0);
    for (int64_t j = 0; j < S; j++) {
      ph->bloom[hs[j] >> 21] |= 1u << ((hs[j] >> 16) & 31);
      bc[hs[j] >> (32 - B)]++;
    }
    for (int b = 0; b < (1 << B); b++) ph->bstart[b + 1] = (uint16_t)(ph->bstart[b] + bc[b]);
    std::vector<int> fillp(ph->bstart.begin(), ph->bstart.end() - 1);
    for (int64_t j = S - 1; j >= 0; j--) {  // descending j inside a bucket -> ascending start
      int b = hs[j] >> (32 - B);
      ph->bent[fillp[b]++] = (uint16_t)j;
    }
    PatDev& d = ph->dev;
    d.S = (int32_t)S;
    d.q = q;
    d.B = B;
    return true;
  }
  return false;
}

// Filter-rate model: expected anchor hits per aligned text word, with byte
// probabilities from the caller's text histogram or, as a proxy, the
// pattern's own byte counts, lightly smoothed (1.28 pseudo-counts spread over
// all 256 bytes: heavier smoothing hides a small alphabet from short patterns).
static void byte_probs(const uint8_t* p, int64_t m, const int64_t* hist, double* pr) {
  if (hist) {
    double tot = 0;
    for (int c = 0; c < 256; c++) tot += (double)hist[c];
    for (int c = 0; c < 256; c++) pr[c] = ((double)hist[c] + 0.5) / (tot + 128.0);
  } else {
    double cnt[256] = {0};
    for (int64_t i = 0; i < m; i++) cnt[p[i]] += 1;
    for (int c = 0; c < 256; c++) pr[c] = (cnt[c] + 0.005) / ((double)m + 1.28);
  }
}
static double gram_prob(const uint8_t* g, const double* pr) { return pr[g[0]] * pr[g[1]] * pr[g[2]] * pr[g[3]]; }

// ALIGNED with nw anchor words: the (4 nw + 3)-byte window minimising
// sum_j prod_w P(p[a+j+4w .. +4)), j = 0..3 (a word k of the text is a
// candidate when words k, k+1, .., k+nw-1 all equal their grams).
static int best_aligned(const uint8_t* p, int64_t m, const double* pr, int nw, double* rate) {
  int best = 0;
  double br = 1e300;
  for (int64_t a = 0; a + 4 * nw + 3 <= m; a++) {
    double r = 0;
    for (int j = 0; j < 4; j++) {
      double g = 1;
      for (int w = 0; w < nw; w++) g *= gram_prob(p + a + j + 4 * w, pr);
      r += g;
    }
    if (r < br * (1 - 1e-12)) br = r, best = (int)a;
  }
  *rate = br;
  return best;
}
// Anchor words for ALIGNED: one more word doubles the filter's compares but
// divides the candidate rate by ~P(gram); worth it once the one-word filter
// would send most segments down the verify path (small alphabets).
static int choose_aligned_words(const uint8_t* p, int64_t m, const double* pr) {
  double r1, r2, r3;
  best_aligned(p, m, pr, 1, &r1);
  if (m < 11 || r1 < MB_ALIGNED2_RATE) return 1;
  best_aligned(p, m, pr, 2, &r2);
  if (m < 15 || r2 < MB_ALIGNED3_RATE) return 2;
  best_aligned(p, m, pr, 3, &r3);
  return r3 < r2 ? 3 : 2;
}
// WIN4: one 4-byte window tested at all 4 byte phases of a word: 4 * P(gram).
static int best_win4(const uint8_t* p, int64_t m, const double* pr, double* rate) {
  int best = 0;
  double br = 1e300;
  for (int64_t a = 0; a + 4 <= m; a++) {
    const double r = 4 * gram_prob(p + a, pr);
    if (r < br * (1 - 1e-12)) br = r, best = (int)a;
  }
  *rate = br;
  return best;
}

// K1G strided q-gram filter: every occurrence s holds exactly one S-aligned
// virtual position x in [s, s + S), and p[x - s .. x - s + Q) lies inside the
// pattern when m >= Q + S - 1.  Variants (S, Q) in order of filter cost; the
// first whose expected true gram hits per 16 text bytes stay below
// GRAM_QUIET_RATE (a hit sends the warp's whole segment down the slow path,
// and a tile's stage is freed only when its slowest warp is done) is taken;
// failing that, the most selective one under GRAM_MAX_RATE or under the
// ALIGNED filter's own candidate rate (the same selectivity for a third of
// the instructions).
#ifndef MB_GRAM_QUIET_RATE
#define MB_GRAM_QUIET_RATE 2e-5
#endif
#ifndef MB_GRAM_MAX_RATE
#define MB_GRAM_MAX_RATE 1e-3
#endif
static bool choose_gram(const uint8_t* p, int64_t m, const double* pr, double aligned_rate16, int* S_out,
                        int* Q_out) {
  static const int variants[4][2] = {{16, 8}, {16, 16}, {8, 8}, {8, 16}};
  double best = 1e300;
  for (int pass = 0; pass < 2; pass++)
    for (const auto& v : variants) {
      const int S = v[0], Q = v[1];
      if (m < Q + S - 1) continue;
      double r = 0;
      for (int j = 0; j < S; j++) {
        double g = 1;
        for (int i = 0; i < Q; i++) g *= pr[p[j + i]];
        r += g;
      }
      r *= 16.0 / S;  // per 16 text bytes
      if (pass == 0 && r <= MB_GRAM_QUIET_RATE) {
        *S_out = S, *Q_out = Q;
        return true;
      }
      if (pass == 1 && r <= std::max(MB_GRAM_MAX_RATE, 2 * aligned_rate16) && r < best * (1 - 1e-9))
        best = r, *S_out = S, *Q_out = Q;
    }
  return best < 1e300;
}
static void build_gram_table(const uint8_t* p, int S, int Q, std::vector<uint32_t>* tab) {
  tab->assign(GRAM_TABLE_WORDS, 0u);
  for (int j = 0; j < S; j++) {
    uint32_t g[4] = {0, 0, 0, 0};
    for (int i = 0; i < Q / 4; i++) g[i] = load_le32(p + j + 4 * i);
    const uint32_t h = gram_bloom_hash(g, Q / 4);
    (*tab)[h >> 25] |= gram_bloom_bits(h);
    (*tab)[GRAM_BLOOM_WORDS + j] = h;
  }
}

// K2 symbol planes: NP text-byte bit positions whose values give the pattern's
// symbols distinct codes where possible -- chosen to minimise the expected
// candidate rate prod_j P(code(text byte) == code(p[j])) under the byte
// probabilities pr.  Returns that rate; bits[] = the chosen bit positions.
static double choose_planes(const uint8_t* p, int64_t m, const double* pr, int np, int* bits) {
  double best = 1e300;
  for (int b0 = 0; b0 < 8; b0++)
    for (int b1 = (np == 2 ? b0 + 1 : 8); b1 < (np == 2 ? 8 : 9); b1++) {
      double cls[4] = {0, 0, 0, 0};
      auto code = [&](int c) { return ((c >> b0) & 1) | (np == 2 ? ((c >> b1) & 1) << 1 : 0); };
      for (int c = 0; c < 256; c++) cls[code(c)] += pr[c];
      double lr = 0;
      for (int64_t j = 0; j < m; j++) lr += std::log(std::max(cls[code(p[j])], 1e-300));
      if (lr < best - 1e-12) best = lr, bits[0] = b0, bits[1] = np == 2 ? b1 : 0;
    }
  return std::exp(best);
}
// one plane while at most two byte values carry the text (each above 1%), else two
static int plane_count(const double* pr) {
  int d = 0;
  for (int c = 0; c < 256; c++) d += pr[c] > 0.01;
  return d <= 2 ? 1 : 2;
}

int build_plan(const uint8_t* pat, int64_t m, const mb_plan_opts* opts, PlanHost* ph, std::string* err) {
  if (m < 1) {
    *err = "pattern must have length >= 1";
    return MB_EINVAL;
  }
  if (m > MB_MAX_M) {
    *err = "pattern longer than MB_MAX_M (" + std::to_string(MB_MAX_M) + ")";
    return MB_EINVAL;
  }
  ph->m = m;
  ph->pat.assign(pat, pat + m);
  horspool_table(pat, m, ph->hor);
  sunday_table(pat, m, ph->sun);
  ph->kmp.assign(m + 1, 0);
  kmp_failure(pat, m, ph->kmp.data());
  ph->period = (int)(m - ph->kmp[m]);

  int fam = opts ? opts->family : MB_FAM_AUTO;
  const int64_t* hist = opts ? opts->hist : nullptr;
  {
    double cnt[256] = {0};
    for (int64_t i = 0; i < m; i++) cnt[pat[i]] += 1;
    ph->entropy = 0;
    for (int c = 0; c < 256; c++)
      if (cnt[c] > 0) ph->entropy -= cnt[c] / m * std::log2(cnt[c] / m);
  }
  if (fam == MB_FAM_AUTO) {
    if (m <= 3)
      fam = MB_FAM_SWAR;
    else if (m <= 6)
      fam = MB_FAM_WIN4;
    else
      fam = MB_FAM_ALIGNED;  // may become SAMPLED or WIN4 below
  }
  const bool auto_long = (opts == nullptr || opts->family == MB_FAM_AUTO) && fam == MB_FAM_ALIGNED;
  bool sampled_ok = false;
  if (fam == MB_FAM_AUTO || fam == MB_FAM_ALIGNED || fam == MB_FAM_SAMPLED) {
    PlanHost tmp;
    sampled_ok = build_sampled(pat, m, ph->period, &tmp);
    if (sampled_ok && (opts == nullptr || opts->family == MB_FAM_AUTO || opts->family == MB_FAM_SAMPLED)) {
      fam = MB_FAM_SAMPLED;
      ph->bloom.swap(tmp.bloom);
      ph->bstart.swap(tmp.bstart);
      ph->bent.swap(tmp.bent);
      ph->dev.S = tmp.dev.S;
      ph->dev.q = tmp.dev.q;
      ph->dev.B = tmp.dev.B;
    }
  }
  // Small alphabets, 5 <= m <= 8: the anchor filters would flag a large share
  // of the words (sigma = 2, m = 8: a quarter of them) and verify each
  // candidate; exact SWAR compares of every byte of every alignment cost ~4
  // operations per text byte instead (config 2 sigma = 2, m = 8).
  if ((opts == nullptr || opts->family == MB_FAM_AUTO) && m >= 5 && m <= 8 &&
      (fam == MB_FAM_WIN4 || fam == MB_FAM_ALIGNED)) {
    double pr[256], r;
    byte_probs(pat, m, hist, pr);
    if (fam == MB_FAM_WIN4)
      best_win4(pat, m, pr, &r);
    else
      best_aligned(pat, m, pr, 1, &r);
    // byte values carrying more than 1% of the text -- only with the caller's text
    // histogram: a 5-byte pattern cannot tell a 4-letter text from a 16-letter one
    // (half of the 5-byte patterns over 16 letters hold <= 4 distinct bytes)
    int nsym = 256;
    if (hist) {
      nsym = 0;
      for (int c = 0; c < 256; c++) nsym += pr[c] > 0.01;
    }
    if (r > MB_SWAR_RATE || (nsym <= 4 && r > MB_SWAR_RATE4)) fam = MB_FAM_SWAR;
  }
  if (auto_long && fam == MB_FAM_ALIGNED) {
    // ALIGNED tests 4 grams of one 7-byte window per word; WIN4 one gram at
    // every byte phase.  When the rare bytes of a pattern fit only one gram
    // (a^(m-1)b: 'aaab' vs three 'aaaa' grams) WIN4 is far more selective.
    double pr[256], ra, rw;
    byte_probs(pat, m, hist, pr);
    const int nw = (opts && opts->anchor_words) ? opts->anchor_words : choose_aligned_words(pat, m, pr);
    // only where ALIGNED would actually be busy (> 1 hit per 1000 words); an
    // invalid forced anchor_words is left for the ALIGNED case to reject
    if (nw >= 1 && nw <= 3 && 4 * nw + 3 <= m) {
      best_aligned(pat, m, pr, nw, &ra);
      best_win4(pat, m, pr, &rw);
      // WIN4 must win by 8x over the cheap one-word filter, by 2x over the
      // wider (costlier) multi-word ones
      const double margin = nw == 1 ? 8.0 : 2.0;
      if (ra > 1e-3 && margin * rw < ra && !(m >= 16 && ph->period <= m / 2)) fam = MB_FAM_WIN4;
    }
  }
  // Small alphabets: the ALIGNED filter needs 2-3 anchor words (8-12 word
  // compares per text word, ALU-bound at ~0.5 of the HBM roofline); the
  // strided gram filter hashes one 8- or 16-byte gram per 8-16 text bytes
  int gram_S = 0, gram_Q = 0;
  if (auto_long && fam == MB_FAM_ALIGNED && !(m >= 16 && ph->period <= m / 2) &&
      !(opts && opts->anchor_words)) {
    double pr[256];
    byte_probs(pat, m, hist, pr);
    double r1, rn;
    best_aligned(pat, m, pr, 1, &r1);  // one-word anchor hits per text word
    const int nw = choose_aligned_words(pat, m, pr);
    best_aligned(pat, m, pr, nw, &rn);
    if ((nw >= 2 || 4 * r1 > 1e-3) && choose_gram(pat, m, pr, 4 * rn, &gram_S, &gram_Q)) fam = MB_FAM_GRAM;
  }
  // K2 where the word filters are busy: exact SWAR at 5 <= m <= 8 (~m/2
  // operations per byte), WIN4 / ALIGNED flagging more than one word in 50,
  // multi-word ALIGNED, or a gram filter above its rate limit -- and two bit
  // planes tell the pattern's symbols apart well enough that the survivors
  // are mostly occurrences.  Periodic patterns keep the break-run test.
  const bool auto_fam = opts == nullptr || opts->family == MB_FAM_AUTO;
  if (auto_fam && m >= 5 && m <= 64 && !(m >= 16 && ph->period <= m / 2) && ph->period > 1 &&
      (fam == MB_FAM_SWAR || fam == MB_FAM_WIN4 || fam == MB_FAM_ALIGNED || fam == MB_FAM_GRAM)) {
    double pr[256], r = 0;
    byte_probs(pat, m, hist, pr);
    bool busy = fam == MB_FAM_SWAR;
    // (m >= 7 on WIN4: a rare byte confined to one gram, a^(m-1)b -- that window is more selective than the model says)
    if (fam == MB_FAM_WIN4) best_win4(pat, m, pr, &r), busy = m <= 6 && r > 2e-2;
    if (fam == MB_FAM_ALIGNED) {
      const int nw = (opts && opts->anchor_words) ? opts->anchor_words : choose_aligned_words(pat, m, pr);
      best_aligned(pat, m, pr, 1, &r);
      busy = !(opts && opts->anchor_words) && (nw >= 2 || r > 2e-2);
    }
    if (fam == MB_FAM_GRAM) {
      double g = 0;
      for (int j = 0; j < gram_S; j++) {
        double x = 1;
        for (int i = 0; i < gram_Q; i++) x *= pr[pat[j + i]];
        g += x;
      }
      busy = g * 16.0 / gram_S > MB_GRAM_MAX_RATE;  // (sigma = 2, m = 16..22: 0.40 ms; quieter variants run at 0.17-0.20)
    }
    if (busy) {
      // measured on 1 GiB texts (profiles/r2/k2_vs_swar_m5_8.json, after the SWAR flag
      // gather): K2 wins from m = 8 -- sigma = 2: 0.379 vs SWAR 0.400 ms (m = 7: 0.479 vs
      // 0.426), sigma = 4: 0.283 vs 0.300 (m = 5: 0.366 vs 0.306, m = 7: 0.291 vs 0.294);
      // m = 12..22 over binary texts 0.24-0.28 vs 0.40-0.44 for two-word ALIGNED
      int bits[2];
      const int np = plane_count(pr);
      const bool len_ok = m >= 8;
      if (len_ok && choose_planes(pat, m, pr, np, bits) <= MB_K2_MAX_CAND) fam = MB_FAM_SHIFTOR;
    }
  }
  if (opts && opts->family == MB_FAM_GRAM) {
    double pr[256];
    byte_probs(pat, m, hist, pr);
    if (!choose_gram(pat, m, pr, 0.0, &gram_S, &gram_Q)) {
      if (m < 15) {
        *err = "gram family needs m >= 15";
        return MB_EINVAL;
      }
      gram_S = 8, gram_Q = 8;
      if (m >= 23) gram_S = 16;
    }
  }
  if (opts && opts->family == MB_FAM_SAMPLED && !sampled_ok) {
    *err = "sampled q-gram family does not apply to this pattern (m < 272, low entropy or periodic)";
    return MB_EINVAL;
  }
  if ((fam == MB_FAM_SWAR && (m == 4 || m > 8)) || (fam == MB_FAM_WIN4 && m < 4) ||
      (fam == MB_FAM_ALIGNED && m < 7) || (fam == MB_FAM_SHIFTOR && m > 64)) {
    *err = "requested kernel family does not apply at this pattern length";
    return MB_EINVAL;
  }
  ph->family = fam;
  PatDev& d = ph->dev;
  {
    const int32_t S = d.S, q = d.q, B = d.B;
    memset(&d, 0, sizeof(d));
    d.S = S;
    d.q = q;
    d.B = B;
  }
  d.m = m;
  d.per = ph->period;
  d.family = fam;
  d.periodic = 0;
  d.L = 0;
  switch (fam) {
    case MB_FAM_SWAR:
      ph->anchor = 0;
      d.delta = 0;
      for (int j = 0; j < 8; j++) d.G[j] = (j < m) ? 0x01010101u * pat[j] : 0u;
      d.exact = 1;
      break;
    case MB_FAM_WIN4: {
      double pr[256], rw;
      byte_probs(pat, m, hist, pr);
      int a = best_win4(pat, m, pr, &rw);
      ph->anchor = a;
      d.delta = a;
      d.G[0] = load_le32(pat + a);
      d.exact = (m == 4);
      // m = 5, 6 (auto): even-offset windows of a 5-byte anchor (FiltWIN4E,
      // two compares per text word instead of four) unless they hit > 4x as often
      if ((opts == nullptr || opts->family == MB_FAM_AUTO) && (m == 5 || m == 6)) {
        int ae = 0;
        double re = 1e300;
        for (int64_t b = 0; b + 5 <= m; b++) {
          const double r = 2 * (gram_prob(pat + b, pr) + gram_prob(pat + b + 1, pr));
          if (r < re * (1 - 1e-12)) re = r, ae = (int)b;
        }
        if (re <= 4 * rw || re < 1e-4) {
          ph->anchor = ae;
          d.nw = 2;  // WIN4E
          d.delta = ae + 1;
          d.G[0] = load_le32(pat + ae);
          d.G[1] = load_le32(pat + ae + 1);
          d.exact = 0;
        }
      }
      break;
    }
    case MB_FAM_ALIGNED: {
      double pr[256], ra;
      byte_probs(pat, m, hist, pr);
      const bool per_verify = m >= 16 && ph->period <= m / 2;  // periodic: break-run test (below) does the work
      int nw = (opts && opts->anchor_words) ? opts->anchor_words : per_verify ? 1 : choose_aligned_words(pat, m, pr);
      if (nw < 1 || nw > 3 || 4 * nw + 3 > m) {
        *err = "anchor_words must be 1..3 with 4 * anchor_words + 3 <= m";
        return MB_EINVAL;
      }
      int a = best_aligned(pat, m, pr, nw, &ra);
      ph->anchor = a;
      d.nw = nw;
      d.delta = a + 3;
      for (int w = 0; w < nw; w++)
        for (int j = 0; j < 4; j++) d.G[4 * w + j] = load_le32(pat + a + j + 4 * w);
      d.exact = 0;
      // Long periodic patterns (a^m, (ab)^k ...) verify through the period /
      // break-run test so dense matches cost O(1) each.
      if (m >= 16 && ph->period <= m / 2) {
        d.periodic = 1;
        d.L = (int)(m - ph->period);
      }
      // c^m (any m this family takes): the exact run filter (FiltRUN1) -- bit b
      // is start b, the nz bitmap needs no anchor and nothing is verified
      if (ph->period == 1 && !(opts && opts->anchor_words)) {
        d.periodic = 1;
        d.L = (int)(m - 1);
        d.nw = 1;
        d.delta = 0;
        d.exact = 1;
        ph->anchor = 0;
      }
      break;
    }
    case MB_FAM_SHIFTOR: {
      // bitparallel.py:66-84 compile_sa on symbol bit planes (FiltSO): G[4 pl + ..] =
      // {byte-bit mask, gather multiplier}; the AND steps cover the D consecutive
      // pattern positions [a, a + D) whose codes are expected to survive at
      // <= 2^-16 (one plane) / 2^-13 (two) of the starts (fewest steps; at most SO_MAX_STEPS), as a
      // table of {shift, plane-A xor mask, plane-B xor mask, 0}: positions < 32
      // first (S entries), then >= 32 (q entries)
      double pr[256];
      byte_probs(pat, m, hist, pr);
      int bits[2];
      const int np = plane_count(pr);
      choose_planes(pat, m, pr, np, bits);
      double cls[4] = {0, 0, 0, 0};
      auto code = [&](int c) { return ((c >> bits[0]) & 1) | (np == 2 ? ((c >> bits[1]) & 1) << 1 : 0); };
      for (int c = 0; c < 256; c++) cls[code(c)] += pr[c];
      // windows reaching the survivor target beat those that do not; then fewer steps; then fewer survivors
      double target = np == 1 ? MB_K2_LOG2_SURVIVORS : MB_K2_LOG2_SURVIVORS + 3.0;
      if (const char* env = getenv("MB_K2_LOG2")) target = atof(env);  // tuning (tools/k2_check.sh)
      int best_a = 0, best_d = 0;
      double best_l = 1;
      bool best_ok = false;
      for (int64_t a = 0; a < m; a++) {
        double l = 0;
        int dd = 0;
        while (a + dd < m && dd < SO_MAX_STEPS && l > target) l += std::log2(std::max(cls[code(pat[a + dd])], 1e-300)), dd++;
        const bool ok = l <= target;
        const bool better = best_d == 0 || (ok && !best_ok) ||
                            (ok == best_ok && (ok ? (dd < best_d || (dd == best_d && l < best_l - 1e-9)) : l < best_l - 1e-9));
        if (better) best_a = (int)a, best_d = dd, best_l = l, best_ok = ok;
      }
      ph->anchor = best_a;
      d.delta = 0;
      d.exact = 0;
      d.nw = np;
      for (int pl = 0; pl < np; pl++) {
        d.G[4 * pl] = 0x01010101u << bits[pl];
        d.G[4 * pl + 1] = ((1u << 28) | (1u << 21) | (1u << 14) | (1u << 7)) >> bits[pl];
      }
      ph->bloom.clear();
      d.S = d.q = 0;
      for (int half = 0; half < 2; half++)
        for (int j = best_a; j < best_a + best_d; j++) {
          if ((j >= 32) != (half == 1)) continue;
          ph->bloom.push_back((uint32_t)(j & 31));
          ph->bloom.push_back(((pat[j] >> bits[0]) & 1) ? 0u : ~0u);
          ph->bloom.push_back(np == 2 && !((pat[j] >> bits[1]) & 1) ? ~0u : 0u);
          ph->bloom.push_back(0u);
          (half ? d.q : d.S)++;
        }
      ph->bstart.clear();
      ph->bent.clear();
      break;
    }
    case MB_FAM_GRAM:
      // as K3: the sample at x covers bits [x, x + S), b = s + S - 1
      ph->anchor = 0;
      d.S = gram_S;
      d.q = gram_Q;
      d.delta = gram_S - 1;
      d.exact = 0;
      build_gram_table(pat, gram_S, gram_Q, &ph->bloom);
      ph->bstart.clear();
      ph->bent.clear();
      break;
    case MB_FAM_SAMPLED:
      // bit b of the sample at x = S*i covers b in [x, x + S): b = s + S - 1
      ph->anchor = 0;
      d.delta = d.S - 1;
      d.exact = 0;
      break;
  }
  d.anchor = ph->anchor;
  // K5 (batched multi-pattern pass) grams: the one-word ALIGNED anchor, for
  // every pattern long enough, so any family can join a batched pass
  if (m >= 7) {
    double pr[256], r1;
    byte_probs(pat, m, hist, pr);
    d.mpa = best_aligned(pat, m, pr, 1, &r1);
    for (int j = 0; j < 4; j++) d.mpG[j] = load_le32(pat + d.mpa + j);
  }
  // staged-tile margins (bytes before / after the tile's bit range)
  d.pre = round16(d.delta);
  d.post = round16(m - d.delta + 40) + 16;
  if (fam == MB_FAM_SHIFTOR) d.post = std::max(d.post, 80);  // the 64-byte plane halo of a tile's last segment
  return MB_OK;
}

}  // namespace mb
