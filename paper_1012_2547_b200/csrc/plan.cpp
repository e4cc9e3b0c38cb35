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

#include <cmath>
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

static inline int round16(int64_t x) { return (int)((x + 15) & ~(int64_t)15); }

// Anchor choice: the window of `len` pattern bytes whose bytes are rarest.  Byte
// rarity comes from the caller's text histogram when given, else from the
// pattern's own byte counts (a proxy: patterns are drawn from the text).  For
// a^(m-1)b in an 'a'-heavy text this picks the window holding 'b', keeping the
// candidate rate near the true match rate.
static int choose_anchor(const uint8_t* p, int64_t m, int len, const int64_t* hist) {
  double w[256];
  if (hist) {
    double tot = 0;
    for (int c = 0; c < 256; c++) tot += (double)hist[c];
    for (int c = 0; c < 256; c++) w[c] = std::log(((double)hist[c] + 0.5) / (tot + 128.0));
  } else {
    int64_t cnt[256] = {0};
    for (int64_t i = 0; i < m; i++) cnt[p[i]]++;
    for (int c = 0; c < 256; c++) w[c] = std::log(((double)cnt[c] + 0.5) / ((double)m + 128.0));
  }
  int best = 0;
  double best_s = 1e300;
  for (int64_t a = 0; a + len <= m; a++) {
    double s = 0;
    for (int k = 0; k < len; k++) s += w[p[a + k]];
    if (s < best_s - 1e-9) {
      best_s = s;
      best = (int)a;
    }
  }
  return best;
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
  if (fam == MB_FAM_AUTO) {
    if (m <= 3)
      fam = MB_FAM_SWAR;
    else if (m <= 6)
      fam = MB_FAM_WIN4;
    else
      fam = MB_FAM_ALIGNED;
  }
  if ((fam == MB_FAM_SWAR && m > 3) || (fam == MB_FAM_WIN4 && m < 4) ||
      (fam == MB_FAM_ALIGNED && m < 7) || (fam == MB_FAM_SHIFTOR && m > 64)) {
    *err = "requested kernel family does not apply at this pattern length";
    return MB_EINVAL;
  }
  ph->family = fam;
  PatDev& d = ph->dev;
  memset(&d, 0, sizeof(d));
  d.m = m;
  d.per = ph->period;
  d.family = fam;
  d.periodic = 0;
  d.L = 0;
  switch (fam) {
    case MB_FAM_SWAR:
      ph->anchor = 0;
      d.delta = 0;
      for (int j = 0; j < 3; j++) d.G[j] = (j < m) ? 0x01010101u * pat[j] : 0u;
      d.exact = 1;
      break;
    case MB_FAM_WIN4: {
      int a = choose_anchor(pat, m, 4, hist);
      ph->anchor = a;
      d.delta = a;
      d.G[0] = load_le32(pat + a);
      d.exact = (m == 4);
      break;
    }
    case MB_FAM_ALIGNED: {
      int a = choose_anchor(pat, m, 7, hist);
      ph->anchor = a;
      d.delta = a + 3;
      for (int j = 0; j < 4; j++) d.G[j] = load_le32(pat + a + j);
      d.exact = 0;
      // Long periodic patterns (a^m, (ab)^k ...) verify through the period /
      // break-run test so dense matches cost O(1) each.
      if (m >= 16 && ph->period <= m / 2) {
        d.periodic = 1;
        d.L = (int)(m - ph->period);
      }
      break;
    }
    case MB_FAM_SHIFTOR:
      ph->anchor = 0;
      d.delta = 0;
      d.exact = 1;
      break;
  }
  d.anchor = ph->anchor;
  // staged-tile margins (bytes before / after the tile's bit range)
  d.pre = round16(d.delta);
  d.post = round16(m - d.delta + 40) + 16;
  return MB_OK;
}

}  // namespace mb
