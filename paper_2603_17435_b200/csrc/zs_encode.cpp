// zs_encode.cpp -- host TCA-TBE compressor (Alg. 1) for libzs.so.
//
// Independent of oracle/ (no shared code).  Parallel over BlockTile rows with a
// deterministic merge: pass 1 counts in-window elements per BlockTile to
// fix every segment offset, pass 2 writes the bit-planes and the H / L segments.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/zs.h"
#include "zs_host.h"

namespace {

int n_workers(int64_t work_items) {
  unsigned hw = std::thread::hardware_concurrency();
  int n = (int)std::max(1u, std::min(hw, 64u));
  return (int)std::max<int64_t>(1, std::min<int64_t>(n, work_items));
}

template <class F>
void parallel_for(int64_t n, F&& f) {
  const int nw = n_workers(n);
  if (nw == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nw);
  for (int w = 0; w < nw; ++w)
    th.emplace_back([&, w]() {
      for (int64_t i = w; i < n; i += nw) f(i);
    });
  for (auto& t : th) t.join();
}

inline int64_t up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Geo {
  int64_t rows, cols, ld, prow, pcol, nbr, nbc, nbt;
};

Geo make_geo(int64_t rows, int64_t cols, int64_t ld) {
  Geo g{rows, cols, ld, up(rows, 64), up(cols, 64), 0, 0, 0};
  g.nbr = g.prow / 64;
  g.nbc = g.pcol / 64;
  g.nbt = g.nbr * g.nbc;
  return g;
}

// number of in-window (H) elements of BlockTile (br, bc); padding counts as in-window
int64_t bt_h_count(const uint16_t* w, const Geo& g, int64_t br, int64_t bc, int lo, int hi) {
  int64_t n = 0;
  const int64_t r0 = br * 64, c0 = bc * 64;
  const int64_t rv = std::min<int64_t>(64, g.rows - r0), cv = std::min<int64_t>(64, g.cols - c0);
  for (int64_t r = 0; r < rv; ++r) {
    const uint16_t* row = w + (r0 + r) * g.ld + c0;
    for (int64_t c = 0; c < cv; ++c) {
      const int e = (row[c] >> 7) & 0xFF;
      n += (e >= lo && e <= hi);
    }
  }
  return n + (64 * 64 - rv * cv);
}

void sizes_from_counts(const Geo& g, const std::vector<int64_t>& hcnt, zs_sizes* s) {
  s->rows = g.rows;
  s->cols = g.cols;
  s->padded_rows = g.prow;
  s->padded_cols = g.pcol;
  s->n_fragtiles = g.nbt * 64;
  s->n_blocktiles = g.nbt;
  int64_t hb = 0, lw = 0, mh = 0, ml = 0;
  for (int64_t b = 0; b < g.nbt; ++b) {
    const int64_t hseg = up(hcnt[b], 16), lseg = up(2 * (4096 - hcnt[b]), 16);
    hb += hseg;
    lw += lseg / 2;
    mh = std::max(mh, hseg);
    ml = std::max(ml, lseg);
  }
  s->h_bytes = hb;
  s->l_words = lw;
  s->max_h_seg_bytes = mh;
  s->max_l_seg_bytes = ml;
}

}  // namespace

namespace zs {

// 7 consecutive exponents with maximum coverage, first start wins ties (Alg. 1 line 3)
int window_start(const int64_t hist[256], int64_t* covered) {
  int64_t run = 0;
  for (int e = 0; e < 7; ++e) run += hist[e];
  int64_t best = run;
  int best_s = 0;
  for (int s = 1; s <= 249; ++s) {
    run += hist[s + 6] - hist[s - 1];
    if (run > best) {
      best = run;
      best_s = s;
    }
  }
  if (covered) *covered = best;
  return best_s;
}

void sizes_and_offsets(int64_t rows, int64_t cols, const uint32_t* hcnt, zs_sizes* s, uint64_t* offsets) {
  const Geo g = make_geo(rows, cols, cols);
  std::vector<int64_t> h(hcnt, hcnt + g.nbt);
  sizes_from_counts(g, h, s);
  if (offsets) {
    uint64_t ho = 0, lo = 0;
    for (int64_t b = 0; b < g.nbt; ++b) {
      offsets[2 * b] = ho;
      offsets[2 * b + 1] = lo;
      ho += (uint64_t)up(hcnt[b], 16);
      lo += (uint64_t)up(2 * (4096 - (int64_t)hcnt[b]), 16);
    }
    offsets[2 * g.nbt] = ho;
    offsets[2 * g.nbt + 1] = lo;
  }
}

}  // namespace zs

extern "C" zs_status zs_encode_bound(int64_t rows, int64_t cols, zs_sizes* s) {
  if (rows < 1 || cols < 1 || !s) return ZS_ERR_INVALID_ARG;
  const Geo g = make_geo(rows, cols, cols);
  s->rows = rows;
  s->cols = cols;
  s->padded_rows = g.prow;
  s->padded_cols = g.pcol;
  s->n_fragtiles = g.nbt * 64;
  s->n_blocktiles = g.nbt;
  s->h_bytes = g.nbt * 4096;
  s->l_words = g.nbt * 4096;
  s->max_h_seg_bytes = 4096;
  s->max_l_seg_bytes = 8192;
  return ZS_OK;
}

extern "C" zs_status zs_encode_measure(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int32_t* base_exp,
                                       int64_t* covered, zs_sizes* exact) {
  if (!w || rows < 1 || cols < 1 || ld < cols || !base_exp || !exact) return ZS_ERR_INVALID_ARG;
  const Geo g = make_geo(rows, cols, ld);
  // Phase I: exponent histogram over logical elements (Alg. 1 line 2)
  const int nw = n_workers(rows);
  std::vector<std::vector<int64_t>> part(nw, std::vector<int64_t>(256, 0));
  {
    std::vector<std::thread> th;
    for (int t = 0; t < nw; ++t)
      th.emplace_back([&, t]() {
        auto& h = part[t];
        for (int64_t r = t; r < rows; r += nw) {
          const uint16_t* row = w + r * ld;
          for (int64_t c = 0; c < cols; ++c) ++h[(row[c] >> 7) & 0xFF];
        }
      });
    for (auto& x : th) x.join();
  }
  int64_t hist[256] = {0};
  for (auto& h : part)
    for (int e = 0; e < 256; ++e) hist[e] += h[e];
  int64_t best = 0;
  const int best_s = zs::window_start(hist, &best);
  *base_exp = best_s - 1;  // line 4
  if (covered) *covered = best;
  std::vector<int64_t> hcnt(g.nbt);
  parallel_for(g.nbr, [&](int64_t br) {
    for (int64_t bc = 0; bc < g.nbc; ++bc) hcnt[br * g.nbc + bc] = bt_h_count(w, g, br, bc, best_s, best_s + 6);
  });
  sizes_from_counts(g, hcnt, exact);
  return ZS_OK;
}

extern "C" zs_status zs_encode(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int32_t base_exp,
                               const zs_sizes* cap, uint64_t* b1, uint64_t* b2, uint64_t* b3, uint8_t* h,
                               uint16_t* l, uint64_t* offsets, zs_sizes* actual, uint16_t* pad_word) {
  if (!w || rows < 1 || cols < 1 || ld < cols || !cap || !b1 || !b2 || !b3 || !offsets || !actual)
    return ZS_ERR_INVALID_ARG;
  if (base_exp < -1 || base_exp > 248) return ZS_ERR_INVALID_ARG;
  const Geo g = make_geo(rows, cols, ld);
  const int lo = base_exp + 1, hi = base_exp + 7;  // window [e_base+1, e_base+7]
  const uint16_t pad = (uint16_t)((base_exp + 1) << 7);

  std::vector<int64_t> hcnt(g.nbt);
  parallel_for(g.nbr, [&](int64_t br) {
    for (int64_t bc = 0; bc < g.nbc; ++bc) hcnt[br * g.nbc + bc] = bt_h_count(w, g, br, bc, lo, hi);
  });
  zs_sizes s;
  sizes_from_counts(g, hcnt, &s);
  if (cap->n_fragtiles < s.n_fragtiles || cap->n_blocktiles < s.n_blocktiles || cap->h_bytes < s.h_bytes ||
      cap->l_words < s.l_words)
    return ZS_ERR_CAPACITY;
  if ((s.h_bytes && !h) || (s.l_words && !l)) return ZS_ERR_INVALID_ARG;

  // offsets: exclusive prefix of padded segment sizes, plus the sentinel pair
  std::vector<int64_t> hoff(g.nbt + 1), loff(g.nbt + 1);
  hoff[0] = loff[0] = 0;
  for (int64_t b = 0; b < g.nbt; ++b) {
    hoff[b + 1] = hoff[b] + up(hcnt[b], 16);
    loff[b + 1] = loff[b] + up(2 * (4096 - hcnt[b]), 16);
  }
  for (int64_t b = 0; b <= g.nbt; ++b) {
    offsets[2 * b] = (uint64_t)hoff[b];
    offsets[2 * b + 1] = (uint64_t)loff[b];
  }

  // Phase II: per BlockTile, FragTiles in canonical order (TCT row-major, FragTile
  // column-major in the 2x2 grid), one byte of every plane per FragTile row.
  parallel_for(g.nbr, [&](int64_t br) {
    uint16_t tile[64][64];
    for (int64_t bc = 0; bc < g.nbc; ++bc) {
      const int64_t bt = br * g.nbc + bc;
      for (int r = 0; r < 64; ++r)
        for (int c = 0; c < 64; ++c) {
          const int64_t gr = br * 64 + r, gc = bc * 64 + c;
          tile[r][c] = (gr < rows && gc < cols) ? w[gr * ld + gc] : pad;
        }
      uint8_t* hp = h + hoff[bt];
      uint16_t* lp = l + loff[bt] / 2;
      int64_t nh = 0, nl = 0;
      for (int tct = 0; tct < 16; ++tct)
        for (int f = 0; f < 4; ++f) {
          const int r0 = (tct >> 2) * 16 + (f & 1) * 8;
          const int c0 = (tct & 3) * 16 + (f >> 1) * 8;
          uint64_t p1 = 0, p2 = 0, p3 = 0;
          for (int rr = 0; rr < 8; ++rr) {
            uint32_t y1 = 0, y2 = 0, y3 = 0;
            for (int cc = 0; cc < 8; ++cc) {
              const uint16_t v = tile[r0 + rr][c0 + cc];
              const int e = (v >> 7) & 0xFF;
              if (e >= lo && e <= hi) {
                const uint32_t code = (uint32_t)(e - base_exp);
                y1 |= (code & 1u) << cc;
                y2 |= ((code >> 1) & 1u) << cc;
                y3 |= ((code >> 2) & 1u) << cc;
                hp[nh++] = (uint8_t)(((v >> 8) & 0x80) | (v & 0x7F));
              } else {
                lp[nl++] = v;
              }
            }
            p1 |= (uint64_t)y1 << (8 * rr);
            p2 |= (uint64_t)y2 << (8 * rr);
            p3 |= (uint64_t)y3 << (8 * rr);
          }
          const int64_t ft = bt * 64 + tct * 4 + f;
          b1[ft] = p1;
          b2[ft] = p2;
          b3[ft] = p3;
        }
      // zero padding up to the 16-byte segment boundary
      for (int64_t i = nh; i < hoff[bt + 1] - hoff[bt]; ++i) hp[i] = 0;
      for (int64_t i = nl; i < (loff[bt + 1] - loff[bt]) / 2; ++i) lp[i] = 0;
    }
  });
  *actual = s;
  if (pad_word) *pad_word = pad;
  return ZS_OK;
}
