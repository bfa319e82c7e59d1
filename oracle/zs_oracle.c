/*
 * zs_oracle.c -- plain, slow, obviously-correct CPU oracle for TCA-TBE / ZipGEMM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the product (paper_2603_17435_b200/).
 *
 * Citations: P:<line> = /root/reference/PAPER.md, S:<line> = /root/reference/SPEC.md
 * (both read while writing; nothing here reads them at run time).
 *
 *   bf16 fields ............ P:164-166 (Sec 2.2)
 *   histogram/window ....... Alg. 1 lines 2-4; S:110-127 (ties -> smallest start)
 *   tile encoding .......... Alg. 1 Phase II; layout ledger S:274-281
 *   canonical order ........ P:361 (FragTiles column-major inside a TensorCoreTile)
 *   sequential decoder ..... S:324-332 (inverse of Alg. 1)
 *   lane (Alg. 2) decoder .. Alg. 2; worked text P:431-437
 *   fp64 GEMM .............. Y = X W^T (north star; paper's Y = W X), fp64 accumulation
 *
 * Everything is done element by element in the paper's order; no blocking or fusion.
 * Return codes: 0 ok, negative = error (documented per function).
 */
#include <stdint.h>
#include <string.h>
#include <math.h>

/* ---------------------------------------------------------------- bf16 fields */
/* sign = bit 15, exponent = bits 14..7, mantissa = bits 6..0 */
int or_split_fields(uint16_t w, int *sign, int *exponent, int *mantissa)
{
    *sign = (w >> 15) & 1;
    *exponent = (w >> 7) & 0xFF;
    *mantissa = w & 0x7F;
    return 0;
}

/* MakeBF16(sign, e, mantissa) (Alg. 2 line 17); -1 on out-of-range fields */
int or_assemble_fields(int sign, int exponent, int mantissa, uint16_t *w)
{
    if (sign < 0 || sign > 1 || exponent < 0 || exponent > 255 || mantissa < 0 || mantissa > 127)
        return -1;
    *w = (uint16_t)((sign << 15) | (exponent << 7) | mantissa);
    return 0;
}

/* Pack(sign, mantissa) (Alg. 1): bit 7 = sign, bits 6..0 = mantissa */
uint8_t or_pack_sm(int sign, int mantissa) { return (uint8_t)((sign << 7) | mantissa); }
void or_unpack_sm(uint8_t b, int *sign, int *mantissa) { *sign = b >> 7; *mantissa = b & 0x7F; }

/* ---------------------------------------------------------------- Phase I (Alg. 1 l.2-4) */
/* ComputeExponentHistogram(W): counts[E] = #words with exponent field E */
void or_histogram(const uint16_t *w, int64_t n, int64_t counts[256])
{
    for (int e = 0; e < 256; e++) counts[e] = 0;
    for (int64_t i = 0; i < n; i++) {
        int s, e, m;
        or_split_fields(w[i], &s, &e, &m);
        counts[e] += 1;
    }
}

/* SelectTop7ConsecutiveExponents: the window [s, s+6] of 7 numerically consecutive
 * exponents with maximum coverage, brute force over all 250 starts,
 * ties -> smallest start.  Returns -1 if the histogram is empty. */
int or_select_window(const int64_t counts[256], int *start, int64_t *covered)
{
    int64_t total = 0;
    for (int e = 0; e < 256; e++) total += counts[e];
    if (total == 0) return -1;
    int best_s = -1;
    int64_t best_cov = -1;
    for (int s = 0; s + 6 <= 255; s++) {
        int64_t cov = 0;
        for (int j = 0; j < 7; j++) cov += counts[s + j];
        if (cov > best_cov) { best_cov = cov; best_s = s; }
    }
    *start = best_s;
    *covered = best_cov;
    return 0;
}

/* ---------------------------------------------------------------- tiling */
/* Position of element `pos` (0..63) of FragTile `f` (0..3, column-major inside the 2x2
 * grid of its TensorCoreTile) of TensorCoreTile `t` (0..15, row-major 4x4 inside the
 * BlockTile) of BlockTile (br, bc): returns padded matrix (row, col). */
static void or_coords(int64_t br, int64_t bc, int t, int f, int pos, int64_t *row, int64_t *col)
{
    int tr = t / 4, tc = t % 4;         /* TCT row-major within BlockTile      */
    int fr = f % 2, fc = f / 2;         /* FragTile column-major within TCT    */
    int er = pos / 8, ec = pos % 8;     /* pos = row*8 + col, LSB first        */
    *row = br * 64 + tr * 16 + fr * 8 + er;
    *col = bc * 64 + tc * 16 + fc * 8 + ec;
}

/* exported for the coordinate pins of S:249-251 */
void or_coords_of(int64_t br, int64_t bc, int t, int f, int pos, int64_t *row, int64_t *col)
{
    or_coords(br, bc, t, f, pos, row, col);
}

/* ---------------------------------------------------------------- Phase II (Alg. 1 l.5-19) */
/*
 * Encode W (rows x cols, row-major, leading dimension = cols) into TCA-TBE.
 *   base_exp_in: INT32_MIN -> choose the window from the histogram (Phase I);
 *                otherwise use this base exponent (e_base in [-1, 248]).
 * Outputs (caller-allocated, see or_encode_bound): B1/B2/B3 (one u64 per FragTile,
 * canonical order), H (bytes), L (u16), offsets (2 u64 per BlockTile: H start byte,
 * L start byte).  info[0..7] = padded_rows, padded_cols, base_exp, pad_word,
 * n_fragtiles, n_blocktiles, h_len_bytes, l_len_words.
 * Errors: -1 empty matrix, -2 bad base_exp, -3 capacity exceeded.
 */
int or_encode(const uint16_t *w, int64_t rows, int64_t cols, int32_t base_exp_in,
              uint64_t *B1, uint64_t *B2, uint64_t *B3,
              uint8_t *H, int64_t h_cap, uint16_t *L, int64_t l_cap,
              uint64_t *offsets, int64_t info[8])
{
    if (rows < 1 || cols < 1) return -1;
    int e_base;
    if (base_exp_in == INT32_MIN) {
        int64_t counts[256], covered;
        int start;
        or_histogram(w, rows * cols, counts);                 /* Alg. 1 line 2 */
        if (or_select_window(counts, &start, &covered)) return -1;   /* line 3 */
        e_base = start - 1;                                   /* line 4: min(E_top) - 1 */
    } else {
        e_base = base_exp_in;
    }
    if (e_base < -1 || e_base > 248) return -2;
    uint16_t pad_word;                                         /* (0, e_base+1, 0) */
    or_assemble_fields(0, e_base + 1, 0, &pad_word);

    int64_t prow = ((rows + 63) / 64) * 64, pcol = ((cols + 63) / 64) * 64;
    int64_t nbr = prow / 64, nbc = pcol / 64;
    int64_t ft = 0, hl = 0, ll = 0, bt = 0;
    for (int64_t br = 0; br < nbr; br++)
        for (int64_t bc = 0; bc < nbc; bc++, bt++) {          /* BlockTile row-major */
            offsets[2 * bt + 0] = (uint64_t)hl;               /* H start, bytes      */
            offsets[2 * bt + 1] = (uint64_t)(ll * 2);         /* L start, bytes      */
            for (int t = 0; t < 16; t++)
                for (int f = 0; f < 4; f++, ft++) {           /* "for each tile t"   */
                    uint64_t b1 = 0, b2 = 0, b3 = 0;          /* line 7              */
                    for (int i = 0; i < 64; i++) {            /* line 8              */
                        int64_t r, c;
                        or_coords(br, bc, t, f, i, &r, &c);
                        uint16_t wv = (r < rows && c < cols) ? w[r * cols + c] : pad_word;
                        int s, e, m;
                        or_split_fields(wv, &s, &e, &m);      /* line 9              */
                        if (e >= e_base + 1 && e <= e_base + 7) {     /* e in E_top   */
                            int code = e - e_base;            /* line 11: c in [1,7] */
                            b1 |= (uint64_t)(code & 1) << i;          /* line 12 */
                            b2 |= (uint64_t)((code >> 1) & 1) << i;
                            b3 |= (uint64_t)((code >> 2) & 1) << i;
                            if (hl >= h_cap) return -3;
                            H[hl++] = or_pack_sm(s, m);       /* line 13: H.Push     */
                        } else {
                            if (ll >= l_cap) return -3;
                            L[ll++] = wv;                     /* line 15: L.Push(w)  */
                        }
                    }
                    B1[ft] = b1; B2[ft] = b2; B3[ft] = b3;    /* line 18             */
                }
            /* 128-bit alignment of each BlockTile's H and L segment, zero padded
             * ("padded offline to ensure 128-bit alignment") */
            while (hl % 16) { if (hl >= h_cap) return -3; H[hl++] = 0; }
            while ((ll * 2) % 16) { if (ll >= l_cap) return -3; L[ll++] = 0; }
        }
    info[0] = prow; info[1] = pcol; info[2] = e_base; info[3] = pad_word;
    info[4] = ft; info[5] = bt; info[6] = hl; info[7] = ll;
    return 0;
}

/* worst-case sizes for or_encode's output buffers */
void or_encode_bound(int64_t rows, int64_t cols, int64_t out[4])
{
    int64_t prow = ((rows + 63) / 64) * 64, pcol = ((cols + 63) / 64) * 64;
    int64_t nbt = (prow / 64) * (pcol / 64);
    out[0] = nbt * 64;        /* fragtiles          */
    out[1] = nbt;             /* blocktiles         */
    out[2] = nbt * 4096;      /* H bytes (all in-window)  */
    out[3] = nbt * 4096;      /* L words (all fallback)   */
}

/* ---------------------------------------------------------------- sequential decoder */
/* Inverse of Alg. 1 in the same canonical order.  out is rows x cols (logical).
 * Errors: -4 a segment overruns its array (corruption). */
int or_decode_sequential(int64_t rows, int64_t cols, int32_t e_base,
                         const uint64_t *B1, const uint64_t *B2, const uint64_t *B3,
                         const uint8_t *H, int64_t h_len, const uint16_t *L, int64_t l_len,
                         const uint64_t *offsets, uint16_t *out)
{
    int64_t prow = ((rows + 63) / 64) * 64, pcol = ((cols + 63) / 64) * 64;
    int64_t nbr = prow / 64, nbc = pcol / 64;
    int64_t ft = 0, bt = 0;
    for (int64_t br = 0; br < nbr; br++)
        for (int64_t bc = 0; bc < nbc; bc++, bt++) {
            int64_t hp = (int64_t)offsets[2 * bt];
            int64_t lp = (int64_t)offsets[2 * bt + 1] / 2;
            for (int t = 0; t < 16; t++)
                for (int f = 0; f < 4; f++, ft++)
                    for (int i = 0; i < 64; i++) {
                        int code = (int)(((B1[ft] >> i) & 1) | (((B2[ft] >> i) & 1) << 1) |
                                         (((B3[ft] >> i) & 1) << 2));
                        uint16_t wv;
                        if (code != 0) {
                            if (hp >= h_len) return -4;
                            int s, m;
                            or_unpack_sm(H[hp++], &s, &m);
                            if (or_assemble_fields(s, e_base + code, m, &wv)) return -4;
                        } else {
                            if (lp >= l_len) return -4;
                            wv = L[lp++];
                        }
                        int64_t r, c;
                        or_coords(br, bc, t, f, i, &r, &c);
                        if (r < rows && c < cols) out[r * cols + c] = wv;
                    }
        }
    return 0;
}

/* ---------------------------------------------------------------- Alg. 2, one lane */
static int or_popc64(uint64_t x) { int n = 0; while (x) { n += (int)(x & 1); x >>= 1; } return n; }

/* Alg. 2 for lane l of one FragTile: both arms are evaluated and the mask bit
 * selects (branch-free reading of P:357/P:431).  w_out[k] for k = 0, 1
 * is the element at p = 2l + k.  Returns -4 on an out-of-segment index. */
int or_decode_lane(uint64_t B1, uint64_t B2, uint64_t B3,
                   const uint8_t *H, int64_t h_start, int64_t h_end,
                   const uint16_t *L, int64_t l_start, int64_t l_end,
                   int32_t e_base, int lane, uint16_t w_out[2])
{
    uint64_t M = B1 | B2 | B3;                          /* Step 1: spatial indicator */
    for (int k = 0; k < 2; k++) {                       /* Step 2 */
        int p = 2 * lane + k;                           /* position in the 8x8 tile */
        uint64_t mask = (p == 0) ? 0 : ((((uint64_t)1) << p) - 1);
        int idx_H = or_popc64(M & mask);                /* Popc(M & mask) */
        int idx_L = p - idx_H;                          /* Case B index */
        int bit = (int)((M >> p) & 1);
        /* Case A: high-frequency path */
        uint16_t wa = 0;
        if (h_start + idx_H < h_end) {
            int s, m;
            or_unpack_sm(H[h_start + idx_H], &s, &m);
            int c = (int)((((B3 >> p) & 1) << 2) | (((B2 >> p) & 1) << 1) | ((B1 >> p) & 1));
            int e = e_base + c;                         /* implicit lookup */
            if (e >= 0 && e <= 255) or_assemble_fields(s, e, m, &wa);
        } else if (bit) return -4;
        /* Case B: fallback path */
        uint16_t wb = 0;
        if (l_start + idx_L < l_end) wb = L[l_start + idx_L];
        else if (!bit) return -4;
        w_out[k] = bit ? wa : wb;                       /* select, no divergence */
    }
    return 0;
}

/* Whole-matrix decode through 32 lockstep lanes per FragTile; per-FragTile segment
 * starts from the popcount prefix scan in canonical order. */
int or_decode_lanes(int64_t rows, int64_t cols, int32_t e_base,
                    const uint64_t *B1, const uint64_t *B2, const uint64_t *B3,
                    const uint8_t *H, int64_t h_len, const uint16_t *L, int64_t l_len,
                    const uint64_t *offsets, uint16_t *out)
{
    int64_t prow = ((rows + 63) / 64) * 64, pcol = ((cols + 63) / 64) * 64;
    int64_t nbr = prow / 64, nbc = pcol / 64;
    int64_t ft = 0, bt = 0;
    for (int64_t br = 0; br < nbr; br++)
        for (int64_t bc = 0; bc < nbc; bc++, bt++) {
            int64_t h_start = (int64_t)offsets[2 * bt];
            int64_t l_start = (int64_t)offsets[2 * bt + 1] / 2;
            for (int t = 0; t < 16; t++)
                for (int f = 0; f < 4; f++, ft++) {
                    uint64_t M = B1[ft] | B2[ft] | B3[ft];
                    int nh = or_popc64(M);
                    for (int lane = 0; lane < 32; lane++) {
                        uint16_t wv[2];
                        int rc = or_decode_lane(B1[ft], B2[ft], B3[ft], H, h_start, h_start + nh,
                                                L, l_start, l_start + (64 - nh), e_base, lane, wv);
                        if (rc) return rc;
                        for (int k = 0; k < 2; k++) {
                            int64_t r, c;
                            or_coords(br, bc, t, f, 2 * lane + k, &r, &c);
                            if (r < rows && c < cols) out[r * cols + c] = wv[k];
                        }
                    }
                    if (h_start + nh > h_len || l_start + (64 - nh) > l_len) return -4;
                    h_start += nh;              /* h advance = popcount(M)      */
                    l_start += 64 - nh;         /* l advance = 64 - popcount(M) */
                }
        }
    return 0;
}

/* ---------------------------------------------------------------- fp64 GEMM */
/* bf16 bit pattern -> exact double (BF16 value formula; subnormals, inf, nan kept) */
double or_bf16_to_double(uint16_t w)
{
    int s, e, m;
    or_split_fields(w, &s, &e, &m);
    double v;
    if (e == 255) v = (m == 0) ? INFINITY : NAN;
    else if (e == 0) v = ldexp((double)m, -126 - 7);            /* subnormal / zero */
    else v = ldexp(1.0 + (double)m / 128.0, e - 127);
    return s ? -v : v;
}

/* Y[m][n] = sum_k X[m][k] * W[n][k], accumulated in fp64 (north star).  X is M x K,
 * W is N x K (both bf16 bit patterns, row-major), Y is M x N doubles. */
void or_gemm_f64(const uint16_t *X, int64_t M, int64_t K, const uint16_t *W, int64_t N, double *Y)
{
    for (int64_t m = 0; m < M; m++)
        for (int64_t n = 0; n < N; n++) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; k++)
                acc += or_bf16_to_double(X[m * K + k]) * or_bf16_to_double(W[n * K + k]);
            Y[m * N + n] = acc;
        }
}

/* Same, but only output columns n in cols[0..ncols) (for sampled checks at full size). */
void or_gemm_f64_cols(const uint16_t *X, int64_t M, int64_t K, const uint16_t *W,
                      const int64_t *cols, int64_t ncols, double *Y)
{
    for (int64_t m = 0; m < M; m++)
        for (int64_t j = 0; j < ncols; j++) {
            double acc = 0.0;
            const uint16_t *wr = W + cols[j] * K;
            for (int64_t k = 0; k < K; k++)
                acc += or_bf16_to_double(X[m * K + k]) * or_bf16_to_double(wr[k]);
            Y[m * ncols + j] = acc;
        }
}

/* Round a double to the nearest bf16 (ties to even), directly from the double. */
uint16_t or_round_bf16(double v)
{
    if (isnan(v)) return 0x7FC0;
    int s = signbit(v) ? 1 : 0;
    double a = fabs(v);
    if (isinf(a)) return (uint16_t)((s << 15) | 0x7F80);
    if (a == 0.0) return (uint16_t)(s << 15);
    int ex;
    frexp(a, &ex);                       /* a = f * 2^ex, f in [0.5, 1) */
    int E = ex - 1;                      /* a in [2^E, 2^(E+1)) */
    if (E < -126) E = -126;              /* subnormal range: fixed quantum */
    double q = ldexp(1.0, E - 7);        /* bf16 quantum at this binade */
    double t = a / q;                    /* exact (power-of-two scaling) */
    double fl = floor(t);
    double fr = t - fl;
    double r = fl;
    if (fr > 0.5 || (fr == 0.5 && fmod(fl, 2.0) != 0.0)) r = fl + 1.0;
    double res = r * q;
    if (res == 0.0) return (uint16_t)(s << 15);   /* underflow to signed zero */
    /* re-encode */
    if (res >= ldexp(1.0, 128)) return (uint16_t)((s << 15) | 0x7F80);
    int E2;
    frexp(res, &E2);
    E2 -= 1;
    uint16_t bits;
    if (E2 < -126) {                     /* subnormal */
        bits = (uint16_t)(int)(res / ldexp(1.0, -133));
    } else {
        int man = (int)((res / ldexp(1.0, E2) - 1.0) * 128.0);
        bits = (uint16_t)(((E2 + 127) << 7) | man);
    }
    return (uint16_t)((s << 15) | bits);
}
