// gfp_fast.cuh -- the transform's hot arithmetic.
//
// fast_mul_lazy: x * y mod p for lazy signed digits, the Z/pZ twiddle,
// pointwise and N^-1 multiply of the transform (the role gfp_mul_fft plays
// for the reference, gfp_mult.py:416-501, paper Alg. 13).  Instead of two
// word-prime NTTs + CRT + LHC, each digit is split as hi * 2^s + lo
// (balanced limbs, |lo| <= 2^(s-1)) and the negacyclic convolution is three
// sub-column sums of 32x32 -> 64 signed IMAD.WIDE products:
//
//   c_m = LL_m + MID_m 2^s + HH_m 2^(2s),   MID = sum (x_lo y_hi + x_hi y_lo),
//   XY_m = sum_{i+j=m} x_i y_j - sum_{i+j=m+k} x_i y_j      (r^k = -1),
//
// with MID from a limb-level Karatsuba product (3 IMAD.WIDE per digit pair).
//
// The host verifies (plan time, exact integers: gfp_elem.cu fast_bounds)
// that every sub-column stays below 2^63 in magnitude for the digit bounds
// the transform guarantees, so the accumulation needs no carries.  The
// quotient of each biased column c' = c + 2^63 r (non-negative, < 2^64 r) by
// r is estimated from floor(c' / 2^w), which is built from the three 64-bit
// sub-columns with shifts only (no 128-bit arithmetic), times a fixed-point
// reciprocal of r; the estimate is at most 3 short, so the remainder is
// exact from the low 64 bits and lies in [0, 4r).  Two cheap carry rounds
// (the balanced normaliser, norm_bal) leave balanced lazy digits in
// [-r/2 - delta, r/2 + delta].
#pragma once
#include "gfp_device.cuh"

// largest k whose multiply uses the fused-accumulate IMAD.WIDE form
#ifndef GFP_CC_MAXK
#define GFP_CC_MAXK 8
#endif

#ifndef GFP_KARA_MAXK
#define GFP_KARA_MAXK 32
#endif

// limb split used by the fast multiply for each k (compile time; the host
// bound check in gfp_elem.cu:fast_bounds verifies it for the given r)
template <int KD>
struct FastSplit {
    static constexpr int S = KD <= 16 ? 29 : 28;
};

// quotient estimate and exact remainder of the biased column
//   c' = HH 2^(2S) + MID 2^S + LL + 2^63 r,  0 <= c' < 2^64 r
template <int S>
GFP_D u64 column_quot(i64 LL, i64 MID, i64 HH, const RadixConsts &rc, u64 &rem)
{
    // floor(c / 2^w) from nested floors of shifts (no 128-bit arithmetic):
    //   w >= 2S:  (HH + (mid >> S)) >> (w - 2S)
    //   w <  2S:  (HH << (2S - w)) + (mid >> (w - S))
    // folded into one branch-free form with sh1 = max(w - 2S, 0),
    // sh2 = max(2S - w, 0) (host-computed)
    // (fast_bounds keeps q_sh1, q_sh2 <= 28; the masks tell the compiler the
    // 64-bit shifts are by less than 32, two SHF each)
    const i64 mid = MID + (LL >> S);  // floor((MID 2^S + LL) / 2^S)
    const i64 t0 =
        ((HH << (rc.q_sh2 & 31)) + (mid >> ((S - rc.q_sh2) & 31))) >> (rc.q_sh1 & 31);
    const u64 t = (u64)t0 + rc.bias_t;  // floor(c' / 2^w), in [0, 2^64)
    const u64 clo = (u64)LL + ((u64)MID << S) + ((u64)HH << (2 * S)) + rc.bias_lo;
    const u64 q = t + __umul64hi(t, rc.m_recip);
    rem = clo - q * rc.r;
    return q;
}

// Mode 2 (r = 2^a + 2^b): with the bias B = 2^62 r (a multiple of 2^a),
// T = floor((c + B) / 2^a) comes from shifts of the sub-columns, and
// 1 / r = 2^-a (1 - 2^(b-a) + ...) gives the quotient estimate
//   q = T - (T >> (a - b)) - 2,  floor((c + B) / r) - q in [0, 3],
// so rem = (c + B) - q r (= low 64 bits minus two shifts) is in [0, 4r)
// without a 64 x 64 multiply.  Returns the signed carry q - 2^62.
// SPARSE == 3: a, b are compile-time (P2Radix<KD>); B mod 2^64 = 0 then.
template <int S, int SPARSE = 2, int KD = 0>
GFP_D i64 column_quot_p2(i64 LL, i64 MID, i64 HH, const RadixConsts &rc, u64 &rem)
{
    const i64 mid = MID + (LL >> S);                // floor(c / 2^S)
    const i64 t2s = HH + (mid >> S);                 // floor(c / 2^(2S))
    if constexpr (SPARSE == 3) {
        constexpr int a = P2Radix<KD>::a, b = P2Radix<KD>::b;
        static_assert(a >= 2 * S && a - 2 * S < 32 && 62 + b - a >= 0, "P2Radix vs S");
        constexpr u64 bias_t = (1ULL << 62) + (1ULL << (62 + b - a));
        const u64 T = (u64)(t2s >> (a - 2 * S)) + bias_t;
        const u64 q = T - (T >> (a - b)) - 2;
        // (2^62 r) mod 2^64 = 0 for a, b >= 2
        const u64 clo = (u64)LL + ((u64)MID << S) + ((u64)HH << (2 * S));
        rem = clo - (q << a) - (q << b);
        return (i64)(q - (1ULL << 62));
    }
    const u64 T = (u64)(t2s >> (rc.p2_sh & 31)) + rc.p2_bias_t;
    const u64 q = T - (T >> (rc.p2_ab & 63)) - 2;
    const u64 clo = (u64)LL + ((u64)MID << S) + ((u64)HH << (2 * S)) + rc.p2_bias_lo;
    rem = clo - (q << (rc.sp_a & 63)) - (q << (rc.p2_b & 63));
    return (i64)(q - (1ULL << 62));
}

// Mode 3 quotient (compile-time r = 2^a + 2^b, P2Radix<KD>), signed: no
// bias.  With T = floor(c / 2^a) (arithmetic shifts of the sub-columns),
//   q = T - floor(T 2^(b-a)) - 1,   c / r - q in (-0.01, 2.01),
// (the second-order term c 2^(2(b-a) - a) is below 1/256 for the paper's
// radices), so rem = c - q r (low 64 bits minus two shifts) lies in
// (-r/100, 2.01 r) and q is the signed carry.
template <int S, int KD>
GFP_D i64 column_quot_p3(i64 LL, i64 MID, i64 HH, u64 &rem)
{
    constexpr int a = P2Radix<KD>::a, b = P2Radix<KD>::b;
    static_assert(a >= 2 * S && a - 2 * S < 32, "P2Radix vs S");
    const i64 mid = MID + (LL >> S);   // floor(c / 2^S) - HH 2^S
    const i64 t2s = HH + (mid >> S);   // floor(c / 2^(2S))
    const i64 T = t2s >> (a - 2 * S);  // floor(c / 2^a)
    const i64 q = T - (T >> (a - b)) - 1;
    const u64 clo = (u64)LL + ((u64)MID << S) + ((u64)HH << (2 * S));
    rem = clo - ((u64)q << a) - ((u64)q << b);
    return q;
}

// Mode 3 quotient with the rounding folded in (k <= GFP_SEQ_MAXK, GFP_P3_ROUNDQ): the
// quotient estimate is taken at a quarter of a digit,
//   T4 = floor(c / 2^(a-2)),  q4 = T4 - floor(T4 2^(b-a)),  4 c / r - q4 in (-1, 1),
// and rounded to the nearest integer, q = floor((q4 + 2) / 4), so
//   c / r - q in (-3/4, 3/4):  rem = c - q r is already a balanced digit,
// |rem| < 3r/4, and the second carry round (norm_bal of the remainder) is
// gone.  Three quarters of r instead of a half costs nothing downstream: four
// lazy radix-2 stages of such digits stay below 12 r + r/2 < 2^63 (the host
// check in make_consts, gfp_elem.cu, proves every bound for the radix).
template <int S, int KD>
GFP_D i64 column_quot_p3r(i64 LL, i64 MID, i64 HH, u64 &rem)
{
    constexpr int a = P2Radix<KD>::a, b = P2Radix<KD>::b;
    static_assert(2 * S >= a - 2 && a - 2 >= S && a - 2 - S < 32 && 2 * S - (a - 2) < 8,
                  "P2Radix vs S (rounding quotient)");
    const i64 mid = MID + (LL >> S);                                       // floor(c / 2^S) - HH 2^S
    const i64 T4 = (HH << (2 * S - (a - 2))) + (mid >> ((a - 2) - S));     // floor(c / 2^(a-2))
    const i64 q4 = T4 - (T4 >> (a - b));
    const i64 q = (q4 + 2) >> 2;
    const u64 clo = (u64)LL + ((u64)MID << S) + ((u64)HH << (2 * S));
    rem = clo - ((u64)q << a) - ((u64)q << b);
    return q;
}

#ifndef GFP_SEQ_MAXK
#define GFP_SEQ_MAXK 32  // largest k whose mode-3 multiply folds the carry into the next column
                         // (with the rounding quotient the serial chain is short enough for
                         // k = 16 / 32 too: C3 multiply passes -3.7%, C5 FFT -1.5%)
#endif
#ifndef GFP_P3_ROUNDQ
#define GFP_P3_ROUNDQ 1  // mode 3, k <= 8: rounding column quotient (no norm_bal per column)
#endif

// The carry rounds of one product, column by column (m = 0 .. k-1), shared
// by the multiply kernels.  Column m's value is c_m = HH 2^(2S) + MID 2^S + LL.
//   modes 0-2:  c_m = q_m r + d_m (column_quot*, d_m in [0, 4r)), then
//               d_m + q_{m-1} = q2_m r + d2_m (norm_bal), digit = d2_m + q2_{m-1}
//   mode 3, k <= GFP_SEQ_MAXK (SEQ): sequential carry: c_m + C_{m-1} = q_m r + rem_m with
//               the rounding quotient (column_quot_p3r): digit = rem_m,
//               |rem_m| < 3r/4, C_m = q_m  [without GFP_P3_ROUNDQ:
//               rem_m = q2_m r + d_m (norm_bal), digit = d_m, C_m = q_m + q2_m]
//               (before the rounding quotient the serial chain across a block of
//               columns cost more than it saved for k >= 16; with it the chain
//               is short enough and every k takes this form)
// with the r^k = -1 wrap at m = 0 resolved by finish() (digits 0 and 1).
template <int S, int SPARSE, int KD>
struct ColReduce {
    static constexpr bool SEQ = SPARSE == 3 && KD <= GFP_SEQ_MAXK;
    i64 q_prev = 0, d0 = 0, f1 = 0;
    int q2_prev = 0;
    // returns true when digit m (>= 2) is final in `out`
    GFP_D bool column(int m, i64 LL, i64 MID, i64 HH, const RadixConsts &rc, i64 &out)
    {
        if constexpr (SEQ) {
            u64 rem;
            i64 d;
            if constexpr (GFP_P3_ROUNDQ) {
                q_prev = column_quot_p3r<S, KD>(LL + q_prev, MID, HH, rem);
                d = (i64)rem;  // |d| < 3r/4
            } else {
                const i64 q = column_quot_p3<S, KD>(LL + q_prev, MID, HH, rem);
                const int q2 = norm_bal<3, KD>((i64)rem, rc, d);
                q_prev = q + q2;
            }
            if (m == 0) {
                d0 = d;
                return false;
            }
            if (m == 1) {
                f1 = d;
                return false;
            }
            out = d;
            return true;
        } else {
            u64 rem;
            i64 carry;
            if (SPARSE >= 2) {
                carry = column_quot_p2<S, SPARSE, KD>(LL, MID, HH, rc, rem);
            } else {
                const u64 qq = column_quot<S>(LL, MID, HH, rc, rem);
                carry = (i64)(qq - (1ULL << 63));
            }
            bool fin = false;
            if (m == 0) {
                d0 = (i64)rem;
            } else {
                i64 d2;
                const int q2 = norm_bal<SPARSE, KD>((i64)rem + q_prev, rc, d2);
                if (m == 1) {
                    f1 = d2;
                } else {
                    out = d2 + q2_prev;
                    fin = true;
                }
                q2_prev = q2;
            }
            q_prev = carry;
            return fin;
        }
    }
    // digits 0 and 1 after the last column (the wrapped carry enters digit 0
    // negated)
    GFP_D void finish(const RadixConsts &rc, i64 &o0, i64 &o1)
    {
        i64 d2_0;
        const int q2_0 = norm_bal<SPARSE, KD>(d0 - q_prev, rc, d2_0);
        if constexpr (SEQ) {
            o0 = d2_0;
        } else {
            o0 = d2_0 - q2_prev;
        }
        o1 = f1 + q2_0;
    }
};

// v or -v by a sign mask m in {0, -1}: (v ^ m) - m, two ALU instructions
// (LOP3 + IADD3).  A multiply by +-1 would sit on the FMA-heavy pipe that the
// IMAD.WIDE products saturate; a literal negation gets folded into the
// products by ptxas (see RadixConsts::neg_one).
GFP_D int cond_neg(int v, int m) { return (v ^ m) - m; }

#ifndef GFP_NEG_X_ALU
#define GFP_NEG_X_ALU 0  // x-limb signs by cond_neg (else a multiply by +-1; measured equal for k = 8)
#endif
#ifndef GFP_NEG_WIN_ALU
#define GFP_NEG_WIN_ALU 0  // window digit signs by cond_neg (else * rc.neg_one; the multiply
                         // measured 2% faster for C3 although it sits on the FMA-heavy pipe)
#endif
GFP_D int sign_x(int v, unsigned bit)
{
    return GFP_NEG_X_ALU ? cond_neg(v, -(int)bit) : v * (1 - 2 * (int)bit);
}
GFP_D int sign_win(int v, int neg_one) { return GFP_NEG_WIN_ALU ? cond_neg(v, neg_one) : v * neg_one; }

// x * y mod p for balanced lazy digits (|digit| <= r/2 + delta), output
// balanced lazy digits.  Limbs are balanced too, x = xh 2^S + xl with
// xl in [-2^(S-1), 2^(S-1)), and the middle sub-column comes from one
// Karatsuba product per digit pair:
//   MID = sum (xl + xh)(yl + yh) - LL - HH,
// so a digit product costs three IMAD.WIDE instead of four.
//
// negx (bit i set: digit i of x enters negated) lets a caller fold a digit
// rotation x * r^a, whose wrapped digits change sign (r^k = -1), into the
// limb split: the negation of a balanced limb pair is again a balanced limb
// pair, so it costs one IMAD per limb instead of a 64-bit negate.
//
// dst != nullptr: each output digit is stored to dst[m] as soon as it is
// final instead of being kept in f (frees registers in the pass kernel).
template <int KD, int SPARSE, bool STORE = false, int DST = 1>
GFP_D void fast_mul_limbs(const int (&xl)[KD], const int (&xh)[KD], const int (&xs)[KD],
                          const int (&yl)[KD], const int (&yh)[KD], const int (&ys)[KD],
                          i64 (&f)[KD], const RadixConsts &rc, i64 *dst = nullptr)
{
    constexpr int S = FastSplit<KD>::S;
    constexpr bool CC = KD <= GFP_CC_MAXK;  // fused-accumulate IMAD.WIDE form (gfp_device.cuh)
    // limb Karatsuba (3 IMAD.WIDE per digit pair, 6 limb registers per
    // digit) up to GFP_KARA_MAXK; above it the schoolbook form (4 IMAD.WIDE,
    // 4 limb registers per digit) keeps the k = 32 operands in registers
    constexpr bool KARA = KD <= GFP_KARA_MAXK;
    // Columns in order, with the two carry rounds streaming behind them:
    //   round 1  c_m = q_m r + d_m                       (column_quot)
    //   round 2  d_m + q_{m-1} = q2_m r + d2_m            (norm_bal)
    //   round 3  f_m = d2_m + q2_{m-1}
    // with the r^k = -1 wrap at m = 0 (q_{-1} = -q_{k-1}).  Only column 0's
    // remainder and digit 1's pending carry wait for the last column.
    ColReduce<S, SPARSE, KD> cr;
#pragma unroll
    for (int m = 0; m < KD; m++) {
        i64 LL = 0, SS = 0, HH = 0, LLn = 0, SSn = 0, HHn = 0;
        if (KARA) {
#pragma unroll
            for (int i = 0; i <= m; i++) {
                LL = mad_wide_s32<CC>(xl[i], yl[m - i], LL);
                SS = mad_wide_s32<CC>(xs[i], ys[m - i], SS);
                HH = mad_wide_s32<CC>(xh[i], yh[m - i], HH);
            }
#pragma unroll
            for (int i = m + 1; i < KD; i++) {  // wrapped terms: r^k = -1
                LLn = mad_wide_s32<CC>(xl[i], yl[m - i + KD], LLn);
                SSn = mad_wide_s32<CC>(xs[i], ys[m - i + KD], SSn);
                HHn = mad_wide_s32<CC>(xh[i], yh[m - i + KD], HHn);
            }
        } else {  // schoolbook limbs: SS accumulates the middle sub-column itself
#pragma unroll
            for (int i = 0; i <= m; i++) {
                LL = mad_wide_s32<CC>(xl[i], yl[m - i], LL);
                SS = mad_wide_s32<CC>(xl[i], yh[m - i], SS);
                SS = mad_wide_s32<CC>(xh[i], yl[m - i], SS);
                HH = mad_wide_s32<CC>(xh[i], yh[m - i], HH);
            }
#pragma unroll
            for (int i = m + 1; i < KD; i++) {
                LLn = mad_wide_s32<CC>(xl[i], yl[m - i + KD], LLn);
                SSn = mad_wide_s32<CC>(xl[i], yh[m - i + KD], SSn);
                SSn = mad_wide_s32<CC>(xh[i], yl[m - i + KD], SSn);
                HHn = mad_wide_s32<CC>(xh[i], yh[m - i + KD], HHn);
            }
        }
        LL -= LLn;
        HH -= HHn;
        const i64 MID = KARA ? (SS - SSn) - LL - HH : SS - SSn;
        i64 v;
        if (cr.column(m, LL, MID, HH, rc, v)) {
            if (STORE)
                dst[m * DST] = v;
            else
                f[m] = v;
        }
    }
    i64 o0, o1;
    cr.finish(rc, o0, o1);
    if (STORE) {
        dst[0] = o0;
        dst[DST] = o1;
    } else {
        f[0] = o0;
        f[1] = o1;
    }
}

// balanced limb split of one digit: v = h 2^S + l, l in [-2^(S-1), 2^(S-1))
template <int S>
GFP_D void split_limbs(i64 v, int &l, int &h)
{
    constexpr i64 half = (i64)1 << (S - 1);
    h = (int)((v + half) >> S);
    l = (int)(v - ((i64)h << S));
}

template <int KD, int SPARSE>
GFP_D void fast_mul_lazy(const i64 (&x)[KD], const i64 (&y)[KD], i64 (&f)[KD],
                         const RadixConsts &rc, unsigned negx = 0)
{
    constexpr int S = FastSplit<KD>::S;
    int xl[KD], xh[KD], xs[KD], yl[KD], yh[KD], ys[KD];
#pragma unroll
    for (int i = 0; i < KD; i++) {
        int l0, h0;
        split_limbs<S>(x[i], l0, h0);
        const unsigned sb = (negx >> i) & 1u;
        xh[i] = sign_x(h0, sb);
        xl[i] = sign_x(l0, sb);
        xs[i] = xl[i] + xh[i];
        split_limbs<S>(y[i], yl[i], yh[i]);
        ys[i] = yl[i] + yh[i];
    }
    fast_mul_limbs<KD, SPARSE>(xl, xh, xs, yl, yh, ys, f, rc);
}

// the same product with y given as pre-split limb pairs (l | h << 32 per
// digit, the plan's limb tables): no split work for the twiddle operand.
// DST: stride in words between the stored digits (STORE; 32 for the
// digit-major tiles of k_pass44t)
template <int KD, int SPARSE, bool STORE = false, int DST = 1>
GFP_D void fast_mul_lazy_ylimbs(const i64 (&x)[KD], const u64 (&ylh)[KD], i64 (&f)[KD],
                                const RadixConsts &rc, unsigned negx = 0, i64 *dst = nullptr)
{
    constexpr int S = FastSplit<KD>::S;
    int xl[KD], xh[KD], xs[KD], yl[KD], yh[KD], ys[KD];
#pragma unroll
    for (int i = 0; i < KD; i++) {
        int l0, h0;
        split_limbs<S>(x[i], l0, h0);
        const unsigned sb = (negx >> i) & 1u;
        xh[i] = sign_x(h0, sb);
        xl[i] = sign_x(l0, sb);
        xs[i] = xl[i] + xh[i];
        yl[i] = (int)(unsigned)ylh[i];
        yh[i] = (int)(unsigned)(ylh[i] >> 32);
        ys[i] = yl[i] + yh[i];
    }
    fast_mul_limbs<KD, SPARSE, STORE, DST>(xl, xh, xs, yl, yh, ys, f, rc, dst);
}

// x * y with the y limbs in a shared-memory column (this thread's int2
// {l, h} per digit at ywin[d * stride]; l + h formed as a digit enters) and only the x limbs in
// registers: columns in blocks of four, x_i times the window
// y_{m0-i} .. y_{m0+3-i} (mod k), one new y digit (negated when its index
// wraps, r^k = -1) entering per step -- the k_mul_wide scheme
// (gfp_mulw.cuh).  Product digits are stored to dst[m] as they become final.
template <int KD, int SPARSE, bool CC>
GFP_D void fast_mul_window_store(const i64 (&x)[KD], unsigned negx, const int2 *ywin, int stride,
                                 i64 *dst, const RadixConsts &rc)
{
    constexpr int S = FastSplit<KD>::S;
    int xl[KD], xh[KD], xs[KD];
#pragma unroll
    for (int i = 0; i < KD; i++) {
        int l0, h0;
        split_limbs<S>(x[i], l0, h0);
        const unsigned sb = (negx >> i) & 1u;
        xh[i] = sign_x(h0, sb);
        xl[i] = sign_x(l0, sb);
        xs[i] = xl[i] + xh[i];
    }
    ColReduce<S, SPARSE, KD> cr;
    // fully unrolled up to k = 16 (compile-time window addresses and wrap
    // signs); k = 32 keeps the block loop to bound the code size
    constexpr int UNR = KD <= 16 ? KD / 4 : 1;
#pragma unroll UNR
    for (int m0 = 0; m0 < KD; m0 += 4) {
        i64 LL[4], SS[4], HH[4];
#pragma unroll
        for (int c = 0; c < 4; c++)
            LL[c] = SS[c] = HH[c] = 0;
        int4 win[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int2 v = ywin[(m0 + c) * stride];
            win[c] = make_int4(v.x, v.y, v.x + v.y, 0);
        }
#pragma unroll
        for (int i = 0; i < KD; i++) {
#pragma unroll
            for (int c = 0; c < 4; c++) {
                LL[c] = mad_wide_s32<CC>(xl[i], win[c].x, LL[c]);
                HH[c] = mad_wide_s32<CC>(xh[i], win[c].y, HH[c]);
                SS[c] = mad_wide_s32<CC>(xs[i], win[c].z, SS[c]);
            }
            if (i + 1 < KD) {
#pragma unroll
                for (int c = 3; c > 0; c--)
                    win[c] = win[c - 1];
                const int j = m0 - i - 1;
                int2 v = ywin[((j + KD) & (KD - 1)) * stride];
                if (j < 0)  // r^k = -1 (rc.neg_one: see RadixConsts)
                    v = make_int2(sign_win(v.x, rc.neg_one), sign_win(v.y, rc.neg_one));
                win[0] = make_int4(v.x, v.y, v.x + v.y, 0);
            }
        }
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const i64 MID = SS[c] - LL[c] - HH[c];
            i64 v;
            if (cr.column(m0 + c, LL[c], MID, HH[c], rc, v))
                dst[m0 + c] = v;
        }
    }
    cr.finish(rc, dst[0], dst[1]);
}
