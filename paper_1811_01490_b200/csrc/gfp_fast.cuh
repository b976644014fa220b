// gfp_fast.cuh -- the transform's hot arithmetic.
//
// fast_mul_lazy: x * y mod p for lazy signed digits, the Z/pZ twiddle,
// pointwise and N^-1 multiply of the transform (the role gfp_mul_fft plays
// for the reference, gfp_mult.py:416-501, paper Alg. 13).  Instead of two
// word-prime NTTs + CRT + LHC, each digit is split as hi * 2^s + lo (|hi|,
// lo < 2^31) and the negacyclic convolution is four sub-column sums of
// 32x32 -> 64 signed IMAD.WIDE products:
//
//   c_m = LL_m + (LH_m + HL_m) 2^s + HH_m 2^(2s),
//   XY_m = sum_{i+j=m} x_i y_j - sum_{i+j=m+k} x_i y_j   (r^k = -1).
//
// The host verifies (plan time, exact integers) that every sub-column stays
// below 2^63 in magnitude for the digit bounds the transform guarantees, so
// the accumulation needs no carries.  Each 128-bit column (biased by 2^63 r
// to be non-negative) gets a quotient estimate from its top 64 bits times a
// fixed-point reciprocal of r (at most 3 short, exact remainder from the low
// word), and two cheap carry rounds leave lazy digits in [-delta, r + delta]
// with delta <= 2^S + k + 8.
#pragma once
#include "gfp_device.cuh"

// 32x32 -> 64 signed multiply-add in one IMAD.WIDE (the compiler otherwise
// widens to a 64x64 multiply)
GFP_D i64 mad_wide_s32(int a, int b, i64 c)
{
    i64 d;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}

// limb split used by the fast multiply for each k (compile time; the host
// bound check in gfp_kernels.cu:fast_bounds verifies it for the given r)
template <int KD>
struct FastSplit {
    static constexpr int S = KD <= 8 ? 30 : 29;
};

// floor(c' / r) for 0 <= c' < 2^64 r, up to 3 short: q in [q* - 3, q*], and
// the exact remainder c' - q r in [0, 4r) from the low word alone.
GFP_D u64 quot_est(u64 hi, u64 lo, const RadixConsts &rc, u64 &rem)
{
    const int w = rc.w;  // bit length of r
    u64 t = (hi << (64 - w)) | (lo >> w);
    u64 q = t + __umul64hi(t, rc.m_recip);
    rem = lo - q * rc.r;
    return q;
}

template <int KD>
GFP_D void fast_mul_lazy(const i64 (&x)[KD], const i64 (&y)[KD], i64 (&f)[KD],
                         const RadixConsts &rc)
{
    constexpr int S = FastSplit<KD>::S;
    constexpr i64 mask = ((i64)1 << S) - 1;
    int xl[KD], xh[KD], yl[KD], yh[KD], nyl[KD], nyh[KD];
#pragma unroll
    for (int i = 0; i < KD; i++) {
        xl[i] = (int)(x[i] & mask);
        xh[i] = (int)(x[i] >> S);
        yl[i] = (int)(y[i] & mask);
        yh[i] = (int)(y[i] >> S);
        nyl[i] = -yl[i];
        nyh[i] = -yh[i];
    }
    const u128 bias = ((u128)rc.bias_hi << 64) | rc.bias_lo;
    i64 q[KD];
    u64 d[KD];
#pragma unroll
    for (int m = 0; m < KD; m++) {
        i64 LL = 0, LH = 0, HL = 0, HH = 0;
#pragma unroll
        for (int i = 0; i < KD; i++) {
            const int j = (m - i + KD) % KD;
            const bool neg = i > m;
            const int a = neg ? nyl[j] : yl[j];
            const int b = neg ? nyh[j] : yh[j];
            LL = mad_wide_s32(xl[i], a, LL);
            LH = mad_wide_s32(xl[i], b, LH);
            HL = mad_wide_s32(xh[i], a, HL);
            HH = mad_wide_s32(xh[i], b, HH);
        }
        // c' = c + 2^63 r, exact and non-negative (host-verified bounds)
        u128 c = bias + (u128)(i128)LL + (u128)((i128)LH << S) + (u128)((i128)HL << S) +
                 (u128)((i128)HH << (2 * S));
        u64 rem;
        u64 qq = quot_est((u64)(c >> 64), (u64)c, rc, rem);
        q[m] = (i64)(qq - (1ULL << 63));
        d[m] = rem;  // in [0, 4r)
    }
    i64 q2[KD], d2[KD];
#pragma unroll
    for (int m = 0; m < KD; m++) {
        i64 cin = m ? q[m - 1] : -q[KD - 1];
        q2[m] = floordiv_small((i64)d[m] + cin, rc, d2[m]);
    }
#pragma unroll
    for (int m = 0; m < KD; m++)
        f[m] = d2[m] + (m ? q2[m - 1] : -q2[KD - 1]);
}
