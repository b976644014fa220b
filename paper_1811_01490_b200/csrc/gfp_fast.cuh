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
// the accumulation needs no carries.  Each 128-bit column is divided by r
// once (Moller-Granlund reciprocal, with a 2^63 r bias to make it
// non-negative), and two cheap carry rounds leave lazy digits in
// [-delta, r + delta] with delta <= k + 2.
#pragma once
#include "gfp_device.cuh"

template <int KD>
GFP_D void fast_mul_lazy(const i64 (&x)[KD], const i64 (&y)[KD], i64 (&f)[KD],
                         const RadixConsts &rc)
{
    const int s = rc.s;
    const i64 mask = ((i64)1 << s) - 1;
    int xl[KD], xh[KD], yl[KD], yh[KD], nyl[KD], nyh[KD];
#pragma unroll
    for (int i = 0; i < KD; i++) {
        xl[i] = (int)(x[i] & mask);
        xh[i] = (int)(x[i] >> s);
        yl[i] = (int)(y[i] & mask);
        yh[i] = (int)(y[i] >> s);
        nyl[i] = -yl[i];
        nyh[i] = -yh[i];
    }
    const i128 bias = (i128)(((u128)rc.bias_hi << 64) | rc.bias_lo);
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
            LL += (i64)xl[i] * a;
            LH += (i64)xl[i] * b;
            HL += (i64)xh[i] * a;
            HH += (i64)xh[i] * b;
        }
        i128 c = (i128)LL + ((i128)LH << s) + ((i128)HL << s) + ((i128)HH << (2 * s)) + bias;
        u128 cu = (u128)c;
        u64 rem;
        u64 qq = div128_by_r((u64)(cu >> 64), (u64)cu, rc, rem);
        q[m] = (i64)(qq - (1ULL << 63));
        d[m] = rem;
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
