// gfp_generic.cuh -- exact thread-serial GF(r^k + 1) multiply for any
// power-of-two k and any 2 <= r < 2^64.
//
// Computes the function of gfp_mul_bigint / gfp_mul_fft (gfp_mult.py:416-512):
// the canonical encoding of x*y mod p.  Mechanism: negacyclic schoolbook
// over radix-r digits with exact 192-bit signed column sums, then a radix-r
// carry pass (128/64 division by a Moller-Granlund reciprocal), then the
// r^k = -1 wrap and the form-A/form-B canonicalisation.  This is the
// general-purpose path (element-wise API, powering, plan tables); the
// transform's hot multiply is the limb-split kernel in gfp_fast.cuh.
#pragma once
#include "gfp_device.cuh"

struct W192 {
    u64 w0, w1, w2;  // two's complement, little-endian
};

GFP_D void w192_add(W192 &a, u64 lo, u64 hi)
{
    u64 t0 = a.w0 + lo;
    u64 c0 = t0 < lo;
    u64 t1 = a.w1 + hi;
    u64 c1 = t1 < hi;
    u64 t1b = t1 + c0;
    c1 |= t1b < t1;
    a.w0 = t0;
    a.w1 = t1b;
    a.w2 += c1;
}

GFP_D void w192_sub(W192 &a, u64 lo, u64 hi)
{
    u64 b0 = a.w0 < lo;
    u64 t0 = a.w0 - lo;
    u64 b1 = a.w1 < hi;
    u64 t1 = a.w1 - hi;
    u64 b1b = t1 < b0;
    t1 -= b0;
    a.w0 = t0;
    a.w1 = t1;
    a.w2 -= (b1 | b1b);
}

GFP_D void w192_add192(W192 &a, const W192 &b)
{
    w192_add(a, b.w0, b.w1);
    a.w2 += b.w2;
}

GFP_D bool w192_neg_p(const W192 &a) { return (i64)a.w2 < 0; }

GFP_D W192 w192_negate(const W192 &a)
{
    W192 z;
    z.w0 = ~a.w0;
    z.w1 = ~a.w1;
    z.w2 = ~a.w2;
    u64 c = 1;
    z.w0 += c;
    c = z.w0 == 0;
    z.w1 += c;
    c = c && z.w1 == 0;
    z.w2 += c;
    return z;
}

// floor divmod of a signed 192-bit value by r: a = q*r + rem, 0 <= rem < r
GFP_D W192 w192_floordiv(const W192 &a, const RadixConsts &rc, u64 &rem)
{
    bool neg = w192_neg_p(a);
    W192 m = neg ? w192_negate(a) : a;
    u64 r0;
    W192 q;
    q.w2 = div128_by_r(0, m.w2, rc, r0);
    q.w1 = div128_by_r(r0, m.w1, rc, r0);
    q.w0 = div128_by_r(r0, m.w0, rc, r0);
    if (neg) {
        if (r0) {
            // -(Q + 1)
            w192_add(q, 1, 0);
            r0 = rc.r - r0;
        }
        q = w192_negate(q);
    }
    rem = r0;
    return q;
}

GFP_D bool w192_small(const W192 &a)
{
    // |a| <= 1
    if (a.w2 == 0 && a.w1 == 0 && a.w0 <= 1)
        return true;
    return a.w2 == ~0ULL && a.w1 == ~0ULL && a.w0 == ~0ULL;
}

// z = x * y mod p; x, y canonical (any form), z canonical.  z may alias.
template <int KD, typename DX, typename DY, typename DZ>
GFP_D void gfp_mul_generic(const DX &x, const DY &y, DZ &z, const RadixConsts &rc)
{
    u64 out[KD];
    W192 C = {0, 0, 0};
    for (int m = 0; m < KD; m++) {
        W192 col = C;
        for (int i = 0; i < KD; i++) {
            int j = m - i;
            bool neg = j < 0;
            if (neg)
                j += KD;
            u64 a = x[i], b = y[j];
            u64 lo = a * b, hi = __umul64hi(a, b);
            if (neg)
                w192_sub(col, lo, hi);
            else
                w192_add(col, lo, hi);
        }
        u64 rem;
        C = w192_floordiv(col, rc, rem);
        out[m] = rem;
    }
    // value = D + C r^k = D - C (mod p)
    while (!w192_small(C)) {
        W192 carry = w192_negate(C);
        for (int m = 0; m < KD; m++) {
            W192 t = carry;
            w192_add(t, out[m], 0);
            u64 rem;
            carry = w192_floordiv(t, rc, rem);
            out[m] = rem;
        }
        C = carry;
    }
    int c = (C.w0 == 0 && C.w2 == 0) ? 0 : (C.w2 == 0 ? 1 : -1);
    finish_canonical(out, KD, rc.r, c);
    for (int m = 0; m < KD; m++)
        z[m] = out[m];
}

// x^e (e as little-endian u64 limbs, shared by all threads), gfp_pow
// (gfp_field.py:164-177) with the exact multiply above.
template <int KD, typename DX, typename DZ>
GFP_D void gfp_pow_generic(const DX &x, const u64 *e, int nbits, DZ &z, const RadixConsts &rc)
{
    u64 acc[KD], base[KD];
    for (int i = 0; i < KD; i++) {
        acc[i] = i == 0 ? 1 : 0;
        base[i] = x[i];
    }
    for (int b = 0; b < nbits; b++) {
        if ((e[b >> 6] >> (b & 63)) & 1)
            gfp_mul_generic<KD>(acc, base, acc, rc);
        if (b + 1 < nbits)
            gfp_mul_generic<KD>(base, base, base, rc);
    }
    for (int i = 0; i < KD; i++)
        z[i] = acc[i];
}
