// gfp_device.cuh -- device arithmetic for GF(p), p = r^k + 1, radix-r digits.
//
// Element representation (reference: gfp_field.py:1-8): k little-endian
// radix-r digits.  Canonical form A has every digit in [0, r); form B is
// (0, ..., 0, r) = p - 1.  Device buffers are digit-major ([k][n] per
// vector) so a warp reading one digit row of consecutive elements issues
// fully coalesced loads.
//
// Two digit regimes are used on the device:
//   * canonical  -- what every public entry point consumes and produces;
//   * lazy       -- signed 64-bit digits in [-delta, r + delta] (delta tiny),
//                   the carry-save form the transform keeps between passes so
//                   butterflies are plain digit-wise adds with no carry chain.
// Multiplication by r^a on any digit vector is exact as a rotation with the
// wrapped digits negated, because r^k = -1, so shifts
// never need normalisation.
#pragma once

// balanced -> canonical digits by carry-lookahead (else a serial chain;
// measured: C4 last pass 1.195 -> 1.070 ms, C2 graph 0.0758 -> 0.0738 ms)
#ifndef GFP_CANON_CLA
#define GFP_CANON_CLA 1
#endif
#include <stdint.h>

#include <type_traits>

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;
typedef __int128 i128;

#define GFP_HD __host__ __device__ __forceinline__
#define GFP_D __device__ __forceinline__

// ---------------------------------------------------------------------------
// Checked build (make checked: GFP_DEBUG=1).  compute-sanitizer is not
// available on the GPU pool, so the library checks itself: GFP_IDX(i, n)
// guards every global / shared index of the pass and exchange kernels
// against the logical extent of the buffer it addresses (a violation prints
// "GFP_CHECK <file>:<line> idx lim" and redirects the access to index 0, so
// the result is also wrong and the oracle comparison fails), and
// GFP_JITTER(site) sleeps a pseudo-random few hundred ns per warp at phase
// boundaries -- perturbing the warps' relative timing so that a missing
// barrier shows up as a wrong result (a timing-perturbation race test).
// Both compile to nothing in the product build.
#ifndef GFP_DEBUG
#define GFP_DEBUG 0
#endif
#if GFP_DEBUG
#include <stdio.h>
static __device__ __noinline__ long long gfp_idx_fail(long long idx, long long lim, const char *file,
                                               int line)
{
    printf("GFP_CHECK %s:%d idx=%lld lim=%lld block=(%d,%d) thread=%d\n", file, line, idx, lim,
           (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);
    return 0;
}
#define GFP_IDX(idx, lim)                                                                       \
    ([&]() -> long long {                                                                       \
        const long long i_ = (long long)(idx), l_ = (long long)(lim);                           \
        return (i_ < 0 || i_ >= l_) ? gfp_idx_fail(i_, l_, __FILE__, __LINE__) : i_;            \
    }())
#define GFP_JITTER(site)                                                                        \
    __nanosleep((unsigned)(((blockIdx.x * 131u + blockIdx.y * 7919u + (threadIdx.x >> 5) * 97u + \
                             (site) * 2654435761u) >> 7) & 511u))
#else
#define GFP_IDX(idx, lim) (idx)
#define GFP_JITTER(site) ((void)0)
#endif

// Per-radix constants, computed once on the host (exact integer arithmetic in
// the Python plan code) and passed by value to every kernel.
struct RadixConsts {
    u64 r;
    u64 d_norm;     // r << sh (top bit set)
    u64 v_recip;    // floor((2^128 - 1) / d_norm) - 2^64  (Moller-Granlund)
    u64 bias_lo;    // 2^63 * r as a 128-bit constant (fast-multiply bias)
    u64 bias_hi;
    double rinv;    // 1.0 / r (quotient estimates for small quotients)
    u64 m_recip;    // floor(2^(64+w) / r) - 2^64 (fast-multiply quotient estimate)
    u64 bias_t;     // (2^63 r) >> w
    i64 sp_mask;    // 2^sp_a - 1
    i64 sp_half;    // 2^(sp_a - 1)
    int sh;         // leading zeros of r
    int w;          // bit length of r (64 - sh)
    int s;          // limb split of the fast multiply (digit = hi 2^s + lo), 0 = no fast path
    int stages_per_norm;  // lazy radix-2 stages allowed between normalisations
    int sp_on;      // sparse radix r = 2^sp_a + sp_eps: shift-based normalisation
    int sp_a;
    int sp_eps;
    int q_sh1;      // max(w - 2S, 0) and max(2S - w, 0) for column_quot
    int q_sh2;
    // mode 2 (r = 2^a + 2^b, the paper's radices): quotients by shifts only
    int p2_ok;      // the mode's bounds hold (fast_bounds)
    int p2_b;       // b = log2(eps)
    int p2_sh;      // a - 2S (column_quot_p2)
    int p2_ab;      // a - b
    u64 p2_bias_t;  // (2^62 r) / 2^a = 2^62 + 2^(62 + b - a)
    u64 p2_bias_lo; // (2^62 r) mod 2^64
    // mode 3: r is the paper's radix for k (P2Radix<k>, compile-time a, b) and
    // the sequential-carry bounds hold (ColReduce, gfp_fast.cuh)
    int p3_ok;
    // -1, passed at run time: a window digit negated with it stays an opaque
    // operand, so ptxas keeps its products as fused IMAD.WIDE (a literal
    // negation is folded into the products, which then split into
    // IMAD + IMAD.HI pairs: measured 360 extra instructions per k = 16 multiply)
    int neg_one;
};

// ---------------------------------------------------------------------------
// 128-by-64 division with a precomputed reciprocal (Moller & Granlund,
// "Improved division by invariant integers", Alg. 4).  d normalised, u1 < d.
GFP_D u64 mg_div(u64 u1, u64 u0, u64 d, u64 v, u64 &rem)
{
    u64 q0 = v * u1;
    u64 q1 = __umul64hi(v, u1);
    u64 t = q0 + u0;
    q1 = q1 + u1 + 1 + (t < q0 ? 1 : 0);
    q0 = t;
    u64 rr = u0 - q1 * d;
    if (rr > q0) {
        q1 -= 1;
        rr += d;
    }
    if (rr >= d) {
        q1 += 1;
        rr -= d;
    }
    rem = rr;
    return q1;
}

// (u1:u0) / r for u1 < r, any r >= 2.
GFP_D u64 div128_by_r(u64 u1, u64 u0, const RadixConsts &rc, u64 &rem)
{
    int sh = rc.sh;
    u64 n1 = sh ? ((u1 << sh) | (u0 >> (64 - sh))) : u1;
    u64 n0 = u0 << sh;
    u64 rn;
    u64 q = mg_div(n1, n0, rc.d_norm, rc.v_recip, rn);
    rem = rn >> sh;
    return q;
}

// floor division of a signed 64-bit value whose quotient is small
// (|v| / r < 2^50); returns q and sets rem in [0, r).
GFP_D i64 floordiv_small(i64 v, const RadixConsts &rc, i64 &rem)
{
    double est = (double)v * rc.rinv;
    i64 q = (i64)floor(est);
    i64 rr = v - q * (i64)rc.r;
    if (rr < 0) {
        q -= 1;
        rr += (i64)rc.r;
    } else if (rr >= (i64)rc.r) {
        q += 1;
        rr -= (i64)rc.r;
    }
    rem = rr;
    return q;
}

// 32x32 -> 64 signed multiply-add, c + a b, as one IMAD.WIDE with a 64-bit
// register addend.  Written as a carry chain over the two 32-bit halves
// (mad.lo.cc.u32 + madc.hi.s32): ptxas fuses that pair into IMAD.WIDE with
// the accumulator, whereas a chain of mad.wide.s32 is re-associated into
// IMAD.WIDE ..., RZ products summed by IADD3 pairs -- one extra ALU
// instruction per product on sm_100a, where the ALU pipe is the limit.
template <bool CC = true>
GFP_D i64 mad_wide_s32(int a, int b, i64 c)
{
    if (!CC) {  // plain form (the k >= 16 kernels keep more registers free with it)
        i64 d;
        asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
        return d;
    }
    unsigned lo = (unsigned)c;
    int hi = (int)(c >> 32);
    asm("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.s32 %1, %2, %3, %1;"
        : "+r"(lo), "+r"(hi)
        : "r"(a), "r"(b));
    return (i64)(((u64)(unsigned)hi << 32) | lo);
}

// Compile-time form of mode 2 for the paper's radices (DEFAULT_RADIX,
// bench_cli.py:36-41): r = 2^a + 2^b with a, b known to the compiler, so
// every shift by a or b and every bias is an immediate (a 64-bit shift by
// a >= 32 is one SHF of the high word) -- SPARSE == 3 in the kernels.  The
// arithmetic is identical to mode 2 (same bounds, fast_bounds).
template <int KD>
struct P2Radix {
    static constexpr int a = 0, b = 0;
};
template <>
struct P2Radix<8> {
    static constexpr int a = 59, b = 16;
};
template <>
struct P2Radix<16> {
    static constexpr int a = 58, b = 10;
};
template <>
struct P2Radix<32> {
    static constexpr int a = 56, b = 21;
};
// r of the compile-time mode for k (0: none)
GFP_HD constexpr u64 p2_radix_of(int k)
{
    return k == 8 ? (1ULL << 59) + (1ULL << 16)
         : k == 16 ? (1ULL << 58) + (1ULL << 10)
         : k == 32 ? (1ULL << 56) + (1ULL << 21) : 0;
}

// Balanced lazy normaliser: v = q r + rem with q small and
// rem in [-r/2 - ex, r/2 + ex] (the host bound check fixes ex).  For the
// paper's sparse radices r = 2^a + eps it is a shift, a mask and one
// IMAD.WIDE:
//   q = (v + 2^(a-1)) >> a,  rem = ((v + 2^(a-1)) mod 2^a) - 2^(a-1) - q eps;
// otherwise a rounded division through a double estimate (one fix-up).
template <int SPARSE, int KD = 0>
GFP_D int norm_bal(i64 v, const RadixConsts &rc, i64 &rem)
{
    if constexpr (SPARSE == 3) {  // compile-time r = 2^a + 2^b
        constexpr int a = P2Radix<KD>::a, b = P2Radix<KD>::b;
        static_assert(a >= 33 && b >= 1 && b < 32, "P2Radix");
        constexpr i64 half = (i64)1 << (a - 1), mask = ((i64)1 << a) - 1;
        const i64 vb = v + half;
        const int q = (int)(vb >> a);
        rem = (vb & mask) - half - ((i64)q << b);
        return q;
    }
    if (SPARSE == 2) {  // eps = 2^b: q eps is a shift (ALU, not the IMAD pipe)
        const i64 vb = v + rc.sp_half;
        const int q = (int)(vb >> rc.sp_a);
        rem = ((vb & rc.sp_mask) - rc.sp_half) - (i64)((u64)(i64)q << rc.p2_b);
        return q;
    }
    if (SPARSE) {
        const i64 vb = v + rc.sp_half;
        const int q = (int)(vb >> rc.sp_a);
        rem = mad_wide_s32(-q, rc.sp_eps, (vb & rc.sp_mask) - rc.sp_half);
        return q;
    }
    const double est = (double)v * rc.rinv;
    i64 q = __double2ll_rn(est);
    i64 rr = v - q * (i64)rc.r;
    const i64 h = (i64)(rc.r >> 1);
    if (rr > h) {
        q += 1;
        rr -= (i64)rc.r;
    } else if (rr < -h) {
        q -= 1;
        rr += (i64)rc.r;
    }
    rem = rr;
    return (int)q;
}

// Canonical digits [0, r] to balanced lazy digits: a digit above r/2 becomes
// d - r with a carry of +1 into the next digit (negated into digit 0, since
// r^k = -1).  The value is unchanged mod p.
template <int KD>
GFP_D void to_balanced(i64 (&x)[KD], u64 r)
{
    const i64 h = (i64)(r >> 1);
    int c[KD];
#pragma unroll
    for (int i = 0; i < KD; i++) {
        c[i] = x[i] > h;
        x[i] -= c[i] ? (i64)r : 0;
    }
#pragma unroll
    for (int i = 0; i < KD; i++)
        x[i] += i ? c[i - 1] : -c[KD - 1];
}

// ---------------------------------------------------------------------------
// Canonical digit arithmetic, thread-serial, exact for any 2 <= r < 2^64.
// These restate gfp_field.py:82-161 digit loop for digit loop, since they are
// the element-wise public API (gfp_add / gfp_sub / gfp_mul_pow_r).

template <typename Digits>
GFP_HD void set_form_b(Digits &z, int k, u64 r)
{
    for (int i = 0; i < k; i++)
        z[i] = 0;
    z[k - 1] = r;
}

// gfp_add (gfp_field.py:82-109)
template <typename DX, typename DY, typename DZ>
GFP_HD void dev_gfp_add(const DX &x, const DY &y, DZ &z, int k, u64 r)
{
    u64 carry = 0;
    for (int i = 0; i < k; i++) {
        u64 a = x[i], b = y[i];
        u64 s = a + b;
        u64 c1 = s < a;
        u64 s2 = s + carry;
        c1 |= (s2 < s);
        bool ge = c1 || s2 >= r;
        z[i] = ge ? s2 - r : s2;
        carry = ge ? 1 : 0;
    }
    if (carry) {
        bool done = false;
        for (int i = 0; i < k; i++) {
            if (!done) {
                if (z[i]) {
                    z[i] -= 1;
                    done = true;
                } else {
                    z[i] = r - 1;
                }
            }
        }
        if (!done)
            set_form_b(z, k, r);
    }
}

// gfp_sub (gfp_field.py:112-135)
template <typename DX, typename DY, typename DZ>
GFP_HD void dev_gfp_sub(const DX &x, const DY &y, DZ &z, int k, u64 r)
{
    u64 borrow = 0;
    for (int i = 0; i < k; i++) {
        u64 a = x[i], b = y[i];
        u64 d = a - b;
        u64 b1 = a < b;
        u64 d2 = d - borrow;
        b1 |= (d < borrow);
        z[i] = b1 ? d2 + r : d2;
        borrow = b1;
    }
    if (borrow) {
        bool done = false;
        for (int i = 0; i < k; i++) {
            if (!done) {
                if (r >= 1 && z[i] < r - 1) {
                    z[i] += 1;
                    done = true;
                } else {
                    z[i] = 0;
                }
            }
        }
        if (!done)
            set_form_b(z, k, r);
    }
}

// ---------------------------------------------------------------------------
// Canonicalisation of a digit vector with digits in [0, r) and a signed
// overflow carry C (value = D + C * r^k = D - C mod p), |C| <= 1.
// x * r^shift on canonical digits, 0 <= shift (taken mod 2k): the
// reference's gfp_mul_pow_r (gfp_field.py:138-161) -- shift >= k negates
// first, then B - A with B the up-shifted digits and A the wrapped top
// digits; a form-B digit r moves one slot up
template <int KD>
GFP_D void dev_mul_pow_r(u64 (&a)[KD], int shift, u64 r)
{
    u64 A[KD], B[KD];
    int s = shift % (2 * KD);
    if (s >= KD) {
        u64 zero[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            zero[d] = 0;
        dev_gfp_sub(zero, a, a, KD, r);
        s -= KD;
    }
    if (s) {
        const bool formb = a[KD - 1] == r;
#pragma unroll
        for (int d = 0; d < KD; d++) {
            const int src = d - s;
            B[d] = src >= 0 ? a[src] : 0;
            A[d] = src < 0 ? a[src + KD] : 0;
        }
        if (formb) {
            // a[k-1] = r lands in A[s-1]; carry it one slot up
            for (int d = 0; d < KD; d++) {
                if (d == s - 1)
                    A[d] -= r;
                if (d == s)
                    A[d] += 1;
            }
        }
        dev_gfp_sub(B, A, a, KD, r);
    }
}

template <typename DZ>
GFP_HD void finish_canonical(DZ &z, int k, u64 r, int C)
{
    if (C == 1) {
        // D - 1; D == 0 -> p - 1 (form B)
        bool done = false;
        for (int i = 0; i < k; i++) {
            if (!done) {
                if (z[i]) {
                    z[i] -= 1;
                    done = true;
                } else {
                    z[i] = r - 1;
                }
            }
        }
        if (!done)
            set_form_b(z, k, r);
    } else if (C == -1) {
        // D + 1; D == r^k - 1 -> r^k = p - 1 (form B)
        bool done = false;
        for (int i = 0; i < k; i++) {
            if (!done) {
                if (z[i] < r - 1) {
                    z[i] += 1;
                    done = true;
                } else {
                    z[i] = 0;
                }
            }
        }
        if (!done)
            set_form_b(z, k, r);
    }
}

// Lazy digits in [-delta, r + delta] (delta < r / 4, host-verified) to the
// canonical encoding.  One carry pass keeps every carry in {-1, 0, 1}; the
// wrap carry C (value = D + C r^k = D - C mod p) is then resolved by
// finish_canonical, including the form-B cases.
template <typename DF, typename DZ>
GFP_D void lazy_to_canonical(const DF &f, DZ &z, int k, const RadixConsts &rc)
{
    const i64 r = (i64)rc.r;
    int C = 0;
    for (int i = 0; i < k; i++) {
        i64 t = (i64)f[i] + C;
        C = 0;
        if (t < 0) {
            t += r;
            C = -1;
        } else if (t >= r) {
            t -= r;
            C = 1;
        }
        z[i] = (u64)t;
    }
    finish_canonical(z, k, rc.r, C);
}

// The same canonicalisation for a compile-time k, branch-free (selects
// instead of the data-dependent loops above): the transform's last pass runs
// it for every output, and the branchy form is ~1000 SASS instructions per
// inlined copy.  Input: lazy digits with |f_i| < r - 1 (balanced or lazy;
// the carry-lookahead form needs only |f_i| < r).
template <int KD>
GFP_D void lazy_to_canonical_bf(const i64 (&f)[KD], u64 (&z)[KD], const RadixConsts &rc)
#if GFP_CANON_CLA
{
    // Balanced digits (|f_i| < r, what the pass kernels hold after their
    // normalisation) need at most one borrow per digit: z_i = f_i - b_i,
    // + r when that is negative, with the borrow into digit i + 1
    //   b_(i+1) = [f_i - b_i < 0] = g_i | (p_i & b_i),  g_i = [f_i < 0], p_i = [f_i = 0].
    // The borrows are a carry-lookahead over two k-bit masks: the carries of
    // the integer sum (g | p) + g (whose generate / propagate bits are g / p)
    // -- no serial dependence between the digits.
    static_assert(KD <= 32, "k + 1 borrow bits must fit the mask");
    using Mask = typename std::conditional<(KD < 32), unsigned, unsigned long long>::type;
    Mask g = 0, p = 0;
#pragma unroll
    for (int i = 0; i < KD; i++) {
        g |= (Mask)(f[i] < 0) << i;
        p |= (Mask)(f[i] == 0) << i;
    }
    // A borrow out of the top digit means the value D is negative and the
    // canonical residue is D + p = (D + 1) + r^k: add the 1 to digit 0 first
    // (still |f_0 + 1| < r) and run the lookahead on the adjusted masks, so the
    // digits below are final -- no carry loop through r - 1 digits afterwards.
    const Mask gp0 = g | p;
    const Mask neg = (((gp0 + g) ^ gp0 ^ g) >> KD) & 1u;
    const i64 f0 = f[0] + (i64)neg;
    g = (g & ~(Mask)1) | (Mask)(f0 < 0);
    p = (p & ~(Mask)1) | (Mask)(f0 == 0);
    const Mask gp = g | p;
    const Mask b = (gp + g) ^ gp ^ g;  // bit i: borrow into digit i (bit k: out of the top)
#pragma unroll
    for (int i = 0; i < KD; i++) {
        const i64 t = (i ? f[i] : f0) - (i64)((b >> i) & 1u);
        z[i] = (u64)(((b >> (i + 1)) & 1u) ? t + (i64)rc.r : t);
    }
    // D = -1: D + 1 = 0 has no borrow left; the residue is p - 1 = r^k (form B)
    if (neg && !((b >> KD) & 1u)) {
#pragma unroll
        for (int i = 0; i < KD - 1; i++)
            z[i] = 0;
        z[KD - 1] = rc.r;
    }
}
#else
{
    const i64 r = (i64)rc.r;
    int C = 0;
#pragma unroll
    for (int i = 0; i < KD; i++) {
        i64 t = f[i] + C;
        const bool neg = t < 0, ge = t >= r;
        t = neg ? t + r : (ge ? t - r : t);
        C = neg ? -1 : (ge ? 1 : 0);
        z[i] = (u64)t;
    }
    // value = Z - C mod p: C = 1 subtracts 1 (borrow through zero digits),
    // C = -1 adds 1 (carry through r - 1 digits); a borrow or carry out of the
    // top digit means the value is p - 1 (form B).  Rare (|C| = 1 needs the
    // top digit to overflow): kept out of the common path.
    if (C != 0) {
        bool bo = C == 1, ca = C == -1;
#pragma unroll
        for (int i = 0; i < KD; i++) {
            const u64 v = z[i];
            const bool z0 = v == 0, zt = v == rc.r - 1;
            z[i] = bo ? (z0 ? rc.r - 1 : v - 1) : (ca ? (zt ? 0 : v + 1) : v);
            bo = bo && z0;
            ca = ca && zt;
        }
        if (bo || ca) {
#pragma unroll
            for (int i = 0; i < KD - 1; i++)
                z[i] = 0;
            z[KD - 1] = rc.r;
        }
    }
}
#endif
