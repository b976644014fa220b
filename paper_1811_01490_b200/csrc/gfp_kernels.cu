// gfp_kernels.cu -- sm_100a kernels and the C-ABI of libgfpfft.so.
//
// Layout: digit-major device vectors ([k][n], [batch][k][N]); see
// include/gfpfft.h and DESIGN.md.  Two kernel families:
//
//   element-wise (thread per element, any power-of-two k <= 128, any r):
//     k_add / k_sub / k_mul_pow_r  restate gfp_field.py:82-161 digit loops;
//     k_mul / k_pow                exact generic multiply (gfp_generic.cuh);
//     k_mul_fast                   limb-split IMAD.WIDE multiply when eligible.
//
//   transform (k in {4, 8, 16, 32}, K = 2k):
//     k_pass  one radix-K Stockham pass: coalesced digit-row loads, the
//             general twiddle (or pointwise / N^-1) multiply in registers,
//             the r^a part of the twiddle folded into the shared-memory store
//             as a digit rotation, the K-point DFT at root r (or 1/r) as
//             lazy radix-2 butterflies with one digit per lane (rotations by
//             r^t are warp shuffles + sign flips), and the store in natural
//             Stockham order.  The last pass canonicalises.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gfp_device.cuh"
#include "gfp_fast.cuh"
#include "gfp_generic.cuh"
#include "gfpfft.h"

#define FULL_MASK 0xffffffffu

// ===========================================================================
// host-side constants
// ===========================================================================

static int ilog2_exact(int64_t v)
{
    int l = 0;
    while (((int64_t)1 << l) < v)
        l++;
    return ((int64_t)1 << l) == v ? l : -1;
}

static bool valid_k(int k) { return k >= 1 && k <= 128 && (k & (k - 1)) == 0; }

static int fast_split_for(int k) { return k <= 16 ? 29 : 28; }  // FastSplit<KD>::S

struct FastPlan {
    int S;        // lazy radix-2 stages between normalisations
    int sp_on;    // sparse-radix normalisation (r = 2^a + eps, |eps| small)
    int sp_a;
    i64 sp_eps;
    u128 delta;   // balanced lazy digits stay in [-r/2 - delta, r/2 + delta]
};

// balanced normaliser (norm_bal) on |v| <= V: the quotient bound and the
// excess it leaves over [-r/2, r/2]
static void norm_bounds(u128 V, u64 r, const FastPlan &fp, u128 *qmax, u128 *ex)
{
    if (fp.sp_on) {
        u128 q = ((V + ((u128)1 << (fp.sp_a - 1))) >> fp.sp_a) + 1;
        u128 e = (u128)(fp.sp_eps < 0 ? -fp.sp_eps : fp.sp_eps);
        *qmax = q;
        *ex = q * (e + 1) + e / 2 + 2;
    } else {
        u128 q = V / r + 2;
        *qmax = q;
        *ex = q + 2;
    }
}

// Fast-path bound check, exact integer arithmetic.  Returns true and fills
// `fp` when every bound of fast_mul_lazy (gfp_fast.cuh) and of the lazy
// butterflies (k_pass) holds for balanced digits |d| <= X = r/2 + delta:
//   * 2^S X + 2^a < 2^63 (S unnormalised radix-2 stages, then norm_bal);
//   * the sub-column sums LL, SS, HH (and MID = SS - LL - HH,
//     MID + (LL >> s)) of the balanced-limb product stay below 2^63;
//   * k X^2 < 2^63 r (the biased column c + 2^63 r is in [0, 2^64 r));
//   * the carry rounds stay within 2^63 and land back inside delta.
static bool fast_bounds(int k, u64 r, FastPlan *out)
{
    if (!(k == 4 || k == 8 || k == 16 || k == 32))
        return false;
    if (r < ((u64)1 << 24) || r >= ((u64)1 << 62) || (r & (r - 1)) == 0)
        return false;
    const u128 two63 = (u128)1 << 63;
    const int K = 2 * k;
    const int logK = ilog2_exact(K);
    const u128 kk = (u128)k;
    FastPlan fp;
    memset(&fp, 0, sizeof(fp));
    // sparse radix: r = 2^a + eps with 2^a the nearest power of two
    int w = 64 - __builtin_clzll(r);
    u64 lo_p = (u64)1 << (w - 1);
    u64 hi_p = (u64)1 << w;
    if (r - lo_p <= hi_p - r) {
        fp.sp_a = w - 1;
        fp.sp_eps = (i64)(r - lo_p);
    } else {
        fp.sp_a = w;
        fp.sp_eps = -(i64)(hi_p - r);
    }
    i64 aeps = fp.sp_eps < 0 ? -fp.sp_eps : fp.sp_eps;
    fp.sp_on = aeps < ((i64)1 << 30) && fp.sp_a >= 40 && (aeps << 20) < ((i64)1 << fp.sp_a);
    const int s = fast_split_for(k);
    const u128 half = (u128)1 << (s - 1);
    const u128 top = (u128)1 << (fp.sp_on ? fp.sp_a : w);
    u128 delta = 2;  // canonical inputs enter through to_balanced (excess <= 1)
    for (int iter = 0; iter < 16; iter++) {
        u128 X = (u128)(r / 2) + delta;
        int S = 0;
        for (int t = 1; t <= logK; t++)
            if ((X << t) + top < two63)
                S = t;
        if (S < 1)
            return false;
        fp.S = S;
        u128 q1, ex1;
        norm_bounds(X << S, r, fp, &q1, &ex1);
        // multiply: balanced limbs, |xl| <= 2^(s-1), |xh| <= H, |xs| <= 2^(s-1) + H
        u128 H = (X + half) >> s;
        u128 Hs = half + H;
        if (Hs >= ((u128)1 << 31))
            return false;
        if (kk * half * half >= two63 || kk * H * H >= two63 || kk * Hs * Hs >= two63)
            return false;
        if (2 * kk * half * H + kk * half * half / ((u128)1 << s) + 2 >= two63)
            return false;
        if (w < 2 * s && ((kk * H * H) << (2 * s - w)) >= two63)
            return false;
        u128 XX = X * X;
        if (XX / r * kk + kk + 8 >= two63)
            return false;
        u128 Q1 = XX / r * kk + kk + 8;  // |column quotient|
        u128 E = 4 * (u128)r + Q1;       // |rem + carry| after round 1
        if (E + top >= two63)
            return false;
        u128 q2, ex2;
        norm_bounds(E, r, fp, &q2, &ex2);
        u128 need = ex1 > ex2 ? ex1 : ex2;
        if (need <= delta)
            break;
        delta = need;
        if (iter == 15)
            return false;
    }
    if (delta * 8 >= r)
        return false;
    fp.delta = delta;
    *out = fp;
    return true;
}

static RadixConsts make_consts(int k, u64 r)
{
    RadixConsts c;
    memset(&c, 0, sizeof(c));
    c.r = r;
    c.sh = __builtin_clzll(r);
    c.d_norm = r << c.sh;
    u128 all = ~(u128)0;
    u128 v = all / c.d_norm;
    c.v_recip = (u64)(v - ((u128)1 << 64));
    u128 bias = (u128)r << 63;
    c.bias_lo = (u64)bias;
    c.bias_hi = (u64)(bias >> 64);
    c.rinv = 1.0 / (double)r;
    c.w = 64 - c.sh;
    if (c.w < 64) {
        u128 m = ((u128)1 << (64 + c.w)) / r;
        c.m_recip = (u64)(m - ((u128)1 << 64));
    }
    FastPlan fp;
    if (fast_bounds(k, r, &fp)) {
        c.s = fast_split_for(k);
        c.stages_per_norm = fp.S;
        c.sp_on = fp.sp_on;
        c.sp_a = fp.sp_a;
        c.sp_eps = (int)fp.sp_eps;
        c.sp_mask = ((i64)1 << fp.sp_a) - 1;
        c.sp_half = (i64)1 << (fp.sp_a - 1);
        c.q_sh1 = c.w > 2 * c.s ? c.w - 2 * c.s : 0;
        c.q_sh2 = c.w < 2 * c.s ? 2 * c.s - c.w : 0;
        c.bias_t = r << (63 - c.w);
    } else {
        c.s = 0;
        c.stages_per_norm = 0;
    }
    return c;
}

// ===========================================================================
// element-wise kernels (grid-stride, thread per element)
// ===========================================================================

template <int KD>
__global__ void k_add(const u64 *__restrict__ x, const u64 *__restrict__ y, u64 *__restrict__ z,
                      int64_t n, u64 r, int sub)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], b[KD], c[KD];
#pragma unroll
        for (int d = 0; d < KD; d++) {
            a[d] = x[d * n + i];
            b[d] = y[d * n + i];
        }
        if (sub)
            dev_gfp_sub(a, b, c, KD, r);
        else
            dev_gfp_add(a, b, c, KD, r);
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

// gfp_mul_pow_r (gfp_field.py:138-161): i >= k negates first, then
// B - A with B the up-shifted digits, A the wrapped top digits; a form-B
// digit r moves one slot up.
template <int KD>
__global__ void k_mul_pow_r(const u64 *__restrict__ x, u64 *__restrict__ z, int64_t n, u64 r,
                            int shift)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], A[KD], B[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            a[d] = x[d * n + i];
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
            bool formb = a[KD - 1] == r;
#pragma unroll
            for (int d = 0; d < KD; d++) {
                int src = d - s;
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
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[d * n + i] = a[d];
    }
}

template <int KD>
__global__ void k_mul_generic(const u64 *__restrict__ x, const u64 *__restrict__ y, int64_t y_inc,
                              u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    int64_t yn = y_inc ? n : 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], b[KD], c[KD];
        int64_t iy = y_inc ? i : 0;
        for (int d = 0; d < KD; d++) {
            a[d] = x[d * n + i];
            b[d] = y[d * yn + iy];
        }
        gfp_mul_generic<KD>(a, b, c, rc);
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

template <int KD, bool SPARSE>
__global__ void k_mul_fast(const u64 *__restrict__ x, const u64 *__restrict__ y, int64_t y_inc,
                           u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    int64_t yn = y_inc ? n : 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        i64 a[KD], b[KD], f[KD];
        u64 c[KD];
        int64_t iy = y_inc ? i : 0;
#pragma unroll
        for (int d = 0; d < KD; d++) {
            a[d] = (i64)x[d * n + i];
            b[d] = (i64)y[d * yn + iy];
        }
        to_balanced<KD>(a, rc.r);
        to_balanced<KD>(b, rc.r);
        fast_mul_lazy<KD, SPARSE>(a, b, f, rc);
        lazy_to_canonical(f, c, KD, rc);
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

template <int KD>
__global__ void k_pow(const u64 *__restrict__ x, const u64 *__restrict__ e, int nbits,
                      u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], c[KD];
        for (int d = 0; d < KD; d++)
            a[d] = x[d * n + i];
        gfp_pow_generic<KD>(a, e, nbits, c, rc);
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

__global__ void k_is_canonical(const u64 *__restrict__ x, uint8_t *__restrict__ out, int64_t n,
                               int k, u64 r)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool all = true, lowzero = true;
        for (int d = 0; d < k; d++) {
            u64 v = x[d * n + i];
            if (v >= r)
                all = false;
            if (d < k - 1 && v)
                lowzero = false;
        }
        out[i] = (all || (lowzero && x[(int64_t)(k - 1) * n + i] == r)) ? 1 : 0;
    }
}

GFP_D u64 splitmix64(u64 z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void k_uniform(u64 *__restrict__ z, int64_t n, int k, u64 r, u64 seed)
{
    int64_t total = n * k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        u64 h = splitmix64(seed * 0x2545F4914F6CDD1DULL + (u64)t);
        z[t] = __umul64hi(h, r);  // uniform in [0, r)
    }
}

// element-major [n][k] -> digit-major [k][n] (dir = 0) or back (dir = 1)
__global__ void k_transpose(const u64 *__restrict__ src, u64 *__restrict__ dst, int64_t n, int k,
                            int dir)
{
    int64_t total = n * k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        // t indexes the destination linearly for coalesced stores
        if (dir == 0) {
            int64_t d = t / n, i = t % n;
            dst[t] = src[i * k + d];
        } else {
            int64_t i = t / k, d = t % k;
            dst[t] = src[d * n + i];
        }
    }
}

// ===========================================================================
// transform pass kernel
// ===========================================================================

struct PassArgs {
    const u64 *in;
    u64 *out;
    const u64 *table;  // element-major [M][k] canonical, omega^b (or omega^b / N)
    const u64 *pre;    // optional pointwise operand, digit-major like `in`
    const u64 *in2;    // optional second set of `batch` vectors (grid.y >= batch)
    u64 *out2;
    int64_t batch_stride;
    int64_t batch;
    int lN, lM, lNs;   // log2 of N, M = N/K and Ns (all powers of two)
    int lG;            // log2 of the groups per CTA
    int neg_exp;   // twiddle exponent N - E (inverse transform)
    int rot_inv;   // base-case root of this execution is 1/r (rotations by r^-t)
    int root_inv;  // the plan's omega^M is 1/r (twiddle split r^-a omega^b)
    int scale;     // every element gets a table multiply (N^-1 folded in)
    int canon;     // canonical output (last pass)
    int in_canon;  // input digits are canonical (convert to balanced on load)
    RadixConsts rc;
};

template <int KD>
GFP_D i64 rot_lane(i64 val, int t, int d, bool inverse)
{
    // multiply the digit vector held one-digit-per-lane by r^t (forward) or
    // r^-t (inverse), 0 < t < k: a rotation with the wrapped digits negated
    int src = inverse ? ((d + t) & (KD - 1)) : ((d - t) & (KD - 1));
    i64 v = __shfl_sync(FULL_MASK, val, src, KD);
    bool neg = inverse ? (d + t >= KD) : (d < t);
    return neg ? -v : v;
}

// one lazy normalisation of a digit held one-digit-per-lane: the quotient
// moves one lane up (negated into digit 0: r^k = -1)
template <int KD, bool SPARSE>
GFP_D void normalize_lane(i64 &v, int d, const RadixConsts &rc)
{
    i64 rem;
    int q = norm_bal<SPARSE>(v, rc, rem);
    int qin = __shfl_sync(FULL_MASK, q, (d - 1) & (KD - 1), KD);
    v = rem + (d == 0 ? -qin : qin);
}

template <int K>
__host__ __device__ constexpr int bitrev_c(int x)
{
    int y = 0;
    for (int b = 1; b < K; b <<= 1) {
        y = (y << 1) | (x & 1);
        x >>= 1;
    }
    return y;
}

// One radix-K Stockham pass over `batch` vectors (grid.y), G = 2^lG groups
// of K elements per CTA.  Group j reads x[j + t M] (t < K), multiplies by
// omega^E, E = t (j mod Ns) (M / Ns), and writes the K-point DFT to
// (j / Ns) Ns K + (j mod Ns) + u Ns.  After log_K N passes the output is the
// natural-order DFT (the reference's dft_general result, fft.py:298-360).
template <int KD, bool SPARSE>
__global__ void __launch_bounds__(256) k_pass(PassArgs A)
{
    constexpr int K = 2 * KD;
    constexpr int LK = KD == 4 ? 3 : KD == 8 ? 4 : KD == 16 ? 5 : 6;
    constexpr int ROW = KD + 1;  // padded smem row (bank spread)
    extern __shared__ i64 sm[];  // [K][G][ROW]
    const int lG = A.lG;
    const int G = 1 << lG;
    const int tid = threadIdx.x;
    // grid.y covers `batch` vectors of (in, out) and then, when in2 is set,
    // `batch` more of (in2, out2): two independent transforms in one launch
    int64_t bidx = blockIdx.y;
    const u64 *in_base = A.in;
    u64 *out_base = A.out;
    if (bidx >= A.batch) {
        bidx -= A.batch;
        in_base = A.in2;
        out_base = A.out2;
    }
    const int64_t j0 = (int64_t)blockIdx.x << lG;
    const int lN = A.lN, lM = A.lM, lNs = A.lNs;
    const int64_t N = (int64_t)1 << lN, M = (int64_t)1 << lM;
    const int64_t nsmask = ((int64_t)1 << lNs) - 1;
    const u64 *in = in_base + bidx * A.batch_stride;
    u64 *out = out_base + bidx * A.batch_stride;
    const u64 *pre = A.pre ? A.pre + bidx * A.batch_stride : nullptr;
    const RadixConsts rc = A.rc;

    // ---- phase A: load K elements per group, twiddle / pointwise multiply
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
        const int g = tid & (G - 1);
        const int t = (tid >> lG) + h * KD;
        const int64_t j = j0 + g;
        i64 x[KD];
        int a = 0;
        if (j < M) {
            const int64_t pos = j + ((int64_t)t << lM);
#pragma unroll
            for (int d = 0; d < KD; d++)
                x[d] = (i64)__ldg(in + ((int64_t)d << lN) + pos);
            if (A.in_canon)
                to_balanced<KD>(x, rc.r);
            if (pre) {
                i64 y[KD];
#pragma unroll
                for (int d = 0; d < KD; d++)
                    y[d] = (i64)__ldg(pre + ((int64_t)d << lN) + pos);
                fast_mul_lazy<KD, SPARSE>(x, y, x, rc);
            }
            // E = t (j mod Ns) (M / Ns) < N; omega^E = (omega^M)^a omega^b
            int64_t E = ((int64_t)t * (j & nsmask)) << (lM - lNs);
            if (A.neg_exp && E)
                E = N - E;
            a = (int)(E >> lM);
            const int64_t b = E & (M - 1);
            // omega^M is r (or 1/r for plans built on an inverse root)
            if (A.root_inv && a)
                a = 2 * KD - a;
            if (b || A.scale) {
                i64 y[KD];
                const ulonglong2 *tp = reinterpret_cast<const ulonglong2 *>(A.table + b * KD);
#pragma unroll
                for (int d = 0; d < KD; d += 2) {
                    ulonglong2 w = __ldg(tp + d / 2);
                    y[d] = (i64)w.x;
                    y[d + 1] = (i64)w.y;
                }
                fast_mul_lazy<KD, SPARSE>(x, y, x, rc);
            }
        } else {
#pragma unroll
            for (int d = 0; d < KD; d++)
                x[d] = 0;
        }
        // x * r^a: rotation by a (0 <= a < 2k), wrapped digits negated
        i64 *row = sm + (((int64_t)t << lG) + g) * ROW;
#pragma unroll
        for (int d = 0; d < KD; d++) {
            int p = d + a;
            i64 v = x[d];
            if (p >= KD) {
                p -= KD;
                v = -v;
            }
            if (p >= KD) {
                p -= KD;
                v = -v;
            }
            row[p] = v;
        }
    }
    __syncthreads();

    // ---- phase B: K-point DFT at root r (or 1/r), one digit per lane
    {
        const int d = tid & (KD - 1);
        const int g = tid / KD;
        const bool inv = A.rot_inv != 0;
        i64 v[K];
#pragma unroll
        for (int t = 0; t < K; t++)
            v[t] = sm[(((int64_t)t << lG) + g) * ROW + d];
        const int S = rc.stages_per_norm;
        int stage = 0;
#pragma unroll
        for (int len = K / 2; len >= 1; len >>= 1) {
#pragma unroll
            for (int st = 0; st < K; st += 2 * len) {
#pragma unroll
                for (int i = 0; i < len; i++) {
                    i64 a0 = v[st + i], b0 = v[st + i + len];
                    v[st + i] = a0 + b0;
                    i64 df = a0 - b0;
                    const int tw = i * (K / (2 * len));  // exponent of the root, < k
                    v[st + i + len] = tw ? rot_lane<KD>(df, tw, d, inv) : df;
                }
            }
            stage++;
            if (len > 1 && stage % S == 0) {
#pragma unroll
                for (int t = 0; t < K; t++)
                    normalize_lane<KD, SPARSE>(v[t], d, rc);
            }
        }
#pragma unroll
        for (int t = 0; t < K; t++)
            normalize_lane<KD, SPARSE>(v[t], d, rc);
        __syncthreads();
#pragma unroll
        for (int t = 0; t < K; t++)
            sm[(((int64_t)bitrev_c<K>(t) << lG) + g) * ROW + d] = v[t];
    }
    __syncthreads();

    // ---- phase C: store in Stockham order (canonicalise on the last pass)
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
        const int g = tid & (G - 1);
        const int u = (tid >> lG) + h * KD;
        const int64_t j = j0 + g;
        if (j >= M)
            continue;
        const int64_t pos = ((j >> lNs) << (lNs + LK)) + (j & nsmask) + ((int64_t)u << lNs);
        const i64 *row = sm + (((int64_t)u << lG) + g) * ROW;
        if (A.canon) {
            i64 f[KD];
            u64 c[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                f[d] = row[d];
            lazy_to_canonical(f, c, KD, rc);
#pragma unroll
            for (int d = 0; d < KD; d++)
                out[((int64_t)d << lN) + pos] = c[d];
        } else {
#pragma unroll
            for (int d = 0; d < KD; d++)
                out[((int64_t)d << lN) + pos] = (u64)row[d];
        }
    }
}

// power table: out[b] = omega^(b * step) for b < n, element-major [n][k]
// (one thread per entry, square-and-multiply over the bits of b with the
// precomputed omega^(2^i step) in `sq`), exact generic multiply.
template <int KD>
__global__ void k_power_table(const u64 *__restrict__ sq, int nsq, u64 *__restrict__ out,
                              int64_t n, RadixConsts rc)
{
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        u64 acc[KD];
        for (int d = 0; d < KD; d++)
            acc[d] = d == 0 ? 1 : 0;
        for (int i = 0; i < nsq; i++) {
            if ((b >> i) & 1) {
                u64 y[KD];
                for (int d = 0; d < KD; d++)
                    y[d] = sq[(int64_t)i * KD + d];
                gfp_mul_generic<KD>(acc, y, acc, rc);
            }
        }
        for (int d = 0; d < KD; d++)
            out[b * KD + d] = acc[d];
    }
}

// sq[i] = omega^(2^i), element-major, single thread (plan time only)
template <int KD>
__global__ void k_squarings(const u64 *__restrict__ omega, u64 *__restrict__ sq, int nsq,
                            RadixConsts rc)
{
    if (blockIdx.x || threadIdx.x)
        return;
    u64 cur[KD];
    for (int d = 0; d < KD; d++)
        cur[d] = omega[d];
    for (int i = 0; i < nsq; i++) {
        for (int d = 0; d < KD; d++)
            sq[(int64_t)i * KD + d] = cur[d];
        gfp_mul_generic<KD>(cur, cur, cur, rc);
    }
}

// element-major table times a constant (element-major [1][k])
template <int KD>
__global__ void k_table_scale(const u64 *__restrict__ tab, const u64 *__restrict__ c,
                              u64 *__restrict__ out, int64_t n, RadixConsts rc)
{
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], y[KD], z[KD];
        for (int d = 0; d < KD; d++) {
            a[d] = tab[b * KD + d];
            y[d] = c[d];
        }
        gfp_mul_generic<KD>(a, y, z, rc);
        for (int d = 0; d < KD; d++)
            out[b * KD + d] = z[d];
    }
}

// element-major canonical table entries -> balanced lazy digits (in place);
// the transform multiplies balanced operands only
template <int KD>
__global__ void k_table_balance(u64 *__restrict__ tab, int64_t n, u64 r)
{
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        i64 x[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            x[d] = (i64)tab[b * KD + d];
        to_balanced<KD>(x, r);
#pragma unroll
        for (int d = 0; d < KD; d++)
            tab[b * KD + d] = (u64)x[d];
    }
}

// Four-step inter-stage twiddle (the sharded transform):
// x is digit-major [batch][k][n] canonical; element (b, i) is multiplied by
// omega^((row0 + b) i) (omega^-(...) when inverse), omega the plan's N-th
// root, using the plan's table omega^j (j < N/K) and the cheap split
// omega^E = (omega^(N/K))^a omega^j as a digit rotation.  Canonical output.
template <int KD, bool SPARSE>
__global__ void k_twiddle_rows(const u64 *__restrict__ x, u64 *__restrict__ out,
                               const u64 *__restrict__ table, int64_t batch, int64_t n,
                               int64_t row0, int lN, int lM, int inverse, int root_inv,
                               RadixConsts rc)
{
    const int64_t total = batch * n;
    const int64_t N = (int64_t)1 << lN, M = (int64_t)1 << lM;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / n, i = t - b * n;
        const u64 *src = x + b * KD * n + i;
        u64 *dst = out + b * KD * n + i;
        i64 v[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            v[d] = (i64)src[d * n];
        int64_t E = ((row0 + b) * i) & (N - 1);
        if (inverse && E)
            E = N - E;
        int a = (int)(E >> lM);
        const int64_t j = E & (M - 1);
        if (root_inv && a)
            a = 2 * KD - a;
        if (j) {
            i64 y[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                y[d] = (i64)table[j * KD + d];
            to_balanced<KD>(v, rc.r);
            fast_mul_lazy<KD, SPARSE>(v, y, v, rc);
        }
        // rotation by a with the wrapped digits negated (r^k = -1), as a
        // log-depth network of compile-time rotations (no local memory)
        i64 w[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            w[d] = v[d];
#pragma unroll
        for (int s = 1; s < 2 * KD; s <<= 1) {
            const bool on = (a & s) != 0;
            i64 rot[KD];
#pragma unroll
            for (int d = 0; d < KD; d++) {
                if (s == KD)
                    rot[d] = -w[d];
                else
                    rot[d] = d >= s ? w[d - s] : -w[d - s + KD];
            }
#pragma unroll
            for (int d = 0; d < KD; d++)
                w[d] = on ? rot[d] : w[d];
        }
        u64 c[KD];
        lazy_to_canonical(w, c, KD, rc);
#pragma unroll
        for (int d = 0; d < KD; d++)
            dst[d * n] = c[d];
    }
}

// ===========================================================================
// C-ABI
// ===========================================================================

static int g_num_sms = 0;

static int num_sms()
{
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0)
            g_num_sms = 148;
    }
    return g_num_sms;
}

static dim3 grid_for(int64_t work, int threads)
{
    int64_t blocks = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * 32;
    if (blocks > cap)
        blocks = cap;
    if (blocks < 1)
        blocks = 1;
    return dim3((unsigned)blocks);
}

static int cuda_status()
{
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GFP_OK : GFP_ECUDA;
}

#define DISPATCH_K(k, CALL)                                                                     \
    switch (k) {                                                                                \
    case 1: { constexpr int KD = 1; CALL; } break;                                              \
    case 2: { constexpr int KD = 2; CALL; } break;                                              \
    case 4: { constexpr int KD = 4; CALL; } break;                                              \
    case 8: { constexpr int KD = 8; CALL; } break;                                              \
    case 16: { constexpr int KD = 16; CALL; } break;                                            \
    case 32: { constexpr int KD = 32; CALL; } break;                                            \
    case 64: { constexpr int KD = 64; CALL; } break;                                            \
    case 128: { constexpr int KD = 128; CALL; } break;                                          \
    default: return GFP_EINVAL;                                                                 \
    }

#define DISPATCH_FAST_K(k, CALL)                                                                \
    switch (k) {                                                                                \
    case 4: { constexpr int KD = 4; CALL; } break;                                              \
    case 8: { constexpr int KD = 8; CALL; } break;                                              \
    case 16: { constexpr int KD = 16; CALL; } break;                                            \
    case 32: { constexpr int KD = 32; CALL; } break;                                            \
    default: return GFP_EUNSUPPORTED;                                                           \
    }

extern "C" {

const char *gfp_strerror(int code)
{
    switch (code) {
    case GFP_OK: return "ok";
    case GFP_EINVAL: return "invalid argument";
    case GFP_ECONFIG: return "configuration not supported by the prime pair";
    case GFP_ECUDA: return "CUDA runtime error";
    case GFP_ENOMEM: return "device allocation failed";
    case GFP_EUNSUPPORTED: return "parameters outside the transform kernels' range";
    default: return "unknown error";
    }
}

int gfp_version(void) { return 1; }

int gfp_check_prime_compat(int k, uint64_t r)
{
    const u64 P1 = 4179340454199820289ULL, P2 = 2485986994308513793ULL;
    if (!valid_k(k) || r < 2)
        return 0;
    u128 limit = ((u128)P1 * P2 - 1) / 2;
    u128 r2 = (u128)r * r;
    if (r2 > limit / (u64)k)
        return 0;
    if ((P1 - 1) % (2 * (u64)k) || (P2 - 1) % (2 * (u64)k))
        return 0;
    return 1;
}

int gfp_fast_path_ok(int k, uint64_t r)
{
    FastPlan fp;
    return fast_bounds(k, r, &fp) ? 1 : 0;
}

static int check_kr(int k, u64 r)
{
    if (!valid_k(k) || r < 2)
        return GFP_EINVAL;
    return GFP_OK;
}

int gfp_vec_add(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k, uint64_t r,
                void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    cudaStream_t st = (cudaStream_t)stream;
    DISPATCH_K(k, (k_add<KD><<<grid_for(n, 256), 256, 0, st>>>(x, y, z, n, r, 0)));
    return cuda_status();
}

int gfp_vec_sub(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k, uint64_t r,
                void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    cudaStream_t st = (cudaStream_t)stream;
    DISPATCH_K(k, (k_add<KD><<<grid_for(n, 256), 256, 0, st>>>(x, y, z, n, r, 1)));
    return cuda_status();
}

int gfp_vec_mul_pow_r(const uint64_t *x, uint64_t *z, int64_t n, int k, uint64_t r, int i,
                      void *stream)
{
    int e = check_kr(k, r);
    if (e)
        return e;
    if (i < 0 || i > 2 * k)
        return GFP_EINVAL;
    if (n <= 0)
        return GFP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DISPATCH_K(k, (k_mul_pow_r<KD><<<grid_for(n, 256), 256, 0, st>>>(x, z, n, r, i)));
    return cuda_status();
}

int gfp_vec_mul(const uint64_t *x, const uint64_t *y, int64_t y_inc, uint64_t *z, int64_t n,
                int k, uint64_t r, void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    cudaStream_t st = (cudaStream_t)stream;
    RadixConsts rc = make_consts(k, r);
    if (rc.stages_per_norm > 0) {
        if (rc.sp_on) {
            DISPATCH_FAST_K(k, (k_mul_fast<KD, true><<<grid_for(n, 128), 128, 0, st>>>(
                                   x, y, y_inc, z, n, rc)));
        } else {
            DISPATCH_FAST_K(k, (k_mul_fast<KD, false><<<grid_for(n, 128), 128, 0, st>>>(
                                   x, y, y_inc, z, n, rc)));
        }
    } else {
        DISPATCH_K(k, (k_mul_generic<KD><<<grid_for(n, 128), 128, 0, st>>>(x, y, y_inc, z, n,
                                                                           rc)));
    }
    return cuda_status();
}

int gfp_vec_pow(const uint64_t *x, const uint64_t *e_limbs, int e_nlimbs, uint64_t *z, int64_t n,
                int k, uint64_t r, void *stream)
{
    int e = check_kr(k, r);
    if (e)
        return e;
    if (n <= 0)
        return GFP_OK;
    if (e_nlimbs < 0)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    int nl = e_nlimbs > 0 ? e_nlimbs : 1;
    u64 *d_e = nullptr;
    if (cudaMallocAsync(&d_e, sizeof(u64) * nl, st) != cudaSuccess)
        return GFP_ENOMEM;
    u64 zero = 0;
    cudaMemcpyAsync(d_e, e_nlimbs ? e_limbs : &zero, sizeof(u64) * nl, cudaMemcpyHostToDevice, st);
    int nbits = 0;
    for (int i = e_nlimbs - 1; i >= 0; i--)
        if (e_limbs[i]) {
            nbits = 64 * i + 64 - __builtin_clzll(e_limbs[i]);
            break;
        }
    RadixConsts rc = make_consts(k, r);
    DISPATCH_K(k, (k_pow<KD><<<grid_for(n, 64), 64, 0, st>>>(x, d_e, nbits, z, n, rc)));
    int rcode = cuda_status();
    cudaStreamSynchronize(st);  // e_limbs is caller host memory
    cudaFreeAsync(d_e, st);
    return rcode;
}

int gfp_vec_is_canonical(const uint64_t *x, uint8_t *out, int64_t n, int k, uint64_t r,
                         void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    k_is_canonical<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, out, n, k, r);
    return cuda_status();
}

int gfp_vec_uniform(uint64_t *z, int64_t n, int k, uint64_t r, uint64_t seed, void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    k_uniform<<<grid_for(n * k, 256), 256, 0, (cudaStream_t)stream>>>(z, n, k, r, seed);
    return cuda_status();
}

int gfp_to_digit_major(const uint64_t *src, uint64_t *dst, int64_t n, int k, void *stream)
{
    if (!valid_k(k))
        return GFP_EINVAL;
    if (n <= 0)
        return GFP_OK;
    k_transpose<<<grid_for(n * k, 256), 256, 0, (cudaStream_t)stream>>>(src, dst, n, k, 0);
    return cuda_status();
}

int gfp_to_element_major(const uint64_t *src, uint64_t *dst, int64_t n, int k, void *stream)
{
    if (!valid_k(k))
        return GFP_EINVAL;
    if (n <= 0)
        return GFP_OK;
    k_transpose<<<grid_for(n * k, 256), 256, 0, (cudaStream_t)stream>>>(src, dst, n, k, 1);
    return cuda_status();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// plans

struct gfp_fft_plan {
    int k, K, e;
    int64_t N, M;
    u64 r;
    RadixConsts rc;
    u64 *table;       // element-major [M][k]: omega^b
    u64 *table_ninv;  // element-major [M][k]: omega^b * N^-1
    // host-path scratch
    u64 *h_dev;
    int64_t h_words;
    int64_t last_launches;
    int root_inv;  // omega^(N/2k) == 1/r (a plan built on an inverse root)
};

static int pass_threads(int k, int64_t M, int *G_out)
{
    // groups per CTA: as many as fit 256 threads, fewer when the transform
    // is too small to give every SM two CTAs
    int Gmax = 256 / k;
    int Gmin = 32 / k > 0 ? 32 / k : 1;
    int G = Gmax;
    while (G > Gmin && (M + G - 1) / G < 2 * (int64_t)num_sms())
        G >>= 1;
    *G_out = G;
    return G * k;
}

template <int KD>
static size_t pass_smem(int G)
{
    return (size_t)(2 * KD) * G * (KD + 1) * sizeof(i64);
}

template <int KD>
static int launch_pass(const gfp_fft_plan *p, const u64 *in, u64 *out, const u64 *in2,
                       u64 *out2, const u64 *pre, int64_t batch, int64_t Ns, int inverse,
                       int scale, int canon, int in_canon, cudaStream_t st)
{
    int G;
    int threads = pass_threads(KD, p->M, &G);
    size_t smem = pass_smem<KD>(G);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_pass<KD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pass_smem<KD>(256 / KD));
        cudaFuncSetAttribute(k_pass<KD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pass_smem<KD>(256 / KD));
        attr_set = true;
    }
    PassArgs A;
    A.in = in;
    A.out = out;
    A.table = scale ? p->table_ninv : p->table;
    A.pre = pre;
    A.batch_stride = (int64_t)KD * p->N;
    A.lN = ilog2_exact(p->N);
    A.lM = ilog2_exact(p->M);
    A.lNs = ilog2_exact(Ns);
    A.lG = ilog2_exact(G);
    A.neg_exp = inverse;
    A.rot_inv = inverse ^ p->root_inv;
    A.root_inv = p->root_inv;
    A.scale = scale;
    A.canon = canon;
    A.in_canon = in_canon;
    A.rc = p->rc;
    A.in2 = in2;
    A.out2 = out2;
    A.batch = batch;
    dim3 grid((unsigned)((p->M + G - 1) / G), (unsigned)(in2 ? 2 * batch : batch));
    if (p->rc.sp_on) {
        k_pass<KD, true><<<grid, threads, smem, st>>>(A);
    } else {
        k_pass<KD, false><<<grid, threads, smem, st>>>(A);
    }
    return cuda_status();
}

// One transform of `batch` vectors (and, when in_b is given, a second
// independent set of `batch` vectors transformed in the same launches).
// in_canon: the input is canonical (user data) and is converted to balanced
// digits on load; out_canon: the last pass canonicalises (user-visible
// output) -- poly_mul keeps its intermediate spectra as balanced lazy digits.
// `pre` is a pointwise operand (balanced lazy) multiplied in on the first
// pass (single set only).
static int run_transform2(gfp_fft_plan *p, const u64 *in, u64 *out, u64 *work, const u64 *in_b,
                          u64 *out_b, u64 *work_b, const u64 *pre, int64_t batch, int inverse,
                          int in_canon, int out_canon, cudaStream_t st)
{
    // ping-pong so that the last pass lands in `out`; inputs are never written
    int e = p->e;
    const u64 *src = in, *src_b = in_b;
    int64_t Ns = 1;
    for (int pass = 0; pass < e; pass++) {
        int remaining = e - pass;  // passes left including this one
        u64 *dst = (remaining % 2 == 1) ? out : work;
        if (dst == src)
            dst = (dst == out) ? work : out;
        u64 *dst_b = nullptr;
        if (in_b) {
            dst_b = (remaining % 2 == 1) ? out_b : work_b;
            if (dst_b == src_b)
                dst_b = (dst_b == out_b) ? work_b : out_b;
        }
        int last = pass == e - 1;
        int scale = inverse && last;
        const u64 *pre_p = pass == 0 ? pre : nullptr;
        int rcode;
        DISPATCH_FAST_K(p->k, (rcode = launch_pass<KD>(p, src, dst, src_b, dst_b, pre_p, batch,
                                                       Ns, inverse, scale, last && out_canon,
                                                       pass == 0 && in_canon, st)));
        if (rcode)
            return rcode;
        p->last_launches++;
        src = dst;
        src_b = dst_b;
        Ns *= p->K;
    }
    if (src != out)
        cudaMemcpyAsync(out, src, sizeof(u64) * (size_t)p->k * p->N * batch,
                        cudaMemcpyDeviceToDevice, st);
    if (in_b && src_b != out_b)
        cudaMemcpyAsync(out_b, src_b, sizeof(u64) * (size_t)p->k * p->N * batch,
                        cudaMemcpyDeviceToDevice, st);
    return cuda_status();
}

static int run_transform(gfp_fft_plan *p, const u64 *in, u64 *out, u64 *work, const u64 *pre,
                         int64_t batch, int inverse, int in_canon, int out_canon,
                         cudaStream_t st)
{
    return run_transform2(p, in, out, work, nullptr, nullptr, nullptr, pre, batch, inverse,
                          in_canon, out_canon, st);
}

extern "C" {

int gfp_fft_plan_create(gfp_fft_plan **plan, int k, uint64_t r, int K, int e,
                        const uint64_t *omega, void *stream)
{
    if (!plan)
        return GFP_EINVAL;
    *plan = nullptr;
    int err = check_kr(k, r);
    if (err)
        return err;
    if (K != 8 && K != 16 && K != 32 && K != 64)
        return GFP_EINVAL;
    if (e < 1)
        return GFP_EINVAL;
    if (K != 2 * k)
        return GFP_EINVAL;
    int64_t N = 1;
    for (int i = 0; i < e; i++) {
        N *= K;
        if (N > ((int64_t)1 << 40))
            return GFP_EINVAL;
    }
    for (int d = 0; d < k; d++)
        if (omega[d] > r)
            return GFP_EINVAL;
    RadixConsts rc = make_consts(k, r);
    if (rc.stages_per_norm <= 0)
        return GFP_EUNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    gfp_fft_plan *p = (gfp_fft_plan *)calloc(1, sizeof(gfp_fft_plan));
    if (!p)
        return GFP_ENOMEM;
    p->k = k;
    p->K = K;
    p->e = e;
    p->N = N;
    p->M = N / K;
    p->r = r;
    p->rc = rc;

    // ---- validate omega like build_plan (fft.py:250-267): omega^N = 1,
    // omega^(N/2) = -1, omega^(N/2k) in {r, r^(2k-1)}
    u64 *d_buf = nullptr;
    size_t words = (size_t)k * 8;
    if (cudaMalloc(&d_buf, sizeof(u64) * words) != cudaSuccess) {
        free(p);
        return GFP_ENOMEM;
    }
    // d_buf: [0] omega (digit-major == element-major for n=1), [1..3] results
    cudaMemcpyAsync(d_buf, omega, sizeof(u64) * k, cudaMemcpyHostToDevice, st);
    u64 exps[3] = {(u64)N, (u64)(N / 2), (u64)(N / (2 * k))};
    for (int i = 0; i < 3; i++) {
        err = gfp_vec_pow(d_buf, &exps[i], 1, d_buf + (size_t)(i + 1) * k, 1, k, r, stream);
        if (err)
            break;
    }
    u64 h_res[3 * 128];
    if (!err && cudaMemcpyAsync(h_res, d_buf + k, sizeof(u64) * 3 * k, cudaMemcpyDeviceToHost,
                                st) != cudaSuccess)
        err = GFP_ECUDA;
    if (!err && cudaStreamSynchronize(st) != cudaSuccess)
        err = GFP_ECUDA;
    if (!err) {
        bool one = true, mone = true, fwd = true, inv = true;
        for (int d = 0; d < k; d++) {
            if (h_res[d] != (u64)(d == 0))
                one = false;
            if (h_res[k + d] != (d == k - 1 ? r : 0))
                mone = false;
            // r as an element: digit 1 = 1 (k >= 2)
            if (h_res[2 * k + d] != (u64)(d == 1))
                fwd = false;
        }
        // 1/r = r^(2k-1) = -(r^(k-1)) = p - r^(k-1) = (r - 1) r^(k-1) + 1
        for (int d = 0; d < k; d++) {
            u64 want = (d == k - 1 ? r - 1 : 0) + (d == 0 ? 1 : 0);
            if (h_res[2 * k + d] != want)
                inv = false;
        }
        if (!one || !mone || !(fwd || inv))
            err = GFP_EINVAL;
        p->root_inv = fwd ? 0 : 1;
    }
    if (err) {
        cudaFree(d_buf);
        free(p);
        return err;
    }

    // ---- twiddle tables: omega^b (b < M) and omega^b * N^-1
    int nsq = 0;
    while (((int64_t)1 << nsq) < p->M)
        nsq++;
    u64 *d_sq = nullptr;
    size_t tbytes = sizeof(u64) * (size_t)k * p->M;
    if (cudaMalloc(&p->table, tbytes) != cudaSuccess ||
        cudaMalloc(&p->table_ninv, tbytes) != cudaSuccess ||
        cudaMalloc(&d_sq, sizeof(u64) * (size_t)k * (nsq + 1)) != cudaSuccess) {
        cudaFree(p->table);
        cudaFree(p->table_ninv);
        cudaFree(d_sq);
        cudaFree(d_buf);
        free(p);
        return GFP_ENOMEM;
    }
    // N^-1 = -(r^k / N) mod p (N | r^k = p - 1): radix-r long division of
    // r^k by N on the host, then negation with the canonical subtract
    u64 q[128], ninv[128], zero[128];
    {
        u128 rem = 1;  // digit k of r^k
        for (int i = k - 1; i >= 0; i--) {
            u128 cur = rem * r;
            q[i] = (u64)(cur / (u64)N);
            rem = cur % (u64)N;
        }
        for (int d = 0; d < k; d++)
            zero[d] = 0;
        dev_gfp_sub(zero, q, ninv, k, r);
    }
    cudaMemcpyAsync(d_buf, ninv, sizeof(u64) * k, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_buf + k, omega, sizeof(u64) * k, cudaMemcpyHostToDevice, st);
    DISPATCH_FAST_K(k, (k_squarings<KD><<<1, 32, 0, st>>>(d_buf + k, d_sq, nsq, rc)));
    DISPATCH_FAST_K(k, (k_power_table<KD><<<grid_for(p->M, 64), 64, 0, st>>>(d_sq, nsq, p->table,
                                                                           p->M, rc)));
    DISPATCH_FAST_K(k, (k_table_scale<KD><<<grid_for(p->M, 64), 64, 0, st>>>(
                           p->table, d_buf, p->table_ninv, p->M, rc)));
    DISPATCH_FAST_K(k, (k_table_balance<KD><<<grid_for(p->M, 128), 128, 0, st>>>(p->table, p->M, r)));
    DISPATCH_FAST_K(k, (k_table_balance<KD><<<grid_for(p->M, 128), 128, 0, st>>>(p->table_ninv, p->M,
                                                                                r)));
    err = cuda_status();
    if (!err && cudaStreamSynchronize(st) != cudaSuccess)
        err = GFP_ECUDA;
    cudaFree(d_sq);
    cudaFree(d_buf);
    if (err) {
        cudaFree(p->table);
        cudaFree(p->table_ninv);
        free(p);
        return err;
    }
    *plan = p;
    return GFP_OK;
}

int gfp_fft_twiddle(const gfp_fft_plan *p, const uint64_t *x, uint64_t *out, int64_t batch,
                    int64_t n, int64_t row0, int inverse, void *stream)
{
    if (!p || !x || !out || batch < 1 || n < 1 || row0 < 0)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int lN = ilog2_exact(p->N), lM = ilog2_exact(p->M);
    dim3 grid = grid_for(batch * n, 128);
    if (p->rc.sp_on) {
        DISPATCH_FAST_K(p->k, (k_twiddle_rows<KD, true><<<grid, 128, 0, st>>>(
                                  x, out, p->table, batch, n, row0, lN, lM, inverse ? 1 : 0,
                                  p->root_inv, p->rc)));
    } else {
        DISPATCH_FAST_K(p->k, (k_twiddle_rows<KD, false><<<grid, 128, 0, st>>>(
                                  x, out, p->table, batch, n, row0, lN, lM, inverse ? 1 : 0,
                                  p->root_inv, p->rc)));
    }
    return cuda_status();
}

int gfp_fft_plan_destroy(gfp_fft_plan *p)
{
    if (!p)
        return GFP_OK;
    cudaFree(p->table);
    cudaFree(p->table_ninv);
    cudaFree(p->h_dev);
    free(p);
    return GFP_OK;
}

int64_t gfp_fft_plan_size(const gfp_fft_plan *p) { return p ? p->N : 0; }

int64_t gfp_fft_workspace_words(const gfp_fft_plan *p, int64_t batch)
{
    return p ? 3 * (int64_t)p->k * p->N * batch : 0;
}

int64_t gfp_fft_plan_last_launches(const gfp_fft_plan *p) { return p ? p->last_launches : 0; }

int gfp_fft_exec(const gfp_fft_plan *cp, const uint64_t *in, uint64_t *out, uint64_t *work,
                 int64_t batch, int inverse, void *stream)
{
    gfp_fft_plan *p = const_cast<gfp_fft_plan *>(cp);
    if (!p || !in || !out || !work || batch < 1)
        return GFP_EINVAL;
    p->last_launches = 0;
    return run_transform(p, in, out, work, nullptr, batch, inverse ? 1 : 0, 1, 1,
                         (cudaStream_t)stream);
}

int gfp_poly_mul(const gfp_fft_plan *cp, const uint64_t *f, const uint64_t *g, uint64_t *out,
                 uint64_t *work, int64_t batch, void *stream)
{
    gfp_fft_plan *p = const_cast<gfp_fft_plan *>(cp);
    if (!p || !f || !g || !out || !work || batch < 1)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    p->last_launches = 0;
    int64_t vw = (int64_t)p->k * p->N * batch;
    u64 *G = work;        // DFT(g)
    u64 *scratch = work + vw;
    u64 *scratch_b = work + 2 * vw;
    // out = DFT(f) and G = DFT(g) in the same launches; the spectra stay
    // balanced lazy digits, only the product is canonicalised
    int err = run_transform2(p, f, out, scratch, g, G, scratch_b, nullptr, batch, 0, 1, 0, st);
    if (!err)  // out = IDFT(out .* G), the pointwise product fused into pass 0
        err = run_transform(p, out, out, scratch, G, batch, 1, 0, 1, st);
    return err;
}

static int ensure_host_scratch(gfp_fft_plan *p, int64_t words)
{
    if (p->h_words >= words)
        return GFP_OK;
    cudaFree(p->h_dev);
    p->h_dev = nullptr;
    p->h_words = 0;
    if (cudaMalloc(&p->h_dev, sizeof(u64) * (size_t)words) != cudaSuccess)
        return GFP_ENOMEM;
    p->h_words = words;
    return GFP_OK;
}

int gfp_fft_exec_host(gfp_fft_plan *p, uint64_t *v, int64_t batch, int inverse, void *stream)
{
    if (!p || !v || batch < 1)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t vw = (int64_t)p->k * p->N * batch;
    int err = ensure_host_scratch(p, 3 * vw);
    if (err)
        return err;
    u64 *a = p->h_dev, *b = a + vw, *w = b + vw;
    cudaMemcpyAsync(a, v, sizeof(u64) * vw, cudaMemcpyHostToDevice, st);
    p->last_launches = 0;
    for (int64_t i = 0; i < batch; i++)
        gfp_to_digit_major(a + i * p->k * p->N, b + i * p->k * p->N, p->N, p->k, st);
    err = run_transform(p, b, b, w, nullptr, batch, inverse ? 1 : 0, 1, 1, st);
    if (err)
        return err;
    for (int64_t i = 0; i < batch; i++)
        gfp_to_element_major(b + i * p->k * p->N, a + i * p->k * p->N, p->N, p->k, st);
    p->last_launches += 2 * batch;
    cudaMemcpyAsync(v, a, sizeof(u64) * vw, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return GFP_ECUDA;
    return cuda_status();
}

int gfp_poly_mul_host(gfp_fft_plan *p, const uint64_t *f, const uint64_t *g, uint64_t *out,
                      int64_t batch, void *stream)
{
    if (!p || !f || !g || !out || batch < 1)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t vw = (int64_t)p->k * p->N * batch;
    int err = ensure_host_scratch(p, 7 * vw);
    if (err)
        return err;
    u64 *hf = p->h_dev, *hg = hf + vw, *df = hg + vw, *dg = df + vw, *w = dg + vw;
    cudaMemcpyAsync(hf, f, sizeof(u64) * vw, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(hg, g, sizeof(u64) * vw, cudaMemcpyHostToDevice, st);
    for (int64_t i = 0; i < batch; i++) {
        gfp_to_digit_major(hf + i * p->k * p->N, df + i * p->k * p->N, p->N, p->k, st);
        gfp_to_digit_major(hg + i * p->k * p->N, dg + i * p->k * p->N, p->N, p->k, st);
    }
    err = gfp_poly_mul(p, df, dg, df, w, batch, st);
    if (err)
        return err;
    for (int64_t i = 0; i < batch; i++)
        gfp_to_element_major(df + i * p->k * p->N, hf + i * p->k * p->N, p->N, p->k, st);
    p->last_launches += 3 * batch;
    cudaMemcpyAsync(out, hf, sizeof(u64) * vw, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return GFP_ECUDA;
    return cuda_status();
}

}  // extern "C"
