// gfp_mulcrt.cu -- the reference's own Z/pZ multiply MECHANISM on the GPU
// (SURVEY 8(f) row 4): gfp_mul_fft, gfp_mult.py:416-501 (paper Alg. 13).
//
// The transforms use the direct exact multiply (gfp_fast.cuh); this kernel
// restates the paper's route for callers that want it step for step:
//   convert_in  x_i, y_i mod q_j, weighted by theta^i in Montgomery form
//               (the _nega_plan in_table, gfp_mult.py:280-305)
//   convolution forward length-k cyclic NTTs of both, pointwise product,
//               inverse NTT (= the negacyclic convolution mod q_j,
//               _convolve gfp_mult.py:351-358), for q_1 = P1, q_2 = P2
//               (word_field.py:15-16)
//   convert_out * theta^-i / k, back to standard form (out_table)
//   crt         the signed coefficient v in [-(P1 P2 - 1)/2, (P1 P2 - 1)/2]
//               (crt_combine, gfp_mult.py:184-198)
//   lhc         |v| = l + h r + c r^2 (lhc_decompose, gfp_mult.py:96-116)
//   final       sum of +-(l + h r + c r^2) r^i, r^k = -1, to the canonical
//               encoding (gfp_mult.py:475-501)
// Thread per element pair, everything in registers.  The residues mod q_j
// are unique and the canonical encoding of the product is unique, so the
// result is bit-identical to the reference (and to gfp_vec_mul); the
// plan constants (theta, the tables) are computed on the host with 128-bit
// integers.  Any primitive 2k-th root theta gives the same convolution.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "gfp_internal.cuh"
#include "gfpfft.h"

namespace {

constexpr u64 CRT_P1 = 4179340454199820289ULL;  // 29 * 2^57 + 1
constexpr u64 CRT_P2 = 2485986994308513793ULL;  // 69 * 2^55 + 1
constexpr int CRT_KMAX = 64;

struct WordC {
    u64 q, qinv;  // qinv = -q^-1 mod 2^64
};

struct CrtConsts {
    WordC w[2];
    u64 in_t[2][CRT_KMAX];   // theta^i R^2 mod q: mont_mul(x, in_t) = x theta^i R
    u64 out_t[2][CRT_KMAX];  // theta^-i / k (standard form)
    u64 pw[2][CRT_KMAX];     // omega^j R (omega = theta^2), Montgomery form
    u64 pwi[2][CRT_KMAX];    // omega^-j R
    u64 m2r1, m1r2;          // (q2^-1 mod q1) R mod q1, (q1^-1 mod q2) R mod q2
    u128 q1q2, half;         // P1 P2 and (P1 P2 - 1) / 2
};

// REDC a b R^-1 mod q (mont_mul, word_field.py:133-140), q < 2^63
__device__ __forceinline__ u64 cm_mul(u64 a, u64 b, const WordC &c)
{
    const u64 lo = a * b, hi = __umul64hi(a, b);
    const u64 d = lo * c.qinv;
    const u64 t = hi + __umul64hi(d, c.q) + (lo != 0);
    return t >= c.q ? t - c.q : t;
}
__device__ __forceinline__ u64 cm_add(u64 a, u64 b, const WordC &c)
{
    const u64 s = a + b;
    return s >= c.q ? s - c.q : s;
}
__device__ __forceinline__ u64 cm_sub(u64 a, u64 b, const WordC &c)
{
    return a >= b ? a - b : a - b + c.q;
}

template <int KD>
__device__ __forceinline__ int brev(int i)
{
    int r = 0;
#pragma unroll
    for (int b = 1; b < KD; b <<= 1)
        r = (r << 1) | ((i & b) ? 1 : 0);
    return r;
}

// in-place cyclic DFT of length KD: X_u = sum_j a_j w^(j u), w^j = pw[j]
template <int KD>
__device__ __forceinline__ void ntt(u64 (&a)[KD], const u64 *pw, const WordC &c)
{
#pragma unroll
    for (int i = 0; i < KD; i++) {
        const int j = brev<KD>(i);
        if (i < j) {
            const u64 t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
#pragma unroll
    for (int len = 2; len <= KD; len <<= 1) {
#pragma unroll
        for (int i = 0; i < KD; i += len) {
#pragma unroll
            for (int jj = 0; jj < len / 2; jj++) {
                const u64 u = a[i + jj];
                const u64 v = jj ? cm_mul(a[i + jj + len / 2], pw[jj * (KD / len)], c)
                                 : a[i + jj + len / 2];
                a[i + jj] = cm_add(u, v, c);
                a[i + jj + len / 2] = cm_sub(u, v, c);
            }
        }
    }
}

// phase clock (profile instantiation only): SM cycle counter, ordered
// against the surrounding code by the asm barrier
__device__ __forceinline__ long long phase_clock()
{
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}

// the crt step for coefficient i: the signed coefficient v in
// [-(P1 P2 - 1)/2, (P1 P2 - 1)/2] as (|v|, sign) (crt_combine, gfp_mult.py:184-198)
__device__ __forceinline__ u128 crt_coeff(u64 a1, u64 a2, const CrtConsts &C, bool &neg)
{
    const u64 r1 = cm_mul(a1, C.m2r1, C.w[0]);  // a1 m2 mod q1
    const u64 r2 = cm_mul(a2, C.m1r2, C.w[1]);  // a2 m1 mod q2
    u128 v = (u128)r1 * C.w[1].q + (u128)r2 * C.w[0].q;
    if (v >= C.q1q2)
        v -= C.q1q2;
    neg = v > C.half;
    if (neg)
        v = C.q1q2 - v;
    return v;
}

// the final step for one LHC triple: +-(l + h r + c r^2) r^i into the
// signed digit accumulators (each wrap past r^k flips the sign, r^k = -1)
template <int KD>
__device__ __forceinline__ void final_accumulate(i64 (&D)[KD], int i, u64 l, u64 h, u64 cc,
                                                 bool neg)
{
    const i64 s = neg ? -1 : 1;
    const i64 terms[3] = {(i64)l * s, (i64)h * s, (i64)cc * s};
#pragma unroll
    for (int t = 0; t < 3; t++) {
        int pos = i + t;
        i64 v_t = terms[t];
        if (pos >= KD) {
            pos -= KD;
            v_t = -v_t;
        }
        if (pos >= KD) {  // k = 1 only: r^2 = (r^1)^2 = +1
            pos -= KD;
            v_t = -v_t;
        }
        D[pos] += v_t;
    }
}

// PROF: the profile instantiation (gfp_mul_fft(profile=), the reference's
// per-step keys, gfp_mult.py:428-500).  It runs the crt, lhc and final steps
// as three separate loops over the coefficients (the product is the same)
// and adds each thread's SM cycles per step into prof[0..5] = convert_in,
// convolution, convert_out, crt, lhc, final.
template <int KD, bool PROF>
__global__ void __launch_bounds__(128) k_mul_crt(const u64 *__restrict__ x, const u64 *__restrict__ y,
                                                 int64_t y_inc, u64 *__restrict__ z, int64_t n,
                                                 const __grid_constant__ CrtConsts C, RadixConsts rc,
                                                 unsigned long long *prof)
{
    const int64_t yn = y_inc ? n : 1;
    long long cyc[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ey = y_inc ? e : 0;
        u64 res[2][KD];
#pragma unroll
        for (int p = 0; p < 2; p++) {
            const WordC &c = C.w[p];
            u64 a[KD], b[KD];
            long long t0 = PROF ? phase_clock() : 0;
            // convert_in
#pragma unroll
            for (int i = 0; i < KD; i++) {
                u64 xv = x[(int64_t)i * n + e], yv = y[(int64_t)i * yn + ey];
                xv = xv >= c.q ? xv % c.q : xv;
                yv = yv >= c.q ? yv % c.q : yv;
                a[i] = cm_mul(xv, C.in_t[p][i], c);
                b[i] = cm_mul(yv, C.in_t[p][i], c);
            }
            if (PROF) {
                const long long t1 = phase_clock();
                cyc[0] += t1 - t0;
                t0 = t1;
            }
            // convolution
            ntt<KD>(a, C.pw[p], c);
            ntt<KD>(b, C.pw[p], c);
#pragma unroll
            for (int i = 0; i < KD; i++)
                a[i] = cm_mul(a[i], b[i], c);
            ntt<KD>(a, C.pwi[p], c);
            if (PROF) {
                const long long t1 = phase_clock();
                cyc[1] += t1 - t0;
                t0 = t1;
            }
            // convert_out
#pragma unroll
            for (int i = 0; i < KD; i++)
                res[p][i] = cm_mul(a[i], C.out_t[p][i], c);
            if (PROF)
                cyc[2] += phase_clock() - t0;
        }
        // crt + lhc + final: signed digit accumulators D (r^k = -1 wraps)
        i64 D[KD];
#pragma unroll
        for (int i = 0; i < KD; i++)
            D[i] = 0;
        long long t0 = PROF ? phase_clock() : 0;
        if constexpr (PROF) {
            u128 v[KD];
            bool neg[KD];
#pragma unroll
            for (int i = 0; i < KD; i++)
                v[i] = crt_coeff(res[0][i], res[1][i], C, neg[i]);
            long long t1 = phase_clock();
            cyc[3] += t1 - t0;
            t0 = t1;
            u64 L[KD], H[KD], Cc[KD];
#pragma unroll
            for (int i = 0; i < KD; i++) {
                const u64 q1 = div128_by_r((u64)(v[i] >> 64), (u64)v[i], rc, L[i]);
                Cc[i] = div128_by_r(0, q1, rc, H[i]);
            }
            t1 = phase_clock();
            cyc[4] += t1 - t0;
            t0 = t1;
#pragma unroll
            for (int i = 0; i < KD; i++)
                final_accumulate<KD>(D, i, L[i], H[i], Cc[i], neg[i]);
        } else {
#pragma unroll
            for (int i = 0; i < KD; i++) {
                bool neg;
                const u128 v = crt_coeff(res[0][i], res[1][i], C, neg);
                // |v| < k r^2 (host-checked gate): v = l + h r + c r^2
                u64 l, h, cc;
                const u64 q1 = div128_by_r((u64)(v >> 64), (u64)v, rc, l);  // v / r < k r < 2^64
                cc = div128_by_r(0, q1, rc, h);
                final_accumulate<KD>(D, i, l, h, cc, neg);
            }
        }
        // carries: digits into [0, r) with a final carry C (value = D - C,
        // r^k = -1); C is folded back into digit 0 until it is in {-1, 0, 1}
        // (one round for the paper's radices), which lazy_to_canonical
        // resolves, form B included
        i64 carry = 0;
        for (int round = 0;; round++) {
            carry = 0;
#pragma unroll
            for (int i = 0; i < KD; i++) {
                i64 rem;
                carry = floordiv_small(D[i] + carry, rc, rem);
                D[i] = rem;
            }
            if ((carry >= -1 && carry <= 1) || round == 6)
                break;
            D[0] -= carry;
        }
        D[0] -= carry;  // in [-1, r]
        u64 out[KD];
        lazy_to_canonical(D, out, KD, rc);
#pragma unroll
        for (int i = 0; i < KD; i++)
            z[(int64_t)i * n + e] = out[i];
        if (PROF)
            cyc[5] += phase_clock() - t0;
    }
    if (PROF) {
#pragma unroll
        for (int s = 0; s < 6; s++)
            atomicAdd(prof + s, (unsigned long long)cyc[s]);
    }
}

// ---- host: 128-bit plan constants
static u64 mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
static u64 powmod(u64 a, u64 e, u64 q)
{
    u64 acc = 1 % q;
    a %= q;
    while (e) {
        if (e & 1)
            acc = mulmod(acc, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return acc;
}
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }  // q prime

static WordC word_c(u64 q)
{
    u64 inv = q;
    for (int i = 0; i < 6; i++)
        inv *= 2 - q * inv;
    WordC c;
    c.q = q;
    c.qinv = (u64)0 - inv;
    return c;
}

static void make_crt_consts(int k, CrtConsts &C)
{
    memset(&C, 0, sizeof(C));
    const u64 qs[2] = {CRT_P1, CRT_P2};
    for (int p = 0; p < 2; p++) {
        const u64 q = qs[p];
        C.w[p] = word_c(q);
        const u64 R = (u64)(((u128)1 << 64) % q);
        // a primitive 2k-th root theta: theta^k = -1
        u64 theta = 1;
        for (u64 g = 2; g < 1000; g++) {
            const u64 t = powmod(g, (q - 1) / (2 * (u64)k), q);
            if (k == 1 ? t == q - 1 : powmod(t, (u64)k, q) == q - 1) {
                theta = t;
                break;
            }
        }
        const u64 omega = mulmod(theta, theta, q);
        const u64 R2 = mulmod(R, R, q);
        const u64 kinv = invmod((u64)k % q, q), tinv = invmod(theta, q), oinv = invmod(omega, q);
        u64 ti = 1, tmi = kinv, oj = 1, oij = 1;
        for (int i = 0; i < k; i++) {
            C.in_t[p][i] = mulmod(ti, R2, q);
            C.out_t[p][i] = tmi;
            C.pw[p][i] = mulmod(oj, R, q);
            C.pwi[p][i] = mulmod(oij, R, q);
            ti = mulmod(ti, theta, q);
            tmi = mulmod(tmi, tinv, q);
            oj = mulmod(oj, omega, q);
            oij = mulmod(oij, oinv, q);
        }
    }
    const u64 m2 = invmod(CRT_P2 % CRT_P1, CRT_P1);  // q2^-1 mod q1
    const u64 m1 = invmod(CRT_P1 % CRT_P2, CRT_P2);  // q1^-1 mod q2
    C.m2r1 = mulmod(m2, (u64)(((u128)1 << 64) % CRT_P1), CRT_P1);
    C.m1r2 = mulmod(m1, (u64)(((u128)1 << 64) % CRT_P2), CRT_P2);
    C.q1q2 = (u128)CRT_P1 * CRT_P2;
    C.half = (C.q1q2 - 1) / 2;
}

}  // namespace

static int mul_crt_run(const uint64_t *x, const uint64_t *y, int64_t y_inc, uint64_t *z,
                       int64_t n, int k, uint64_t r, unsigned long long *prof, cudaStream_t st)
{
    int e = check_kr(k, r);
    if (e)
        return e;
    if (!gfp_check_prime_compat(k, r))  // gfp_mult.check_prime_compat: k r^2, 2k | q - 1
        return GFP_ECONFIG;
    if (k > CRT_KMAX)
        return GFP_EUNSUPPORTED;
    if (n <= 0)
        return GFP_OK;
    // the plan constants depend on k only: built once per k (log2 k < 7)
    static CrtConsts cache[7];
    static bool have[7] = {false, false, false, false, false, false, false};
    static std::mutex mu;
    int lk = 0;
    while ((1 << lk) < k)
        lk++;
    CrtConsts C;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!have[lk]) {
            make_crt_consts(k, cache[lk]);
            have[lk] = true;
        }
        C = cache[lk];
    }
    const RadixConsts rc = make_consts(k, r);
    const dim3 grid = grid_for(n, 128);
#define MUL_CRT(KK)                                                                           \
    if (prof)                                                                                 \
        k_mul_crt<KK, true><<<grid, 128, 0, st>>>(x, y, y_inc, z, n, C, rc, prof);            \
    else                                                                                      \
        k_mul_crt<KK, false><<<grid, 128, 0, st>>>(x, y, y_inc, z, n, C, rc, nullptr);
    switch (k) {
    case 1: MUL_CRT(1) break;
    case 2: MUL_CRT(2) break;
    case 4: MUL_CRT(4) break;
    case 8: MUL_CRT(8) break;
    case 16: MUL_CRT(16) break;
    case 32: MUL_CRT(32) break;
    default: MUL_CRT(64) break;
    }
#undef MUL_CRT
    return cuda_status();
}

extern "C" int gfp_vec_mul_crt(const uint64_t *x, const uint64_t *y, int64_t y_inc, uint64_t *z,
                               int64_t n, int k, uint64_t r, void *stream)
{
    return mul_crt_run(x, y, y_inc, z, n, k, r, nullptr, (cudaStream_t)stream);
}

extern "C" int gfp_vec_mul_crt_profile(const uint64_t *x, const uint64_t *y, int64_t y_inc,
                                       uint64_t *z, int64_t n, int k, uint64_t r,
                                       uint64_t *step_cycles, float *ms, void *stream)
{
    if (!step_cycles)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *d = nullptr;
    if (cudaMalloc(&d, 6 * sizeof(unsigned long long)) != cudaSuccess)
        return GFP_ENOMEM;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEventCreate(&ev[0]);
    cudaEventCreate(&ev[1]);
    cudaMemsetAsync(d, 0, 6 * sizeof(unsigned long long), st);
    cudaEventRecord(ev[0], st);
    int err = mul_crt_run(x, y, y_inc, z, n, k, r, d, st);
    cudaEventRecord(ev[1], st);
    if (!err && cudaMemcpyAsync(step_cycles, d, 6 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, st) != cudaSuccess)
        err = GFP_ECUDA;
    if (!err && cudaStreamSynchronize(st) != cudaSuccess)
        err = GFP_ECUDA;
    if (!err && ms)
        cudaEventElapsedTime(ms, ev[0], ev[1]);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    cudaFree(d);
    return err;
}
