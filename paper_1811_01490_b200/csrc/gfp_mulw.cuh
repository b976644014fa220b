// gfp_mulw.cuh -- element-wise Z/pZ multiply for wide elements (k = 32):
// the C5 configuration's 2^22 independent products (gfp_mul_fft /
// gfp_mul_bigint, gfp_mult.py:416-512, applied element by element).
//
// Same arithmetic as fast_mul_lazy (gfp_fast.cuh: balanced 2^S limbs, limb
// Karatsuba, three sub-columns per output column, column_quot + two carry
// rounds), reorganised so a k = 32 product fits the register file: the x
// limbs (3 x 32) stay in registers, the y limbs live in this thread's
// shared-memory column ([digit][thread] int4 {l, h, l + h}, conflict-free),
// and the columns are produced in blocks of four.  For block m0..m0+3 the
// thread walks i = 0..k-1 and multiplies x_i by the window
// y_{m0-i}, ..., y_{m0+3-i} (mod k); one new y digit enters the window per
// step, so a product triple costs one LDS.128 per four columns.  y digits
// with a negative index wrap negated (r^k = -1): the sign is applied when the
// digit enters the window.  Lazy output digits go to `z` as scratch and are
// canonicalised in a second sweep by the same thread.
#pragma once
#include "gfp_internal.cuh"
#include "gfp_fast.cuh"

#ifndef GFP_MULW_CC
#define GFP_MULW_CC true  // fused-accumulate IMAD.WIDE form (gfp_device.cuh)
#endif

template <int KD, int SPARSE>
__global__ void __launch_bounds__(128, 3)
    k_mul_wide(const u64 *__restrict__ x, const u64 *__restrict__ y, int64_t y_inc,
               u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    static_assert(KD % 4 == 0, "column blocks of four");
    constexpr int S = FastSplit<KD>::S;
    extern __shared__ int4 ysm[];  // [KD][blockDim.x]
    const int nt = blockDim.x;
    int4 *my = ysm + threadIdx.x;
    const int64_t yn = y_inc ? n : 1;
    for (int64_t e = blockIdx.x * (int64_t)nt + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * nt) {
        const int64_t ey = y_inc ? e : 0;
        // ---- y: canonical -> balanced -> limbs in shared memory
        {
            i64 v[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                v[d] = (i64)y[d * yn + ey];
            to_balanced<KD>(v, rc.r);
#pragma unroll
            for (int d = 0; d < KD; d++) {
                int l, h;
                split_limbs<S>(v[d], l, h);
                my[d * nt] = make_int4(l, h, l + h, 0);
            }
        }
        // ---- x: canonical -> balanced -> limbs in registers
        int xl[KD], xh[KD], xs[KD];
        {
            i64 v[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                v[d] = (i64)x[d * n + e];
            to_balanced<KD>(v, rc.r);
#pragma unroll
            for (int d = 0; d < KD; d++) {
                split_limbs<S>(v[d], xl[d], xh[d]);
                xs[d] = xl[d] + xh[d];
            }
        }
        // ---- column blocks; carry rounds as in fast_mul_limbs
        ColReduce<S, SPARSE, KD> cr;
#pragma unroll 1
        for (int m0 = 0; m0 < KD; m0 += 4) {
            i64 LL[4], SS[4], HH[4];
#pragma unroll
            for (int c = 0; c < 4; c++)
                LL[c] = SS[c] = HH[c] = 0;
            int4 win[4];  // win[c] = +-y_{m0 + c - i}
#pragma unroll
            for (int c = 0; c < 4; c++)
                win[c] = my[(m0 + c) * nt];
#pragma unroll
            for (int i = 0; i < KD; i++) {
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    LL[c] = mad_wide_s32<GFP_MULW_CC>(xl[i], win[c].x, LL[c]);
                    HH[c] = mad_wide_s32<GFP_MULW_CC>(xh[i], win[c].y, HH[c]);
                    SS[c] = mad_wide_s32<GFP_MULW_CC>(xs[i], win[c].z, SS[c]);
                }
                if (i + 1 < KD) {
#pragma unroll
                    for (int c = 3; c > 0; c--)
                        win[c] = win[c - 1];
                    // y_{m0 - i - 1}: wraps negated when m0 - i - 1 < 0
                    const int j = m0 - i - 1;
                    int4 v = my[((j + KD) & (KD - 1)) * nt];
                    if (j < 0)
                        v = make_int4(-v.x, -v.y, -v.z, 0);
                    win[0] = v;
                }
            }
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const i64 MID = SS[c] - LL[c] - HH[c];
                i64 v;
                if (cr.column(m0 + c, LL[c], MID, HH[c], rc, v))
                    z[(m0 + c) * n + e] = (u64)v;  // lazy digit, scratch
            }
        }
        // ---- wrap carries into digits 0, 1; canonicalise
        i64 f[KD];
        cr.finish(rc, f[0], f[1]);
#pragma unroll
        for (int d = 2; d < KD; d++)
            f[d] = (i64)z[d * n + e];
        u64 c[KD];
        lazy_to_canonical(f, c, KD, rc);
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[d * n + e] = c[d];
    }
}

// launcher for k_mul_wide (k = 32): returns 1 when it handled the call
static inline int launch_mul_wide(int k, const u64 *x, const u64 *y, int64_t y_inc, u64 *z,
                                  int64_t n, const RadixConsts &rc, cudaStream_t st)
{
    if (k != 32 || rc.stages_per_norm <= 0)
        return 0;
    const int nt = 128;
    const size_t smem = sizeof(int4) * 32 * nt;
    static unsigned long long attr = 0;  // per device
    once_per_device(attr, [&] {
        cudaFuncSetAttribute(k_mul_wide<32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_mul_wide<32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_mul_wide<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_mul_wide<32, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    });
    int64_t blocks = (n + nt - 1) / nt;
    const int64_t cap = (int64_t)num_sms() * 3 * 8;
    if (blocks > cap)
        blocks = cap;
    if (rc.p3_ok)
        k_mul_wide<32, 3><<<(unsigned)blocks, nt, smem, st>>>(x, y, y_inc, z, n, rc);
    else if (rc.p2_ok)
        k_mul_wide<32, 2><<<(unsigned)blocks, nt, smem, st>>>(x, y, y_inc, z, n, rc);
    else if (rc.sp_on)
        k_mul_wide<32, 1><<<(unsigned)blocks, nt, smem, st>>>(x, y, y_inc, z, n, rc);
    else
        k_mul_wide<32, 0><<<(unsigned)blocks, nt, smem, st>>>(x, y, y_inc, z, n, rc);
    return 1;
}
