// gfp_generic_pass.cu -- the transform for radices outside the fast path.
//
// The pass kernels (k_pass44, k_pass) keep digits lazy between butterflies
// and multiply with 32-bit limbs; both need headroom in a 64-bit word that
// radices close to 2^64 do not leave (RadixConsts::stages_per_norm == 0,
// e.g. the reference's (8, 2^63 + 2^34) and (4, 2^64 - 2^50) fields,
// tests/test_gfp_field.py:15-24).  The reference's build_plan accepts any
// such prime (fft.py:237-275), so these plans run here instead: radix-2
// Stockham passes on CANONICAL digits with the reference's own element
// algorithms -- gfp_add / gfp_sub (gfp_field.py:82-135), gfp_mul_pow_r
// (:138-161) for the r^a part of each twiddle and the exact 192-bit-column
// multiply (gfp_generic.cuh) for the omega^b part, the cheap-twiddle split of
// fft.py:84-103.  Slower than the fast path (one butterfly per thread, a
// generic multiply per twiddle), exact for every r < 2^64 and
// k in {4, 8, 16, 32}; the output is the unique canonical DFT, so it equals
// the reference's dft_general bit for bit.
#include "gfp_internal.cuh"
#include "gfp_generic.cuh"

// One radix-2 Stockham pass (the radix-K pass of gfp_pass.cuh with K = 2):
// butterfly j < N/2 reads x[j], x[j + N/2], multiplies the second by
// omega^E, E = (j mod Ns) N / (2 Ns) (N - E for the inverse), and writes
// x0 + y to (j / Ns) 2 Ns + (j mod Ns) and x0 - y to that + Ns.
template <int KD>
__global__ void __launch_bounds__(128) k_pass_generic(const u64 *__restrict__ in,
                                                      u64 *__restrict__ out,
                                                      const u64 *__restrict__ table, int64_t batch,
                                                      int lN, int lM, int lNs, int inverse,
                                                      int root_inv, RadixConsts rc)
{
    const int64_t N = (int64_t)1 << lN, M = (int64_t)1 << lM, H = N >> 1;
    const int64_t nsmask = ((int64_t)1 << lNs) - 1;
    const int64_t total = batch * H;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / H, j = t - b * H;
        const u64 *src = in + b * KD * N;
        u64 *dst = out + b * KD * N;
        u64 x0[KD], x1[KD];
#pragma unroll
        for (int d = 0; d < KD; d++) {
            x0[d] = src[GFP_IDX(((int64_t)d << lN) + j, (int64_t)KD << lN)];
            x1[d] = src[GFP_IDX(((int64_t)d << lN) + j + H, (int64_t)KD << lN)];
        }
        int64_t E = (j & nsmask) << (lN - 1 - lNs);
        if (inverse && E)
            E = N - E;
        int a = (int)(E >> lM);
        const int64_t bb = E & (M - 1);
        if (root_inv && a)  // omega^M = 1/r: r^a walks backwards
            a = 2 * KD - a;
        if (bb) {
            u64 w[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                w[d] = table[GFP_IDX(bb * KD + d, M * KD)];
            gfp_mul_generic<KD>(x1, w, x1, rc);
        }
        if (a)
            dev_mul_pow_r<KD>(x1, a, rc.r);
        u64 s[KD], df[KD];
        dev_gfp_add(x0, x1, s, KD, rc.r);
        dev_gfp_sub(x0, x1, df, KD, rc.r);
        const int64_t pos = ((j >> lNs) << (lNs + 1)) + (j & nsmask);
#pragma unroll
        for (int d = 0; d < KD; d++) {
            dst[GFP_IDX(((int64_t)d << lN) + pos, (int64_t)KD << lN)] = s[d];
            dst[GFP_IDX(((int64_t)d << lN) + pos + ((int64_t)1 << lNs), (int64_t)KD << lN)] = df[d];
        }
    }
}

// element-wise product by a single element c (N^-1 of the inverse, or the
// pointwise spectrum product with c_inc = 1)
template <int KD>
__global__ void __launch_bounds__(128) k_scale_generic(const u64 *__restrict__ x,
                                                       const u64 *__restrict__ c, int64_t c_inc,
                                                       u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], y[KD];
#pragma unroll
        for (int d = 0; d < KD; d++) {
            a[d] = x[(int64_t)d * n + i];
            y[d] = c_inc ? c[(int64_t)d * n + i] : c[d];
        }
        gfp_mul_generic<KD>(a, y, a, rc);
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[(int64_t)d * n + i] = a[d];
    }
}

// log2 N radix-2 passes in ping-pong, the last one landing in `out`, then the
// N^-1 scale for the inverse; in may equal out
int run_generic(gfp_fft_plan *p, const u64 *in, u64 *out, u64 *work, int64_t batch, int inverse,
                cudaStream_t st)
{
    const int lN = ilog2_exact(p->N), lM = ilog2_exact(p->M);
    const u64 *src = in;
    for (int pass = 0; pass < lN; pass++) {
        const int remaining = lN - pass;
        u64 *dst = (remaining % 2 == 1) ? out : work;
        if (dst == src)
            dst = (dst == out) ? work : out;
        const dim3 grid = grid_for(batch * (p->N >> 1), 128);
        DISPATCH_FAST_K(p->k, (k_pass_generic<KD><<<grid, 128, 0, st>>>(
                                  src, dst, p->table, batch, lN, lM, pass, inverse, p->root_inv,
                                  p->rc)));
        p->last_launches++;
        src = dst;
    }
    if (src != out)
        cudaMemcpyAsync(out, src, sizeof(u64) * (size_t)p->k * p->N * batch,
                        cudaMemcpyDeviceToDevice, st);
    if (inverse) {
        for (int64_t b = 0; b < batch; b++) {
            u64 *v = out + b * (int64_t)p->k * p->N;
            DISPATCH_FAST_K(p->k, (k_scale_generic<KD><<<grid_for(p->N, 128), 128, 0, st>>>(
                                      v, p->ninv_dev, 0, v, p->N, p->rc)));
        }
        p->last_launches += batch;
    }
    return cuda_status();
}

// out = in .* G element-wise ([batch][k][N] digit-major)
int generic_pointwise(gfp_fft_plan *p, const u64 *in, const u64 *G, u64 *out, int64_t batch,
                      cudaStream_t st)
{
    const int64_t n = p->N;
    for (int64_t b = 0; b < batch; b++) {
        const int64_t off = b * (int64_t)p->k * n;
        DISPATCH_FAST_K(p->k, (k_scale_generic<KD><<<grid_for(n, 128), 128, 0, st>>>(
                                  in + off, G + off, 1, out + off, n, p->rc)));
    }
    p->last_launches += batch;
    return cuda_status();
}
