// gfp_probe.cu -- instrumentation: measured integer-pipe peak for the
// roofline ("IMAD.WIDE.U32 peak: to be measured on the box").
// Each thread runs NCH independent chains of 32x32 -> 64 products (one
// IMAD.WIDE each, nothing else in the loop); the result is stored so nothing
// is dead.  ops = grid * block * iters * NCH IMAD.WIDE per launch.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gfpfft.h"
#include "gfp_internal.cuh"

#define NCH 8

__global__ void k_probe_imad_wide(int64_t iters, int a0, int b0, int64_t *out)
{
    // NCH independent chains of pure IMAD.WIDE: each 32x32 -> 64 product's
    // high and low halves are the next multiplier and multiplicand, so ptxas
    // emits exactly one IMAD.WIDE per product and nothing else in the loop
    // (an accumulating mad.wide.s32 compiles on sm_100a to IMAD.WIDE + a
    // 64-bit IADD3 pair, which would measure the ALU pipe as well).  This is
    // the issue rate of the pipe the transform's limb products run on:
    // 32 per clock per SM on B200.
    int a[NCH], b[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++) {
        a[c] = a0 + c + threadIdx.x;
        b[c] = (b0 ^ blockIdx.x) + c;
    }
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            int64_t d;
            asm volatile("mul.wide.s32 %0, %1, %2;" : "=l"(d) : "r"(a[c]), "r"(b[c]));
            a[c] = (int)(d >> 32);
            b[c] = (int)d;
        }
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < NCH; c++)
        s ^= a[c] ^ b[c];
    if (s == 0x12345678)
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

extern "C" int gfp_probe_imad_wide(int64_t iters, int blocks, int threads, float *ms_out,
                                   double *ops_out, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    int64_t *out = nullptr;
    if (cudaMalloc(&out, sizeof(int64_t) * (size_t)blocks * threads) != cudaSuccess)
        return GFP_ENOMEM;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_probe_imad_wide<<<blocks, threads, 0, st>>>(iters / 10 + 1, 3, 5, out);  // warm-up
    cudaEventRecord(e0, st);
    k_probe_imad_wide<<<blocks, threads, 0, st>>>(iters, 3, 5, out);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    *ms_out = ms;
    *ops_out = (double)blocks * threads * (double)iters * NCH;
    return cudaGetLastError() == cudaSuccess ? GFP_OK : GFP_ECUDA;
}

// ---- the checked build's self-test (gfp_debug_build / gfp_debug_selftest)
__global__ void k_debug_selftest(uint64_t *out, int64_t lim)
{
    // one guarded index past its extent: the checked build prints GFP_CHECK
    out[GFP_IDX(lim + threadIdx.x, lim)] = 1;
}

extern "C" int gfp_debug_build(void) { return GFP_DEBUG; }

extern "C" int gfp_debug_selftest(void *stream)
{
    if (!GFP_DEBUG)
        return GFP_EUNSUPPORTED;
    uint64_t *buf = nullptr;
    if (cudaMalloc(&buf, 4 * sizeof(uint64_t)) != cudaSuccess)
        return GFP_ENOMEM;
    k_debug_selftest<<<1, 1, 0, (cudaStream_t)stream>>>(buf, 4);
    const int err = cudaStreamSynchronize((cudaStream_t)stream) == cudaSuccess ? GFP_OK : GFP_ECUDA;
    cudaFree(buf);
    return err;
}
