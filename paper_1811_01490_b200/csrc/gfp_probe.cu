// gfp_probe.cu -- instrumentation: measured integer-pipe peak for the
// roofline ("IMAD.WIDE.U32 peak: to be measured on the box").
// Each thread runs NCH independent mad.wide.s32 chains; the operands stay
// 32-bit so ptxas cannot fold them, and the result is stored so nothing is
// dead.  ops = grid * block * iters * NCH IMAD.WIDE per launch.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gfpfft.h"

#define NCH 8

__global__ void k_probe_imad_wide(int64_t iters, int a0, int b0, int64_t *out)
{
    int b = b0 ^ blockIdx.x;
    int64_t acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; c++)
        acc[c] = c + a0 + threadIdx.x;
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            // the multiplicand depends on the running accumulator, so the
            // product cannot be hoisted out of the loop
            int64_t d;
            asm volatile("{\n\t.reg .u32 t;\n\tcvt.u32.u64 t, %1;\n\t"
                         "mad.wide.s32 %0, t, %2, %1;\n\t}"
                         : "=l"(d) : "l"(acc[c]), "r"(b + c));
            acc[c] = d;
        }
    }
    int64_t s = 0;
#pragma unroll
    for (int c = 0; c < NCH; c++)
        s ^= acc[c];
    if (s == 0x123456789)
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
