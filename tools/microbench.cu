// Integer-pipe microbenchmarks for the roofline (B200, sm_100a).
// Each kernel runs NCH independent dependent chains per thread; the
// multiplicand depends on the chain so nothing is hoisted.  Prints
// ops/clk/SM assuming the clock read from nvidia-smi is supplied.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
typedef unsigned long long u64;

__global__ void k_madwide_s32(int64_t iters, int b0, int64_t *out) {
    int64_t acc[NCH];
    for (int c = 0; c < NCH; c++) acc[c] = c + threadIdx.x;
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            int64_t d;
            asm volatile("{\n\t.reg .u32 t;\n\tcvt.u32.u64 t, %1;\n\tmad.wide.s32 %0, t, %2, %1;\n\t}" : "=l"(d) : "l"(acc[c]), "r"(b0 + c));
            acc[c] = d;
        }
    int64_t s = 0; for (int c = 0; c < NCH; c++) s ^= acc[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

__global__ void k_madwide_u32(int64_t iters, int b0, int64_t *out) {
    u64 acc[NCH];
    for (int c = 0; c < NCH; c++) acc[c] = c + threadIdx.x;
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            u64 d;
            asm volatile("{\n\t.reg .u32 t;\n\tcvt.u32.u64 t, %1;\n\tmad.wide.u32 %0, t, %2, %1;\n\t}" : "=l"(d) : "l"(acc[c]), "r"(b0 + c));
            acc[c] = d;
        }
    u64 s = 0; for (int c = 0; c < NCH; c++) s ^= acc[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

// unsigned wide mad where the multiplicand comes from a separate register
// that also evolves (mimics x_i * y_j with independent operands)
__global__ void k_madwide_u32_ind(int64_t iters, unsigned b0, int64_t *out) {
    u64 acc[NCH];
    unsigned a[NCH];
    for (int c = 0; c < NCH; c++) { acc[c] = c + threadIdx.x; a[c] = threadIdx.x * 7 + c; }
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            u64 d;
            asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a[c]), "r"(b0 + c), "l"(acc[c]));
            acc[c] = d;
            a[c] ^= (unsigned)d;  // LOP3 on the ALU pipe, keeps a[] live
        }
    u64 s = 0; for (int c = 0; c < NCH; c++) s ^= acc[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

__global__ void k_imad32(int64_t iters, int b0, int64_t *out) {
    int acc[NCH];
    for (int c = 0; c < NCH; c++) acc[c] = c + threadIdx.x;
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            int d;
            asm volatile("mad.lo.s32 %0, %1, %2, %1;" : "=r"(d) : "r"(acc[c]), "r"(b0 + c));
            acc[c] = d;
        }
    int s = 0; for (int c = 0; c < NCH; c++) s ^= acc[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

__global__ void k_iadd3(int64_t iters, int b0, int64_t *out) {
    int acc[NCH];
    for (int c = 0; c < NCH; c++) acc[c] = c + threadIdx.x;
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            int d;
            asm volatile("add.s32 %0, %1, %2;" : "=r"(d) : "r"(acc[c]), "r"(b0 + c));
            acc[c] = d;
        }
    int s = 0; for (int c = 0; c < NCH; c++) s ^= acc[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

__global__ void k_add64(int64_t iters, int b0, int64_t *out) {
    int64_t acc[NCH];
    for (int c = 0; c < NCH; c++) acc[c] = c + threadIdx.x;
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            int64_t d;
            asm volatile("add.s64 %0, %1, %2;" : "=l"(d) : "l"(acc[c]), "l"((int64_t)(b0 + c)));
            acc[c] = d;
        }
    int64_t s = 0; for (int c = 0; c < NCH; c++) s ^= acc[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

// pure IMAD.WIDE issue rate: each wide product's halves become the next
// operands (no ALU work; ptxas emits one IMAD.WIDE per product)
__global__ void k_wide_rz(int64_t iters, int b0, int64_t *out) {
    int a[NCH], b[NCH];
    for (int c = 0; c < NCH; c++) { a[c] = threadIdx.x + c; b[c] = b0 + c; }
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            int64_t d;
            asm volatile("mul.wide.s32 %0, %1, %2;" : "=l"(d) : "r"(a[c]), "r"(b[c]));
            a[c] = (int)(d >> 32);
            b[c] = (int)d;
        }
    int s = 0; for (int c = 0; c < NCH; c++) s ^= a[c] ^ b[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

// product accumulated into 64 bits as ptxas compiles it on sm_100a:
// IMAD.WIDE with RZ plus a 64-bit add (IADD3 + IADD3.X / IMAD.X)
__global__ void k_wide_acc(int64_t iters, int b0, int64_t *out) {
    int64_t acc[NCH]; int a[NCH];
    for (int c = 0; c < NCH; c++) { acc[c] = threadIdx.x + c; a[c] = threadIdx.x * 3 + c; }
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            asm volatile("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc[c]) : "r"(a[c]), "r"(b0 + c));
            a[c] = (int)(acc[c] >> 32);
        }
    int64_t s = 0; for (int c = 0; c < NCH; c++) s ^= acc[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

// IMAD.WIDE with a 64-bit register addend (the carry-chain formulation ptxas
// fuses): independent accumulators, multiplier fed from the accumulator
__global__ void k_wide_cc(int64_t iters, int b0, int64_t *out) {
    unsigned lo[NCH]; int hi[NCH], a[NCH];
    for (int c = 0; c < NCH; c++) { lo[c] = threadIdx.x + c; hi[c] = 0; a[c] = threadIdx.x * 3 + c; }
    for (int64_t i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < NCH; c++) {
            asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.s32 %1, %2, %3, %1;"
                         : "+r"(lo[c]), "+r"(hi[c]) : "r"(a[c]), "r"(b0 + c));
            a[c] = hi[c];
        }
    int64_t s = 0; for (int c = 0; c < NCH; c++) s ^= ((int64_t)hi[c] << 32) | lo[c];
    if (s == 0x1234567) out[threadIdx.x] = s;
}

template <typename F>
double run(F kern, const char *name, int sms, double mhz) {
    int64_t *out; cudaMalloc(&out, 1 << 20);
    int blocks = sms * 8, threads = 256; int64_t iters = 4000;
    kern<<<blocks, threads>>>(100, 3, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0); kern<<<blocks, threads>>>(iters, 3, out); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double ops = (double)blocks * threads * iters * NCH;
    double rate = ops / (best * 1e-3);
    printf("%-22s %8.3f ms  %9.3f Tops/s  %7.2f ops/clk/SM @%.0f MHz\n", name, best, rate / 1e12, rate / (sms * mhz * 1e6), mhz);
    cudaFree(out);
    return rate;
}

int main(int argc, char **argv) {
    double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run(k_wide_rz, "IMAD.WIDE only", sms, mhz);
    run(k_wide_acc, "IMAD.WIDE+64b add", sms, mhz);
    run(k_wide_cc, "IMAD.WIDE reg addend", sms, mhz);
    run(k_madwide_s32, "mad.wide.s32 chain", sms, mhz);
    run(k_madwide_u32, "mad.wide.u32 chain", sms, mhz);
    run(k_madwide_u32_ind, "mad.wide.u32 ind+lop", sms, mhz);
    run(k_imad32, "mad.lo.s32 chain", sms, mhz);
    run(k_iadd3, "add.s32 chain", sms, mhz);
    run(k_add64, "add.s64 chain", sms, mhz);
    return 0;
}
