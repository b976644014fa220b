// gfp_internal.cuh -- declarations shared by the translation units of
// libgfpfft.so (host helpers, the pass-kernel arguments, the plan object).
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gfp_device.cuh"
#include "gfpfft.h"

#define FULL_MASK 0xffffffffu

int ilog2_exact(int64_t v);
bool valid_k(int k);
RadixConsts make_consts(int k, u64 r);
bool fast_path_bounds_ok(int k, u64 r);
int num_sms();
dim3 grid_for(int64_t work, int threads);
int cuda_status();
int check_kr(int k, u64 r);
// Two-stream pipeline of the host entry points: chunk i of a large call runs
// on stream s[i % 2] (its copies and kernels in order), so one chunk's H2D
// overlaps the other's kernels and D2H (PCIe is full duplex).  begin makes
// both streams wait for the caller's stream; end makes the caller's stream
// wait for both and releases them.
struct HostPipe {
    cudaStream_t s[2] = {nullptr, nullptr};
    cudaEvent_t ev = nullptr;
};
int host_pipe_begin(HostPipe &hp, cudaStream_t caller);
int host_pipe_end(HostPipe &hp, cudaStream_t caller);
// words of one pipeline chunk (128 MiB)
constexpr int64_t HOST_CHUNK_WORDS = (int64_t)1 << 24;

// element-major [B][n_em][k] <-> digit-major [B][k][n_dm] (to_dm: zero-pad
// i >= n_em; else write i < n_em only), tiled through shared memory
int transpose_batched(const u64 *src, u64 *dst, int64_t batch, int64_t n_em, int64_t n_dm, int k,
                      int to_dm, cudaStream_t st);

// Run f once per CUDA device (function attributes such as the dynamic
// shared-memory limit apply per device context); `mask` holds one bit per
// device id.  A benign race only repeats the idempotent f.
template <typename F>
inline void once_per_device(unsigned long long &mask, F &&f)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & bit)
        return;
    f();
    __atomic_fetch_or(&mask, bit, __ATOMIC_ACQ_REL);
}

struct gfp_fft_plan;

// pass launches served by k_pass44t (gfp_tma_pass_launches)
extern long long g_tma_pass_launches;

#define GFP_MAX_GRID_Y 65535  // pass kernels put the batch in grid.y
#define GFP_MAX_TIMED 64  // pass launches timed per call (gfp_fft_plan_pass_times)

struct PassArgs {
    const u64 *in;
    u64 *out;
    const u64 *table;  // element-major [M][k] balanced, omega^b (or omega^b / N)
    const u64 *table_lh;  // the same entries as limb pairs l | h << 32 (k_pass44)
    const u64 *pre;    // optional pointwise operand, digit-major like `in`
    const u64 *in2;    // optional second set of `batch` vectors (grid.y >= batch)
    u64 *out2;
    int64_t batch_stride;
    int64_t batch;
    int lN, lM, lNs;   // log2 of N, M = N/K and Ns (all powers of two)
    int lG;            // log2 of the groups per CTA (k_pass)
    int gpc;           // groups per CTA, 1..32 (k_pass44; 32 unless the grid is under two waves)
    int neg_exp;   // twiddle exponent N - E (inverse transform)
    int rot_inv;   // base-case root of this execution is 1/r (rotations by r^-t)
    int root_inv;  // the plan's omega^M is 1/r (twiddle split r^-a omega^b)
    int scale;     // every element gets a table multiply (N^-1 folded in)
    int canon;     // canonical output (last pass)
    int in_canon;  // input digits are canonical (convert to balanced on load)
    RadixConsts rc;
    // element-major I/O (the host entry points; k_pass44 only): when set, the
    // first pass reads element (b, pos) from in_em + (b n_in + pos) k (zero
    // for pos >= n_in) instead of `in`, and the last pass writes element
    // (b, pos < n_out) to out_em + (b n_out + pos) k instead of `out`.  The
    // pointers may be mapped pinned host memory (zero-copy over PCIe).
    const u64 *in_em;
    const u64 *in2_em;
    int64_t n_in, n_in2;
    u64 *out_em;
    int64_t n_out;
    // four-step twiddle on the first pass (PassIO::ft): table (limb pairs),
    // log2 of its plan's N and M, row offset, direction, plan root form
    const u64 *ft_lh;
    int ft_lN, ft_lM, ft_inv, ft_root_inv;
    int64_t ft_row0;
    // four-step exchange fused into the last pass (k_pass44, PassIO::xdst):
    // element (b, pos) of this rank's batch goes to rank g = pos >> lxb at
    //   xdst[g] + ((pos & (2^lxb - 1)) k + d) xg xA + xrank xA + b
    // (gfp_exchange_transpose's layout); xg = 0: off
    u64 *xdst[8];
    int xg, xrank, lxb;
    int64_t xA;
};

// Extras of one transform's first / last pass (k_pass44 only):
// element-major endpoints (see PassArgs), and the four-step inter-stage
// twiddle folded into the first pass: element (b, i) of the batch is
// multiplied by w^(+-(ft_row0 + b) i), w the root of the plan `ft` (the
// D_{N1,N2} stage of a sharded transform, fft.py:62-103).
struct PassIO {
    const u64 *in;
    const u64 *in2;
    int64_t n_in, n_in2;
    u64 *out;
    int64_t n_out;
    const gfp_fft_plan *ft;
    int64_t ft_row0;
    int ft_inv;
    // the last pass stores into the four-step exchange's receive buffers
    // (xg ranks, up to 8) instead of `out`
    u64 *const *xdst;
    int xg, xrank;
};

// ---------------------------------------------------------------------------
// plans

struct gfp_fft_plan {
    int k, K, e;
    int64_t N, M;
    u64 r;
    RadixConsts rc;
    u64 *table;       // element-major [M][k]: omega^b
    u64 *table_ninv;  // element-major [M][k]: omega^b * N^-1
    u64 *table_lh;    // both tables as balanced limb pairs (k_pass44 only, else null)
    u64 *table_ninv_lh;
    // host-path scratch
    u64 *h_dev;
    int64_t h_words;
    int64_t last_launches;
    int root_inv;  // omega^(N/2k) == 1/r (a plan built on an inverse root)
    // per-launch timing of the last call (gfp_fft_plan_set_timing)
    int generic;    // radix without the fast path's headroom: gfp_generic_pass.cu
    u64 *ninv_dev;  // N^-1 (canonical, device) for the generic path's final scale
    int timing, n_ev;
    cudaEvent_t ev[GFP_MAX_TIMED + 1];
    int ev_pass[GFP_MAX_TIMED];
};

// the generic-radix transform (gfp_generic_pass.cu): radix-2 passes on
// canonical digits, in -> out (in may equal out), N^-1 included when inverse;
// and the element-wise product out = in .* G of [batch][k][N] vectors
int run_generic(gfp_fft_plan *p, const u64 *in, u64 *out, u64 *work, int64_t batch, int inverse,
                cudaStream_t st);
int generic_pointwise(gfp_fft_plan *p, const u64 *in, const u64 *G, u64 *out, int64_t batch,
                      cudaStream_t st);

// one radix-K Stockham pass (gfp_pass.cuh), instantiated per k in gfp_pass_k*.cu
// true when the pass kernels of this plan take element-major I/O (PassIO)
bool em_io_supported(const gfp_fft_plan *p);

// em: element-major first-pass input / last-pass output (nullptr: none);
// returns GFP_EUNSUPPORTED when em is requested but the kernel for this k
// cannot do it (the caller then stages through digit-major buffers)
template <int KD>
int launch_pass(const gfp_fft_plan *p, const u64 *in, u64 *out, const u64 *in2, u64 *out2,
                const u64 *pre, int64_t batch, int64_t Ns, int inverse, int scale, int canon,
                int in_canon, const PassIO *em, cudaStream_t st);


// The middle of a k = 8 poly-multiply as one kernel (gfp_pmid44t.cuh): the
// forward last pass of both operands, the pointwise product and the inverse
// first pass.  f_in / g_in: the operands after the forward passes 0 .. e-2;
// out: the inverse's first-pass output (balanced lazy digits).
bool poly_mid_supported(const gfp_fft_plan *p);
int launch_poly_mid(const gfp_fft_plan *p, const u64 *f_in, const u64 *g_in, u64 *out,
                    int64_t batch, cudaStream_t st);

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
