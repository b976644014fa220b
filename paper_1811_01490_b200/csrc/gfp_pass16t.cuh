// gfp_pass16t.cuh -- the multiply-free first pass for k = 16 (K = 2k = 32) on
// TMA tiles: the butterfly pass of C3 (64 transforms of 2^20 points).
//
// The first pass of a transform (Ns = 1) has no level twiddle, no pointwise
// operand and no N^-1: group j reads x[j + t M] (t < 32) and writes the
// 32-point DFT at root rho = r (or 1/r) to 32 j + u (dft_base of the
// reference: dft2 butterflies and r^t shifts, fft.py:114-193).  k_pass<16>
// computes it with one digit per lane and warp shuffles for every rotation
// (1270 instructions per element, mio_throttle-bound, 0.54 of the HBM copy
// peak).  Here the DFT is three sweeps over digit-major shared-memory tiles in
// which every rotation is a row index known at compile time:
//
//   32 = 4 x 4 x 2:  t = t1 + 8 t2,  t1 = s1 + 2 s2,  u = u0 + 4 v0 + 16 v1
//     S1  Y[t1][u0] = sum_t2 w^(t2 u0) x[t1 + 8 t2]             w = rho^8
//     S2  Z[s1][v0] = sum_s2 w^(s2 v0) rho^(t1 u0) Y[t1][u0]
//     S3  X[u]      = Z[0][v0] + (-1)^v1 rho^(4 v0) Z[1][v0]
//
//   * a CTA owns 16 consecutive groups; tile t = [16 digits][16 groups] (2 KB)
//     is one TMA box, all 32 tiles requested at kernel start (64 KB in flight
//     per CTA, 3 CTAs per SM);
//   * S1 / S2: two lanes per group-element, lane half h holding the digits
//     {4h .. 4h+3} and {8+4h .. 11+4h}: the radix-4 butterfly's factor
//     w = r^8 pairs digit d with d + 8, both in the same thread, so the
//     butterfly is pure register arithmetic; the factor rho^(t1 u0) is the
//     row the digit is read from (u0 = the warp, t1 unrolled).  Results go
//     back to the same tiles in place;
//   * S3: lane = output index u, a thread holds all 16 digits of X[u] of one
//     group -- the radix-2 step (rho^(4 v0) moves blocks of four digits), the
//     balanced normalisation without any cross-thread carry, and row stores in
//     which the 32 lanes write 32 consecutive columns.  S2 stores tile T at
//     column g ^ swz(T) so these reads (16 tiles, one column) are conflict-free.
#pragma once
#include "gfp_pass44t.cuh"

#ifndef P16T
#define P16T 1  // 0: the first pass of k = 16 stays on k_pass<16, ., NOMUL> (A/B builds)
#endif

namespace p16t {

constexpr int KD = 16, K = 32, W = 16;
constexpr int TILE = KD * W;  // words
constexpr size_t SMEM = (size_t)K * TILE * 8 + K * 8;

// row of the thread's digit c (0..7) for half h
__host__ __device__ constexpr int drow(int h, int c) { return c < 4 ? 4 * h + c : 4 + 4 * h + c; }

// exponent of rho^e as a power of r (rho = r or 1/r)
template <bool INV>
__host__ __device__ constexpr int rexp(int e)
{
    return INV ? (32 - (e % 32)) % 32 : e % 32;
}

// 4-point DFT at w = rho^8 (w^2 = -1) of four half-elements held as digits
// {4h + c, 8 + 4h + c}: (w t)[d] = -t[d + 8] (d < 8), t[d - 8] (d >= 8) for
// rho = r; the opposite signs for rho = 1/r (r^-8 = -r^8).  In place:
// x_u = sum_t w^(t u) x_t.
template <bool INV>
GFP_D void bfly4(i64 (&x0)[8], i64 (&x1)[8], i64 (&x2)[8], i64 (&x3)[8])
{
    i64 s0[8], d0[8], s1[8], t[8], d1[8];
#pragma unroll
    for (int c = 0; c < 8; c++) {
        s0[c] = x0[c] + x2[c];
        d0[c] = x0[c] - x2[c];
        s1[c] = x1[c] + x3[c];
        t[c] = x1[c] - x3[c];
    }
#pragma unroll
    for (int c = 0; c < 4; c++) {
        d1[c] = INV ? t[c + 4] : -t[c + 4];
        d1[c + 4] = INV ? -t[c] : t[c];
    }
#pragma unroll
    for (int c = 0; c < 8; c++) {
        x0[c] = s0[c] + s1[c];
        x2[c] = s0[c] - s1[c];
        x1[c] = d0[c] + d1[c];
        x3[c] = d0[c] - d1[c];
    }
}

// the thread's eight digits of (tile element) * r^R, R in [0, 32): digit d
// comes from row (d - R) mod 16, negated when it wrapped xor R >= 16
template <int H, int R>
GFP_D void load_rot(const i64 *col, i64 (&a)[8])
{
    constexpr int s = R & 15;
    constexpr bool negall = R >= 16;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        const int d = drow(H, c);
        const int src = (d - s + 16) & 15;
        const bool neg = (d < s) != negall;
        const i64 v = col[src * W];
        a[c] = neg ? -v : v;
    }
}

// column swizzle of tile T in the S2 -> S3 hand-off: the sixteen tiles one
// S3 lane group reads (T = 8 u0 + 2 v0 + s1) get sixteen different columns
__host__ __device__ constexpr int swz(int T) { return ((T >> 3) << 2) | ((T >> 1) & 3); }

// S2: the butterfly (u0, s1) over s2 -- inputs rho^(t1 u0) Y[t1][u0],
// t1 = s1 + 2 s2, from tiles 8 u0 + t1; outputs Z[s1][v0] to tiles
// 8 u0 + s1 + 2 v0 (the same four tiles) at their swizzled column
template <bool INV, int U0, int S1>
GFP_D void bfly_s2(i64 *sm, int g, int h)
{
    i64 a[4][8];
    // the two halves read different rows: each takes its own (compile-time) path
    if (h == 0) {
        load_rot<0, rexp<INV>((S1 + 0) * U0)>(sm + (8 * U0 + S1 + 0) * TILE + g, a[0]);
        load_rot<0, rexp<INV>((S1 + 2) * U0)>(sm + (8 * U0 + S1 + 2) * TILE + g, a[1]);
        load_rot<0, rexp<INV>((S1 + 4) * U0)>(sm + (8 * U0 + S1 + 4) * TILE + g, a[2]);
        load_rot<0, rexp<INV>((S1 + 6) * U0)>(sm + (8 * U0 + S1 + 6) * TILE + g, a[3]);
    } else {
        load_rot<1, rexp<INV>((S1 + 0) * U0)>(sm + (8 * U0 + S1 + 0) * TILE + g, a[0]);
        load_rot<1, rexp<INV>((S1 + 2) * U0)>(sm + (8 * U0 + S1 + 2) * TILE + g, a[1]);
        load_rot<1, rexp<INV>((S1 + 4) * U0)>(sm + (8 * U0 + S1 + 4) * TILE + g, a[2]);
        load_rot<1, rexp<INV>((S1 + 6) * U0)>(sm + (8 * U0 + S1 + 6) * TILE + g, a[3]);
    }
    __syncwarp();  // both halves have read these four tiles
    bfly4<INV>(a[0], a[1], a[2], a[3]);
#pragma unroll
    for (int v0 = 0; v0 < 4; v0++) {
        const int T = 8 * U0 + S1 + 2 * v0;
        i64 *col = sm + T * TILE + (g ^ swz(T)) + 4 * h * W;
#pragma unroll
        for (int c = 0; c < 8; c++)
            col[(c < 4 ? c : 4 + c) * W] = a[v0][c];
    }
}

template <bool INV, int U0>
GFP_D void sweep2(i64 *sm, int g, int h)
{
    bfly_s2<INV, U0, 0>(sm, g, h);
    bfly_s2<INV, U0, 1>(sm, g, h);
}

}  // namespace p16t

template <int SPARSE, bool INV>
__global__ void __launch_bounds__(128, 3)
    k_first16t(const __grid_constant__ PassArgs A, const __grid_constant__ PassTma T)
{
    using namespace p16t;
    extern __shared__ __align__(128) i64 sm[];  // [K][TILE] tiles, then K mbarriers
    u64 *bar = reinterpret_cast<u64 *>(sm + K * TILE);
    const int lane = threadIdx.x & 31;
    const int w = __shfl_sync(FULL_MASK, threadIdx.x >> 5, 0);
    const bool leader = p44t::elect_one();
    const int g = lane & 15, h = lane >> 4;

    int bidx = blockIdx.y;
    const CUtensorMap *tin = &T.in;
    u64 *out = A.out;
    if (bidx >= A.batch) {
        bidx -= (int)A.batch;
        tin = &T.in2;
        out = A.out2;
    }
    out += (int64_t)bidx * A.batch_stride;
    const int lN = A.lN, lM = A.lM;
    const RadixConsts rc = A.rc;
    const int j0 = blockIdx.x * W;  // M % 16 == 0

    if (threadIdx.x == 0) {
#pragma unroll
        for (int t = 0; t < K; t++)
            p44t::mbar_init(&bar[t], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const u64 pol = p44t::evict_first_policy();
    if (leader) {  // tiles t = w + 4 i: the ones this warp's S1 butterflies read
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int t = w + 4 * i;
            p44t::mbar_expect_tx(&bar[t], TILE * 8);
            p44t::tma_load(sm + t * TILE, tin, &bar[t], j0 + (t << lM), bidx, pol);
        }
    }

    // ---- S1: butterflies t1 = w, w + 4 over t2 (tiles t1 + 8 t2), in place
    const i64 half = (i64)(rc.r >> 1);
#pragma unroll 1
    for (int b = 0; b < 2; b++) {
        const int t1 = w + 4 * b;
        i64 a[4][8];
#pragma unroll
        for (int t2 = 0; t2 < 4; t2++) {
            const int t = t1 + 8 * t2;
            p44t::mbar_wait(&bar[t], 0);
            const i64 *col = sm + GFP_IDX(t * TILE + g, K * TILE);
            const i64 *ph = col + 4 * h * W;
#pragma unroll
            for (int c = 0; c < 8; c++)
                a[t2][c] = ph[(c < 4 ? c : 4 + c) * W];
            if (A.in_canon) {
                // canonical digits [0, r] to balanced: d - r with a carry into
                // the next digit when d > r / 2 (negated into digit 0); the
                // carries into the thread's two runs come from the other
                // half's rows 4h - 1 (mod 16) and 4h + 7
                const i64 p0 = col[(h ? 3 : 15) * W], p1 = ph[7 * W];
                int cin0 = p0 > half, cin1 = p1 > half;
                cin0 = h ? cin0 : -cin0;
                int cy[8];
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    cy[c] = a[t2][c] > half;
                    a[t2][c] -= cy[c] ? (i64)rc.r : 0;
                }
#pragma unroll
                for (int c = 0; c < 8; c++)
                    a[t2][c] += c == 0 ? cin0 : c == 4 ? cin1 : cy[c - 1];
            }
        }
        __syncwarp();  // the other half has read its carry rows
        bfly4<INV>(a[0], a[1], a[2], a[3]);
#pragma unroll
        for (int u0 = 0; u0 < 4; u0++) {
            i64 *ph = sm + GFP_IDX((t1 + 8 * u0) * TILE + g, K * TILE) + 4 * h * W;
#pragma unroll
            for (int c = 0; c < 8; c++)
                ph[(c < 4 ? c : 4 + c) * W] = a[u0][c];
        }
    }
    GFP_JITTER(1);
    __syncthreads();

    // ---- S2: warp u0 = w, tiles 8 u0 .. 8 u0 + 7
    switch (w) {
    case 0: sweep2<INV, 0>(sm, g, h); break;
    case 1: sweep2<INV, 1>(sm, g, h); break;
    case 2: sweep2<INV, 2>(sm, g, h); break;
    default: sweep2<INV, 3>(sm, g, h); break;
    }
    GFP_JITTER(2);
    __syncthreads();

    // ---- S3: lane = u, groups g = w + 4 i: X[u] = Z[0][v0] +- rho^(4 v0) Z[1][v0],
    // normalise, store column 32 (j0 + g) + u of every digit row
    {
        const int u = lane, u0 = u & 3, v0 = (u >> 2) & 3, v1 = u >> 4;
        const int T0 = 8 * u0 + 2 * v0;
        const int R = INV ? (32 - 4 * v0) & 31 : 4 * v0;  // rho^(4 v0) as a power of r
        const int bs = (R >> 2) & 3;                      // block shift (four digits per block)
        const int na = R >= 16;
#pragma unroll 1
        for (int i = 0; i < 4; i++) {
            const int gg = w + 4 * i;
            const i64 *p0 = sm + GFP_IDX(T0 * TILE + (gg ^ (4 * u0 + v0)), K * TILE);
            const i64 *p1 = p0 + TILE;
            i64 X[KD];
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const int sb = (b - bs) & 3;
                const int neg = ((b < bs) ^ na) ^ v1;  // sign of the Z[1] term
                const i64 m = -(i64)neg;
                const i64 *q1 = p1 + 4 * sb * W;
#pragma unroll
                for (int i4 = 0; i4 < 4; i4++)
                    X[4 * b + i4] = p0[(4 * b + i4) * W] + ((q1[i4 * W] ^ m) + neg);
            }
            p44::normalize_el<KD, SPARSE>(X, rc);
            u64 *op = out + (((int64_t)(j0 + gg)) << 5) + u;
#pragma unroll
            for (int d = 0; d < KD; d++)
                __stcs(op + GFP_IDX((int64_t)d << lN, ((int64_t)KD << lN) - (((int64_t)(j0 + gg)) << 5) - u),
                       (u64)X[d]);
        }
    }
}

// the first pass of a k = 16 transform with nothing to multiply (the NOMUL
// case of launch_pass) on at least 16 groups, for the compile-time radix
static inline bool p16t_takes(const PassArgs &A, int64_t M)
{
    return P16T && A.rc.p3_ok && A.rc.stages_per_norm >= 5 && (M & 15) == 0 && A.lN <= 30 &&
           A.lNs == 0 && !A.pre && !A.scale && !A.canon;
}

// returns 1 when the pass was launched
static inline int launch_first16t(const PassArgs &A, int64_t M, int64_t nsets, cudaStream_t st)
{
    PassTma T;
    const int64_t N = (int64_t)1 << A.lN;
    if (!p44t_make_map(&T.in, A.in, N, 16, A.batch, A.batch_stride, 16))
        return 0;
    T.in2 = T.in;
    if (A.in2 && !p44t_make_map(&T.in2, A.in2, N, 16, A.batch, A.batch_stride, 16))
        return 0;
    T.out = T.in;  // unused: the stores are plain row stores
    T.out2 = T.in2;
    void (*kern)(const PassArgs, const PassTma) =
        A.rot_inv ? k_first16t<3, true> : k_first16t<3, false>;
    static unsigned long long set_on = 0;
    once_per_device(set_on, [&] {
        cudaFuncSetAttribute(k_first16t<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)p16t::SMEM);
        cudaFuncSetAttribute(k_first16t<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)p16t::SMEM);
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(M / p16t::W), (unsigned)nsets);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = p16t::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, A, T);
    __atomic_fetch_add(&g_tma_pass_launches, 1, __ATOMIC_RELAXED);
    return 1;
}
