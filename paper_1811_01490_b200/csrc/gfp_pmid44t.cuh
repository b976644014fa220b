// gfp_pmid44t.cuh -- the middle of a k = 8 polynomial multiply as ONE kernel:
// the forward transforms' last pass (both operands), the pointwise Z/pZ
// product and the inverse transform's first pass.
//
// Group j of the forward last pass (Ns = M) writes its outputs to j + u M,
// u < 16 -- exactly the elements group j of the inverse's first pass (Ns = 1)
// reads.  So the spectra F, G of SURVEY 3.4's composition (dft_general twice,
// fft.py:298-360; the pointwise gfp_mul, gfp_mult.py:416-512; dft_inverse,
// fft.py:363-370) never have to leave the SM: a CTA takes 32 consecutive
// groups of both operands as TMA tiles (2 x 16 tiles, 64 KB), runs the
// twiddle multiplies and the 16-point DFTs of the forward last pass on both,
// normalises, multiplies H_u = F_u G_u element by element, runs the
// inverse's first 16-point DFT on H and stores it in first-pass order.  One
// launch, one global round trip and one pass of tile latencies less than the
// two-kernel form; the arithmetic is the same function by function
// (k_pass44t's phase A / stage 1 / stage 2, the pointwise multiply of
// k_pass44's `pre` path), so the result is bit-identical.
//
// CTA = 16 warps x 32 lanes (lane = group): warp w twiddles element t = w of
// both operands (one table entry for both), stage 1 runs on warps 0-3 (f)
// and 4-7 (g), stage 2 and the normalisation on all 16 (operand x u0 x output
// half), the pointwise product on all 16 (u = w), the inverse's stage 1 on
// warps 0-3 and its stage 2 on all 16 (u0 x output).
#pragma once
#include "gfp_pass44t.cuh"

#ifndef PMID_FUSE
#define PMID_FUSE 1  // 0: poly-multiply keeps the two-kernel middle (A/B builds)
#endif

template <int KD, int SPARSE, bool FINV>
__global__ void __launch_bounds__(512, 1)
    k_pmid44t(const __grid_constant__ PassArgs A, const __grid_constant__ PassTma T)
{
    static_assert(KD == 8, "radix 4 x 4 pass is for K = 16");
    constexpr int K = 2 * KD;
    constexpr int TILE = KD * 32;
    constexpr bool IINV = !FINV;  // the inverse transform's base-case root
    extern __shared__ __align__(128) i64 sm[];  // tiles 0..15: f (then H), 16..31: g; 32 mbarriers
    u64 *bar = reinterpret_cast<u64 *>(sm + 2 * K * TILE);
    const int lane = threadIdx.x & 31;
    const int w = __shfl_sync(FULL_MASK, threadIdx.x >> 5, 0);
    const bool leader = p44t::elect_one();
    const int bidx = blockIdx.y;
    const int lN = A.lN, lM = A.lM;
    const int64_t M = (int64_t)1 << lM;
    const RadixConsts rc = A.rc;
    const int j0 = blockIdx.x * 32;
    const int64_t j = j0 + lane;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int t = 0; t < 2 * K; t++)
            p44t::mbar_init(&bar[t], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const u64 pol = p44t::evict_first_policy();
    if (leader) {
        p44t::mbar_expect_tx(&bar[w], TILE * 8);
        p44t::tma_load(sm + w * TILE, &T.in, &bar[w], j0 + (w << lM), bidx, pol);
        p44t::mbar_expect_tx(&bar[K + w], TILE * 8);
        p44t::tma_load(sm + (K + w) * TILE, &T.in2, &bar[K + w], j0 + (w << lM), bidx, pol);
    }

    // ---- forward last pass, phase A: element t = w of f and of g times
    // omega^E, E = t j (Ns = M): one table entry serves both operands
    {
        const int t = w;
        const unsigned E = (unsigned)t * (unsigned)j;  // < 16 M = N
        p44::Twiddle tw;
        {
            int a = (int)(E >> lM);
            tw.b = E & ((1u << lM) - 1u);
            if (A.root_inv && a)
                a = 2 * KD - a;
            tw.as = a & (KD - 1);
            tw.negx = ((1u << tw.as) - 1u) ^ (a >= KD ? ((1u << KD) - 1u) : 0u);
        }
        const bool mul_tw = __any_sync(FULL_MASK, tw.b != 0);
        u64 ylh[KD];
        if (mul_tw) {
            const ulonglong2 *tp =
                reinterpret_cast<const ulonglong2 *>(A.table_lh + GFP_IDX(tw.b, M) * KD);
#pragma unroll
            for (int d = 0; d < KD; d += 2) {
                const ulonglong2 v = __ldg(tp + d / 2);
                ylh[d] = v.x;
                ylh[d + 1] = v.y;
            }
        }
#pragma unroll 1
        for (int op = 0; op < 2; op++) {
            i64 *tile = sm + GFP_IDX((op * K + t) * TILE + lane, 2 * K * TILE);
            p44t::mbar_wait(&bar[op * K + t], 0);
            i64 x[KD], f[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                x[d] = tile[((d - tw.as) & (KD - 1)) * 32];
            if (mul_tw) {
                fast_mul_lazy_ylimbs<KD, SPARSE, true, 32>(x, ylh, f, rc, tw.negx, tile);
            } else {
#pragma unroll
                for (int d = 0; d < KD; d++)
                    tile[d * 32] = ((tw.negx >> d) & 1u) ? -x[d] : x[d];
            }
        }
    }
    GFP_JITTER(1);
    __syncthreads();

    // ---- forward stage 1: warps 0-3 on f, 4-7 on g (t1 = w mod 4)
    i64 e[4][KD];
    if (w < 8) {
        const int base = (w >> 2) * K, t1 = w & 3;
#pragma unroll
        for (int t2 = 0; t2 < 4; t2++) {
            const i64 *tile = sm + GFP_IDX((base + t1 + 4 * t2) * TILE + lane, 2 * K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[t2][d] = tile[d * 32];
        }
        p44::dft4<KD, FINV, 0>(e[0], e[1], e[2], e[3]);
#pragma unroll
        for (int u0 = 0; u0 < 4; u0++) {
            i64 *tile = sm + GFP_IDX((base + 4 * u0 + t1) * TILE + lane, 2 * K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                tile[d * 32] = e[u0][d];
        }
    }
    GFP_JITTER(2);
    __syncthreads();

    // ---- forward stage 2: warp = (u0, operand, output half); the two
    // outputs u = u0 + 4 u1, u1 = 2 hf + q, normalised, go to tile u of the
    // operand (natural order: the pointwise product pairs F_u with G_u)
    {
        const int u0 = w & 3, base = ((w >> 2) & 1) * K, hf = w >> 3;
#pragma unroll
        for (int t1 = 0; t1 < 4; t1++) {
            const i64 *tile = sm + GFP_IDX((base + 4 * u0 + t1) * TILE + lane, 2 * K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[t1][d] = tile[d * 32];
        }
        switch (u0) {
        case 0: p44::dft4<KD, FINV, 0>(e[0], e[1], e[2], e[3]); break;
        case 1: p44::dft4<KD, FINV, 1>(e[0], e[1], e[2], e[3]); break;
        case 2: p44::dft4<KD, FINV, 2>(e[0], e[1], e[2], e[3]); break;
        default: p44::dft4<KD, FINV, 3>(e[0], e[1], e[2], e[3]); break;
        }
#pragma unroll
        for (int q = 0; q < 2; q++) {
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[q][d] = hf ? e[2 + q][d] : e[q][d];
            p44::normalize_el<KD, SPARSE>(e[q], rc);
        }
        GFP_JITTER(3);
        __syncthreads();  // every warp has read its stage-1 tiles
#pragma unroll
        for (int q = 0; q < 2; q++) {
            i64 *tile = sm + GFP_IDX((base + u0 + 4 * (2 * hf + q)) * TILE + lane, 2 * K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                tile[d * 32] = e[q][d];
        }
    }
    GFP_JITTER(4);
    __syncthreads();

    // ---- pointwise product H_u = F_u G_u, u = w, into f's tile u
    {
        constexpr int S = FastSplit<KD>::S;
        i64 *ft = sm + GFP_IDX(w * TILE + lane, 2 * K * TILE);
        const i64 *gt = sm + GFP_IDX((K + w) * TILE + lane, 2 * K * TILE);
        i64 x[KD], f[KD];
        u64 ylh[KD];
#pragma unroll
        for (int d = 0; d < KD; d++) {
            x[d] = ft[d * 32];
            int l, h;
            split_limbs<S>(gt[d * 32], l, h);
            ylh[d] = (u64)(unsigned)l | ((u64)(unsigned)h << 32);
        }
        fast_mul_lazy_ylimbs<KD, SPARSE, true, 32>(x, ylh, f, rc, 0u, ft);
    }
    GFP_JITTER(5);
    __syncthreads();

    // ---- inverse first pass (no twiddle at Ns = 1), stage 1 on warps 0-3
    if (w < 4) {
#pragma unroll
        for (int t2 = 0; t2 < 4; t2++) {
            const i64 *tile = sm + GFP_IDX((w + 4 * t2) * TILE + lane, 2 * K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[t2][d] = tile[d * 32];
        }
        p44::dft4<KD, IINV, 0>(e[0], e[1], e[2], e[3]);
#pragma unroll
        for (int u0 = 0; u0 < 4; u0++) {
            i64 *tile = sm + GFP_IDX((4 * u0 + w) * TILE + lane, 2 * K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                tile[d * 32] = e[u0][d];
        }
    }
    GFP_JITTER(6);
    __syncthreads();

    // ---- inverse stage 2: warp = (u0, u1); output u = u0 + 4 u1 of group j
    // goes to column 16 j + u: park as [d][g][u ^ (g mod 16)] over the g tiles
    // (free since the product) and write every digit row's 512 columns
    {
        const int u0 = w & 3, u1 = w >> 2;
#pragma unroll
        for (int t1 = 0; t1 < 4; t1++) {
            const i64 *tile = sm + GFP_IDX((4 * u0 + t1) * TILE + lane, 2 * K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[t1][d] = tile[d * 32];
        }
        switch (u0) {
        case 0: p44::dft4<KD, IINV, 0>(e[0], e[1], e[2], e[3]); break;
        case 1: p44::dft4<KD, IINV, 1>(e[0], e[1], e[2], e[3]); break;
        case 2: p44::dft4<KD, IINV, 2>(e[0], e[1], e[2], e[3]); break;
        default: p44::dft4<KD, IINV, 3>(e[0], e[1], e[2], e[3]); break;
        }
#pragma unroll
        for (int d = 0; d < KD; d++) {
            i64 v = e[0][d];
            v = u1 == 1 ? e[1][d] : v;
            v = u1 == 2 ? e[2][d] : v;
            v = u1 == 3 ? e[3][d] : v;
            e[0][d] = v;
        }
        p44::normalize_el<KD, SPARSE>(e[0], rc);
        i64 *park = sm + K * TILE;  // the g tiles: not read any more
        const int u = u0 + 4 * u1;
#pragma unroll
        for (int d = 0; d < KD; d++)
            park[GFP_IDX(d * 512 + lane * 16 + (u ^ (lane & 15)), K * TILE)] = e[0][d];
        GFP_JITTER(7);
        __syncthreads();
        u64 *out = A.out + (int64_t)bidx * A.batch_stride + ((int64_t)j0 << 4);
        const int c = threadIdx.x;  // column 16 j0 + c
        const int g = c >> 4, uu = c & 15;
#pragma unroll
        for (int d = 0; d < KD; d++)
            __stcs(out + GFP_IDX(((int64_t)d << lN) + c, ((int64_t)KD << lN) - ((int64_t)j0 << 4)),
                   (u64)park[GFP_IDX(d * 512 + g * 16 + (uu ^ (g & 15)), K * TILE)]);
    }
}

// the fused middle serves k = 8 plans of at least two passes whose groups fill
// whole CTAs, on the fast (lazy-digit) path
static inline bool pmid_takes(const gfp_fft_plan *p)
{
    return PMID_FUSE && p->k == 8 && p->e >= 2 && (p->M & 31) == 0 && p->N <= ((int64_t)1 << 30) &&
           !p->generic && pass44_enabled(p->k, p->rc) && p->table_lh && p44t_encoder() != nullptr;
}

// f_in, g_in: the operands after the forward passes 0 .. e-2 ([batch][k][N],
// balanced lazy); out: the inverse transform's first-pass output.  Returns 1
// when launched.
static inline int launch_pmid44t(const gfp_fft_plan *p, const u64 *f_in, const u64 *g_in, u64 *out,
                                 int64_t batch, cudaStream_t st)
{
    constexpr int KD = 8;
    PassArgs A;
    memset(&A, 0, sizeof(A));
    A.in = f_in;
    A.in2 = g_in;
    A.out = out;
    A.table_lh = p->table_lh;
    A.batch_stride = (int64_t)p->k * p->N;
    A.batch = batch;
    A.lN = ilog2_exact(p->N);
    A.lM = ilog2_exact(p->M);
    A.lNs = A.lM;
    A.root_inv = p->root_inv;
    A.rot_inv = p->root_inv;  // the forward's base-case root; the inverse uses the other
    A.rc = p->rc;
    PassTma T;
    if (!p44t_make_map(&T.in, f_in, p->N, KD, batch, A.batch_stride) ||
        !p44t_make_map(&T.in2, g_in, p->N, KD, batch, A.batch_stride))
        return 0;
    T.out = T.in;
    T.out2 = T.in2;
    void (*kern)(const PassArgs, const PassTma) = nullptr;
    const bool finv = A.rot_inv != 0;
    if (A.rc.p3_ok)
        kern = finv ? k_pmid44t<KD, 3, true> : k_pmid44t<KD, 3, false>;
    else if (A.rc.p2_ok)
        kern = finv ? k_pmid44t<KD, 2, true> : k_pmid44t<KD, 2, false>;
    else
        kern = finv ? k_pmid44t<KD, 0, true> : k_pmid44t<KD, 0, false>;
    constexpr size_t smem = (size_t)4 * KD * (KD * 32) * 8 + 4 * KD * 8;
    static unsigned long long set_on = 0;
    once_per_device(set_on, [&] {
        cudaFuncSetAttribute(k_pmid44t<KD, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_pmid44t<KD, 3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_pmid44t<KD, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_pmid44t<KD, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_pmid44t<KD, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_pmid44t<KD, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p->M / 32), (unsigned)batch);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
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
