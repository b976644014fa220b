// gfp_pass44t.cuh -- the k = 8 radix-16 Stockham pass for large transforms
// with TMA tile movement (sm_100a: cp.async.bulk.tensor + mbarrier).
//
// Same pass and the same arithmetic as k_pass44 (gfp_pass44.cuh; the
// reference's dft_general level, fft.py:298-360, with the level twiddle split
// r^a omega^b of fft.py:84-103), for the passes that carry the bulk of a large
// transform: digit-major input and output, every group of the CTA present
// (M % 32 == 0); NW warps per CTA as in
// k_pass44 (4 for grids that fill the GPU, 8 / 16 for small transforms).  What changes is how the
// digit rows move:
//
//   * the vectors are 3-D tensors [batch][k][N] of u64; one TMA box
//     {32 columns, k rows, 1} is the 2 KB tile "element t of 32 consecutive
//     groups, all digits".  Lane 0 of warp w issues the four tile loads of the
//     warp's elements t = w + 4 i at kernel start -- 8 KB in flight per warp
//     with no registers or address arithmetic spent on them (the LDG form
//     spends ~65 of the pass's ~1020 instructions per element on it and has
//     one element's rows in flight) -- each completing on its own mbarrier;
//   * shared memory holds the 16 tiles digit-major ([t][d][lane], 32 KB, no
//     padding: a thread only ever touches its own column, and a warp's
//     64-bit accesses to one digit row are conflict-free).  The rotation r^a
//     is the row index of the tile read, the product digits go back to the
//     same tile, stage 1 / stage 2 exchange through the tiles in place;
//   * the outputs X[u0 + 4 u1] of warp u0 are written back into the warp's
//     own four tiles and leave as four TMA box stores (Ns >= 32: the 32
//     groups' outputs are 32 consecutive columns; Ns = 16: two boxes of 16).
#pragma once
#include <cuda.h>

#include "gfp_pass44.cuh"

#ifndef P44_TMA
#define P44_TMA 1  // 0: large transforms stay on k_pass44<NW = 4> (A/B builds)
#endif
#ifndef P44T_MINB
#define P44T_MINB 6  // CTAs per SM the NW = 4 kernel is register-bounded for (32 KB tiles
                     // each): 80 registers with 192 B of spills beats 5 CTAs at 96 since the
                     // rounding column quotient (C4 passes 0.698 -> 0.678 ms); 4 CTAs at 126
                     // registers: 0.70 ms
#endif
#ifndef P44T_EARLY_TABLE_MINEPT
#define P44T_EARLY_TABLE_MINEPT 4  // elements per thread from which the table entry is loaded
                                   // before the tile wait
#endif
#ifndef P44T_TRACE
#define P44T_TRACE 0  // timeline of one CTA by printf (tools/trace_c2.py only)
#endif
#if P44T_TRACE
#define P44T_T(i) do { if (trace_on) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[i])); } while (0)
#else
#define P44T_T(i) ((void)0)
#endif

// tensor maps of one pass launch: the two vector sets' inputs and outputs
struct PassTma {
    CUtensorMap in, in2;    // box {32, k, 1}
    CUtensorMap out, out2;  // box {32, k, 1}; {16, k, 1} for the Ns = 16 pass
};

namespace p44t {

GFP_D unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

GFP_D void mbar_init(u64 *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
GFP_D void mbar_expect_tx(u64 *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// wait for the barrier's phase `parity` to complete (try_wait suspends the
// thread for a bounded time per attempt)
GFP_D void mbar_wait(u64 *bar, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "P44T_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra P44T_DONE;\n"
        "bra P44T_WAIT;\n"
        "P44T_DONE:\n"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
GFP_D bool elect_one()
{
    unsigned pred;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}"
        : "=r"(pred));
    return pred != 0;
}
GFP_D u64 evict_first_policy()
{
    u64 pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// box {c0 .. c0 + 31, all rows, batch c2} -> dst, completion on bar
GFP_D void tma_load(void *dst, const CUtensorMap *map, u64 *bar, int c0, int c2, u64 pol)
{
    // streamed tiles carry an L2 evict-first policy: the twiddle tables stay
    // (without it: C4 4.35 -> 4.51 ms)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(0), "r"(c2), "l"(pol)
        : "memory");
}
GFP_D void tma_store(const CUtensorMap *map, const void *src, int c0, int c2, u64 pol)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint"
                 " [%0, {%2, %3, %4}], [%1], %5;" ::"l"(map),
                 "r"(smem_u32(src)), "r"(c0), "r"(0), "r"(c2), "l"(pol)
                 : "memory");
}

}  // namespace p44t

template <int KD, int SPARSE, bool INV, int NW>
__global__ void __launch_bounds__(NW * 32, NW == 4 ? P44T_MINB : NW == 8 ? 2 : 1)
    k_pass44t(const __grid_constant__ PassArgs A, const __grid_constant__ PassTma T)
{
    static_assert(KD == 8, "radix 4 x 4 pass is for K = 16");
    constexpr int K = 2 * KD;
    constexpr int TILE = KD * 32;  // words of one tile: [d][lane]
    constexpr int EPT = K / NW;    // phase-A elements per thread
    __shared__ __align__(128) i64 sm[K * TILE];
    __shared__ __align__(8) u64 bar[K];
    const int lane = threadIdx.x & 31;
    // elements t = w + NW i; broadcast so the compiler keeps w (and the TMA
    // operands derived from it) in uniform registers
    const int w = __shfl_sync(FULL_MASK, threadIdx.x >> 5, 0);
    const bool leader = p44t::elect_one();  // one lane issues the warp's TMA operations

    int bidx = blockIdx.y;
    const CUtensorMap *tin = &T.in, *tout = &T.out;
    if (bidx >= A.batch) {
        bidx -= (int)A.batch;
        tin = &T.in2;
        tout = &T.out2;
    }
    const int lN = A.lN, lM = A.lM, lNs = A.lNs;
    const int64_t N = (int64_t)1 << lN, M = (int64_t)1 << lM;
    const int64_t nsmask = ((int64_t)1 << lNs) - 1;
    const RadixConsts rc = A.rc;
    const int j0 = blockIdx.x * 32;  // M % 32 == 0: every lane has a group
    const int64_t j = j0 + lane;

#if P44T_TRACE
    unsigned long long tr[10] = {0};
    const bool trace_on = blockIdx.x == 1 && blockIdx.y == 0 && threadIdx.x == 0;
#endif
    P44T_T(0);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int t = 0; t < K; t++)
            p44t::mbar_init(&bar[t], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // programmatic dependent launch (see k_pass44): the previous pass's
    // writes are visible after the wait, before the first tile load
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    P44T_T(1);
    const u64 pol = p44t::evict_first_policy();
    if (leader) {
#pragma unroll
        for (int i = 0; i < EPT; i++) {
            const int t = w + NW * i;
            p44t::mbar_expect_tx(&bar[t], TILE * 8);
            p44t::tma_load(sm + t * TILE, tin, &bar[t], j0 + (t << lM), bidx, pol);
        }
    }

    // ---- phase A: element t = w + NW i of the lane's group times omega^E =
    // r^a omega^b; r^a is the row the digit is read from (and a sign folded
    // into the multiply's limb split), omega^b one general multiply whose
    // digits go back to the tile as they become final
#pragma unroll 1
    for (int i = 0; i < EPT; i++) {
        const int t = w + NW * i;
        i64 *tile = sm + GFP_IDX(t * TILE + lane, K * TILE);
        // omega^E = r^a omega^b, E = t (j mod Ns)(M / Ns) < N <= 2^30: 32-bit
        // arithmetic; the first pass of a four-step row transform carries the
        // enclosing transform's twiddle w^(+-(row0 + b) pos) instead (its own
        // is trivial)
        unsigned E = ((unsigned)t * ((unsigned)j & (unsigned)nsmask)) << (lM - lNs);
        if (A.neg_exp && E)
            E = (unsigned)N - E;
        int tlM = lM, troot_inv = A.root_inv;
        const u64 *tab = A.table_lh;
        if (A.ft_lh) {
            const int64_t Nf = (int64_t)1 << A.ft_lN;
            int64_t Ef = ((A.ft_row0 + bidx) * (j + ((int64_t)t << lM))) & (Nf - 1);
            if (A.ft_inv && Ef)
                Ef = Nf - Ef;
            E = (unsigned)Ef;
            tlM = A.ft_lM;
            troot_inv = A.ft_root_inv;
            tab = A.ft_lh;
        }
        p44::Twiddle tw;
        {
            int a = (int)(E >> tlM);
            tw.b = E & ((1u << tlM) - 1u);
            if (troot_inv && a)
                a = 2 * KD - a;
            tw.as = a & (KD - 1);
            tw.negx = ((1u << tw.as) - 1u) ^ (a >= KD ? ((1u << KD) - 1u) : 0u);
        }
        // warp-uniform multiply: lanes with b = 0 multiply by table[0] = 1
        const bool mul_tw = __any_sync(FULL_MASK, tw.b || A.scale);
        // With four elements per thread (large transforms) the table entry is
        // requested before the wait for the tile, so the two latencies overlap
        // (C4 passes 0.718 -> 0.708 ms); with one or two (C1 / C2) the sixteen
        // registers held across the wait cost more than the overlap gains
        // (C2 graph 0.0717 -> 0.0737 ms), so those load it after the wait.
        constexpr bool EARLY = EPT >= P44T_EARLY_TABLE_MINEPT;
        u64 ylh[KD];
        const ulonglong2 *tp =
            reinterpret_cast<const ulonglong2 *>(tab + GFP_IDX(tw.b, (int64_t)1 << tlM) * KD);
        if (EARLY && mul_tw) {
#pragma unroll
            for (int d = 0; d < KD; d += 2) {
                const ulonglong2 v = __ldg(tp + d / 2);
                ylh[d] = v.x;
                ylh[d + 1] = v.y;
            }
        }
        p44t::mbar_wait(&bar[t], 0);
        if (i == 0)
            P44T_T(2);
        i64 x[KD], f[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            x[d] = tile[((d - tw.as) & (KD - 1)) * 32];
        if (A.in_canon)  // first pass only, where a = 0
            to_balanced<KD>(x, rc.r);
        if (mul_tw) {
            if (!EARLY) {
#pragma unroll
                for (int d = 0; d < KD; d += 2) {
                    const ulonglong2 v = __ldg(tp + d / 2);
                    ylh[d] = v.x;
                    ylh[d + 1] = v.y;
                }
            }
            fast_mul_lazy_ylimbs<KD, SPARSE, true, 32>(x, ylh, f, rc, tw.negx, tile);
        } else {  // r^a alone (t = 0: the identity)
#pragma unroll
            for (int d = 0; d < KD; d++)
                tile[d * 32] = ((tw.negx >> d) & 1u) ? -x[d] : x[d];
        }
    }

    P44T_T(3);
    GFP_JITTER(1);
    // ---- stage 1 (warps w < 4, t1 = w): 4-point DFT over t2 of tiles
    // t1 + 4 t2, outputs u0 back into tiles t1 + 4 u0 -- the same four tiles.
    // With NW = 4 they are this thread's own phase-A columns: no barrier.
    i64 e[4][KD];
    if (NW > 4)
        __syncthreads();
    P44T_T(4);
    if (w < 4) {
#pragma unroll
        for (int t2 = 0; t2 < 4; t2++) {
            const i64 *tile = sm + GFP_IDX((w + 4 * t2) * TILE + lane, K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[t2][d] = tile[d * 32];
        }
        p44::dft4<KD, INV, 0>(e[0], e[1], e[2], e[3]);
#pragma unroll
        for (int u0 = 0; u0 < 4; u0++) {
            i64 *tile = sm + GFP_IDX((4 * u0 + w) * TILE + lane, K * TILE);
#pragma unroll
            for (int d = 0; d < KD; d++)
                tile[d * 32] = e[u0][d];
        }
    }
    P44T_T(5);
    GFP_JITTER(2);
    __syncthreads();
    P44T_T(6);

    // ---- stage 2 over SPL = NW / 4 warps per u0: every warp gathers
    // Y[t1][u0] from tiles 4 u0 + t1, applies rho^(t1 u0) as a compile-time
    // rotation and runs the (cheap, lazy) DFT over t1, then normalises and
    // stores only its NU = 4 / SPL outputs u1 in [h NU, h NU + NU)
    constexpr int SPL = NW / 4, NU = 4 / SPL;
    const int u0 = w & 3;
    const int h = w >> 2;
#pragma unroll
    for (int t1 = 0; t1 < 4; t1++) {
        const i64 *tile = sm + GFP_IDX((4 * u0 + t1) * TILE + lane, K * TILE);
#pragma unroll
        for (int d = 0; d < KD; d++)
            e[t1][d] = tile[d * 32];
    }
    switch (u0) {
    case 0: p44::dft4<KD, INV, 0>(e[0], e[1], e[2], e[3]); break;
    case 1: p44::dft4<KD, INV, 1>(e[0], e[1], e[2], e[3]); break;
    case 2: p44::dft4<KD, INV, 2>(e[0], e[1], e[2], e[3]); break;
    default: p44::dft4<KD, INV, 3>(e[0], e[1], e[2], e[3]); break;
    }
    if (SPL > 1) {
        if (h > 0) {  // this warp's outputs into e[0 .. NU-1] (static indices)
#pragma unroll
            for (int q = 0; q < NU; q++) {
#pragma unroll
                for (int d = 0; d < KD; d++) {
                    i64 v = e[q][d];
#pragma unroll
                    for (int hh = 1; hh < SPL; hh++)
                        v = h == hh ? e[hh * NU + q][d] : v;
                    e[q][d] = v;
                }
            }
        }
        // tiles 4 u0 + t1 are read by all SPL warps of this u0 and rewritten
        // below
        GFP_JITTER(3);
        __syncthreads();
    }
    if (lNs == 0) {
        // First pass (Ns = 1): output u of group j goes to column 16 j + u, so
        // the CTA's outputs are 512 consecutive columns of every digit row.
        // Park them over the tiles as [d][g][u ^ (g mod 16)] (the XOR keeps
        // both the lane-per-group writes and the lane-per-column reads
        // conflict-free without padding) and write each row lane-contiguously.
        constexpr int NT = NW * 32;
        u64 *out = (blockIdx.y >= A.batch ? A.out2 : A.out) + (int64_t)bidx * A.batch_stride;
        if (SPL == 1)
            __syncthreads();  // every warp's stage-2 reads done: the park spans all tiles
#pragma unroll
        for (int q = 0; q < NU; q++) {
            p44::normalize_el<KD, SPARSE>(e[q], rc);
            if (A.canon) {
                u64 c[KD];
                lazy_to_canonical_bf<KD>(e[q], c, rc);
#pragma unroll
                for (int d = 0; d < KD; d++)
                    e[q][d] = (i64)c[d];
            }
            const int u = u0 + 4 * (h * NU + q);
#pragma unroll
            for (int d = 0; d < KD; d++)
                sm[GFP_IDX(d * 512 + lane * 16 + (u ^ (lane & 15)), K * TILE)] = e[q][d];
        }
        GFP_JITTER(4);
        __syncthreads();
        u64 *obase = out + ((int64_t)j0 << 4);
#pragma unroll
        for (int q4 = 0; q4 < 512 / NT; q4++) {
            const int c = threadIdx.x + NT * q4;  // column 16 j0 + c
            const int g = c >> 4, u = c & 15;
#pragma unroll
            for (int d = 0; d < KD; d++)
                __stcs(obase + GFP_IDX(((int64_t)d << lN) + c, ((int64_t)KD << lN) - ((int64_t)j0 << 4)),
                       (u64)sm[GFP_IDX(d * 512 + g * 16 + (u ^ (g & 15)), K * TILE)]);
        }
        return;
    }
    // One balanced normalisation per output, the canonical form on the last
    // pass; X[u0 + 4 u1] = e[q] goes back to tile 4 u0 + u1 as the source of
    // its box store.  Output u of group j lives at
    // (j / Ns) Ns K + (j mod Ns) + u Ns: for Ns >= 32 the warp's 32 groups
    // are 32 consecutive columns (one {32, k} box, the tile as it is); for
    // Ns = 16 they are two runs of 16 columns 256 apart (two {16, k} boxes:
    // the tile holds them as [half][d][16]).
    __syncwarp();  // Ns = 16 writes other lanes' (already read) columns
    const bool wide = lNs >= 5;
    const int ob = wide ? lane : (lane >> 4) * (KD * 16) + (lane & 15);
    const int os = wide ? 32 : 16;
#pragma unroll
    for (int q = 0; q < NU; q++) {
        p44::normalize_el<KD, SPARSE>(e[q], rc);
        i64 *tile = sm + GFP_IDX((4 * u0 + h * NU + q) * TILE + ob, K * TILE);
        if (A.canon) {
            u64 c[KD];
            lazy_to_canonical_bf<KD>(e[q], c, rc);
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[q][d] = (i64)c[d];
        }
#pragma unroll
        for (int d = 0; d < KD; d++)
            tile[GFP_IDX(d * os, TILE - ob)] = e[q][d];
    }
    P44T_T(7);
    // generic-proxy writes -> async proxy (TMA) reads
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (leader) {
        const int64_t base = (((int64_t)j0 >> lNs) << (lNs + 4)) + (j0 & nsmask);
#pragma unroll
        for (int q = 0; q < NU; q++) {
            const int u1 = h * NU + q;
            const i64 *tile = sm + (4 * u0 + u1) * TILE;
            const int c0 = (int)(base + ((int64_t)(u0 + 4 * u1) << lNs));
            if (wide) {
                p44t::tma_store(tout, tile, c0, bidx, pol);
            } else {  // groups j0 + 16 .. j0 + 31 are the next block of Ns K columns
                p44t::tma_store(tout, tile, c0, bidx, pol);
                p44t::tma_store(tout, tile + KD * 16, c0 + (1 << (lNs + 4)), bidx, pol);
            }
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // the tiles must stay until the stores have read them
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
#if P44T_TRACE
    P44T_T(8);
    if (trace_on)
        printf("P44T_TRACE NW=%d lNs=%d start=%llu init+pdlwait=%llu tilewait=%llu phaseA=%llu bar1=%llu stage1=%llu bar2=%llu stage2=%llu store=%llu\n",
               NW, lNs, tr[0], tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3], tr[5] - tr[4],
               tr[6] - tr[5], tr[7] - tr[6], tr[8] - tr[7]);
#endif
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link
// dependency on libcuda); nullptr when the driver does not offer it
typedef CUresult (*p44t_encode_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static inline p44t_encode_fn p44t_encoder()
{
    static p44t_encode_fn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return (p44t_encode_fn)p;
    }();
    return fn;
}

// tensor map of a digit-major vector set: [batch][k][N] u64, box {cols, k, 1}
static inline bool p44t_encode_map(CUtensorMap *m, const u64 *base, int64_t N, int k, int64_t batch,
                                 int64_t batch_stride, int cols = 32)
{
    p44t_encode_fn enc = p44t_encoder();
    if (!enc || ((uintptr_t)base & 15))
        return false;
    const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)k, (cuuint64_t)batch};
    const cuuint64_t strides[2] = {(cuuint64_t)N * 8, (cuuint64_t)batch_stride * 8};
    const cuuint32_t box[3] = {(cuuint32_t)cols, (cuuint32_t)k, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, (void *)base, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

// The same through a small per-thread cache: a descriptor depends only on the
// base address and the shape, and a transform's passes alternate between a
// few buffers, so repeated calls (C1 / C2 are launch-bound when launched
// from a stream) encode nothing.
static inline bool p44t_make_map(CUtensorMap *m, const u64 *base, int64_t N, int k, int64_t batch,
                                 int64_t batch_stride, int cols = 32)
{
    struct Entry {
        const u64 *base;
        int64_t N, batch, stride;
        int k, cols, valid;
        CUtensorMap map;
    };
    constexpr int NE = 32;
    static thread_local Entry cache[NE];
    static thread_local int next = 0;
    for (int i = 0; i < NE; i++) {
        const Entry &c = cache[i];
        if (c.valid && c.base == base && c.N == N && c.batch == batch && c.stride == batch_stride &&
            c.k == k && c.cols == cols) {
            *m = c.map;
            return true;
        }
    }
    if (!p44t_encode_map(m, base, N, k, batch, batch_stride, cols))
        return false;
    Entry &c = cache[next];
    next = (next + 1) % NE;
    c.base = base;
    c.N = N;
    c.batch = batch;
    c.stride = batch_stride;
    c.k = k;
    c.cols = cols;
    c.map = *m;
    c.valid = 1;
    return true;
}

// the passes k_pass44t takes: the digit-major k = 8 passes of transforms
// with at least 32 groups (not the pointwise-product, host-memory or
// fused-exchange forms of the first / last pass)
static inline bool p44t_takes(const PassArgs &A, int64_t M)
{
    return P44_TMA && (M & 31) == 0 && (A.lNs >= 4 || A.lNs == 0) &&
           A.lN <= 30 && A.ft_lN <= 30 && !A.in_em && !A.out_em && !A.xg && !A.pre;
}

template <int KD, int SP, bool IV>
static inline void (*p44t_kernel(int nw))(const PassArgs, const PassTma)
{
    return nw == 4 ? k_pass44t<KD, SP, IV, 4> : nw == 8 ? k_pass44t<KD, SP, IV, 8>
                                                        : k_pass44t<KD, SP, IV, 16>;
}

// returns 1 when the pass was launched
template <int KD>
static int launch_pass44t(const PassArgs &A, int64_t M, int64_t nsets, cudaStream_t st)
{
    if constexpr (KD != 8) {
        return 0;
    } else {
        PassTma T;
        const int64_t N = (int64_t)1 << A.lN;
        const int64_t bs = A.batch_stride;
        // the stores are {32, k} boxes for Ns >= 32, {16, k} boxes for Ns = 16
        // (and plain row stores in the first pass)
        const int ocols = A.lNs == 4 ? 16 : 32;
        if (!p44t_make_map(&T.in, A.in, N, KD, A.batch, bs) ||
            !p44t_make_map(&T.out, A.out, N, KD, A.batch, bs, ocols))
            return 0;
        T.in2 = T.in;
        T.out2 = T.out;
        if (A.in2 && (!p44t_make_map(&T.in2, A.in2, N, KD, A.batch, bs) ||
                      !p44t_make_map(&T.out2, A.out2, N, KD, A.batch, bs, ocols)))
            return 0;
        // elements per thread in phase A as in launch_pass44: 4 when the grid
        // fills the GPU, fewer (more warps per CTA) for small transforms
        const int64_t ctas = (M / 32) * nsets;
        const int nw = ctas >= 4 * (int64_t)num_sms() ? 4 : ctas >= (int64_t)num_sms() ? 8 : 16;
        void (*kern)(const PassArgs, const PassTma) = nullptr;
        const bool inv = A.rot_inv != 0;
        if (A.rc.p3_ok)
            kern = inv ? p44t_kernel<KD, 3, true>(nw) : p44t_kernel<KD, 3, false>(nw);
        else if (A.rc.p2_ok)
            kern = inv ? p44t_kernel<KD, 2, true>(nw) : p44t_kernel<KD, 2, false>(nw);
        else
            kern = inv ? p44t_kernel<KD, 0, true>(nw) : p44t_kernel<KD, 0, false>(nw);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(M / 32), (unsigned)nsets);
        cfg.blockDim = dim3(nw * 32);
        cfg.dynamicSmemBytes = 0;
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
}
