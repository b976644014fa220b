// gfp_pass256.cuh -- two radix-16 Stockham stages in one kernel (radix 256 =
// 16 x 16) for k = 8 in the compile-time radix mode: half the launches and
// half the HBM round trips of k_pass44 for the same arithmetic.
//
// Pass at Ns (a power of 16): group J of M2 = N/256 reads x[J + T M2]
// (T < 256), multiplies by omega^(T (J mod Ns) (M2/Ns)) and writes its
// 256-point DFT at rho = omega^(N/256) to (J/Ns) Ns 256 + (J mod Ns) + U Ns:
// exactly two consecutive k_pass44 passes (Ns and 16 Ns).  The 256-point DFT
// is 16 x 16 (T = t1 + 16 t2, U = uA + 16 uB):
//   stage A   DFT16 over t2 for every t1           -> Y[t1][uA]
//   twiddle   Y[t1][uA] *= rho^(t1 uA) = r^a omega^b (the reference's cheap
//             split, fft.py:84-103: a digit rotation and one general multiply)
//   stage B   DFT16 over t1 for every uA           -> X[uA + 16 uB]
// Each DFT16 is pass44's 4 x 4 scheme (p44::dft4, compile-time rotations)
// run by four warps' worth of quarter-threads over shared-memory slots.
//
// CTA: 4 consecutive groups (1024 elements, 83 KB of slots), 256 threads,
// thread per element in the load / twiddle / store phases (4 each).
#pragma once
#include "gfp_pass44.cuh"

namespace p256 {

constexpr int G = 4;         // groups per CTA
constexpr int SLOT = 10;     // i64 words per element slot (80 B)
constexpr int NSLOT = G * 256;

// slot index (g, T) = 4 T + g, padded by one slot every 64 (bank spread for
// the stride-4 stage-B access)
GFP_D i64 *slot_ptr(i64 *sm, int sidx) { return sm + (sidx + (sidx >> 6)) * SLOT; }

GFP_D void ld_el(const i64 *p, i64 (&x)[8])
{
#pragma unroll
    for (int d = 0; d < 8; d += 2) {
        const longlong2 v = *reinterpret_cast<const longlong2 *>(p + d);
        x[d] = v.x;
        x[d + 1] = v.y;
    }
}
GFP_D void st_el(i64 *p, const i64 (&x)[8])
{
#pragma unroll
    for (int d = 0; d < 8; d += 2)
        *reinterpret_cast<longlong2 *>(p + d) = make_longlong2(x[d], x[d + 1]);
}

// omega^E = r^a omega^b for E in [0, N): rotation (as, negx) and table index b
struct Tw {
    int64_t b;
    int as;
    unsigned negx;
};
GFP_D Tw split_tw(int64_t E, int lN, int lM, int neg_exp, int root_inv)
{
    const int64_t N = (int64_t)1 << lN;
    if (neg_exp && E)
        E = N - E;
    int a = (int)(E >> lM);
    Tw tw;
    tw.b = E & (((int64_t)1 << lM) - 1);
    if (root_inv && a)
        a = 16 - a;
    tw.as = a & 7;
    tw.negx = ((1u << tw.as) - 1u) ^ (a >= 8 ? 0xffu : 0u);
    return tw;
}

// One DFT16 over the slots base + i * stride (i < 16), natural order in
// place, normalised; q = this thread's quarter (warp-uniform).  Three block
// barriers (every thread of the CTA calls it the same way).
template <int SPARSE, bool INV>
GFP_D void dft16(i64 *sm, int base, int stride, int q, const RadixConsts &rc)
{
    constexpr int KD = 8;
    i64 e[4][KD];
    // 4-point DFT over i = q + 4 i2 at rho^4; output u0 back to slot q + 4 u0
#pragma unroll
    for (int i2 = 0; i2 < 4; i2++)
        ld_el(slot_ptr(sm, base + (q + 4 * i2) * stride), e[i2]);
    p44::dft4<KD, INV, 0>(e[0], e[1], e[2], e[3]);
#pragma unroll
    for (int u0 = 0; u0 < 4; u0++)
        st_el(slot_ptr(sm, base + (q + 4 * u0) * stride), e[u0]);
    __syncthreads();
    // u0 = q: gather Y[i1][u0] (slot i1 + 4 u0), rotation rho^(i1 u0),
    // 4-point DFT over i1 -> X[u0 + 4 u1]
#pragma unroll
    for (int i1 = 0; i1 < 4; i1++)
        ld_el(slot_ptr(sm, base + (i1 + 4 * q) * stride), e[i1]);
    switch (q) {
    case 0: p44::dft4<KD, INV, 0>(e[0], e[1], e[2], e[3]); break;
    case 1: p44::dft4<KD, INV, 1>(e[0], e[1], e[2], e[3]); break;
    case 2: p44::dft4<KD, INV, 2>(e[0], e[1], e[2], e[3]); break;
    default: p44::dft4<KD, INV, 3>(e[0], e[1], e[2], e[3]); break;
    }
#pragma unroll
    for (int u1 = 0; u1 < 4; u1++)
        p44::normalize_el<KD, SPARSE>(e[u1], rc);
    __syncthreads();
#pragma unroll
    for (int u1 = 0; u1 < 4; u1++)
        st_el(slot_ptr(sm, base + (q + 4 * u1) * stride), e[u1]);
    __syncthreads();
}

// x (balanced digits, x * r^a folded in as rotation as / signs negx) times
// omega^b from the limb table -> slot; b == 0 lanes multiply by table[0] = 1
// when any lane of the warp multiplies (warp-uniform multiply)
template <int SPARSE>
GFP_D void twiddle_to_slot(const i64 (&x)[8], const Tw &tw, bool any, bool active,
                           const u64 *table_lh, i64 *slot, const RadixConsts &rc)
{
    constexpr int KD = 8;
    if (any) {
        u64 ylh[KD];
        const ulonglong2 *tp = reinterpret_cast<const ulonglong2 *>(table_lh + tw.b * KD);
#pragma unroll
        for (int d = 0; d < KD; d += 2) {
            const ulonglong2 v = __ldg(tp + d / 2);
            ylh[d] = v.x;
            ylh[d + 1] = v.y;
        }
        i64 f[KD];
        fast_mul_lazy_ylimbs<KD, SPARSE, true>(x, ylh, f, rc, tw.negx, slot);
    } else {
        i64 f[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            f[d] = !active ? 0 : ((tw.negx >> d) & 1u) ? -x[d] : x[d];
        st_el(slot, f);
    }
}

}  // namespace p256

template <int SPARSE, bool INV>
__global__ void __launch_bounds__(256, 2) k_pass256(PassArgs A)
{
    constexpr int KD = 8;
    extern __shared__ __align__(16) i64 sm256[];
    i64 *sm = sm256;
    const int tid = threadIdx.x;
    const int lane = tid & 31, w = tid >> 5;

    int64_t bidx = blockIdx.y;
    const u64 *in_base = A.in;
    u64 *out_base = A.out;
    if (bidx >= A.batch) {
        bidx -= A.batch;
        in_base = A.in2;
        out_base = A.out2;
    }
    const int lN = A.lN, lM = A.lM, lNs = A.lNs;
    const int lM2 = lN - 8;
    const int64_t nsmask = ((int64_t)1 << lNs) - 1;
    const u64 *in = in_base + bidx * A.batch_stride;
    u64 *out = out_base + bidx * A.batch_stride;
    const u64 *pre = A.pre ? A.pre + bidx * A.batch_stride : nullptr;
    const RadixConsts rc = A.rc;
    const int64_t J0 = (int64_t)blockIdx.x * p256::G;
    const unsigned rowN = 1u << lN;

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- phase 1: load element (g, T), outer twiddle, slot 4 T + g
#pragma unroll 1
    for (int i = 0; i < 4; i++) {
        const int e = tid + 256 * i;
        const int g = e & 3, T = e >> 2;
        const int64_t J = J0 + g;
        const int64_t pos = J + ((int64_t)T << lM2);
        const p256::Tw tw =
            p256::split_tw(((int64_t)T * (J & nsmask)) << (lM2 - lNs), lN, lM, A.neg_exp,
                           A.root_inv);
        i64 x[KD];
        const u64 *src = in + pos;
#pragma unroll
        for (int d = 0; d < KD; d++)
            x[d] = (i64)__ldcs(src + (unsigned)((d - tw.as) & (KD - 1)) * rowN);
        if (A.in_canon)  // first pass only, a = 0
            to_balanced<KD>(x, rc.r);
        i64 *slot = p256::slot_ptr(sm, e);
        const bool any = __any_sync(FULL_MASK, tw.b != 0);
        if (pre) {  // first pass only (a = b = 0): pointwise product
            u64 ylh[KD];
            constexpr int S = FastSplit<KD>::S;
#pragma unroll
            for (int d = 0; d < KD; d++) {
                int l, h;
                split_limbs<S>((i64)__ldg(pre + ((int64_t)d << lN) + pos), l, h);
                ylh[d] = (u64)(unsigned)l | ((u64)(unsigned)h << 32);
            }
            i64 f[KD];
            fast_mul_lazy_ylimbs<KD, SPARSE, true>(x, ylh, f, rc, 0u, slot);
        } else {
            p256::twiddle_to_slot<SPARSE>(x, tw, any, true, A.table_lh_plain, slot, rc);
        }
    }
    __syncthreads();

    // ---- stage A: DFT16 over t2 (slots 4 (t1 + 16 t2) + g) for the 64 (g, t1)
    const int q = w & 3;
    const int s = lane + 32 * (w >> 2);  // DFT id, < 64
    p256::dft16<SPARSE, INV>(sm, s, 64, q, rc);  // base 4 t1 + g = s, stride 64

    // ---- inner twiddle rho^(t1 uA) (and N^-1 on the last pass: table_lh is
    // then the omega^b N^-1 table and every element multiplies)
#pragma unroll 1
    for (int i = 0; i < 4; i++) {
        const int e = tid + 256 * i;  // slot 4 (t1 + 16 uA) + g
        const int T = e >> 2, t1 = T & 15, uA = T >> 4;
        const p256::Tw tw = p256::split_tw((int64_t)(t1 * uA) << lM2, lN, lM, A.neg_exp,
                                           A.root_inv);
        i64 *slot = p256::slot_ptr(sm, e);
        i64 x[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            x[d] = slot[(d - tw.as) & (KD - 1)];
        const bool any = __any_sync(FULL_MASK, tw.b != 0 || A.scale);
        __syncwarp();  // every lane has read its slot before any lane rewrites it
        p256::twiddle_to_slot<SPARSE>(x, tw, any, true, A.table_lh, slot, rc);
    }
    __syncthreads();

    // ---- stage B: DFT16 over t1 (slots 4 (t1 + 16 uA) + g) for the 64 (g, uA)
    // (s = g + 4 uA: base 64 uA + g, stride 4)
    p256::dft16<SPARSE, INV>(sm, 64 * (s >> 2) + (s & 3), 4, q, rc);

    // ---- store X[U], U = uA + 16 uB, from slot 4 (uB + 16 uA) + g
    const bool first = lNs == 0;
#pragma unroll 1
    for (int i = 0; i < 4; i++) {
        const int e = tid + 256 * i;
        int g, U;
        if (first) {  // outputs of the CTA are 1024 consecutive positions
            g = e >> 8;
            U = e & 255;
        } else {
            g = e & 3;
            U = e >> 2;
        }
        const int uA = U & 15, uB = U >> 4;
        const int64_t J = J0 + g;
        const int64_t pos = ((J >> lNs) << (lNs + 8)) + (J & nsmask) + ((int64_t)U << lNs);
        i64 v[KD];
        p256::ld_el(p256::slot_ptr(sm, 4 * (uB + 16 * uA) + g), v);
        if (A.canon) {
            u64 c[KD];
            lazy_to_canonical_bf<KD>(v, c, rc);
#pragma unroll
            for (int d = 0; d < KD; d++)
                __stcs(out + ((int64_t)d << lN) + pos, c[d]);
        } else {
#pragma unroll
            for (int d = 0; d < KD; d++)
                __stcs(out + ((int64_t)d << lN) + pos, (u64)v[d]);
        }
    }
}

// k_pass256 can serve a pair of passes for k = 8 in mode 3 when the transform
// has at least 4 groups of 256 (N >= 1024).  Opt-in (GFP_PASS256=1): measured
// slower than two k_pass44 launches -- C4 forward 5.05 -> 5.25 ms (eight block
// barriers per CTA, 32-byte global segments, the rotated shared-memory reads
// of the inner twiddle), C2 0.079 -> 0.101 ms (1024 elements per CTA leave a
// 2^16-point transform 128 CTAs: fewer than the SMs).
static inline bool pass256_enabled(int k, const RadixConsts &rc, int64_t N)
{
    static int enabled = -1;
    if (enabled < 0) {
        const char *e = getenv("GFP_PASS256");
        enabled = (e && e[0] == '1') ? 1 : 0;
    }
    return enabled && k == 8 && rc.p3_ok && rc.stages_per_norm >= 4 && N >= 1024;
}

static inline int launch_pass256(const PassArgs &A, int64_t N, int64_t nsets, cudaStream_t st)
{
    const int64_t M2 = N >> 8;
    const size_t smem = (size_t)(p256::NSLOT + p256::NSLOT / 64) * p256::SLOT * sizeof(i64);
    static bool set = false;
    if (!set) {
        cudaFuncSetAttribute(k_pass256<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_pass256<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        set = true;
    }
    dim3 grid((unsigned)(M2 / p256::G), (unsigned)nsets);
    if (A.rot_inv)
        launch_pdl(k_pass256<3, true>, grid, 256, st, A, smem);
    else
        launch_pdl(k_pass256<3, false>, grid, 256, st, A, smem);
    return 1;
}
