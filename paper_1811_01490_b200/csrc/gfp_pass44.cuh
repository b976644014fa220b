// gfp_pass44.cuh -- radix-16 Stockham pass for k = 8 (K = 2k = 16), thread
// per element throughout (no warp shuffles).
//
// Same pass as k_pass (gfp_pass.cuh): group j of M = N/K groups reads
// x[j + t M] (t < K), multiplies element t by omega^E,
// E = t (j mod Ns) (M / Ns), and writes the K-point DFT at root rho = r (or
// 1/r) to (j / Ns) Ns K + (j mod Ns) + u Ns.  The reference computes the
// same transform with dft_general (fft.py:298-360): base-case blocks of
// dft2 / r^t shifts (fft.py:114-193) and level twiddles split as
// r^a * omega^b (_twiddle_level_cheap, fft.py:84-103).
//
// Mapping (CTA = 4 warps x 32 lanes, 32 consecutive groups, lane = group):
//   phase A   warp w loads elements t = w + 4 t2 (t2 < 4) of its lane's
//             group.  r^a is folded into the digit addressing of the load
//             (digit d comes from row (d - a) mod k) and the wrapped digits'
//             sign into the multiply's limb split; omega^b is one general
//             multiply (fast_mul_lazy) by the table entry.
//             Each finished element is parked in the thread's own smem slot
//             (keeping four in registers across the multiplies halves occupancy).
//   stage 1   4-point DFT over t2 at root rho^4 (a rotation by k/2 digits):
//             pure adds with compile-time digit renaming, in registers.
//   exchange  outputs Y[w][u0] through shared memory (one 80 B slot each).
//   stage 2   warp w = u0 gathers Y[t1][u0], applies rho^(t1 u0) as a
//             compile-time rotation (warp-uniform switch on u0) whose sign
//             flips fold into the adds, and runs the 4-point DFT over t1:
//             X[u0 + 4 u1].  One balanced normalisation per element, the
//             canonical form on the last pass, coalesced digit-row stores.
// K = 16 = 4 x 4 needs 4 lazy radix-2 stages without normalisation; the
// launcher only selects this kernel when the host bound check allows it
// (RadixConsts::stages_per_norm >= 4).
//
// Since round 2 the digit-major passes of transforms with >= 32 groups run as
// k_pass44t (gfp_pass44t.cuh: the same pass on TMA tiles).  This kernel keeps
// what that one does not take: the pointwise-product pass of a poly-multiply,
// the element-major (host-memory) first / last passes, the fused four-step
// exchange, and transforms under 512 points.
#pragma once
#include "gfp_internal.cuh"
#include "gfp_fast.cuh"

// register bounds (CTAs per SM) of the instantiations: NW = 4 at 5 CTAs/SM
// (96 registers; C4), its fused-exchange variant at 4 (128 registers: 5
// spilled and measured slower), NW = 8 at 2, NW = 16 at 1 (2 CTAs/SM at 64
// registers spilled: C2 0.076 -> 0.100 ms)
#define P44_MINB 5
#define P44_XCH_MINB 4
#define P44_MINB16 1
// stage 2's outputs split over all NW warps when NW > 4
#define P44_SPLIT2 1
// transforms per CTA in the fused-exchange pass: 8 -> 64 B store segments
// (measured at 1 GPU: sharded C4 5.237 ms with 4, 5.218 ms with 8)
#define P44_XT 8
// smallest NW that stages the next element with cp.async (NW = 4 keeps
// 40 KB smem for 5 CTAs / SM: measured 1.5% faster on C4)
#define P44_PF_MINNW 8

namespace p44 {

// digit rotation a (0 <= a < 2k) of element t of group j in a pass:
// omega^E = r^a omega^b, E = t (j mod Ns)(M / Ns)
struct Twiddle {
    int64_t b;
    int as;
    unsigned negx;
};
template <int KD>
GFP_D Twiddle twiddle_of(int t, int64_t j, int64_t nsmask, int lM, int lNs, int64_t N,
                         int64_t M, int neg_exp, int root_inv)
{
    Twiddle tw;
    int64_t E = ((int64_t)t * (j & nsmask)) << (lM - lNs);
    if (neg_exp && E)
        E = N - E;
    int a = (int)(E >> lM);
    tw.b = E & (M - 1);
    if (root_inv && a)
        a = 2 * KD - a;
    // x * r^a: digit d comes from row (d - a) mod k, negated when it
    // wrapped (d < a mod k) xor a >= k
    tw.as = a & (KD - 1);
    tw.negx = ((1u << tw.as) - 1u) ^ (a >= KD ? ((1u << KD) - 1u) : 0u);
    return tw;
}

// y = x * r^S for a compile-time S in [0, 2k): digit renaming, wrapped
// digits negated (r^k = -1)
template <int KD, int S>
GFP_D void rot_c(const i64 (&x)[KD], i64 (&y)[KD])
{
    constexpr int s = S % KD;
    constexpr bool negall = ((S / KD) & 1) != 0;
#pragma unroll
    for (int d = 0; d < KD; d++) {
        const int src = (d - s + KD) % KD;
        const bool wrap = d < s;
        y[d] = (wrap != negall) ? -x[src] : x[src];
    }
}

// exponent of rho^e as a power of r: rho = r (forward) or 1/r = r^(2k-1)
template <int KD, bool INV>
__host__ __device__ constexpr int rexp(int e)
{
    return INV ? (2 * KD - (e % (2 * KD))) % (2 * KD) : e % (2 * KD);
}

// in-place 4-point DFT at root w = rho^(K/4) (w^2 = -1):
//   Z0 = (x0 + x2) + (x1 + x3)   Z2 = (x0 + x2) - (x1 + x3)
//   Z1 = (x0 - x2) + w(x1 - x3)  Z3 = (x0 - x2) - w(x1 - x3)
// x1 and x3 may first be multiplied by rho^(T1) and rho^(3 T1), x2 by
// rho^(2 T1) (stage 2's inter-stage twiddle, T1 = u0), as compile-time
// rotations whose sign flips the compiler folds into the adds.
template <int KD, bool INV, int TW>
GFP_D void dft4(i64 (&x0)[KD], i64 (&x1)[KD], i64 (&x2)[KD], i64 (&x3)[KD])
{
    i64 a1[KD], a2[KD], a3[KD];
    rot_c<KD, rexp<KD, INV>(TW)>(x1, a1);
    rot_c<KD, rexp<KD, INV>(2 * TW)>(x2, a2);
    rot_c<KD, rexp<KD, INV>(3 * TW)>(x3, a3);
    i64 s0[KD], d0[KD], s1[KD], t[KD], d1[KD];
#pragma unroll
    for (int d = 0; d < KD; d++) {
        s0[d] = x0[d] + a2[d];
        d0[d] = x0[d] - a2[d];
        s1[d] = a1[d] + a3[d];
        t[d] = a1[d] - a3[d];
    }
    rot_c<KD, rexp<KD, INV>(KD / 2)>(t, d1);  // w = rho^(K/4) = rho^(k/2)
#pragma unroll
    for (int d = 0; d < KD; d++) {
        x0[d] = s0[d] + s1[d];
        x2[d] = s0[d] - s1[d];
        x1[d] = d0[d] + d1[d];
        x3[d] = d0[d] - d1[d];
    }
}

// one balanced normalisation of a lazy element: digit quotients move one
// digit up, the top one wraps negated into digit 0 (r^k = -1)
template <int KD, int SPARSE>
GFP_D void normalize_el(i64 (&v)[KD], const RadixConsts &rc)
{
    if constexpr (SPARSE == 3) {
        // compile-time r = 2^a + 2^b: digit d becomes
        //   ((v_d + 2^(a-1)) mod 2^a) - 2^(a-1) + (q_{d-1} - q_d 2^b)
        // with the small correction q_{d-1} - q_d 2^b formed in 32 bits (one
        // IMAD) and added once (|q| <= 2^5, so it fits easily)
        constexpr int a = P2Radix<KD>::a, b = P2Radix<KD>::b;
        constexpr i64 half = (i64)1 << (a - 1), mask = ((i64)1 << a) - 1;
        int q[KD];
        i64 m[KD];
#pragma unroll
        for (int d = 0; d < KD; d++) {
            const i64 vb = v[d] + half;
            q[d] = (int)(vb >> a);
            m[d] = vb & mask;
        }
#pragma unroll
        for (int d = 0; d < KD; d++) {
            const int cin = d ? q[d - 1] : -q[KD - 1];
            v[d] = m[d] - half + (i64)(cin - (q[d] << b));
        }
        return;
    }
    int q[KD];
    i64 rem[KD];
#pragma unroll
    for (int d = 0; d < KD; d++)
        q[d] = norm_bal<SPARSE, KD>(v[d], rc, rem[d]);
    v[0] = rem[0] - q[KD - 1];
#pragma unroll
    for (int d = 1; d < KD; d++)
        v[d] = rem[d] + q[d - 1];
}

}  // namespace p44

template <int KD, int SPARSE, bool INV, int NW, bool XCH = false>
__global__ void __launch_bounds__(NW * 32, NW == 4 ? (XCH ? P44_XCH_MINB : P44_MINB) : NW == 8 ? 2 : P44_MINB16)
    k_pass44(PassArgs A)
{
    static_assert(KD == 8, "radix 4 x 4 pass is for K = 16");
    constexpr int K = 2 * KD;
    constexpr int SLOT = KD + 2;  // 80 B element slot: conflict-free 128-bit smem access
    __shared__ __align__(16) i64 sm[K * 32 * SLOT];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;  // t1 in stage 1, u0 in stage 2 (warp-uniform)

    // fused four-step exchange (last pass, A.xg ranks): a CTA spans P44_XT
    // transforms x 32/P44_XT groups (lane = (32/P44_XT) ts + jl) so the transposed stores
    // (consecutive transforms adjacent) fill whole 32 B sectors
    constexpr bool xch = XCH;  // A.xg != 0 (a separate instantiation: lane-dependent
                               // batch pointers cost registers)
    int64_t bidx = xch ? (int64_t)blockIdx.y * P44_XT + lane / (32 / P44_XT) : blockIdx.y;
    const u64 *in_base = A.in;
    u64 *out_base = A.out;
    const u64 *em_in = A.in_em;
    int64_t n_in = A.n_in;
    if (bidx >= A.batch) {
        bidx -= A.batch;
        in_base = A.in2;
        out_base = A.out2;
        em_in = A.in2_em;
        n_in = A.n_in2;
    }
    if (em_in)
        em_in += bidx * n_in * KD;
    u64 *em_out = A.out_em ? A.out_em + bidx * A.n_out * KD : nullptr;
    const int lN = A.lN, lM = A.lM, lNs = A.lNs;
    const int64_t N = (int64_t)1 << lN, M = (int64_t)1 << lM;
    const int64_t nsmask = ((int64_t)1 << lNs) - 1;
    const u64 *in = in_base + bidx * A.batch_stride;
    u64 *out = out_base + bidx * A.batch_stride;
    const u64 *pre = A.pre ? A.pre + bidx * A.batch_stride : nullptr;
    const RadixConsts rc = A.rc;
    // gpc consecutive groups per CTA (32, or fewer to spread a small grid
    // over every SM: launch_pass44)
    const int gpc = A.gpc;
    const int64_t j0 = (int64_t)blockIdx.x * gpc;
    const int64_t j = j0 + (xch ? (lane & (32 / P44_XT - 1)) : lane);
    const bool active = (xch || lane < gpc) && j < M;

    // programmatic dependent launch: let the next pass's CTAs be scheduled
    // as this grid drains, and wait for the previous pass's writes before the
    // first global access (no-ops when launched without the attribute)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- phase A: load + twiddle elements t = w + NW i (16 / NW per thread)
    // With two or more elements per thread the digit-major loads of element
    // i + 1 are issued (cp.async, 8 B per digit row, coalesced across the
    // warp) into this warp's staging rows while element i is multiplied, so
    // the HBM latency hides behind the multiply (was ~20% of the stall
    // samples); the rotation r^a is applied when the row is read back.
    extern __shared__ __align__(16) u64 pf_stage[];  // [NW][KD][32]
    constexpr bool PF = NW <= 8 && NW >= P44_PF_MINNW;
    const bool pf = PF && !em_in;
    u64 *stg = pf_stage + w * (KD * 32) + lane;
    auto prefetch = [&](int i) {
        if (active) {
            const int64_t e0 = j + ((int64_t)(w + NW * i) << lM);
#pragma unroll
            for (int r_ = 0; r_ < KD; r_++) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(stg + r_ * 32);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa),
                             "l"(in + GFP_IDX(e0 + ((int64_t)r_ << lN), (int64_t)KD << lN))
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (pf)
        prefetch(0);
    i64 e[4][KD];
    for (int i = 0; i < 16 / NW; i++) {
        const int t = w + NW * i;
        i64 f[KD], x[KD];
        int64_t b = 0;
        unsigned negx = 0;
        const int64_t pos = j + ((int64_t)t << lM);
        if (em_in) {
            // first pass (Ns = 1, a = 0), element-major input, possibly mapped
            // host memory: the warp's 32 elements (j0 .. j0 + 31, t) are 2 KB
            // contiguous; read them with lane-contiguous 16 B loads (full
            // 512 B requests over PCIe) into this row's smem slots
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int e = (lane >> 2) + 8 * q, dp = (lane & 3) * 2;
                ulonglong2 v = make_ulonglong2(0, 0);
                if (e < gpc && j0 + e < M && j0 + e + ((int64_t)t << lM) < n_in)
                    v = reinterpret_cast<const ulonglong2 *>(
                        em_in)[GFP_IDX(((j0 + ((int64_t)t << lM)) * KD) / 2 + lane + 32 * q,
                                       n_in * KD / 2)];
                *reinterpret_cast<ulonglong2 *>(sm + GFP_IDX((t * 32 + e) * SLOT + dp, (K * 32 * SLOT))) = v;
            }
            __syncwarp();
        }
        if (active) {
            p44::Twiddle tw = p44::twiddle_of<KD>(t, j, nsmask, lM, lNs, N, M,
                                                  A.neg_exp, A.root_inv);
            if (A.ft_lh) {
                // first pass (own twiddle trivial): the four-step twiddle
                // w^(+-(row0 + b) pos) of the enclosing transform instead
                const int64_t Nf = (int64_t)1 << A.ft_lN;
                int64_t E = ((A.ft_row0 + bidx) * pos) & (Nf - 1);
                if (A.ft_inv && E)
                    E = Nf - E;
                int a = (int)(E >> A.ft_lM);
                tw.b = E & (((int64_t)1 << A.ft_lM) - 1);
                if (A.ft_root_inv && a)
                    a = 2 * KD - a;
                tw.as = a & (KD - 1);
                tw.negx = ((1u << tw.as) - 1u) ^ (a >= KD ? ((1u << KD) - 1u) : 0u);
            }
            b = tw.b;
            negx = tw.negx;
            if (em_in) {
                const i64 *slot = sm + GFP_IDX((t * 32 + lane) * SLOT, (K * 32 * SLOT));
#pragma unroll
                for (int d = 0; d < KD; d += 2) {
                    const longlong2 v = *reinterpret_cast<const longlong2 *>(slot + d);
                    x[d] = v.x;
                    x[d + 1] = v.y;
                }
            } else if (pf) {
                asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
                for (int d = 0; d < KD; d++)
                    x[d] = (i64)stg[((d - tw.as) & (KD - 1)) * 32];
                if (i + 1 < 16 / NW)  // own rows, already read: refill them
                    prefetch(i + 1);
            } else {
                // rows are N words apart; k N words fit 32-bit offsets (N <= 2^26)
                const u64 *src = in + pos;
                const unsigned rowN = 1u << lN;
#pragma unroll
                for (int d = 0; d < KD; d++)  // streamed once: evict-first, keep the tables in L2
                    x[d] = (i64)__ldcs(src + GFP_IDX((unsigned)((d - tw.as) & (KD - 1)) * rowN,
                                                     (int64_t)KD * N - pos));
            }
            if (A.in_canon)  // pass 0 only, where a = 0
                to_balanced<KD>(x, rc.r);
        }
        // element t parks in slot t: holding four elements in registers
        // across the multiplies would cost occupancy
        i64 *slot = sm + GFP_IDX((t * 32 + lane) * SLOT, (K * 32 * SLOT));
        // Up to two multiplies through ONE inlined copy of the multiply (the
        // kernel's code size matters: ~2/3 of it would be multiplies): the
        // pointwise product by `pre` (pass 0 only, a = b = 0), then the
        // twiddle omega^b.  The twiddle multiply is warp-uniform: lanes whose
        // twiddle is a pure power of r (b = 0) multiply by table[0] = 1
        // instead of diverging.  Each product digit is stored to the slot as
        // soon as it is final; a second multiply reloads it.
        const bool mul_tw = __any_sync(FULL_MASK, active && (b || A.scale));
        const int nmul = (pre ? 1 : 0) + (mul_tw ? 1 : 0);
#pragma unroll 1
        for (int mi = 0; mi < nmul; mi++) {
            const bool use_pre = pre && mi == 0;
            if (mi > 0) {  // own slot: no cross-lane ordering needed
#pragma unroll
                for (int d = 0; d < KD; d += 2) {
                    const longlong2 v = *reinterpret_cast<const longlong2 *>(slot + d);
                    x[d] = v.x;
                    x[d + 1] = v.y;
                }
            }
            if (active) {
                u64 ylh[KD];
                if (use_pre) {
                    constexpr int S = FastSplit<KD>::S;
#pragma unroll
                    for (int d = 0; d < KD; d++) {
                        int l, h;
                        split_limbs<S>((i64)__ldg(pre + GFP_IDX(((int64_t)d << lN) + pos,
                                                                (int64_t)KD << lN)), l, h);
                        ylh[d] = (u64)(unsigned)l | ((u64)(unsigned)h << 32);
                    }
                } else {
                    const ulonglong2 *tp = reinterpret_cast<const ulonglong2 *>(
                        (A.ft_lh ? A.ft_lh : A.table_lh) +
                        GFP_IDX(b, A.ft_lh ? ((int64_t)1 << A.ft_lM) : M) * KD);
#pragma unroll
                    for (int d = 0; d < KD; d += 2) {
                        const ulonglong2 v = __ldg(tp + d / 2);
                        ylh[d] = v.x;
                        ylh[d + 1] = v.y;
                    }
                }
                fast_mul_lazy_ylimbs<KD, SPARSE, true>(x, ylh, f, rc, use_pre ? 0u : negx, slot);
            }
        }
        if (!mul_tw || !active) {
            // no twiddle multiply: r^a alone (a digit renaming) or an idle lane
            if (pre && active) {  // own slot (divergent: no warp barrier here)
#pragma unroll
                for (int d = 0; d < KD; d += 2) {
                    const longlong2 v = *reinterpret_cast<const longlong2 *>(slot + d);
                    x[d] = v.x;
                    x[d + 1] = v.y;
                }
            }
#pragma unroll
            for (int d = 0; d < KD; d++)
                f[d] = !active ? 0 : ((negx >> d) & 1u) ? -x[d] : x[d];
#pragma unroll
            for (int d = 0; d < KD; d += 2)
                *reinterpret_cast<longlong2 *>(slot + d) = make_longlong2(f[d], f[d + 1]);
        }
    }

    GFP_JITTER(1);
    // ---- stage 1 (warps w < 4, t1 = w): 4-point DFT over t2 (root rho^4) of
    // slots t1 + 4 t2, outputs u0 = 0..3 back into slots t1 + 4 u0 (the same
    // slots: no other thread touches them).  With NW = 4 the thread reads
    // its own phase-A slots and needs no barrier.
    if (NW > 4)
        __syncthreads();
    if (w < 4) {
#pragma unroll
    for (int t2 = 0; t2 < 4; t2++) {
        const i64 *slot = sm + GFP_IDX(((t2 * 4 + w) * 32 + lane) * SLOT, (K * 32 * SLOT));
#pragma unroll
        for (int d = 0; d < KD; d += 2) {
            const longlong2 v = *reinterpret_cast<const longlong2 *>(slot + d);
            e[t2][d] = v.x;
            e[t2][d + 1] = v.y;
        }
    }
    p44::dft4<KD, INV, 0>(e[0], e[1], e[2], e[3]);
#pragma unroll
    for (int u0 = 0; u0 < 4; u0++) {
        i64 *slot = sm + GFP_IDX(((u0 * 4 + w) * 32 + lane) * SLOT, (K * 32 * SLOT));
#pragma unroll
        for (int d = 0; d < KD; d += 2)
            *reinterpret_cast<longlong2 *>(slot + d) = make_longlong2(e[u0][d], e[u0][d + 1]);
    }
    }
    GFP_JITTER(2);
    __syncthreads();
    // Stage 2 over SPL = NW / 4 warps per u0 (P44_SPLIT2): every warp gathers
    // its u0's four slots and computes the (cheap, lazy) 4-point DFT, then
    // normalises / canonicalises / stores only its 4 / SPL outputs u1 -- the
    // expensive per-output work spread over all NW warps instead of 4.
    constexpr int SPL = (P44_SPLIT2 && NW > 4) ? NW / 4 : 1;
    constexpr int NU = 4 / SPL;  // outputs per warp
    if (SPL == 1 && w >= 4)
        return;
    const int u0 = w & 3;
    const int h = SPL == 1 ? 0 : w >> 2;  // output block u1 in [h NU, h NU + NU)

    // ---- stage 2: gather Y[t1][u0], twiddle rho^(t1 u0), DFT over t1
#pragma unroll
    for (int t1 = 0; t1 < 4; t1++) {
        const i64 *slot = sm + GFP_IDX(((u0 * 4 + t1) * 32 + lane) * SLOT, (K * 32 * SLOT));
#pragma unroll
        for (int d = 0; d < KD; d += 2) {
            const longlong2 v = *reinterpret_cast<const longlong2 *>(slot + d);
            e[t1][d] = v.x;
            e[t1][d + 1] = v.y;
        }
    }
    switch (u0) {
    case 0: p44::dft4<KD, INV, 0>(e[0], e[1], e[2], e[3]); break;
    case 1: p44::dft4<KD, INV, 1>(e[0], e[1], e[2], e[3]); break;
    case 2: p44::dft4<KD, INV, 2>(e[0], e[1], e[2], e[3]); break;
    default: p44::dft4<KD, INV, 3>(e[0], e[1], e[2], e[3]); break;
    }
    if (SPL > 1 && h > 0) {  // this warp's outputs into e[0 .. NU-1] (static indices)
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
    // one balanced normalisation per output, then (last pass) the canonical
    // form, once for all three store paths below (keeps the kernel's code
    // small: the store paths only move digits)
    const bool canon = A.canon || em_out;
#pragma unroll
    for (int q = 0; q < NU; q++) {
        p44::normalize_el<KD, SPARSE>(e[q], rc);
        if (canon) {
            u64 c[KD];
            lazy_to_canonical_bf<KD>(e[q], c, rc);
#pragma unroll
            for (int d = 0; d < KD; d++)
                e[q][d] = (i64)c[d];
        }
    }
    if (em_out) {
        // last pass (Ns = M: output u of group j at j + u M), element-major,
        // possibly mapped host memory: park the canonical outputs in the
        // stage-2 slots (rows 4 u0 + u1), then write each u's 32 elements
        // (2 KB contiguous) with lane-contiguous 16 B stores
        GFP_JITTER(3);
        if (SPL > 1)  // the u0 slots are read by every warp of the u0 above
            asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
#pragma unroll
        for (int q = 0; q < NU; q++) {
            const int u1 = h * NU + q;
            i64 *slot = sm + GFP_IDX(((4 * u0 + u1) * 32 + lane) * SLOT, (K * 32 * SLOT));
#pragma unroll
            for (int d = 0; d < KD; d += 2)
                *reinterpret_cast<longlong2 *>(slot + d) = make_longlong2(e[q][d], e[q][d + 1]);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NU; q++) {
            const int u1 = h * NU + q;
            const int64_t ubase = j0 + ((int64_t)(u0 + 4 * u1) << lM);
#pragma unroll
            for (int qq = 0; qq < 4; qq++) {
                const int e = (lane >> 2) + 8 * qq, dp = (lane & 3) * 2;
                const longlong2 v =
                    *reinterpret_cast<const longlong2 *>(
                        sm + GFP_IDX(((4 * u0 + u1) * 32 + e) * SLOT + dp, (K * 32 * SLOT)));
                if (e < gpc && j0 + e < M && ubase + e < A.n_out)
                    reinterpret_cast<ulonglong2 *>(
                        em_out)[GFP_IDX(ubase * KD / 2 + lane + 32 * qq, A.n_out * KD / 2)] =
                        make_ulonglong2((u64)v.x, (u64)v.y);
            }
        }
        return;
    }
    if (lNs == 0) {
        // first pass (Ns = 1): output u of group j goes to 16 j + u, so a
        // lane-per-group store would scatter 8 B per 128 B line.  Park the
        // outputs digit-major ([d][g][u], row pitch 17: conflict-free both
        // ways) over the slots, then write each digit row's 512 consecutive
        // positions lane-contiguously.
        constexpr int NT = SPL * 128;  // threads in stage 2
        i64 *park = sm;
        GFP_JITTER(4);
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");  // stage-2 slot reads done
#pragma unroll
        for (int q = 0; q < NU; q++) {
            const int u = u0 + 4 * (h * NU + q);
#pragma unroll
            for (int d = 0; d < KD; d++)
                park[GFP_IDX((d * 32 + lane) * 17 + u, (K * 32 * SLOT))] = e[q][d];
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
        const int tid = threadIdx.x;  // < NT: the stage-2 warps
        u64 *obase = out + (j0 << 4);
#pragma unroll
        for (int q4 = 0; q4 < 512 / NT; q4++) {
            const int q = tid + NT * q4;       // position 16 j0 + q
            const int g = q >> 4, u = q & 15;  // group j0 + g, output u
            if (g < gpc && j0 + g < M) {
#pragma unroll
                for (int d = 0; d < KD; d++)
                    __stcs(obase + GFP_IDX(((int64_t)d << lN) + q, ((int64_t)KD << lN) - (j0 << 4)),
                           (u64)park[GFP_IDX((d * 32 + g) * 17 + u, (K * 32 * SLOT))]);
            }
        }
        return;
    }
    if (!active)
        return;
    // X[u0 + 4 u1] = e[u1] -> (j / Ns) Ns K + (j mod Ns) + u Ns
    const int64_t base = ((j >> lNs) << (lNs + 4)) + (j & nsmask);
    if (xch) {  // straight into the owner's receive buffer (peer pointer or local)
        const int64_t GA = (int64_t)A.xg * A.xA;
        const int64_t col = (int64_t)A.xrank * A.xA + bidx;
        const int64_t bmask = ((int64_t)1 << A.lxb) - 1;
#pragma unroll
        for (int q = 0; q < NU; q++) {
            const int64_t pos = base + ((int64_t)(u0 + 4 * (h * NU + q)) << lNs);
            const int g = (int)(pos >> A.lxb);
            u64 *dp = A.xdst[0];
#pragma unroll
            for (int gg = 1; gg < 8; gg++)
                dp = g == gg ? A.xdst[gg] : dp;
            (void)GFP_IDX(g, A.xg);
            dp += (pos & bmask) * KD * GA + col;
#pragma unroll
            for (int d = 0; d < KD; d++)
                __stcs(dp + GFP_IDX(d * GA, ((bmask + 1) * KD - (pos & bmask) * KD) * GA - col),
                       (u64)e[q][d]);
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < NU; q++) {
        const int64_t pos = base + ((int64_t)(u0 + 4 * (h * NU + q)) << lNs);
#pragma unroll
        for (int d = 0; d < KD; d++)
            __stcs(out + GFP_IDX(((int64_t)d << lN) + pos, (int64_t)KD << lN), (u64)e[q][d]);
    }
}

// k_pass44 serves k = 8 when 4 lazy radix-2 stages fit the digit bounds
static inline bool pass44_enabled(int k, const RadixConsts &rc)
{
    return k == 8 && rc.stages_per_norm >= 4;
}

// launch with programmatic stream serialisation (PDL): the kernel may start
// while the previous kernel on the stream drains; it orders itself with
// griddepcontrol.wait
static inline void launch_pdl(void (*kern)(PassArgs), dim3 grid, int threads, cudaStream_t st,
                              const PassArgs &A, size_t smem = 0)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, A);
}

// NW <= 8: dynamic shared memory for the cp.async staging rows ([NW][k][32]);
// the attribute is per device context, so it is set once per device
template <int KD, int SP, bool IV, int NW, bool XCH = false>
static inline void launch_p44(dim3 grid, cudaStream_t st, const PassArgs &A)
{
    const size_t smem = NW >= P44_PF_MINNW ? (size_t)NW * KD * 32 * sizeof(u64) : 0;
    static unsigned long long set_on = 0;
    once_per_device(set_on, [&] {
        cudaFuncSetAttribute(k_pass44<KD, SP, IV, NW, XCH>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    launch_pdl(k_pass44<KD, SP, IV, NW, XCH>, grid, NW * 32, st, A, smem);
}

// launcher: returns 1 when it handled the pass
template <int KD>
static int launch_pass44(const PassArgs &A0, int64_t M, int64_t nsets, cudaStream_t st)
{
    if constexpr (KD != 8) {
        return 0;
    } else {
        if (!pass44_enabled(KD, A0.rc))
            return 0;
        const int64_t ctas = ((M + 31) / 32) * nsets;
        // elements per thread in phase A: 4 when the grid fills the GPU,
        // fewer (more warps per CTA) for small transforms (C1, C2).  Groups
        // per CTA: 32 (spreading a grid under two waves over every SM with
        // fewer was measured: no gain for C1 / C2, latency-bound per CTA).
        const int nw = ctas >= 4 * (int64_t)num_sms() ? 4 : ctas >= (int64_t)num_sms() ? 8 : 16;
        int gpc = 32;
        PassArgs A = A0;
        if (A.xg)  // fused exchange: 8 groups x 4 transforms per CTA
            gpc = 32 / P44_XT;
        A.gpc = gpc;
        dim3 grid((unsigned)((M + gpc - 1) / gpc), (unsigned)(A.xg ? nsets / P44_XT : nsets));
        const bool inv = A.rot_inv != 0;
#define P44_LAUNCH(SP, IV)                                                                    \
    if (A.xg) {                                                                               \
        launch_p44<KD, SP, IV, 4, true>(grid, st, A);                                         \
        return 1;                                                                             \
    }                                                                                         \
    switch (nw) {                                                                             \
    case 4: launch_p44<KD, SP, IV, 4>(grid, st, A); break;                                     \
    case 8: launch_p44<KD, SP, IV, 8>(grid, st, A); break;                                     \
    default: launch_pdl(k_pass44<KD, SP, IV, 16>, grid, 512, st, A); break;                   \
    }
        // mode 2 (shift quotients) for r = 2^a + 2^b, else the generic mode
        if (A.rc.p3_ok) {
            if (inv) {
                P44_LAUNCH(3, true)
            } else {
                P44_LAUNCH(3, false)
            }
        } else if (A.rc.p2_ok) {
            if (inv) {
                P44_LAUNCH(2, true)
            } else {
                P44_LAUNCH(2, false)
            }
        } else {
            if (inv) {
                P44_LAUNCH(0, true)
            } else {
                P44_LAUNCH(0, false)
            }
        }
#undef P44_LAUNCH
        return 1;
    }
}
