// gfp_pass.cuh -- the transform's pass kernel (k_pass) and its launcher.
//
// k_pass  one radix-K Stockham pass: coalesced digit-row loads, the
//         general twiddle (or pointwise / N^-1) multiply in registers,
//         the r^a part of the twiddle folded into the shared-memory store
//         as a digit rotation, the K-point DFT at root r (or 1/r) as
//         lazy radix-2 butterflies with one digit per lane (rotations by
//         r^t are warp shuffles + sign flips), and the store in natural
//         Stockham order.  The last pass canonicalises.
#pragma once
#include "gfp_internal.cuh"
#include "gfp_fast.cuh"
#include "gfp_pass44.cuh"
#include "gfp_pass44t.cuh"
#include "gfp_pass16t.cuh"

// k values whose pass multiply keeps the twiddle limbs in shared memory
// (fast_mul_window_store) instead of registers
#ifndef PASS_WINDOW_MINK
#define PASS_WINDOW_MINK 16
#endif
#ifndef PASS_WINDOW_MAXK
#define PASS_WINDOW_MAXK 32  // k = 32 too (200 registers, no spills: C5 FFT 0.61 -> 0.52 ms)
#endif
#define PASS_WINDOW(KD) ((KD) >= PASS_WINDOW_MINK && (KD) <= PASS_WINDOW_MAXK)
#ifndef GFP_WINDOW_CC
#define GFP_WINDOW_CC true
#endif
#ifndef PRE_WINDOW_MINK
#define PRE_WINDOW_MINK 16  // smallest k whose pointwise multiply goes through the window
                           // (k = 16: 168 -> 148 registers, C3 1% faster)
#endif
#ifndef P32_SPLIT
#define P32_SPLIT 1  // k = 32: the 64-point DFT as 8 x 8 (eight live values per lane)
#endif
#ifndef PASS32_MINB
#define PASS32_MINB 2
#endif
#ifndef PASS16_MINB
#define PASS16_MINB 3  // CTAs per SM the k = 16 pass is register-bounded for
#endif
#ifndef PASS_NOMUL_MINB
#define PASS_NOMUL_MINB 5  // the multiply-free first pass (NOMUL) for k >= 16
#endif

template <int KD>
GFP_D i64 rot_lane(i64 val, int t, int d, bool inverse)
{
    // multiply the digit vector held one-digit-per-lane by r^t (forward) or
    // r^-t (inverse), 0 < t < k: a rotation with the wrapped digits negated
    int src = inverse ? ((d + t) & (KD - 1)) : ((d - t) & (KD - 1));
    i64 v = __shfl_sync(FULL_MASK, val, src, KD);
    bool neg = inverse ? (d + t >= KD) : (d < t);
    return neg ? -v : v;
}

// one lazy normalisation of a digit held one-digit-per-lane: the quotient
// moves one lane up (negated into digit 0: r^k = -1)
template <int KD, int SPARSE>
GFP_D void normalize_lane(i64 &v, int d, const RadixConsts &rc)
{
    i64 rem;
    int q = norm_bal<SPARSE, KD>(v, rc, rem);
    int qin = __shfl_sync(FULL_MASK, q, (d - 1) & (KD - 1), KD);
    v = rem + (d == 0 ? -qin : qin);
}

// x * r^e for any 0 <= e < 2k on a digit held one-digit-per-lane
// (r^k = -1: e >= k negates)
template <int KD>
GFP_D i64 rot_lane_any(i64 val, int e, int d, bool inverse)
{
    const bool flip = (e & KD) != 0;
    const int t = e & (KD - 1);
    i64 v = t ? rot_lane<KD>(val, t, d, inverse) : val;
    return flip ? -v : v;
}

// 8-point DFT at root r^(8 s) -- s = rstep / 8 -- of digit lanes, natural
// order in and out (decimation in frequency, compile-time bit reversal)
template <int KD, int RSTEP>
GFP_D void dft8_lane(i64 (&v)[8], int d, bool inverse)
{
#pragma unroll
    for (int len = 4; len >= 1; len >>= 1) {
#pragma unroll
        for (int st = 0; st < 8; st += 2 * len) {
#pragma unroll
            for (int i = 0; i < len; i++) {
                const i64 a0 = v[st + i], b0 = v[st + i + len];
                v[st + i] = a0 + b0;
                const int e = RSTEP * i * (8 / (2 * len));  // < 2k
                v[st + i + len] = e ? rot_lane_any<KD>(a0 - b0, e, d, inverse) : a0 - b0;
            }
        }
    }
    i64 w[8];
#pragma unroll
    for (int t = 0; t < 8; t++)
        w[t] = v[t];
#pragma unroll
    for (int t = 0; t < 8; t++)
        v[((t & 1) << 2) | (t & 2) | ((t >> 2) & 1)] = w[t];
}

template <int K>
__host__ __device__ constexpr int bitrev_c(int x)
{
    int y = 0;
    for (int b = 1; b < K; b <<= 1) {
        y = (y << 1) | (x & 1);
        x >>= 1;
    }
    return y;
}

// One radix-K Stockham pass over `batch` vectors (grid.y), G = 2^lG groups
// of K elements per CTA.  Group j reads x[j + t M] (t < K), multiplies by
// omega^E, E = t (j mod Ns) (M / Ns), and writes the K-point DFT to
// (j / Ns) Ns K + (j mod Ns) + u Ns.  After log_K N passes the output is the
// natural-order DFT (the reference's dft_general result, fft.py:298-360).
//
// NOMUL: the instantiation for a pass with nothing to multiply (the first
// pass: no twiddle at Ns = 1, no pointwise operand, no N^-1) -- a pure
// HBM stream without the multiply's registers, so more CTAs per SM.
template <int KD, int SPARSE, bool NOMUL = false>
__global__ void __launch_bounds__(KD >= 16 ? 128 : 256,
                                  NOMUL && KD == 16 ? PASS_NOMUL_MINB
                                  : NOMUL && KD == 32 ? 3  /* 68 KB smem: 3 CTAs / SM */
                                  : KD == 16 ? PASS16_MINB : KD == 32 ? PASS32_MINB : 1)
    k_pass(PassArgs A)
{
    constexpr int K = 2 * KD;
    constexpr int LK = KD == 4 ? 3 : KD == 8 ? 4 : KD == 16 ? 5 : 6;
    constexpr int ROW = KD + 1;  // padded smem row (bank spread)
    extern __shared__ i64 sm[];  // [K][G][ROW]
    const int lG = A.lG;
    const int G = 1 << lG;
    const int tid = threadIdx.x;
    // grid.y covers `batch` vectors of (in, out) and then, when in2 is set,
    // `batch` more of (in2, out2): two independent transforms in one launch
    int64_t bidx = blockIdx.y;
    const u64 *in_base = A.in;
    u64 *out_base = A.out;
    if (bidx >= A.batch) {
        bidx -= A.batch;
        in_base = A.in2;
        out_base = A.out2;
    }
    const int64_t j0 = (int64_t)blockIdx.x << lG;
    const int lN = A.lN, lM = A.lM, lNs = A.lNs;
    const int64_t N = (int64_t)1 << lN, M = (int64_t)1 << lM;
    const int64_t nsmask = ((int64_t)1 << lNs) - 1;
    const u64 *in = in_base + bidx * A.batch_stride;
    u64 *out = out_base + bidx * A.batch_stride;
    const u64 *pre = A.pre ? A.pre + bidx * A.batch_stride : nullptr;
    const RadixConsts rc = A.rc;
    // programmatic dependent launch (see k_pass44)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- phase A: load K elements per group, twiddle / pointwise multiply.
    // omega^E = r^a omega^b: r^a is folded into the digit addressing of the
    // load (digit d comes from row (d - a) mod k) and the wrapped digits'
    // signs into the multiply's limb split (fast_mul_lazy negx); the product
    // digits go straight to the element's shared-memory row.
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
        const int g = tid & (G - 1);
        const int t = (tid >> lG) + h * KD;
        const int64_t j = j0 + g;
        const bool active = j < M;
        const int64_t pos = j + ((int64_t)t << lM);
        i64 x[KD];
        int64_t b = 0;
        unsigned negx = 0;
        if (active) {
            const u64 *src = in + pos;
            const unsigned rowN = 1u << lN;
            if constexpr (NOMUL) {
                // first pass (Ns = 1): E = 0, no rotation, no sign -- plain
                // digit-row loads (streamed once: evict-first)
#pragma unroll
                for (int d = 0; d < KD; d++)
                    x[d] = (i64)__ldcs(src + GFP_IDX((size_t)d * rowN, (int64_t)KD * N - pos));
            } else {
                // E = t (j mod Ns) (M / Ns) < N; omega^E = (omega^M)^a omega^b
                int64_t E = ((int64_t)t * (j & nsmask)) << (lM - lNs);
                if (A.neg_exp && E)
                    E = N - E;
                int a = (int)(E >> lM);
                b = E & (M - 1);
                // omega^M is r (or 1/r for plans built on an inverse root)
                if (A.root_inv && a)
                    a = 2 * KD - a;
                const int as = a & (KD - 1);
                negx = (unsigned)(((1ull << as) - 1ull) ^
                                  (a >= KD ? ((1ull << KD) - 1ull) : 0ull));
#pragma unroll
                for (int d = 0; d < KD; d++)
                    x[d] = (i64)__ldg(src + GFP_IDX((size_t)((unsigned)((d - as) & (KD - 1)) * rowN),
                                                    (int64_t)KD * N - pos));
            }
            if (A.in_canon)  // pass 0 only, where a = 0
                to_balanced<KD>(x, rc.r);
            if (!NOMUL && pre) {  // pass 0 only (a = b = 0)
                if constexpr (KD >= PRE_WINDOW_MINK && PASS_WINDOW(KD)) {
                    // through the window (registers: x only), product parked in
                    // the element's row and read back
                    constexpr int S = FastSplit<KD>::S;
                    unsigned long long *yw =
                        reinterpret_cast<unsigned long long *>(sm + ((size_t)K << lG) * ROW) + tid;
                    const int nt = (int)blockDim.x;
#pragma unroll
                    for (int d = 0; d < KD; d++) {
                        int l, h;
                        split_limbs<S>((i64)__ldg(pre + GFP_IDX(((int64_t)d << lN) + pos,
                                                                (int64_t)KD << lN)), l, h);
                        yw[d * nt] = (u64)(unsigned)l | ((u64)(unsigned)h << 32);
                    }
                    i64 *prow = sm + (((int64_t)t << lG) + g) * ROW;
                    fast_mul_window_store<KD, SPARSE, GFP_WINDOW_CC>(
                        x, 0u, reinterpret_cast<const int2 *>(yw), nt, prow, rc);
#pragma unroll
                    for (int d = 0; d < KD; d++)
                        x[d] = prow[d];
                } else {
                    i64 y[KD];
#pragma unroll
                    for (int d = 0; d < KD; d++)
                        y[d] = (i64)__ldg(pre + GFP_IDX(((int64_t)d << lN) + pos, (int64_t)KD << lN));
                    fast_mul_lazy<KD, SPARSE>(x, y, x, rc);
                }
            }
        } else {
#pragma unroll
            for (int d = 0; d < KD; d++)
                x[d] = 0;
        }
        i64 *row = sm + (((int64_t)t << lG) + g) * ROW;
        // warp-uniform multiply: lanes with b = 0 multiply by table[0] = 1
        if (!NOMUL && __any_sync(FULL_MASK, active && (b || A.scale))) {
            if (active) {
                const ulonglong2 *tp =
                    reinterpret_cast<const ulonglong2 *>(A.table_lh + GFP_IDX(b, M) * KD);
                if (PASS_WINDOW(KD)) {
                    // twiddle limbs staged in this thread's smem column,
                    // multiplied through the sliding window (registers: x only)
                    // (a limb pair l | h << 32 is the int2 {l, h} bit for bit)
                    unsigned long long *yw =
                        reinterpret_cast<unsigned long long *>(sm + ((size_t)K << lG) * ROW) + tid;
                    const int nt = (int)blockDim.x;
#pragma unroll
                    for (int d = 0; d < KD; d += 2) {
                        const ulonglong2 w = __ldg(tp + d / 2);
                        yw[d * nt] = w.x;
                        yw[(d + 1) * nt] = w.y;
                    }
                    fast_mul_window_store<KD, SPARSE, GFP_WINDOW_CC>(
                        x, negx, reinterpret_cast<const int2 *>(yw), nt, row, rc);
                } else {
                    u64 ylh[KD];
#pragma unroll
                    for (int d = 0; d < KD; d += 2) {
                        const ulonglong2 w = __ldg(tp + d / 2);
                        ylh[d] = w.x;
                        ylh[d + 1] = w.y;
                    }
                    i64 f[KD];
                    fast_mul_lazy_ylimbs<KD, SPARSE, true>(x, ylh, f, rc, negx, row);
                }
            } else {
#pragma unroll
                for (int d = 0; d < KD; d++)
                    row[d] = 0;
            }
        } else if (NOMUL) {
#pragma unroll
            for (int d = 0; d < KD; d++)
                row[d] = x[d];
        } else {
#pragma unroll
            for (int d = 0; d < KD; d++)
                row[d] = ((negx >> d) & 1u) ? -x[d] : x[d];
        }
    }
    GFP_JITTER(1);
    __syncthreads();

    // ---- phase B: K-point DFT at root r (or 1/r), one digit per lane
    if constexpr (KD == 32 && P32_SPLIT && SPARSE == 3) {  // mode 3: S = 6 (p3_ok)
        // K = 64 = 8 x 8 (t = t1 + 8 t2, u = u0 + 8 u1): 8-point DFTs over t2
        // in place, the factor rho^(t1 u0) (a lane rotation), 8-point DFTs
        // over t1 with X[u0 + 8 u1] left in slot u1 + 8 u0 (the slots this
        // step read); eight values per lane live at a time instead of 64.
        // One warp owns a group's slots: warp barriers only.
        const int d = tid & (KD - 1);
        const int g = tid / KD;
        const bool inv = A.rot_inv != 0;
        i64 *gs = sm + (int64_t)g * ROW + d;  // slot t at gs[(t << lG) * ROW]
#pragma unroll 1
        for (int t1 = 0; t1 < 8; t1++) {
            i64 v[8];
#pragma unroll
            for (int t2 = 0; t2 < 8; t2++)
                v[t2] = gs[((int64_t)(t1 + 8 * t2) << lG) * ROW];
            dft8_lane<KD, 8>(v, d, inv);
#pragma unroll
            for (int u0 = 0; u0 < 8; u0++)
                gs[((int64_t)(t1 + 8 * u0) << lG) * ROW] = v[u0];
        }
        __syncwarp();
#pragma unroll 1
        for (int u0 = 0; u0 < 8; u0++) {
            i64 v[8];
#pragma unroll
            for (int t1 = 0; t1 < 8; t1++) {
                const i64 y = gs[((int64_t)(t1 + 8 * u0) << lG) * ROW];
                v[t1] = t1 ? rot_lane_any<KD>(y, (t1 * u0) & (2 * KD - 1), d, inv) : y;
            }
            dft8_lane<KD, 8>(v, d, inv);
#pragma unroll
            for (int u1 = 0; u1 < 8; u1++) {
                normalize_lane<KD, SPARSE>(v[u1], d, rc);
                gs[((int64_t)(u1 + 8 * u0) << lG) * ROW] = v[u1];
            }
        }
    } else {
        const int d = tid & (KD - 1);
        const int g = tid / KD;
        const bool inv = A.rot_inv != 0;
        i64 v[K];
#pragma unroll
        for (int t = 0; t < K; t++)
            v[t] = sm[GFP_IDX((((int64_t)t << lG) + g) * ROW + d, ((int64_t)K << lG) * ROW)];
        const int S = rc.stages_per_norm;
        int stage = 0;
#pragma unroll
        for (int len = K / 2; len >= 1; len >>= 1) {
#pragma unroll
            for (int st = 0; st < K; st += 2 * len) {
#pragma unroll
                for (int i = 0; i < len; i++) {
                    i64 a0 = v[st + i], b0 = v[st + i + len];
                    v[st + i] = a0 + b0;
                    i64 df = a0 - b0;
                    const int tw = i * (K / (2 * len));  // exponent of the root, < k
                    v[st + i + len] = tw ? rot_lane<KD>(df, tw, d, inv) : df;
                }
            }
            stage++;
            if (len > 1 && stage % S == 0) {
#pragma unroll
                for (int t = 0; t < K; t++)
                    normalize_lane<KD, SPARSE>(v[t], d, rc);
            }
        }
#pragma unroll
        for (int t = 0; t < K; t++)
            normalize_lane<KD, SPARSE>(v[t], d, rc);
        __syncthreads();
#pragma unroll
        for (int t = 0; t < K; t++)
            sm[GFP_IDX((((int64_t)bitrev_c<K>(t) << lG) + g) * ROW + d,
                       ((int64_t)K << lG) * ROW)] = v[t];
    }
    GFP_JITTER(2);
    __syncthreads();

    // ---- phase C: store in Stockham order (canonicalise on the last pass)
    // (the k = 32 split DFT leaves X[u0 + 8 u1] in slot u1 + 8 u0).  On the
    // first pass (Ns = 1) output u of group j goes to K j + u: lanes take
    // consecutive u there, so each digit row is written in contiguous runs of
    // K words (else lanes take consecutive groups: contiguous for Ns >= G)
    const bool ufast = lNs == 0;
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
        const int idx = tid + h * (G * KD);  // (g, u) pair over both iterations: G K outputs
        const int g = ufast ? idx >> LK : tid & (G - 1);
        const int u = ufast ? idx & (K - 1) : (tid >> lG) + h * KD;
        const int64_t j = j0 + g;
        if (j >= M)
            continue;
        const int64_t pos = ((j >> lNs) << (lNs + LK)) + (j & nsmask) + ((int64_t)u << lNs);
        const int us = (KD == 32 && P32_SPLIT && SPARSE == 3) ? ((u >> 3) | ((u & 7) << 3)) : u;
        const i64 *row = sm + (((int64_t)us << lG) + g) * ROW;
        if (A.canon) {
            i64 f[KD];
            u64 c[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                f[d] = row[d];
            lazy_to_canonical_bf<KD>(f, c, rc);  // balanced digits (phase B)
#pragma unroll
            for (int d = 0; d < KD; d++)
                out[GFP_IDX(((int64_t)d << lN) + pos, (int64_t)KD << lN)] = c[d];
        } else {
#pragma unroll
            for (int d = 0; d < KD; d++)
                out[GFP_IDX(((int64_t)d << lN) + pos, (int64_t)KD << lN)] = (u64)row[d];
        }
    }
}

static int pass_threads(int k, int64_t M, int *G_out)
{
    // groups per CTA: as many as fit 256 threads (128 for k >= 16, whose
    // multiply needs ~170 registers), fewer when the transform is too small
    // to give every SM two CTAs
    int Gmax = (k >= 16 ? 128 : 256) / k;
    int Gmin = 32 / k > 0 ? 32 / k : 1;
    int G = Gmax;
    while (G > Gmin && (M + G - 1) / G < 2 * (int64_t)num_sms())
        G >>= 1;
    *G_out = G;
    return G * k;
}

template <int KD>
static size_t pass_smem(int G, bool nomul = false)
{
    // [K][G][k + 1] element rows, plus the window multiply's y-limb columns
    // (k int2 per thread, G k threads) when it is on for this k
    return (size_t)(2 * KD) * G * (KD + 1) * sizeof(i64) +
           (PASS_WINDOW(KD) && !nomul ? (size_t)KD * G * KD * sizeof(int2) : 0);
}

// the pass-kernel arguments shared by k_pass and k_pass44
static inline int make_pass_args(const gfp_fft_plan *p, const u64 *in, u64 *out, const u64 *in2,
                                 u64 *out2, const u64 *pre, int64_t batch, int64_t Ns,
                                 int inverse, int scale, int canon, int in_canon,
                                 const PassIO *em, int G, PassArgs &A)
{
    A.gpc = 32;
    A.in = in;
    A.out = out;
    A.table = scale ? p->table_ninv : p->table;
    A.table_lh = scale ? p->table_ninv_lh : p->table_lh;
    A.pre = pre;
    A.batch_stride = (int64_t)p->k * p->N;
    A.lN = ilog2_exact(p->N);
    A.lM = ilog2_exact(p->M);
    A.lNs = ilog2_exact(Ns);
    A.lG = ilog2_exact(G);
    A.neg_exp = inverse;
    A.rot_inv = inverse ^ p->root_inv;
    A.root_inv = p->root_inv;
    A.scale = scale;
    A.canon = canon;
    A.in_canon = in_canon;
    A.rc = p->rc;
    A.in2 = in2;
    A.out2 = out2;
    A.batch = batch;
    A.in_em = A.in2_em = nullptr;
    A.out_em = nullptr;
    A.n_in = A.n_in2 = A.n_out = 0;
    A.ft_lh = nullptr;
    A.ft_lN = A.ft_lM = A.ft_inv = A.ft_root_inv = 0;
    A.ft_row0 = 0;
    A.xg = A.xrank = A.lxb = 0;
    A.xA = 0;
    for (int g = 0; g < 8; g++)
        A.xdst[g] = nullptr;
    if (em) {
        if (Ns == 1 && em->ft && (scale || in_canon))
            return GFP_EUNSUPPORTED;  // first pass with N^-1 or canonical input
        if (Ns == 1 && em->ft) {
            A.ft_lh = em->ft->table_lh;
            A.ft_lN = ilog2_exact(em->ft->N);
            A.ft_lM = ilog2_exact(em->ft->M);
            A.ft_inv = em->ft_inv;
            A.ft_root_inv = em->ft->root_inv;
            A.ft_row0 = em->ft_row0;
        }
        if (Ns == 1 && em->in) {
            A.in_em = em->in;
            A.in2_em = em->in2;
            A.n_in = em->n_in;
            A.n_in2 = em->n_in2;
        }
        if (canon && em->out) {
            A.out_em = em->out;
            A.n_out = em->n_out;
        }
        if (em->xg && Ns * p->K == p->N) {  // last pass: stores go to the exchange
            if (Ns == 1 || em->xg > 8 || (em->xg & (em->xg - 1)) || batch % 8 || in2 || pre)
                return GFP_EUNSUPPORTED;
            A.xg = em->xg;
            A.xrank = em->xrank;
            A.lxb = ilog2_exact(p->N / em->xg);
            A.xA = batch;
            for (int g = 0; g < em->xg; g++)
                A.xdst[g] = em->xdst[g];
        }
    }
    return GFP_OK;
}

template <int KD>
int launch_pass(const gfp_fft_plan *p, const u64 *in, u64 *out, const u64 *in2,
                       u64 *out2, const u64 *pre, int64_t batch, int64_t Ns, int inverse,
                       int scale, int canon, int in_canon, const PassIO *em, cudaStream_t st)
{
    int G;
    int threads = pass_threads(KD, p->M, &G);
    size_t smem = pass_smem<KD>(G);
    static unsigned long long attr_set = 0;  // per device
    once_per_device(attr_set, [&] {
        for (int m = 0; m < 3; m++) {
            const void *fn = m == 0 ? (const void *)k_pass<KD, 0>
                             : m == 1 ? (const void *)k_pass<KD, 1> : (const void *)k_pass<KD, 2>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pass_smem<KD>(256 / KD));
        }
        if constexpr (P2Radix<KD>::a != 0) {
            cudaFuncSetAttribute((const void *)k_pass<KD, 3>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pass_smem<KD>(256 / KD));
            cudaFuncSetAttribute((const void *)k_pass<KD, 3, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pass_smem<KD>(256 / KD, true));
        }
    });
    if ((in2 ? 2 : 1) * batch > GFP_MAX_GRID_Y)  // the batch is grid.y (callers chunk)
        return GFP_EINVAL;
    PassArgs A;
    int err = make_pass_args(p, in, out, in2, out2, pre, batch, Ns, inverse, scale, canon, in_canon,
                             em, G, A);
    if (err)
        return err;
    // large k = 8 transforms: the TMA form of the pass for every pass it takes
    if (pass44_enabled(KD, A.rc) &&
        p44t_takes(A, p->M) &&
        launch_pass44t<KD>(A, p->M, in2 ? 2 * batch : batch, st))
        return cuda_status();
    if (launch_pass44<KD>(A, p->M, in2 ? 2 * batch : batch, st))
        return cuda_status();
    if (A.in_em || A.out_em || A.ft_lh || A.xg)
        return GFP_EUNSUPPORTED;
    if constexpr (KD == 16) {  // the multiply-free first pass on TMA tiles
        if (p16t_takes(A, p->M) && launch_first16t(A, p->M, in2 ? 2 * batch : batch, st))
            return cuda_status();
    }
    dim3 grid((unsigned)((p->M + G - 1) / G), (unsigned)(in2 ? 2 * batch : batch));
    if constexpr (P2Radix<KD>::a != 0) {
        if (p->rc.p3_ok) {
            if (Ns == 1 && !pre && !scale)  // nothing to multiply in this pass
                launch_pdl(k_pass<KD, 3, true>, grid, threads, st, A, pass_smem<KD>(G, true));
            else
                launch_pdl(k_pass<KD, 3>, grid, threads, st, A, smem);
            return cuda_status();
        }
    }
    if (p->rc.p2_ok) {
        launch_pdl(k_pass<KD, 2>, grid, threads, st, A, smem);
    } else if (p->rc.sp_on) {
        launch_pdl(k_pass<KD, 1>, grid, threads, st, A, smem);
    } else {
        launch_pdl(k_pass<KD, 0>, grid, threads, st, A, smem);
    }
    return cuda_status();
}
