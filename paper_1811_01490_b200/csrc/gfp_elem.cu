// gfp_elem.cu -- element-wise kernels (thread per element, any power-of-two
// k <= 128, any r), the radix constants and the element-wise C-ABI.
//
//   k_add / k_sub / k_mul_pow_r  restate gfp_field.py:82-161 digit loops;
//   k_mul / k_pow                exact generic multiply (gfp_generic.cuh);
//   k_mul_fast                   limb-split IMAD.WIDE multiply when eligible.
#include "gfp_internal.cuh"
#include "gfp_fast.cuh"
#include "gfp_generic.cuh"
#include "gfp_mulw.cuh"

// ===========================================================================
// host-side constants
// ===========================================================================

int ilog2_exact(int64_t v)
{
    int l = 0;
    while (((int64_t)1 << l) < v)
        l++;
    return ((int64_t)1 << l) == v ? l : -1;
}

bool valid_k(int k) { return k >= 1 && k <= 128 && (k & (k - 1)) == 0; }

static int fast_split_for(int k) { return k <= 16 ? 29 : 28; }  // FastSplit<KD>::S

struct FastPlan {
    int S;        // lazy radix-2 stages between normalisations
    int sp_on;    // sparse-radix normalisation (r = 2^a + eps, |eps| small)
    int sp_a;
    i64 sp_eps;
    u128 delta;   // balanced lazy digits stay in [-r/2 - delta, r/2 + delta]
};

// balanced normaliser (norm_bal) on |v| <= V: the quotient bound and the
// excess it leaves over [-r/2, r/2]
static void norm_bounds(u128 V, u64 r, const FastPlan &fp, u128 *qmax, u128 *ex)
{
    if (fp.sp_on) {
        u128 q = ((V + ((u128)1 << (fp.sp_a - 1))) >> fp.sp_a) + 1;
        u128 e = (u128)(fp.sp_eps < 0 ? -fp.sp_eps : fp.sp_eps);
        *qmax = q;
        *ex = q * (e + 1) + e / 2 + 2;
    } else {
        u128 q = V / r + 2;
        *qmax = q;
        *ex = q + 2;
    }
}

// Fast-path bound check, exact integer arithmetic.  Returns true and fills
// `fp` when every bound of fast_mul_lazy (gfp_fast.cuh) and of the lazy
// butterflies (k_pass) holds for balanced digits |d| <= X = r/2 + delta:
//   * 2^S X + 2^a < 2^63 (S unnormalised radix-2 stages, then norm_bal);
//   * the sub-column sums LL, SS, HH (and MID = SS - LL - HH,
//     MID + (LL >> s)) of the balanced-limb product stay below 2^63;
//   * k X^2 < 2^63 r (the biased column c + 2^63 r is in [0, 2^64 r));
//   * the carry rounds stay within 2^63 and land back inside delta.
static bool fast_bounds(int k, u64 r, FastPlan *out)
{
    if (!(k == 4 || k == 8 || k == 16 || k == 32))
        return false;
    if (r < ((u64)1 << 24) || r >= ((u64)1 << 62) || (r & (r - 1)) == 0)
        return false;
    const u128 two63 = (u128)1 << 63;
    const int K = 2 * k;
    const int logK = ilog2_exact(K);
    const u128 kk = (u128)k;
    FastPlan fp;
    memset(&fp, 0, sizeof(fp));
    // sparse radix: r = 2^a + eps with 2^a the nearest power of two
    int w = 64 - __builtin_clzll(r);
    u64 lo_p = (u64)1 << (w - 1);
    u64 hi_p = (u64)1 << w;
    if (r - lo_p <= hi_p - r) {
        fp.sp_a = w - 1;
        fp.sp_eps = (i64)(r - lo_p);
    } else {
        fp.sp_a = w;
        fp.sp_eps = -(i64)(hi_p - r);
    }
    i64 aeps = fp.sp_eps < 0 ? -fp.sp_eps : fp.sp_eps;
    fp.sp_on = aeps < ((i64)1 << 30) && fp.sp_a >= 40 && (aeps << 20) < ((i64)1 << fp.sp_a);
    const int s = fast_split_for(k);
    // column_quot's shifts: 2s - w and w - 2s must stay below 29
    if (w + 28 < 2 * s || w > 2 * s + 28)
        return false;
    const u128 half = (u128)1 << (s - 1);
    const u128 top = (u128)1 << (fp.sp_on ? fp.sp_a : w);
    u128 delta = 2;  // canonical inputs enter through to_balanced (excess <= 1)
    for (int iter = 0; iter < 16; iter++) {
        u128 X = (u128)(r / 2) + delta;
        int S = 0;
        for (int t = 1; t <= logK; t++)
            if ((X << t) + top < two63)
                S = t;
        if (S < 1)
            return false;
        fp.S = S;
        u128 q1, ex1;
        // the digits entering the S lazy stages: normalised ones, or -- mode 3
        // with the rounding column quotient (k <= GFP_SEQ_MAXK, gfp_fast.cuh) -- products
        // of magnitude up to 3r/4
        u128 Vn = X << S;
        if (k <= GFP_SEQ_MAXK && r == p2_radix_of(k)) {
            const u128 Xm = 3 * ((u128)r / 4) + 16;
            if ((Xm << S) + top >= two63)
                return false;
            if ((Xm << S) > Vn)
                Vn = Xm << S;
        }
        norm_bounds(Vn, r, fp, &q1, &ex1);
        // multiply: balanced limbs, |xl| <= 2^(s-1), |xh| <= H, |xs| <= 2^(s-1) + H
        u128 H = (X + half) >> s;
        u128 Hs = half + H;
        if (Hs >= ((u128)1 << 31))
            return false;
        if (kk * half * half >= two63 || kk * H * H >= two63 || kk * Hs * Hs >= two63)
            return false;
        if (2 * kk * half * H + kk * half * half / ((u128)1 << s) + 2 >= two63)
            return false;
        if (w < 2 * s && ((kk * H * H) << (2 * s - w)) >= two63)
            return false;
        u128 XX = X * X;
        if (XX / r * kk + kk + 8 >= two63)
            return false;
        u128 Q1 = XX / r * kk + kk + 8;  // |column quotient|
        u128 E = 4 * (u128)r + Q1;       // |rem + carry| after round 1
        if (E + top >= two63)
            return false;
        u128 q2, ex2;
        norm_bounds(E, r, fp, &q2, &ex2);
        u128 need = ex1 > ex2 ? ex1 : ex2;
        if (need <= delta)
            break;
        delta = need;
        if (iter == 15)
            return false;
    }
    if (delta * 8 >= r)
        return false;
    fp.delta = delta;
    *out = fp;
    return true;
}

RadixConsts make_consts(int k, u64 r)
{
    RadixConsts c;
    memset(&c, 0, sizeof(c));
    c.r = r;
    c.sh = __builtin_clzll(r);
    c.d_norm = r << c.sh;
    u128 all = ~(u128)0;
    u128 v = all / c.d_norm;
    c.v_recip = (u64)(v - ((u128)1 << 64));
    u128 bias = (u128)r << 63;
    c.bias_lo = (u64)bias;
    c.bias_hi = (u64)(bias >> 64);
    c.rinv = 1.0 / (double)r;
    c.neg_one = -1;
    c.w = 64 - c.sh;
    if (c.w < 64) {
        u128 m = ((u128)1 << (64 + c.w)) / r;
        c.m_recip = (u64)(m - ((u128)1 << 64));
    }
    FastPlan fp;
    if (fast_bounds(k, r, &fp)) {
        c.s = fast_split_for(k);
        c.stages_per_norm = fp.S;
        c.sp_on = fp.sp_on;
        c.sp_a = fp.sp_a;
        c.sp_eps = (int)fp.sp_eps;
        c.sp_mask = ((i64)1 << fp.sp_a) - 1;
        c.sp_half = (i64)1 << (fp.sp_a - 1);
        c.q_sh1 = c.w > 2 * c.s ? c.w - 2 * c.s : 0;
        c.q_sh2 = c.w < 2 * c.s ? 2 * c.s - c.w : 0;
        c.bias_t = r << (63 - c.w);
        // mode 2: r = 2^a + 2^b, quotients by shifts (gfp_fast.cuh column_quot_p2)
        const int a = fp.sp_a, S = c.s;
        const i64 eps = fp.sp_eps;
        if (fp.sp_on && eps > 0 && (eps & (eps - 1)) == 0 && a >= 2 * S && a - 2 * S < 32) {
            const int b = __builtin_ctzll((u64)eps);
            const u128 X = (u128)(r / 2) + fp.delta;
            const u128 two62r = (u128)r << 62;
            // |c| <= k X^2 < 2^62 r keeps c + 2^62 r in [0, 2^63 r): T < 2^64
            if (62 + b - a >= 0 && (u128)k * X * X < two62r) {
                c.p2_ok = 1;
                c.p2_b = b;
                c.p2_sh = a - 2 * S;
                c.p2_ab = a - b;
                c.p2_bias_t = ((u64)1 << 62) + ((u64)1 << (62 + b - a));
                c.p2_bias_lo = (u64)two62r;
            }
        }
        // mode 3 (ColReduce): column c_m + C_{m-1} with the running carry
        // |C| <= k X^2 / r + small folded into LL before the signed quotient
        if (c.p2_ok && r == p2_radix_of(k)) {
            const int b = c.p2_b;
            const u128 two63 = (u128)1 << 63;
            const u128 X = (u128)(r / 2) + fp.delta;
            const u128 half = (u128)1 << (S - 1);
            const u128 H = (X + half) >> S;
            const u128 kk = (u128)k;
            const u128 cmax = kk * X * X / r + (kk * X * X / r >> 30) + 16;
            const u128 cabs = kk * X * X + cmax;
            const int e2 = a + 2 * (a - b) - 8;  // second-order term < 1/256
            bool ok = kk * half * half + cmax < two63 &&
                      2 * kk * half * H + (kk * half * half + cmax) / ((u128)1 << S) + 2 < two63 &&
                      (cabs >> (2 * S)) < (two63 >> 1) && (cabs >> a) < ((u128)1 << 62) &&
                      (e2 >= 127 || cabs < ((u128)1 << e2));
            // digit bounds: m >= 2 from norm_bal(rem), rem in (-r/100, 2.01 r);
            // digit 0 from norm_bal(d_0 - C); digit 1 gets digit 0's carry
            u128 q2, ex2, q0, ex0;
            norm_bounds(3 * (u128)r, r, fp, &q2, &ex2);
            norm_bounds(X + cmax, r, fp, &q0, &ex0);
            ok = ok && ex0 <= fp.delta && ex2 + q0 <= fp.delta;
            // k <= GFP_SEQ_MAXK: the rounding column quotient (column_quot_p3r).  A multiply's
            // x operand is a normalised digit vector or an earlier product
            // (|x| <= Xm = 3r/4 + 16), its y operand a table entry or a
            // normalised vector (|y| <= X)
            if (k <= GFP_SEQ_MAXK && ok) {
                const u128 Xm = 3 * ((u128)r / 4) + 16;
                const u128 Hx = (Xm + half) >> S, Hy = (X + half) >> S;
                const u128 cr = kk * Xm * X / r + 16;                  // |carry|
                const u128 llc = kk * half * half + cr;                // |LL + C|
                const u128 mid = kk * half * (Hx + Hy) + (llc >> S) + 2;  // |MID + (LL >> S)|
                const u128 cabs2 = kk * Xm * X + cr;
                const int e2r = a - 2 + 2 * (a - b) - 8;
                ok = 2 * S >= a - 2 && a - 2 >= S && llc < two63 &&
                     kk * (half + Hx) * (half + Hy) < two63 &&          // SS, SS - SSn
                     mid < two63 &&
                     ((kk * Hx * Hy) << (2 * S - (a - 2))) + (mid >> (a - 2 - S)) + 4 < two63 &&  // T4, q4 + 2
                     (e2r >= 127 || (cabs2 >> e2r) == 0) &&             // second-order term < 1/256
                     Xm + cr + ((u128)1 << (a - 1)) < two63 &&          // digit 0: norm_bal(d_0 - C)
                     (Xm << fp.S) + ((u128)1 << (a - 1)) < two63;       // lazy stages + normalize_el
                // digit 0 comes out of norm_bal (balanced, within delta); digit 1
                // gets its carry on top of a product digit
                u128 q0r, ex0r;
                norm_bounds(Xm + cr, r, fp, &q0r, &ex0r);
                ok = ok && ex0r <= fp.delta && q0r + 3 * ((u128)r / 4) + 2 <= Xm;
            }
            // the k = 32 mode-3 pass runs its 64-point DFT without a mid normalisation
            ok = ok && (k != 32 || fp.S >= 6);
            c.p3_ok = ok ? 1 : 0;
        }
    } else {
        c.s = 0;
        c.stages_per_norm = 0;
    }
    return c;
}

bool fast_path_bounds_ok(int k, u64 r)
{
    FastPlan fp;
    return fast_bounds(k, r, &fp);
}

// ===========================================================================
// element-wise kernels (grid-stride, thread per element)
// ===========================================================================

template <int KD>
__global__ void k_add(const u64 *__restrict__ x, const u64 *__restrict__ y, u64 *__restrict__ z,
                      int64_t n, u64 r, int sub)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], b[KD], c[KD];
#pragma unroll
        for (int d = 0; d < KD; d++) {
            a[d] = x[d * n + i];
            b[d] = y[d * n + i];
        }
        if (sub)
            dev_gfp_sub(a, b, c, KD, r);
        else
            dev_gfp_add(a, b, c, KD, r);
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

// gfp_mul_pow_r (gfp_field.py:138-161): i >= k negates first, then
// B - A with B the up-shifted digits, A the wrapped top digits; a form-B
// digit r moves one slot up.
template <int KD>
__global__ void k_mul_pow_r(const u64 *__restrict__ x, u64 *__restrict__ z, int64_t n, u64 r,
                            int shift)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            a[d] = x[d * n + i];
        dev_mul_pow_r<KD>(a, shift, r);
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[d * n + i] = a[d];
    }
}

template <int KD>
__global__ void k_mul_generic(const u64 *__restrict__ x, const u64 *__restrict__ y, int64_t y_inc,
                              u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    int64_t yn = y_inc ? n : 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], b[KD], c[KD];
        int64_t iy = y_inc ? i : 0;
        for (int d = 0; d < KD; d++) {
            a[d] = x[d * n + i];
            b[d] = y[d * yn + iy];
        }
        gfp_mul_generic<KD>(a, b, c, rc);
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

template <int KD, int SPARSE>
__global__ void k_mul_fast(const u64 *__restrict__ x, const u64 *__restrict__ y, int64_t y_inc,
                           u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    int64_t yn = y_inc ? n : 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        i64 a[KD], b[KD], f[KD];
        u64 c[KD];
        int64_t iy = y_inc ? i : 0;
#pragma unroll
        for (int d = 0; d < KD; d++) {
            a[d] = (i64)x[d * n + i];
            b[d] = (i64)y[d * yn + iy];
        }
        to_balanced<KD>(a, rc.r);
        to_balanced<KD>(b, rc.r);
        fast_mul_lazy<KD, SPARSE>(a, b, f, rc);
        lazy_to_canonical(f, c, KD, rc);
#pragma unroll
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

template <int KD>
__global__ void k_pow(const u64 *__restrict__ x, const u64 *__restrict__ e, int nbits,
                      u64 *__restrict__ z, int64_t n, RadixConsts rc)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], c[KD];
        for (int d = 0; d < KD; d++)
            a[d] = x[d * n + i];
        gfp_pow_generic<KD>(a, e, nbits, c, rc);
        for (int d = 0; d < KD; d++)
            z[d * n + i] = c[d];
    }
}

__global__ void k_is_canonical(const u64 *__restrict__ x, uint8_t *__restrict__ out, int64_t n,
                               int k, u64 r)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        bool all = true, lowzero = true;
        for (int d = 0; d < k; d++) {
            u64 v = x[d * n + i];
            if (v >= r)
                all = false;
            if (d < k - 1 && v)
                lowzero = false;
        }
        out[i] = (all || (lowzero && x[(int64_t)(k - 1) * n + i] == r)) ? 1 : 0;
    }
}

GFP_D u64 splitmix64(u64 z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void k_uniform(u64 *__restrict__ z, int64_t n, int k, u64 r, u64 seed)
{
    int64_t total = n * k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        u64 h = splitmix64(seed * 0x2545F4914F6CDD1DULL + (u64)t);
        z[t] = __umul64hi(h, r);  // uniform in [0, r)
    }
}

// element-major [n][k] -> digit-major [k][n] (dir = 0) or back (dir = 1)
__global__ void k_transpose(const u64 *__restrict__ src, u64 *__restrict__ dst, int64_t n, int k,
                            int dir)
{
    int64_t total = n * k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        // t indexes the destination linearly for coalesced stores
        if (dir == 0) {
            int64_t d = t / n, i = t % n;
            dst[t] = src[i * k + d];
        } else {
            int64_t i = t / k, d = t % k;
            dst[t] = src[d * n + i];
        }
    }
}

// Batched, tiled layout conversion between element-major [B][n_em][k] and
// digit-major [B][k][n_dm] (the host entry points' staging): a CTA moves
// tiles of 32 elements x k digits through shared memory, so both the
// element-major side (32 k contiguous words) and every digit row (32
// contiguous words) are accessed coalesced.  to_dm: element-major -> digit-
// major, elements i >= n_em written as 0 (zero padding to the transform
// length); otherwise digit-major -> element-major for i < n_em (truncation
// to the product length).  n_dm >= n_em.
template <int KD>
__global__ void __launch_bounds__(256) k_transpose_tiles(const u64 *__restrict__ src,
                                                         u64 *__restrict__ dst, int64_t batch,
                                                         int64_t n_em, int64_t n_dm, int to_dm)
{
    __shared__ u64 tile[32 * (KD + 1)];
    const int64_t tiles_per = (n_dm + 31) / 32;
    const int64_t ntiles = batch * tiles_per;
    for (int64_t tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
        const int64_t b = tt / tiles_per;
        const int64_t i0 = (tt - b * tiles_per) * 32;
        if (!to_dm && i0 >= n_em)
            continue;
        const u64 *s_em = src + b * n_em * KD;  // element-major side (to_dm)
        const u64 *s_dm = src + b * n_dm * KD;  // digit-major side (!to_dm)
        u64 *d_em = dst + b * n_em * KD;
        u64 *d_dm = dst + b * n_dm * KD;
        __syncthreads();
        for (int w = threadIdx.x; w < 32 * KD; w += blockDim.x) {
            if (to_dm) {  // w = e k + d over the 32 elements' contiguous words
                const int e = w / KD, d = w % KD;
                tile[e * (KD + 1) + d] = i0 + e < n_em ? s_em[(i0 + e) * KD + d] : 0;
            } else {      // w = d 32 + e: digit rows
                const int d = w / 32, e = w % 32;
                tile[e * (KD + 1) + d] = i0 + e < n_dm ? s_dm[(int64_t)d * n_dm + i0 + e] : 0;
            }
        }
        __syncthreads();
        for (int w = threadIdx.x; w < 32 * KD; w += blockDim.x) {
            if (to_dm) {
                const int d = w / 32, e = w % 32;
                if (i0 + e < n_dm)
                    d_dm[(int64_t)d * n_dm + i0 + e] = tile[e * (KD + 1) + d];
            } else {
                const int e = w / KD, d = w % KD;
                if (i0 + e < n_em)
                    d_em[(i0 + e) * KD + d] = tile[e * (KD + 1) + d];
            }
        }
    }
}

int transpose_batched(const u64 *src, u64 *dst, int64_t batch, int64_t n_em, int64_t n_dm, int k,
                      int to_dm, cudaStream_t st)
{
    if (batch <= 0 || n_dm <= 0)
        return GFP_OK;
    const int64_t tiles = batch * ((n_dm + 31) / 32);
    const int64_t cap = (int64_t)num_sms() * 8;
    const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
    DISPATCH_K(k, (k_transpose_tiles<KD><<<grid, 256, 0, st>>>(src, dst, batch, n_em, n_dm, to_dm)));
    return cuda_status();
}

int host_pipe_begin(HostPipe &hp, cudaStream_t caller)
{
    if (cudaEventCreateWithFlags(&hp.ev, cudaEventDisableTiming) != cudaSuccess)
        return GFP_ECUDA;
    cudaEventRecord(hp.ev, caller);
    for (int i = 0; i < 2; i++) {
        if (cudaStreamCreateWithFlags(&hp.s[i], cudaStreamNonBlocking) != cudaSuccess)
            return GFP_ECUDA;
        cudaStreamWaitEvent(hp.s[i], hp.ev, 0);
    }
    return cuda_status();
}

int host_pipe_end(HostPipe &hp, cudaStream_t caller)
{
    for (int i = 0; i < 2; i++) {
        if (!hp.s[i])
            continue;
        cudaEventRecord(hp.ev, hp.s[i]);
        cudaStreamWaitEvent(caller, hp.ev, 0);
        cudaStreamDestroy(hp.s[i]);  // released once its queued work completes
        hp.s[i] = nullptr;
    }
    if (hp.ev)
        cudaEventDestroy(hp.ev);
    hp.ev = nullptr;
    return cuda_status();
}

static int g_num_sms[64];  // per device id (0 = not queried yet)

int num_sms()
{
    int dev = 0;
    cudaGetDevice(&dev);
    int &n = g_num_sms[dev & 63];
    if (!n) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n = v > 0 ? v : 148;
    }
    return n;
}

dim3 grid_for(int64_t work, int threads)
{
    int64_t blocks = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * 32;
    if (blocks > cap)
        blocks = cap;
    if (blocks < 1)
        blocks = 1;
    return dim3((unsigned)blocks);
}

int cuda_status()
{
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GFP_OK : GFP_ECUDA;
}


extern "C" {

const char *gfp_strerror(int code)
{
    switch (code) {
    case GFP_OK: return "ok";
    case GFP_EINVAL: return "invalid argument";
    case GFP_ECONFIG: return "configuration not supported by the prime pair";
    case GFP_ECUDA: return "CUDA runtime error";
    case GFP_ENOMEM: return "device allocation failed";
    case GFP_EUNSUPPORTED: return "parameters outside the transform kernels' range";
    default: return "unknown error";
    }
}

int gfp_version(void) { return 1; }

int gfp_check_prime_compat(int k, uint64_t r)
{
    const u64 P1 = 4179340454199820289ULL, P2 = 2485986994308513793ULL;
    if (!valid_k(k) || r < 2)
        return 0;
    u128 limit = ((u128)P1 * P2 - 1) / 2;
    u128 r2 = (u128)r * r;
    if (r2 > limit / (u64)k)
        return 0;
    if ((P1 - 1) % (2 * (u64)k) || (P2 - 1) % (2 * (u64)k))
        return 0;
    return 1;
}

int gfp_fast_path_ok(int k, uint64_t r)
{
    return fast_path_bounds_ok(k, r) ? 1 : 0;
}

}  // extern "C"

int check_kr(int k, u64 r)
{
    if (!valid_k(k) || r < 2)
        return GFP_EINVAL;
    return GFP_OK;
}

extern "C" {

int gfp_radix_mode(int k, uint64_t r)
{
    if (check_kr(k, r))
        return -2;
    const RadixConsts c = make_consts(k, r);
    if (c.stages_per_norm <= 0)
        return -1;
    return c.p3_ok ? 3 : c.p2_ok ? 2 : c.sp_on ? 1 : 0;
}

int gfp_vec_add(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k, uint64_t r,
                void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    cudaStream_t st = (cudaStream_t)stream;
    DISPATCH_K(k, (k_add<KD><<<grid_for(n, 256), 256, 0, st>>>(x, y, z, n, r, 0)));
    return cuda_status();
}

int gfp_vec_sub(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k, uint64_t r,
                void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    cudaStream_t st = (cudaStream_t)stream;
    DISPATCH_K(k, (k_add<KD><<<grid_for(n, 256), 256, 0, st>>>(x, y, z, n, r, 1)));
    return cuda_status();
}

int gfp_vec_mul_pow_r(const uint64_t *x, uint64_t *z, int64_t n, int k, uint64_t r, int i,
                      void *stream)
{
    int e = check_kr(k, r);
    if (e)
        return e;
    if (i < 0 || i > 2 * k)
        return GFP_EINVAL;
    if (n <= 0)
        return GFP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DISPATCH_K(k, (k_mul_pow_r<KD><<<grid_for(n, 256), 256, 0, st>>>(x, z, n, r, i)));
    return cuda_status();
}

int gfp_vec_mul(const uint64_t *x, const uint64_t *y, int64_t y_inc, uint64_t *z, int64_t n,
                int k, uint64_t r, void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    cudaStream_t st = (cudaStream_t)stream;
    RadixConsts rc = make_consts(k, r);
    if (launch_mul_wide(k, x, y, y_inc, z, n, rc, st))
        return cuda_status();
    if (rc.stages_per_norm > 0) {
        // (mode 2 costs k = 32 registers it does not have: spills)
        if (rc.p2_ok && k != 32) {
            DISPATCH_FAST_K(k, (k_mul_fast<KD, 2><<<grid_for(n, 128), 128, 0, st>>>(
                                   x, y, y_inc, z, n, rc)));
        } else if (rc.sp_on) {
            DISPATCH_FAST_K(k, (k_mul_fast<KD, 1><<<grid_for(n, 128), 128, 0, st>>>(
                                   x, y, y_inc, z, n, rc)));
        } else {
            DISPATCH_FAST_K(k, (k_mul_fast<KD, false><<<grid_for(n, 128), 128, 0, st>>>(
                                   x, y, y_inc, z, n, rc)));
        }
    } else {
        DISPATCH_K(k, (k_mul_generic<KD><<<grid_for(n, 128), 128, 0, st>>>(x, y, y_inc, z, n,
                                                                           rc)));
    }
    return cuda_status();
}

int gfp_vec_pow(const uint64_t *x, const uint64_t *e_limbs, int e_nlimbs, uint64_t *z, int64_t n,
                int k, uint64_t r, void *stream)
{
    int e = check_kr(k, r);
    if (e)
        return e;
    if (n <= 0)
        return GFP_OK;
    if (e_nlimbs < 0)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    int nl = e_nlimbs > 0 ? e_nlimbs : 1;
    u64 *d_e = nullptr;
    if (cudaMallocAsync(&d_e, sizeof(u64) * nl, st) != cudaSuccess)
        return GFP_ENOMEM;
    u64 zero = 0;
    cudaMemcpyAsync(d_e, e_nlimbs ? e_limbs : &zero, sizeof(u64) * nl, cudaMemcpyHostToDevice, st);
    int nbits = 0;
    for (int i = e_nlimbs - 1; i >= 0; i--)
        if (e_limbs[i]) {
            nbits = 64 * i + 64 - __builtin_clzll(e_limbs[i]);
            break;
        }
    RadixConsts rc = make_consts(k, r);
    DISPATCH_K(k, (k_pow<KD><<<grid_for(n, 64), 64, 0, st>>>(x, d_e, nbits, z, n, rc)));
    int rcode = cuda_status();
    cudaStreamSynchronize(st);  // e_limbs is caller host memory
    cudaFreeAsync(d_e, st);
    return rcode;
}

int gfp_vec_is_canonical(const uint64_t *x, uint8_t *out, int64_t n, int k, uint64_t r,
                         void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    k_is_canonical<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, out, n, k, r);
    return cuda_status();
}

int gfp_vec_uniform(uint64_t *z, int64_t n, int k, uint64_t r, uint64_t seed, void *stream)
{
    int e = check_kr(k, r);
    if (e || n <= 0)
        return e;
    k_uniform<<<grid_for(n * k, 256), 256, 0, (cudaStream_t)stream>>>(z, n, k, r, seed);
    return cuda_status();
}

int gfp_vec_mul_host(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k,
                     uint64_t r, void *stream)
{
    int e = check_kr(k, r);
    if (e)
        return e;
    if (!x || !y || !z || n < 0)
        return GFP_EINVAL;
    if (n == 0)
        return GFP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    // chunks of ~128 MiB per operand through the two-stream pipeline: the
    // H2D of one chunk overlaps the kernels and D2H of the other
    const int64_t chunk = HOST_CHUNK_WORDS / k < n ? HOST_CHUNK_WORDS / k : n;
    const int64_t nchunks = (n + chunk - 1) / chunk;
    const size_t cw = (size_t)chunk * k;
    const int nst = nchunks > 1 ? 2 : 1;
    u64 *buf = nullptr;
    if (cudaMalloc(&buf, (size_t)nst * 4 * cw * sizeof(u64)) != cudaSuccess) {
        cudaGetLastError();
        return GFP_ENOMEM;
    }
    HostPipe hp;
    if (nst > 1)
        e = host_pipe_begin(hp, st);
    for (int64_t c = 0; c < nchunks && !e; c++) {
        cudaStream_t s = nst > 1 ? hp.s[c & 1] : st;
        u64 *hx = buf + (size_t)(c & (nst - 1)) * 4 * cw, *hy = hx + cw, *dx = hy + cw,
            *dy = dx + cw;
        const int64_t i0 = c * chunk, m = n - i0 < chunk ? n - i0 : chunk;
        const size_t bytes = (size_t)m * k * sizeof(u64);
        cudaMemcpyAsync(hx, x + i0 * k, bytes, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(hy, y + i0 * k, bytes, cudaMemcpyHostToDevice, s);
        e = transpose_batched(hx, dx, 1, m, m, k, 1, s);
        if (!e)
            e = transpose_batched(hy, dy, 1, m, m, k, 1, s);
        if (!e)
            e = gfp_vec_mul(dx, dy, 1, dx, m, k, r, s);
        if (!e)
            e = transpose_batched(dx, hx, 1, m, m, k, 0, s);
        if (!e)
            cudaMemcpyAsync(z + i0 * k, hx, bytes, cudaMemcpyDeviceToHost, s);
    }
    if (nst > 1) {
        const int e2 = host_pipe_end(hp, st);
        e = e ? e : e2;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && !e)
        e = GFP_ECUDA;
    cudaFree(buf);
    return e ? e : cuda_status();
}

int gfp_to_digit_major(const uint64_t *src, uint64_t *dst, int64_t n, int k, void *stream)
{
    if (!valid_k(k))
        return GFP_EINVAL;
    if (n <= 0)
        return GFP_OK;
    k_transpose<<<grid_for(n * k, 256), 256, 0, (cudaStream_t)stream>>>(src, dst, n, k, 0);
    return cuda_status();
}

int gfp_to_element_major(const uint64_t *src, uint64_t *dst, int64_t n, int k, void *stream)
{
    if (!valid_k(k))
        return GFP_EINVAL;
    if (n <= 0)
        return GFP_OK;
    k_transpose<<<grid_for(n * k, 256), 256, 0, (cudaStream_t)stream>>>(src, dst, n, k, 1);
    return cuda_status();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// One element operation on host digit tuples (the reference's scalar API:
// gfp_add, gfp_sub, gfp_mul_pow_r, gfp_mul_fft / gfp_mul_bigint, gfp_pow):
// one H2D of the operands through a persistent pinned staging buffer, one
// kernel, one D2H, one stream synchronisation -- instead of a tensor
// allocation and two synchronising copies per operand in the Python layer.
#include <mutex>

namespace {
struct ScalarStage {
    u64 *host = nullptr;  // pinned: [x k][y k][e limbs][z k]
    u64 *dev = nullptr;
};
constexpr int SCALAR_WORDS = 3 * 128 + 64;  // x, y, z (k <= 128) + 64 exponent limbs
ScalarStage g_scalar[64];
std::mutex g_scalar_mu;
}  // namespace

extern "C" int gfp_scalar_op(int op, const uint64_t *x, const uint64_t *y, int64_t arg,
                             uint64_t *z, int k, uint64_t r, void *stream)
{
    int e = check_kr(k, r);
    if (e)
        return e;
    if (!x || !z || op < 0 || op > 5 || ((op <= 1 || op == 3 || op == 4 || op == 5) && !y))
        return GFP_EINVAL;
    if (op == 2 && (arg < 0 || arg > 2 * k))
        return GFP_EINVAL;
    if (op == 5 && (arg < 0 || arg > 64))
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_scalar_mu);
    ScalarStage &S = g_scalar[dev & 63];
    if (!S.host) {
        if (cudaMallocHost(&S.host, sizeof(u64) * SCALAR_WORDS) != cudaSuccess ||
            cudaMalloc(&S.dev, sizeof(u64) * SCALAR_WORDS) != cudaSuccess) {
            cudaGetLastError();
            return GFP_ENOMEM;
        }
    }
    u64 *hx = S.host, *hy = hx + 128, *he = hy + 128, *hz = he + 64;
    u64 *dx = S.dev, *dy = dx + 128, *de = dy + 128, *dz = de + 64;
    memcpy(hx, x, sizeof(u64) * k);
    const int ny = op == 5 ? (int)arg : (op == 2 ? 0 : k);
    if (ny)
        memcpy(op == 5 ? he : hy, y, sizeof(u64) * ny);
    cudaMemcpyAsync(dx, hx, sizeof(u64) * (128 + 128 + 64), cudaMemcpyHostToDevice, st);
    const RadixConsts rc = make_consts(k, r);
    switch (op) {
    case 0:
    case 1:
        DISPATCH_K(k, (k_add<KD><<<1, 32, 0, st>>>(dx, dy, dz, 1, r, op)));
        break;
    case 2:
        DISPATCH_K(k, (k_mul_pow_r<KD><<<1, 32, 0, st>>>(dx, dz, 1, r, (int)arg)));
        break;
    case 3:
        e = gfp_vec_mul(dx, dy, 1, dz, 1, k, r, st);
        break;
    case 4:
        e = gfp_vec_mul_crt(dx, dy, 1, dz, 1, k, r, st);
        break;
    default: {
        int nbits = 0;
        for (int i = (int)arg - 1; i >= 0; i--)
            if (he[i]) {
                nbits = 64 * i + 64 - __builtin_clzll(he[i]);
                break;
            }
        DISPATCH_K(k, (k_pow<KD><<<1, 32, 0, st>>>(dx, de, nbits, dz, 1, rc)));
    }
    }
    if (e)
        return e;
    cudaMemcpyAsync(hz, dz, sizeof(u64) * k, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return GFP_ECUDA;
    memcpy(z, hz, sizeof(u64) * k);
    return cuda_status();
}
