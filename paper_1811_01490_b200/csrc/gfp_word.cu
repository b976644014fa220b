// gfp_word.cu -- the word-prime transform: DFT over Z/qZ for an odd prime
// q < 2^63 on Montgomery residues (R = 2^64), and the cyclic / negacyclic
// convolutions built on it.
//
// Reference: word_field.py:103-200 (WordPrime, mont_mul REDC, word_pow,
// mont_inv), fft.py:376-421 (MontField: the field dft_general runs on for
// the word primes), gfp_mult.py:230-386 (_make_plan / _nega_plan /
// _cyclic_plan / _convolve, cyclic_convolution, negacyclic_convolution).
// In the reference these are the inner transforms of gfp_mul_fft over the
// prime pair P1 = 29 2^57 + 1, P2 = 69 2^55 + 1 (word_field.py:15-16).
//
// Residues in [0, q) are unique, so every exact DFT at the same root gives
// the reference's bits; the GPU uses its own schedule:
//   * Stockham autosort passes of radix R in {16, 8, 4, 2} (R = 16 while
//     four or more factors of two remain): group j of M = N/R reads
//     x[j + t M], multiplies by w^E, E = t (j mod Ns) (M / Ns), runs the
//     R-point DFT in registers and writes (j / Ns) Ns R + (j mod Ns) + u Ns
//     -- the natural-order DFT after the last pass, like k_pass (gfp_pass.cuh);
//   * the R-point DFT is radix-2 with the butterfly factors w^(N/R)^m read
//     from the plan's power table (L1-resident);
//   * optional element weights fused into the first pass (x_i * win_i and a
//     pointwise operand) and the last pass (X_u * wout_u or a scalar):
//     the convolution is 3 transforms and no separate element-wise kernels.
// Thread per group, digit-free 64-bit words: each pass streams 2 x 8 N
// bytes, so the transform is HBM-bound for large N (REDC: 3 64-bit products).
#include "gfp_internal.cuh"

struct WordConsts {
    u64 q;
    u64 qinv;  // -q^-1 mod 2^64
    u64 r2;    // 2^128 mod q
    u64 one;   // 2^64 mod q (Montgomery 1)
};

// REDC product a b 2^-64 mod q, inputs and output in [0, q) (mont_mul,
// word_field.py:133-140); q < 2^63 keeps t < 2q < 2^64.
GFP_HD u64 w_mul(u64 a, u64 b, const WordConsts &c)
{
#ifdef __CUDA_ARCH__
    const u64 lo = a * b, hi = __umul64hi(a, b);
    const u64 d = lo * c.qinv;
    const u64 t = hi + __umul64hi(d, c.q) + (lo != 0);
#else
    const u128 ab = (u128)a * b;
    const u64 lo = (u64)ab, hi = (u64)(ab >> 64);
    const u64 d = lo * c.qinv;
    const u64 t = hi + (u64)(((u128)d * c.q) >> 64) + (lo != 0);
#endif
    return t >= c.q ? t - c.q : t;
}
GFP_HD u64 w_add(u64 a, u64 b, const WordConsts &c)
{
    const u64 s = a + b;
    return s >= c.q ? s - c.q : s;
}
GFP_HD u64 w_sub(u64 a, u64 b, const WordConsts &c) { return a >= b ? a - b : a - b + c.q; }

GFP_HD u64 w_pow(u64 a, u64 e, const WordConsts &c)
{
    u64 acc = c.one;
    while (e) {
        if (e & 1)
            acc = w_mul(acc, a, c);
        a = w_mul(a, a, c);
        e >>= 1;
    }
    return acc;
}

// x * w mod q for a constant w (standard form) with its Shoup factor
// ws = floor(w 2^64 / q): one high and two low 64-bit products instead of
// REDC's three wide ones.  With w = the standard value of a Montgomery
// constant w_m (w = w_m R^-1), x * w = mont_mul(x, w_m): the same residue,
// so Montgomery-form data keeps its form.
GFP_D u64 w_mul_shoup(u64 x, ulonglong2 w, const WordConsts &c)
{
    const u64 hi = __umul64hi(x, w.y);
    const u64 r = x * w.x - hi * c.q;  // in [0, 2q)
    return r >= c.q ? r - c.q : r;
}

struct WordPassArgs {
    const u64 *in;
    u64 *out;
    const ulonglong2 *tw;  // {w^i (standard form), Shoup factor}, i < N
    const u64 *w_in;   // pass 0: x_i <- x_i * w_in[i] (nullptr: none)
    const u64 *pre;    // pass 0: x_i <- x_i * pre[b][i] (pointwise operand)
    const u64 *w_out;  // last pass: X_u <- X_u * w_out[u]
    u64 scale;         // last pass: X_u <- X_u * scale (0: none)
    int64_t batch_stride;
    int lN, lNs;
    WordConsts c;
};

// w^(e) for the R-point DFT factor, e in units of N / R
template <int R>
GFP_D ulonglong2 w_root(const WordPassArgs &A, int e)
{
    return __ldg(A.tw + ((int64_t)e << (A.lN - (R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1))));
}

// y[t] = x[bitreverse(t)] for t < 2^LR, resolved at compile time
template <int LR, int T>
struct Brev {
    static constexpr int v = ((T & 1) << (LR - 1)) | Brev<LR - 1, (T >> 1)>::v;
};
template <int T>
struct Brev<0, T> {
    static constexpr int v = 0;
};
template <int LR, int T = 0>
GFP_D void brev_copy(const u64 (&x)[1 << LR], u64 (&y)[1 << LR])
{
    if constexpr (T < (1 << LR)) {
        y[T] = x[Brev<LR, T>::v];
        brev_copy<LR, T + 1>(x, y);
    }
}

template <int R>
__global__ void __launch_bounds__(256) k_word_pass(WordPassArgs A)
{
    constexpr int LR = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
    const int64_t M = ((int64_t)1 << A.lN) >> LR;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (j >= M)
        return;
    const int64_t boff = (int64_t)blockIdx.y * A.batch_stride;
    const u64 *in = A.in + boff;
    u64 *out = A.out + boff;
    const WordConsts c = A.c;
    const int64_t nsmask = ((int64_t)1 << A.lNs) - 1;
    const int64_t js = j & nsmask;
    u64 x[R];
#pragma unroll
    for (int t = 0; t < R; t++)
        x[t] = __ldcs(in + j + t * M);
    if (A.w_in) {  // first pass only (uniform branches: the loops stay unrolled)
#pragma unroll
        for (int t = 0; t < R; t++)
            x[t] = w_mul(x[t], __ldg(A.w_in + j + t * M), c);
    }
    if (A.pre) {
#pragma unroll
        for (int t = 0; t < R; t++)
            x[t] = w_mul(x[t], __ldg(A.pre + boff + j + t * M), c);
    }
    if (js) {  // w^(t js M / Ns)
#pragma unroll
        for (int t = 1; t < R; t++)
            x[t] = w_mul_shoup(x[t], __ldg(A.tw + (((int64_t)t * js) << (A.lN - LR - A.lNs))), c);
    }
    // R-point DFT at root w^(N/R): decimation in time, bit-reversed input
    // order resolved at compile time
    u64 y[R];
    brev_copy<LR>(x, y);
#pragma unroll
    for (int s = 1; s <= LR; s++) {
#pragma unroll
        for (int bi = 0; bi < R / 2; bi++) {
            const int half = 1 << (s - 1);
            const int m = bi & (half - 1);
            const int lo = ((bi >> (s - 1)) << s) + m;
            u64 u = y[lo], v = y[lo + half];
            const int e = m << (LR - s);  // w_R^(m R / 2^s)
            if (e)
                v = w_mul_shoup(v, w_root<R>(A, e), c);
            y[lo] = w_add(u, v, c);
            y[lo + half] = w_sub(u, v, c);
        }
    }
    const int64_t obase = ((j >> A.lNs) << (A.lNs + LR)) + js;
    if (A.w_out) {
#pragma unroll
        for (int u = 0; u < R; u++)
            y[u] = w_mul(y[u], __ldg(A.w_out + obase + ((int64_t)u << A.lNs)), c);
    }
    if (A.scale) {
#pragma unroll
        for (int u = 0; u < R; u++)
            y[u] = w_mul(y[u], A.scale, c);
    }
    if (R == 16 && A.lNs == 0 && (j | 31) < M) {
        // first pass: thread j writes positions 16 j .. 16 j + 15 -- stage the
        // warp's 512 outputs in shared memory and store them contiguously
        // (a lane-per-group store touches 32 lines with 8 bytes each)
        __shared__ u64 stage[8][32 * 17];
        const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
        u64 *st = stage[wq];
#pragma unroll
        for (int u = 0; u < R; u++)
            st[lane * 17 + u] = y[u];
        __syncwarp();
        u64 *ob = out + ((j - lane) << 4);
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const int q = lane + 32 * i;  // position 16 (j - lane) + q
            __stcs(ob + q, st[(q >> 4) * 17 + (q & 15)]);
        }
        return;
    }
#pragma unroll
    for (int u = 0; u < R; u++)
        __stcs(out + obase + ((int64_t)u << A.lNs), y[u]);
}

template <>
__global__ void __launch_bounds__(256) k_word_pass<1>(WordPassArgs A)
{
    // n = 1: the DFT is the identity; weights and scale still apply
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x || blockIdx.x)
        return;
    const int64_t boff = (int64_t)blockIdx.y * A.batch_stride;
    u64 v = A.in[boff];
    if (A.w_in)
        v = w_mul(v, A.w_in[0], A.c);
    if (A.pre)
        v = w_mul(v, A.pre[boff], A.c);
    if (A.w_out)
        v = w_mul(v, A.w_out[0], A.c);
    if (A.scale)
        v = w_mul(v, A.scale, A.c);
    A.out[boff] = v;
}

// table[i] = mont_mul(base^i, post) for i < n (base, post Montgomery or any
// word: post = one gives the powers themselves)
__global__ void k_word_powers(u64 *table, int64_t n, u64 base, u64 post, WordConsts c)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        table[i] = w_mul(w_pow(base, (u64)i, c), post, c);
}

// table[i] = {w, floor(w 2^64 / q)} with w = base^i in standard form
// (base Montgomery); the quotient by restoring long division (plan time)
__global__ void k_word_shoup_powers(ulonglong2 *table, int64_t n, u64 base, WordConsts c)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const u64 w = w_mul(w_pow(base, (u64)i, c), 1, c);  // standard form
        u64 rem = w, quo = 0;  // (w 2^64) / q, one quotient bit per step
        for (int b = 0; b < 64; b++) {
            const bool top = rem >> 63;
            rem <<= 1;
            quo <<= 1;
            if (top || rem >= c.q) {
                rem -= c.q;
                quo |= 1;
            }
        }
        table[i] = make_ulonglong2(w, quo);
    }
}

__global__ void k_word_mul(const u64 *a, const u64 *b, u64 *z, int64_t n, WordConsts c)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        z[i] = w_mul(a[i], b[i], c);
}

__global__ void k_word_check(const u64 *x, int64_t n, u64 q, int *bad)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (x[i] >= q)
            atomicOr(bad, 1);
}

struct gfp_word_plan {
    WordConsts c;
    int64_t n;
    int lN;
    ulonglong2 *tw_fwd, *tw_inv;  // {w^i, Shoup}, {w^-i, Shoup} (i < n), standard form
    u64 ninv;              // n^-1 in Montgomery form
    u64 *w_in, *w_out;     // convolution weights (standard-form in/out), or null
    u64 *scratch;
    int64_t scratch_words;
    int *d_bad;  // input range flag (device) and its pinned host copy
    int *h_bad;
};

static WordConsts word_consts(u64 q)
{
    WordConsts c;
    c.q = q;
    // -q^-1 mod 2^64 by Newton (q odd)
    u64 inv = q;  // correct to 3 bits
    for (int i = 0; i < 6; i++)
        inv *= 2 - q * inv;
    c.qinv = (u64)0 - inv;
    const u128 R1 = ((u128)1 << 64) % q;
    c.one = (u64)R1;
    c.r2 = (u64)(((u128)c.one * c.one) % q);
    return c;
}

static bool word_q_ok(u64 q) { return q >= 3 && (q & 1) && q < ((u64)1 << 63); }

// Stockham schedule over N = 2^lN: radix 16 while >= 4 factors remain
static int word_run(const gfp_word_plan *p, const u64 *in, u64 *out, int64_t batch, int inverse,
                    const u64 *w_in, const u64 *pre, const u64 *w_out, u64 scale, u64 *work,
                    cudaStream_t st)
{
    if (batch > GFP_MAX_GRID_Y)  // the batch is the pass kernels' grid.y
        return GFP_EINVAL;
    const int lN = p->lN;
    int radices[64], np = 0, rem = lN;
    while (rem >= 4) {
        radices[np++] = 4;
        rem -= 4;
    }
    if (rem)
        radices[np++] = rem;
    if (np == 0)
        radices[np++] = 0;  // n = 1
    const u64 *src = in;
    int lNs = 0;
    for (int pi = 0; pi < np; pi++) {
        const bool last = pi == np - 1;
        u64 *dst = ((np - pi) % 2 == 1) ? out : work;
        if (dst == src)
            dst = dst == out ? work : out;
        WordPassArgs A;
        A.in = src;
        A.out = dst;
        A.tw = inverse ? p->tw_inv : p->tw_fwd;
        A.w_in = pi == 0 ? w_in : nullptr;
        A.pre = pi == 0 ? pre : nullptr;
        A.w_out = last ? w_out : nullptr;
        A.scale = last ? scale : 0;
        A.batch_stride = p->n;
        A.lN = lN;
        A.lNs = lNs;
        A.c = p->c;
        const int lr = radices[pi];
        const int64_t M = lr ? (p->n >> lr) : 1;
        const int threads = 256;
        dim3 grid((unsigned)((M + threads - 1) / threads), (unsigned)batch);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(threads);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        switch (lr) {
        case 4: cudaLaunchKernelEx(&cfg, k_word_pass<16>, A); break;
        case 3: cudaLaunchKernelEx(&cfg, k_word_pass<8>, A); break;
        case 2: cudaLaunchKernelEx(&cfg, k_word_pass<4>, A); break;
        case 1: cudaLaunchKernelEx(&cfg, k_word_pass<2>, A); break;
        default: cudaLaunchKernelEx(&cfg, k_word_pass<1>, A); break;
        }
        src = dst;
        lNs += lr;
    }
    if (src != out)
        cudaMemcpyAsync(out, src, sizeof(u64) * (size_t)p->n * batch, cudaMemcpyDeviceToDevice,
                        st);
    return cuda_status();
}

static int ensure_scratch(gfp_word_plan *p, int64_t words)
{
    if (p->scratch_words >= words)
        return GFP_OK;
    if (p->scratch)
        cudaFree(p->scratch);
    p->scratch = nullptr;
    p->scratch_words = 0;
    if (cudaMalloc(&p->scratch, sizeof(u64) * (size_t)words) != cudaSuccess)
        return GFP_ENOMEM;
    p->scratch_words = words;
    return GFP_OK;
}

extern "C" {

int gfp_word_consts(uint64_t q, uint64_t *qinv, uint64_t *r2, uint64_t *one)
{
    if (!word_q_ok(q))
        return GFP_EINVAL;
    WordConsts c = word_consts(q);
    if (qinv)
        *qinv = c.qinv;
    if (r2)
        *r2 = c.r2;
    if (one)
        *one = c.one;
    return GFP_OK;
}

int gfp_word_vec_mont_mul(uint64_t q, const uint64_t *a, const uint64_t *b, uint64_t *z,
                          int64_t n, void *stream)
{
    if (!word_q_ok(q) || n < 0)
        return GFP_EINVAL;
    if (n == 0)
        return GFP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_word_mul<<<grid_for(n, 256), 256, 0, st>>>(a, b, z, n, word_consts(q));
    return cuda_status();
}

int gfp_word_plan_create(gfp_word_plan **plan, uint64_t q, int64_t n, uint64_t omega,
                         int negacyclic, uint64_t theta, void *stream)
{
    if (!plan)
        return GFP_EINVAL;
    *plan = nullptr;
    if (!word_q_ok(q) || n < 1 || (n & (n - 1)) || omega >= q || theta >= q)
        return GFP_EINVAL;
    const int lN = ilog2_exact(n);
    WordConsts c = word_consts(q);
    // omega must be a primitive n-th root (fft.py:250-254): w^n = 1 and,
    // for n > 1, w^(n/2) = -1; q - 1 must be divisible by n
    if ((q - 1) % (u64)n)
        return GFP_EINVAL;
    const u64 minus_one = w_mul(q - 1, c.r2, c);
    if (w_pow(omega, (u64)n, c) != c.one || (n > 1 && w_pow(omega, (u64)n / 2, c) != minus_one))
        return GFP_EINVAL;
    if (negacyclic && (w_pow(theta, 2 * (u64)n, c) != c.one ||
                       w_pow(theta, (u64)n, c) != minus_one || w_mul(theta, theta, c) != omega))
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    gfp_word_plan *p = (gfp_word_plan *)calloc(1, sizeof(gfp_word_plan));
    if (!p)
        return GFP_ENOMEM;
    p->c = c;
    p->n = n;
    p->lN = lN;
    const u64 omega_inv = w_pow(omega, (u64)n - 1, c);
    const u64 n_m = w_mul((u64)(n % (int64_t)q), c.r2, c);
    p->ninv = w_pow(n_m, q - 2, c);  // (n^-1) R
    if (cudaMalloc(&p->tw_fwd, sizeof(ulonglong2) * n) != cudaSuccess ||
        cudaMalloc(&p->tw_inv, sizeof(ulonglong2) * n) != cudaSuccess ||
        cudaMalloc(&p->w_in, sizeof(u64) * n) != cudaSuccess ||
        cudaMalloc(&p->w_out, sizeof(u64) * n) != cudaSuccess) {
        gfp_word_plan_destroy(p);
        return GFP_ENOMEM;
    }
    const dim3 g = grid_for(n, 256);
    k_word_shoup_powers<<<g, 256, 0, st>>>(p->tw_fwd, n, omega, c);
    k_word_shoup_powers<<<g, 256, 0, st>>>(p->tw_inv, n, omega_inv, c);
    // convolution weights (gfp_mult.py:280-323): standard-form inputs enter
    // Montgomery form with the weight, outputs leave it with the 1/n scale
    //   cyclic:     in_i = R^2,             out_i = n^-1          (standard)
    //   negacyclic: in_i = theta^i R^2,     out_i = theta^-i n^-1 (standard)
    const u64 ninv_std = w_mul(p->ninv, 1, c);
    if (negacyclic) {
        const u64 theta_inv = w_pow(theta, 2 * (u64)n - 1, c);
        k_word_powers<<<g, 256, 0, st>>>(p->w_in, n, theta, c.r2, c);
        k_word_powers<<<g, 256, 0, st>>>(p->w_out, n, theta_inv, ninv_std, c);
    } else {
        k_word_powers<<<g, 256, 0, st>>>(p->w_in, n, c.one, c.r2, c);
        k_word_powers<<<g, 256, 0, st>>>(p->w_out, n, c.one, ninv_std, c);
    }
    int err = cuda_status();
    if (err) {
        gfp_word_plan_destroy(p);
        return err;
    }
    *plan = p;
    return GFP_OK;
}

int gfp_word_plan_destroy(gfp_word_plan *p)
{
    if (!p)
        return GFP_OK;
    cudaFree(p->tw_fwd);
    cudaFree(p->tw_inv);
    cudaFree(p->w_in);
    cudaFree(p->w_out);
    cudaFree(p->scratch);
    cudaFree(p->d_bad);
    if (p->h_bad)
        cudaFreeHost(p->h_bad);
    free(p);
    return GFP_OK;
}

int gfp_word_ntt_exec(gfp_word_plan *p, const uint64_t *in, uint64_t *out, int64_t batch,
                      int inverse, void *stream)
{
    if (!p || batch < 1 || !in || !out)
        return GFP_EINVAL;
    int err = ensure_scratch(p, p->n * batch);
    if (err)
        return err;
    return word_run(p, in, out, batch, inverse, nullptr, nullptr, nullptr,
                    inverse ? p->ninv : 0, p->scratch, (cudaStream_t)stream);
}

int gfp_word_convolve(gfp_word_plan *p, const uint64_t *x, const uint64_t *y, uint64_t *out,
                      int64_t batch, void *stream)
{
    if (!p || batch < 1 || !x || !y || !out)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t words = p->n * batch;
    int err = ensure_scratch(p, 3 * words);
    if (err)
        return err;
    if (!p->d_bad) {
        if (cudaMalloc((void **)&p->d_bad, sizeof(int)) != cudaSuccess ||
            cudaMallocHost((void **)&p->h_bad, sizeof(int)) != cudaSuccess)
            return GFP_ENOMEM;
    }
    // range check queued with the work; one synchronisation at the end
    cudaMemsetAsync(p->d_bad, 0, sizeof(int), st);
    k_word_check<<<grid_for(words, 256), 256, 0, st>>>(x, words, p->c.q, p->d_bad);
    k_word_check<<<grid_for(words, 256), 256, 0, st>>>(y, words, p->c.q, p->d_bad);
    u64 *a = p->scratch, *b = p->scratch + words, *work = p->scratch + 2 * words;
    // forward of both weighted operands, then the inverse with the pointwise
    // product fused into its first pass and the out weights into its last
    err = word_run(p, x, a, batch, 0, p->w_in, nullptr, nullptr, 0, work, st);
    if (!err)
        err = word_run(p, y, b, batch, 0, p->w_in, nullptr, nullptr, 0, work, st);
    if (!err)
        err = word_run(p, a, out, batch, 1, nullptr, b, p->w_out, 0, work, st);
    if (err)
        return err;
    cudaMemcpyAsync(p->h_bad, p->d_bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return cuda_status();
    // "inputs must be reduced mod q" (gfp_mult.py:361-366); out is unspecified then
    return *p->h_bad ? GFP_EINVAL : GFP_OK;
}

}  // extern "C"
