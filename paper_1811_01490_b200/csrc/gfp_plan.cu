// gfp_plan.cu -- transform plans (omega validation, twiddle tables built on
// the device with the exact multiply), the four-step inter-stage twiddle,
// transform orchestration (Stockham pass sequence, poly-multiply) and the
// transform C-ABI.
#include "gfp_internal.cuh"
#include "gfp_fast.cuh"
#include "gfp_generic.cuh"

// power table: out[b] = omega^(b * step) for b < n, element-major [n][k]
// (one thread per entry, square-and-multiply over the bits of b with the
// precomputed omega^(2^i step) in `sq`), exact generic multiply.
template <int KD>
__global__ void k_power_table(const u64 *__restrict__ sq, int nsq, u64 *__restrict__ out,
                              int64_t n, RadixConsts rc)
{
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        u64 acc[KD];
        for (int d = 0; d < KD; d++)
            acc[d] = d == 0 ? 1 : 0;
        for (int i = 0; i < nsq; i++) {
            if ((b >> i) & 1) {
                u64 y[KD];
                for (int d = 0; d < KD; d++)
                    y[d] = sq[(int64_t)i * KD + d];
                gfp_mul_generic<KD>(acc, y, acc, rc);
            }
        }
        for (int d = 0; d < KD; d++)
            out[b * KD + d] = acc[d];
    }
}

// sq[i] = omega^(2^i), element-major, single thread (plan time only)
template <int KD>
__global__ void k_squarings(const u64 *__restrict__ omega, u64 *__restrict__ sq, int nsq,
                            RadixConsts rc)
{
    if (blockIdx.x || threadIdx.x)
        return;
    u64 cur[KD];
    for (int d = 0; d < KD; d++)
        cur[d] = omega[d];
    for (int i = 0; i < nsq; i++) {
        for (int d = 0; d < KD; d++)
            sq[(int64_t)i * KD + d] = cur[d];
        gfp_mul_generic<KD>(cur, cur, cur, rc);
    }
}

// element-major table times a constant (element-major [1][k])
template <int KD>
__global__ void k_table_scale(const u64 *__restrict__ tab, const u64 *__restrict__ c,
                              u64 *__restrict__ out, int64_t n, RadixConsts rc)
{
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        u64 a[KD], y[KD], z[KD];
        for (int d = 0; d < KD; d++) {
            a[d] = tab[b * KD + d];
            y[d] = c[d];
        }
        gfp_mul_generic<KD>(a, y, z, rc);
        for (int d = 0; d < KD; d++)
            out[b * KD + d] = z[d];
    }
}

// element-major canonical table entries -> balanced lazy digits (in place);
// the transform multiplies balanced operands only
template <int KD>
__global__ void k_table_balance(u64 *__restrict__ tab, int64_t n, u64 r)
{
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        i64 x[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            x[d] = (i64)tab[b * KD + d];
        to_balanced<KD>(x, r);
#pragma unroll
        for (int d = 0; d < KD; d++)
            tab[b * KD + d] = (u64)x[d];
    }
}

// balanced table entries -> limb pairs (l | h << 32, v = h 2^S + l) for the
// k_pass44 twiddle multiply (fast_mul_lazy_ylimbs)
template <int KD>
__global__ void k_table_limbs(const u64 *__restrict__ tab, u64 *__restrict__ out, int64_t n)
{
    constexpr int S = FastSplit<KD>::S;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int d = 0; d < KD; d++) {
            int l, h;
            split_limbs<S>((i64)tab[b * KD + d], l, h);
            out[b * KD + d] = (u64)(unsigned)l | ((u64)(unsigned)h << 32);
        }
    }
}

// Four-step inter-stage twiddle (the sharded transform):
// x is digit-major [batch][k][n] canonical; element (b, i) is multiplied by
// omega^((row0 + b) i) (omega^-(...) when inverse), omega the plan's N-th
// root, using the plan's table omega^j (j < N/K) and the cheap split
// omega^E = (omega^(N/K))^a omega^j as a digit rotation.  Canonical output.
template <int KD, int SPARSE>
__global__ void k_twiddle_rows(const u64 *__restrict__ x, u64 *__restrict__ out,
                               const u64 *__restrict__ table, int64_t batch, int64_t n,
                               int64_t row0, int lN, int lM, int inverse, int root_inv,
                               RadixConsts rc)
{
    const int64_t total = batch * n;
    const int64_t N = (int64_t)1 << lN, M = (int64_t)1 << lM;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / n, i = t - b * n;
        const u64 *src = x + b * KD * n + i;
        u64 *dst = out + b * KD * n + i;
        i64 v[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            v[d] = (i64)src[d * n];
        int64_t E = ((row0 + b) * i) & (N - 1);
        if (inverse && E)
            E = N - E;
        int a = (int)(E >> lM);
        const int64_t j = E & (M - 1);
        if (root_inv && a)
            a = 2 * KD - a;
        if (j) {
            i64 y[KD];
#pragma unroll
            for (int d = 0; d < KD; d++)
                y[d] = (i64)table[j * KD + d];
            to_balanced<KD>(v, rc.r);
            fast_mul_lazy<KD, SPARSE>(v, y, v, rc);
        }
        // rotation by a with the wrapped digits negated (r^k = -1), as a
        // log-depth network of compile-time rotations (no local memory)
        i64 w[KD];
#pragma unroll
        for (int d = 0; d < KD; d++)
            w[d] = v[d];
#pragma unroll
        for (int s = 1; s < 2 * KD; s <<= 1) {
            const bool on = (a & s) != 0;
            i64 rot[KD];
#pragma unroll
            for (int d = 0; d < KD; d++) {
                if (s == KD)
                    rot[d] = -w[d];
                else
                    rot[d] = d >= s ? w[d - s] : -w[d - s + KD];
            }
#pragma unroll
            for (int d = 0; d < KD; d++)
                w[d] = on ? rot[d] : w[d];
        }
        u64 c[KD];
        lazy_to_canonical(w, c, KD, rc);
#pragma unroll
        for (int d = 0; d < KD; d++)
            dst[d * n] = c[d];
    }
}

// Per-launch device timing (gfp_fft_plan_set_timing): with timing on, an
// event is recorded on the launching stream before the first pass launch of
// a call and after every pass launch, so consecutive events bracket exactly
// one pass kernel.  pass >= 0 labels the launch just completed.
static void timing_mark(gfp_fft_plan *p, cudaStream_t st, int pass)
{
    if (!p->timing)
        return;
    if (pass < 0 && p->n_ev > 0)  // before a launch: only the call's first one needs a start
        return;
    if (p->n_ev >= GFP_MAX_TIMED + 1)
        return;
    if (!p->ev[p->n_ev] && cudaEventCreate(&p->ev[p->n_ev]) != cudaSuccess)
        return;
    cudaEventRecord(p->ev[p->n_ev], st);
    if (pass >= 0 && p->n_ev > 0)
        p->ev_pass[p->n_ev - 1] = pass;
    p->n_ev++;
}

// start of an API call on the plan: launch count and timing marks reset
static void begin_call(gfp_fft_plan *p)
{
    p->last_launches = 0;
    p->n_ev = 0;
}

// One transform of `batch` vectors (and, when in_b is given, a second
// independent set of `batch` vectors transformed in the same launches).
// in_canon: the input is canonical (user data) and is converted to balanced
// digits on load; out_canon: the last pass canonicalises (user-visible
// output) -- poly_mul keeps its intermediate spectra as balanced lazy digits.
// `pre` is a pointwise operand (balanced lazy) multiplied in on the first
// pass (single set only).
static int run_transform2(gfp_fft_plan *p, const u64 *in, u64 *out, u64 *work, const u64 *in_b,
                          u64 *out_b, u64 *work_b, const u64 *pre, int64_t batch, int inverse,
                          int in_canon, int out_canon, cudaStream_t st, const PassIO *em = nullptr)
{
    // one Stockham pass per launch; ping-pong so that the last launch lands
    // in `out`; inputs are never written
    const int e = p->e;
    const u64 *src = in, *src_b = in_b;
    int64_t Ns = 1;
    for (int pass = 0; pass < e; pass++) {
        const int remaining = e - pass;  // launches left including this one
        u64 *dst = (remaining % 2 == 1) ? out : work;
        if (dst == src)
            dst = (dst == out) ? work : out;
        u64 *dst_b = nullptr;
        if (in_b) {
            dst_b = (remaining % 2 == 1) ? out_b : work_b;
            if (dst_b == src_b)
                dst_b = (dst_b == out_b) ? work_b : out_b;
        }
        const int last = pass + 1 == e;
        const int scale = inverse && last;
        const u64 *pre_p = pass == 0 ? pre : nullptr;
        int rcode = GFP_EUNSUPPORTED;
        timing_mark(p, st, -1);
        DISPATCH_FAST_K(p->k, (rcode = launch_pass<KD>(p, src, dst, src_b, dst_b, pre_p, batch, Ns,
                                                       inverse, scale, last && out_canon,
                                                       pass == 0 && in_canon, em, st)));
        if (rcode)
            return rcode;
        timing_mark(p, st, pass);
        p->last_launches++;
        src = dst;
        src_b = dst_b;
        Ns *= p->K;
    }
    if (em && ((em->out && out_canon) || em->xg))
        return cuda_status();  // the last pass wrote the element-major output / the exchange
    if (src != out)
        cudaMemcpyAsync(out, src, sizeof(u64) * (size_t)p->k * p->N * batch,
                        cudaMemcpyDeviceToDevice, st);
    if (in_b && src_b != out_b)
        cudaMemcpyAsync(out_b, src_b, sizeof(u64) * (size_t)p->k * p->N * batch,
                        cudaMemcpyDeviceToDevice, st);
    return cuda_status();
}

static int run_transform(gfp_fft_plan *p, const u64 *in, u64 *out, u64 *work, const u64 *pre,
                         int64_t batch, int inverse, int in_canon, int out_canon,
                         cudaStream_t st, const PassIO *em = nullptr)
{
    if (p->generic) {  // canonical digits throughout: the forms do not matter
        if (em)
            return GFP_EUNSUPPORTED;
        int err = GFP_OK;
        if (pre) {
            err = generic_pointwise(p, in, pre, work, batch, st);
            in = work;
            if (!err && work == out)
                return GFP_EINVAL;
            // the transform ping-pongs between out and a second buffer:
            // the spectra product sits in work, so copy it to out first
            if (!err) {
                cudaMemcpyAsync(out, work, sizeof(u64) * (size_t)p->k * p->N * batch,
                                cudaMemcpyDeviceToDevice, st);
                in = out;
            }
        }
        return err ? err : run_generic(p, in, out, work, batch, inverse, st);
    }
    return run_transform2(p, in, out, work, nullptr, nullptr, nullptr, pre, batch, inverse,
                          in_canon, out_canon, st, em);
}

extern "C" {

int gfp_fft_plan_create(gfp_fft_plan **plan, int k, uint64_t r, int K, int e,
                        const uint64_t *omega, void *stream)
{
    if (!plan)
        return GFP_EINVAL;
    *plan = nullptr;
    int err = check_kr(k, r);
    if (err)
        return err;
    if (K != 8 && K != 16 && K != 32 && K != 64)
        return GFP_EINVAL;
    if (e < 1)
        return GFP_EINVAL;
    if (K != 2 * k)
        return GFP_EINVAL;
    int64_t N = 1;
    for (int i = 0; i < e; i++) {
        N *= K;
        if (N > ((int64_t)1 << 40))
            return GFP_EINVAL;
    }
    for (int d = 0; d < k; d++)
        if (omega[d] > r)
            return GFP_EINVAL;
    RadixConsts rc = make_consts(k, r);
    cudaStream_t st = (cudaStream_t)stream;
    gfp_fft_plan *p = (gfp_fft_plan *)calloc(1, sizeof(gfp_fft_plan));
    if (!p)
        return GFP_ENOMEM;
    // radices without the fast path's headroom: canonical radix-2 passes
    // (gfp_generic_pass.cu)
    p->generic = rc.stages_per_norm <= 0 ? 1 : 0;
    p->k = k;
    p->K = K;
    p->e = e;
    p->N = N;
    p->M = N / K;
    p->r = r;
    p->rc = rc;

    // ---- validate omega like build_plan (fft.py:250-267): omega^N = 1,
    // omega^(N/2) = -1, omega^(N/2k) in {r, r^(2k-1)}
    u64 *d_buf = nullptr;
    size_t words = (size_t)k * 8;
    if (cudaMalloc(&d_buf, sizeof(u64) * words) != cudaSuccess) {
        free(p);
        return GFP_ENOMEM;
    }
    // d_buf: [0] omega (digit-major == element-major for n=1), [1..3] results
    cudaMemcpyAsync(d_buf, omega, sizeof(u64) * k, cudaMemcpyHostToDevice, st);
    u64 exps[3] = {(u64)N, (u64)(N / 2), (u64)(N / (2 * k))};
    for (int i = 0; i < 3; i++) {
        err = gfp_vec_pow(d_buf, &exps[i], 1, d_buf + (size_t)(i + 1) * k, 1, k, r, stream);
        if (err)
            break;
    }
    u64 h_res[3 * 128];
    if (!err && cudaMemcpyAsync(h_res, d_buf + k, sizeof(u64) * 3 * k, cudaMemcpyDeviceToHost,
                                st) != cudaSuccess)
        err = GFP_ECUDA;
    if (!err && cudaStreamSynchronize(st) != cudaSuccess)
        err = GFP_ECUDA;
    if (!err) {
        bool one = true, mone = true, fwd = true, inv = true;
        for (int d = 0; d < k; d++) {
            if (h_res[d] != (u64)(d == 0))
                one = false;
            if (h_res[k + d] != (d == k - 1 ? r : 0))
                mone = false;
            // r as an element: digit 1 = 1 (k >= 2)
            if (h_res[2 * k + d] != (u64)(d == 1))
                fwd = false;
        }
        // 1/r = r^(2k-1) = -(r^(k-1)) = p - r^(k-1) = (r - 1) r^(k-1) + 1
        for (int d = 0; d < k; d++) {
            u64 want = (d == k - 1 ? r - 1 : 0) + (d == 0 ? 1 : 0);
            if (h_res[2 * k + d] != want)
                inv = false;
        }
        if (!one || !mone || !(fwd || inv))
            err = GFP_EINVAL;
        p->root_inv = fwd ? 0 : 1;
    }
    if (err) {
        cudaFree(d_buf);
        free(p);
        return err;
    }

    // ---- twiddle tables: omega^b (b < M) and omega^b * N^-1
    int nsq = 0;
    while (((int64_t)1 << nsq) < p->M)
        nsq++;
    u64 *d_sq = nullptr;
    size_t tbytes = sizeof(u64) * (size_t)k * p->M;
    if (cudaMalloc(&p->table, tbytes) != cudaSuccess ||
        cudaMalloc(&p->table_ninv, tbytes) != cudaSuccess ||
        cudaMalloc(&d_sq, sizeof(u64) * (size_t)k * (nsq + 1)) != cudaSuccess) {
        cudaFree(p->table);
        cudaFree(p->table_ninv);
        cudaFree(d_sq);
        cudaFree(d_buf);
        free(p);
        return GFP_ENOMEM;
    }
    // N^-1 = -(r^k / N) mod p (N | r^k = p - 1): radix-r long division of
    // r^k by N on the host, then negation with the canonical subtract
    u64 q[128], ninv[128], zero[128];
    {
        u128 rem = 1;  // digit k of r^k
        for (int i = k - 1; i >= 0; i--) {
            u128 cur = rem * r;
            q[i] = (u64)(cur / (u64)N);
            rem = cur % (u64)N;
        }
        for (int d = 0; d < k; d++)
            zero[d] = 0;
        dev_gfp_sub(zero, q, ninv, k, r);
    }
    cudaMemcpyAsync(d_buf, ninv, sizeof(u64) * k, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_buf + k, omega, sizeof(u64) * k, cudaMemcpyHostToDevice, st);
    DISPATCH_FAST_K(k, (k_squarings<KD><<<1, 32, 0, st>>>(d_buf + k, d_sq, nsq, rc)));
    DISPATCH_FAST_K(k, (k_power_table<KD><<<grid_for(p->M, 64), 64, 0, st>>>(d_sq, nsq, p->table,
                                                                           p->M, rc)));
    DISPATCH_FAST_K(k, (k_table_scale<KD><<<grid_for(p->M, 64), 64, 0, st>>>(
                           p->table, d_buf, p->table_ninv, p->M, rc)));
    if (p->generic) {  // canonical table, N^-1 kept for the final scale
        if (cudaMalloc(&p->ninv_dev, sizeof(u64) * k) != cudaSuccess)
            err = GFP_ENOMEM;
        else
            cudaMemcpyAsync(p->ninv_dev, ninv, sizeof(u64) * k, cudaMemcpyHostToDevice, st);
    } else {
        DISPATCH_FAST_K(k, (k_table_balance<KD><<<grid_for(p->M, 128), 128, 0, st>>>(p->table,
                                                                                    p->M, r)));
        DISPATCH_FAST_K(k, (k_table_balance<KD><<<grid_for(p->M, 128), 128, 0, st>>>(
                               p->table_ninv, p->M, r)));
    }
    err = err ? err : cuda_status();
    if (!err && !p->generic) {  // limb-pair tables: the twiddle operand of every pass kernel
        if (cudaMalloc(&p->table_lh, tbytes) != cudaSuccess ||
            cudaMalloc(&p->table_ninv_lh, tbytes) != cudaSuccess) {
            err = GFP_ENOMEM;
        } else {
            DISPATCH_FAST_K(k, (k_table_limbs<KD><<<grid_for(p->M, 128), 128, 0, st>>>(
                                   p->table, p->table_lh, p->M)));
            DISPATCH_FAST_K(k, (k_table_limbs<KD><<<grid_for(p->M, 128), 128, 0, st>>>(
                                   p->table_ninv, p->table_ninv_lh, p->M)));
            err = cuda_status();
        }
    }
    if (!err && cudaStreamSynchronize(st) != cudaSuccess)
        err = GFP_ECUDA;
    cudaFree(d_sq);
    cudaFree(d_buf);
    if (err) {
        cudaFree(p->table);
        cudaFree(p->table_ninv);
        cudaFree(p->table_lh);
        cudaFree(p->table_ninv_lh);
        cudaFree(p->ninv_dev);
        free(p);
        return err;
    }
    *plan = p;
    return GFP_OK;
}

int gfp_fft_twiddle(const gfp_fft_plan *p, const uint64_t *x, uint64_t *out, int64_t batch,
                    int64_t n, int64_t row0, int inverse, void *stream)
{
    if (!p || !x || !out || batch < 1 || n < 1 || row0 < 0)
        return GFP_EINVAL;
    if (p->generic)
        return GFP_EUNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    const int lN = ilog2_exact(p->N), lM = ilog2_exact(p->M);
    dim3 grid = grid_for(batch * n, 128);
    if (p->rc.p2_ok) {
        DISPATCH_FAST_K(p->k, (k_twiddle_rows<KD, 2><<<grid, 128, 0, st>>>(
                                  x, out, p->table, batch, n, row0, lN, lM, inverse ? 1 : 0,
                                  p->root_inv, p->rc)));
    } else if (p->rc.sp_on) {
        DISPATCH_FAST_K(p->k, (k_twiddle_rows<KD, true><<<grid, 128, 0, st>>>(
                                  x, out, p->table, batch, n, row0, lN, lM, inverse ? 1 : 0,
                                  p->root_inv, p->rc)));
    } else {
        DISPATCH_FAST_K(p->k, (k_twiddle_rows<KD, false><<<grid, 128, 0, st>>>(
                                  x, out, p->table, batch, n, row0, lN, lM, inverse ? 1 : 0,
                                  p->root_inv, p->rc)));
    }
    return cuda_status();
}

int gfp_fft_plan_destroy(gfp_fft_plan *p)
{
    if (!p)
        return GFP_OK;
    cudaFree(p->table);
    cudaFree(p->table_ninv);
    cudaFree(p->table_lh);
    cudaFree(p->table_ninv_lh);
    cudaFree(p->h_dev);
    cudaFree(p->ninv_dev);
    for (int i = 0; i <= GFP_MAX_TIMED; i++)
        if (p->ev[i])
            cudaEventDestroy(p->ev[i]);
    free(p);
    return GFP_OK;
}

int64_t gfp_fft_plan_size(const gfp_fft_plan *p) { return p ? p->N : 0; }

int64_t gfp_fft_workspace_words(const gfp_fft_plan *p, int64_t batch)
{
    return p ? 3 * (int64_t)p->k * p->N * batch : 0;
}

int64_t gfp_fft_plan_last_launches(const gfp_fft_plan *p) { return p ? p->last_launches : 0; }

long long g_tma_pass_launches = 0;
int64_t gfp_tma_pass_launches(void) { return __atomic_load_n(&g_tma_pass_launches, __ATOMIC_RELAXED); }

int gfp_fft_plan_caps(const gfp_fft_plan *p)
{
    if (!p || !em_io_supported(p))
        return 0;
    return GFP_CAP_EM_IO | (p->e >= 2 ? GFP_CAP_FT | GFP_CAP_XCH : 0);
}

int gfp_fft_plan_set_timing(gfp_fft_plan *p, int on)
{
    if (!p)
        return GFP_EINVAL;
    p->timing = on ? 1 : 0;
    p->n_ev = 0;
    return GFP_OK;
}

int gfp_fft_plan_pass_times(gfp_fft_plan *p, float *ms, int *pass, int max)
{
    if (!p || max < 0)
        return -GFP_EINVAL;
    const int n = p->n_ev > 0 ? p->n_ev - 1 : 0;
    if (n == 0)
        return 0;
    if (cudaEventSynchronize(p->ev[n]) != cudaSuccess)
        return -GFP_ECUDA;
    int i = 0;
    for (; i < n && i < max; i++) {
        if (ms && cudaEventElapsedTime(&ms[i], p->ev[i], p->ev[i + 1]) != cudaSuccess)
            return -GFP_ECUDA;
        if (pass)
            pass[i] = p->ev_pass[i];
    }
    return i;
}

int gfp_fft_exec(const gfp_fft_plan *cp, const uint64_t *in, uint64_t *out, uint64_t *work,
                 int64_t batch, int inverse, void *stream)
{
    gfp_fft_plan *p = const_cast<gfp_fft_plan *>(cp);
    if (!p || !in || !out || !work || batch < 1)
        return GFP_EINVAL;
    begin_call(p);
    // the batch is the pass kernels' grid.y: chunks of at most 65535 vectors
    const int64_t vw = (int64_t)p->k * p->N;
    for (int64_t b0 = 0; b0 < batch; b0 += GFP_MAX_GRID_Y) {
        const int64_t nb = batch - b0 < GFP_MAX_GRID_Y ? batch - b0 : GFP_MAX_GRID_Y;
        const int err = run_transform(p, in + b0 * vw, out + b0 * vw, work, nullptr, nb,
                                      inverse ? 1 : 0, 1, 1, (cudaStream_t)stream);
        if (err)
            return err;
    }
    return GFP_OK;
}

int gfp_fft_exec_ex(const gfp_fft_plan *cp, const uint64_t *in, uint64_t *out, uint64_t *work,
                    int64_t batch, int inverse, int in_canon, int out_canon,
                    const gfp_fft_plan *ft, int64_t ft_row0, int ft_inverse, void *stream)
{
    gfp_fft_plan *p = const_cast<gfp_fft_plan *>(cp);
    if (!p || !in || !out || !work || batch < 1 || ft_row0 < 0)
        return GFP_EINVAL;
    if (ft && (in_canon || ft->k != p->k || !em_io_supported(p)))
        return ft->k != p->k || in_canon ? GFP_EINVAL : GFP_EUNSUPPORTED;
    begin_call(p);
    PassIO io = {nullptr, nullptr, 0, 0, nullptr, 0, ft, ft_row0, ft_inverse ? 1 : 0};
    return run_transform(p, in, out, work, nullptr, batch, inverse ? 1 : 0, in_canon ? 1 : 0,
                         out_canon ? 1 : 0, (cudaStream_t)stream, ft ? &io : nullptr);
}

int gfp_fft_exec_exchange(const gfp_fft_plan *cp, const uint64_t *in, uint64_t *scratch,
                          uint64_t *work, int64_t batch, int inverse, int in_canon, int out_canon,
                          uint64_t *const *dst, int world, int rank, void *stream)
{
    gfp_fft_plan *p = const_cast<gfp_fft_plan *>(cp);
    if (!p || !in || !scratch || !work || !dst || batch < 1 || world < 1 || rank < 0 ||
        rank >= world || p->N % world)
        return GFP_EINVAL;
    for (int g = 0; g < world; g++)
        if (!dst[g])
            return GFP_EINVAL;
    if (p->k != 8 || p->e < 2 || world > 8 || (world & (world - 1)) || batch % 8 ||
        !em_io_supported(p))
        return GFP_EUNSUPPORTED;
    begin_call(p);
    PassIO io = {nullptr, nullptr, 0, 0, nullptr, 0, nullptr, 0, 0, dst, world, rank};
    return run_transform(p, in, scratch, work, nullptr, batch, inverse ? 1 : 0, in_canon ? 1 : 0,
                         out_canon ? 1 : 0, (cudaStream_t)stream, &io);
}

// poly-multiply with the fused middle kernel: buffers o (the result), G,
// scratch, scratch_b hold `nb` vectors each; f and g are never written
static int poly_mul_fused(gfp_fft_plan *p, const u64 *f, const u64 *g, u64 *o, u64 *G, u64 *scratch,
                          u64 *scratch_b, int64_t nb, cudaStream_t st,
                          const PassIO *em_fwd = nullptr, const PassIO *em_inv = nullptr)
{
    const int e = p->e;
    const u64 *sf = f, *sg = g;
    u64 *bf[2] = {o, scratch}, *bg[2] = {G, scratch_b};
    int64_t Ns = 1;
    int rcode = GFP_OK;
    for (int pass = 0; pass + 1 < e; pass++) {  // forward passes 0 .. e-2
        u64 *df = bf[pass & 1] == sf ? bf[(pass & 1) ^ 1] : bf[pass & 1];
        u64 *dg = bg[pass & 1] == sg ? bg[(pass & 1) ^ 1] : bg[pass & 1];
        timing_mark(p, st, -1);
        rcode = launch_pass<8>(p, sf, df, sg, dg, nullptr, nb, Ns, 0, 0, 0, pass == 0, em_fwd, st);
        if (rcode)
            return rcode;
        timing_mark(p, st, pass);
        p->last_launches++;
        sf = df;
        sg = dg;
        Ns *= p->K;
    }
    // fused middle: (sf, sg) -> the buffer of {o, scratch} that is not sf,
    // chosen so that the inverse's remaining e - 1 passes end in o
    // (ping-pong: the last launch must land in o)
    const int rem = e - 1;  // inverse launches after the fused one
    u64 *dm = (rem % 2 == 0) ? o : scratch;
    if (dm == sf)  // (e.g. e = 2: the forward pass 0 wrote o): use the other and copy at the end
        dm = dm == o ? scratch : o;
    timing_mark(p, st, -1);
    rcode = launch_poly_mid(p, sf, sg, dm, nb, st);
    if (rcode)
        return rcode;
    timing_mark(p, st, e - 1);
    p->last_launches++;
    const u64 *src = dm;
    Ns = p->K;
    for (int pass = 1; pass < e; pass++) {  // inverse passes 1 .. e-1
        u64 *dst = src == o ? scratch : o;
        const int last = pass + 1 == e;
        timing_mark(p, st, -1);
        rcode = launch_pass<8>(p, src, dst, nullptr, nullptr, nullptr, nb, Ns, 1, last, last, 0,
                               em_inv, st);
        if (rcode)
            return rcode;
        timing_mark(p, st, pass);
        p->last_launches++;
        src = dst;
        Ns *= p->K;
    }
    if (em_inv && em_inv->out)
        return cuda_status();  // the last pass wrote the element-major output
    if (src != o)
        cudaMemcpyAsync(o, src, sizeof(u64) * (size_t)p->k * p->N * nb, cudaMemcpyDeviceToDevice,
                        st);
    return cuda_status();
}

int gfp_poly_mul(const gfp_fft_plan *cp, const uint64_t *f, const uint64_t *g, uint64_t *out,
                 uint64_t *work, int64_t batch, void *stream)
{
    gfp_fft_plan *p = const_cast<gfp_fft_plan *>(cp);
    if (!p || !f || !g || !out || !work || batch < 1)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    begin_call(p);
    // both operands share grid.y: chunks of at most 32767 products
    constexpr int64_t CH = GFP_MAX_GRID_Y / 2;
    const int64_t ew = (int64_t)p->k * p->N;
    int err = GFP_OK;
    for (int64_t b0 = 0; b0 < batch && !err; b0 += CH) {
        const int64_t nb = batch - b0 < CH ? batch - b0 : CH;
        const int64_t vw = ew * nb;
        u64 *G = work;  // DFT(g)
        u64 *scratch = work + vw;
        u64 *scratch_b = work + 2 * vw;
        u64 *o = out + b0 * ew;
        // o = DFT(f) and G = DFT(g) in the same launches; the spectra stay
        // balanced lazy digits, only the product is canonicalised
        if (p->generic) {
            err = run_generic(p, f + b0 * ew, o, scratch, nb, 0, st);
            if (!err)
                err = run_generic(p, g + b0 * ew, G, scratch_b, nb, 0, st);
        } else if (poly_mid_supported(p) &&
                   !(((uintptr_t)o | (uintptr_t)G | (uintptr_t)scratch | (uintptr_t)scratch_b) & 15)) {
            // forward passes 0 .. e-2 of both operands, then ONE kernel for the
            // forward last pass + pointwise product + inverse first pass, then
            // the inverse passes 1 .. e-1 (2 e - 1 launches instead of 2 e)
            err = poly_mul_fused(p, f + b0 * ew, g + b0 * ew, o, G, scratch, scratch_b, nb, st);
            continue;
        } else {
            err = run_transform2(p, f + b0 * ew, o, scratch, g + b0 * ew, G, scratch_b, nullptr,
                                 nb, 0, 1, 0, st);
        }
        if (!err)  // o = IDFT(o .* G), the pointwise product fused into pass 0
            err = run_transform(p, o, o, scratch, G, nb, 1, 0, 1, st);
    }
    return err;
}

static int ensure_host_scratch(gfp_fft_plan *p, int64_t words)
{
    if (p->h_words >= words)
        return GFP_OK;
    cudaFree(p->h_dev);
    p->h_dev = nullptr;
    p->h_words = 0;
    if (cudaMalloc(&p->h_dev, sizeof(u64) * (size_t)words) != cudaSuccess)
        return GFP_ENOMEM;
    p->h_words = words;
    return GFP_OK;
}

// Device alias of a host pointer: pinned (cudaHostAlloc / cudaHostRegister)
// memory is mapped into the device address space, so the first and last
// transform passes read and write it directly over PCIe (no staging copy,
// no transpose kernel).  Pageable memory returns nullptr: the caller stages.
static u64 *mapped_alias(const void *h)
{
    // the pass kernels access element-major host rows with 16 B vectors
    if ((uintptr_t)h & 15)
        return nullptr;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type == cudaMemoryTypeHost && at.devicePointer)
        return (u64 *)at.devicePointer;
    return nullptr;
}

// the staged route for kernels without element-major I/O (k != 8): one copy
// of each operand's nf / ng elements, one batched transpose that zero-pads to
// N, the product, one batched transpose of its first n_out elements, one copy
// back -- O(1) copies and launches per call, whatever the batch
static int poly_mul_host_staged(gfp_fft_plan *p, const u64 *f, int64_t nf, const u64 *g,
                                int64_t ng, u64 *out, int64_t n_out, int64_t batch,
                                cudaStream_t st)
{
    const int k = p->k;
    const int64_t N = p->N, vw = (int64_t)k * N * batch;
    int err = ensure_host_scratch(p, 7 * vw);  // staging, operands, poly_mul workspace (3 vw)
    if (err)
        return err;
    u64 *hf = p->h_dev, *hg = hf + vw, *df = hg + vw, *dg = df + vw, *w = dg + vw;
    cudaMemcpyAsync(hf, f, sizeof(u64) * k * nf * batch, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(hg, g, sizeof(u64) * k * ng * batch, cudaMemcpyHostToDevice, st);
    err = transpose_batched(hf, df, batch, nf, N, k, 1, st);
    if (!err)
        err = transpose_batched(hg, dg, batch, ng, N, k, 1, st);
    if (!err)
        err = gfp_poly_mul(p, df, dg, df, w, batch, st);
    if (err)
        return err;
    const int64_t launches = p->last_launches;
    err = transpose_batched(df, hf, batch, n_out, N, k, 0, st);
    if (err)
        return err;
    cudaMemcpyAsync(out, hf, sizeof(u64) * k * n_out * batch, cudaMemcpyDeviceToHost, st);
    p->last_launches = launches + 3;
    return GFP_OK;
}

int gfp_poly_mul_host2(gfp_fft_plan *p, const uint64_t *f, int64_t nf, const uint64_t *g,
                       int64_t ng, uint64_t *out, int64_t batch, void *stream)
{
    if (!p || !f || !g || !out || batch < 1 || nf < 1 || ng < 1 || nf > p->N || ng > p->N)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = p->k;
    const int64_t N = p->N, vw = (int64_t)k * N * batch;
    const int64_t n_out = nf + ng - 1 < N ? nf + ng - 1 : N;
    begin_call(p);
    if (!em_io_supported(p)) {
        int err = poly_mul_host_staged(p, f, nf, g, ng, out, n_out, batch, st);
        if (err)
            return err;
        if (cudaStreamSynchronize(st) != cudaSuccess)
            return GFP_ECUDA;
        return cuda_status();
    }
    const u64 *mf = mapped_alias(f), *mg = mapped_alias(g);
    u64 *mo = mapped_alias(out);
    // device workspace: the two spectra, two ping-pong buffers, and staging
    // for whichever operand is not mapped
    const int64_t stage_words = (mf ? 0 : k * nf * batch) + (mg ? 0 : k * ng * batch) +
                                (mo ? 0 : k * n_out * batch);
    int err = ensure_host_scratch(p, 4 * vw + stage_words);
    if (err)
        return err;
    u64 *F = p->h_dev, *G = F + vw, *s1 = G + vw, *s2 = s1 + vw, *stg = s2 + vw;
    if (!mf) {
        cudaMemcpyAsync(stg, f, sizeof(u64) * k * nf * batch, cudaMemcpyHostToDevice, st);
        mf = stg;
        stg += k * nf * batch;
    }
    if (!mg) {
        cudaMemcpyAsync(stg, g, sizeof(u64) * k * ng * batch, cudaMemcpyHostToDevice, st);
        mg = stg;
        stg += k * ng * batch;
    }
    u64 *dout = mo ? mo : stg;
    // forward transforms of both operands in the same launches; pass 0 reads
    // the element-major operands (zero past nf / ng); spectra stay lazy
    PassIO e1 = {mf, mg, nf, ng, nullptr, 0, nullptr, 0, 0};
    PassIO e2 = {nullptr, nullptr, 0, 0, dout, n_out, nullptr, 0, 0};
    if (poly_mid_supported(p) &&  // the middle as one kernel (gfp_pmid44t.cuh; TMA: 16 B alignment)
        !(((uintptr_t)F | (uintptr_t)G | (uintptr_t)s1 | (uintptr_t)s2) & 15)) {
        err = poly_mul_fused(p, F, G, F, G, s1, s2, batch, st, &e1, &e2);
    } else {
        err = run_transform2(p, F, F, s1, G, G, s2, nullptr, batch, 0, 1, 0, st, &e1);
        if (!err) {
            // inverse of F .* G (pointwise product fused into pass 0, N^-1 into
            // the last pass), which writes the first n_out elements element-major
            err = run_transform(p, F, F, s1, G, batch, 1, 0, 1, st, &e2);
        }
    }
    if (!err && !mo) {
        cudaMemcpyAsync(out, dout, sizeof(u64) * k * n_out * batch, cudaMemcpyDeviceToHost, st);
    }
    if (err)
        return err;
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return GFP_ECUDA;
    return cuda_status();
}

int gfp_poly_mul_host(gfp_fft_plan *p, const uint64_t *f, const uint64_t *g, uint64_t *out,
                      int64_t batch, void *stream)
{
    if (!p)
        return GFP_EINVAL;
    return gfp_poly_mul_host2(p, f, p->N, g, p->N, out, batch, stream);
}

// one chunk of gfp_fft_exec_host: transforms [b0, b0 + nb) of the host
// array v (element-major), on stream s with device buffers a / b / w (+ stg
// for pageable input), nb k N words each
static int exec_host_chunk(gfp_fft_plan *p, uint64_t *v, u64 *mv, int64_t b0, int64_t nb,
                           int inverse, u64 *a, u64 *b, u64 *w, u64 *stg, cudaStream_t s)
{
    const int k = p->k;
    const int64_t N = p->N, ew = (int64_t)k * N, vw = ew * nb;
    const u64 *src;
    if (mv) {
        src = mv + b0 * ew;
    } else {
        cudaMemcpyAsync(stg, v + b0 * ew, sizeof(u64) * vw, cudaMemcpyHostToDevice, s);
        src = stg;
    }
    int err;
    if (!em_io_supported(p)) {
        // no element-major kernel for this k: one batched transpose on each
        // side of the transform
        err = transpose_batched(src, b, nb, N, N, k, 1, s);
        if (!err)
            err = run_transform(p, b, b, w, nullptr, nb, inverse ? 1 : 0, 1, 1, s);
        if (!err)
            err = transpose_batched(b, a, nb, N, N, k, 0, s);
        if (err)
            return err;
        p->last_launches += 2;
        cudaMemcpyAsync(v + b0 * ew, a, sizeof(u64) * vw, cudaMemcpyDeviceToHost, s);
        return GFP_OK;
    }
    // a single-pass transform would read and write v in the same launch:
    // stage its output
    const bool stage_out = !mv || p->e == 1;
    PassIO em = {src, nullptr, N, 0, stage_out ? a : mv + b0 * ew, N, nullptr, 0, 0};
    err = run_transform(p, b, b, w, nullptr, nb, inverse ? 1 : 0, 1, 1, s, &em);
    if (err)
        return err;
    if (stage_out)
        cudaMemcpyAsync(v + b0 * ew, a, sizeof(u64) * vw, cudaMemcpyDeviceToHost, s);
    return GFP_OK;
}

int gfp_fft_exec_host(gfp_fft_plan *p, uint64_t *v, int64_t batch, int inverse, void *stream)
{
    if (!p || !v || batch < 1)
        return GFP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = p->k;
    const int64_t N = p->N, ew = (int64_t)k * N;
    begin_call(p);
    u64 *mv = em_io_supported(p) ? mapped_alias(v) : nullptr;
    // batches of more than ~128 MiB go through the two-stream pipeline in
    // chunks of transforms: one chunk's host traffic overlaps the other's
    // kernels (and H2D overlaps D2H)
    int64_t per = HOST_CHUNK_WORDS / ew;
    if (per < 1)
        per = 1;
    if (per > batch)
        per = batch;
    if (per > GFP_MAX_GRID_Y)
        per = GFP_MAX_GRID_Y;
    const int64_t nchunks = (batch + per - 1) / per;
    const int nst = nchunks > 1 ? 2 : 1;
    const int64_t cw = ew * per;  // words of one chunk buffer
    int err = ensure_host_scratch(p, (int64_t)nst * 4 * cw);
    if (err)
        return err;
    HostPipe hp;
    if (nst > 1)
        err = host_pipe_begin(hp, st);
    for (int64_t c = 0; c < nchunks && !err; c++) {
        cudaStream_t s = nst > 1 ? hp.s[c & 1] : st;
        u64 *a = p->h_dev + (c & (nst - 1)) * 4 * cw, *b = a + cw, *w = b + cw, *stg = w + cw;
        const int64_t b0 = c * per, nb = batch - b0 < per ? batch - b0 : per;
        err = exec_host_chunk(p, v, mv, b0, nb, inverse, a, b, w, stg, s);
    }
    if (nst > 1) {
        const int e2 = host_pipe_end(hp, st);
        err = err ? err : e2;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && !err)
        err = GFP_ECUDA;
    return err ? err : cuda_status();
}

}  // extern "C"
