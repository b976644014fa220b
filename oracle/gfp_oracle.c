/*
 * gfp_oracle.c -- CPU restatement of the reference `gfpfft` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_1811_01490_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It is
 * never linked into, called by, or used as a fallback for the product.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * vectors produced by running the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py, which imports /root/reference/pkg/src).
 *
 * Layout: elements are element-major, k little-endian u64 radix-r digits per
 * element (the reference's tuple order, and the GFPV payload order of
 * bench_cli.py:88-116).
 *
 * What is restated, with the reference file:line it follows:
 *   MT19937 seeding / getrandbits / randrange   CPython `random` (the input
 *                                               convention of bench_cli.py:383,394)
 *   gfp_encode                                  gfp_field.py:69-79
 *   gfp_add / gfp_sub / gfp_mul_pow_r           gfp_field.py:82-161
 *   word primes + Montgomery                    word_field.py:15-16, 102-171
 *   word_primitive_root                         word_field.py:174-196
 *   negacyclic convolution (theta-weighted)     gfp_mult.py:280-305, 335-378
 *   crt_combine                                 gfp_mult.py:184-198
 *   lhc_decompose                               gfp_mult.py:96-116
 *   gfp_mul_fft final shift-and-add             gfp_mult.py:416-501
 *   check_prime_compat                          gfp_mult.py:207-226
 *   base_case_ops (_gen_layers + swap cycles)   fft.py:114-168
 *   stride_permutation                          fft.py:34-56
 *   _twiddle_level_cheap                        fft.py:84-103
 *   FftPlan / build_plan                        fft.py:199-275
 *   dft_general / dft_inverse                   fft.py:298-370
 *   gfp_find_nth_root / gfp_primitive_root      gfp_field.py:164-237
 *   _gfp_root                                   bench_cli.py:398-402
 *   poly multiply (composition, no ref symbol)
 *
 * The reference is single-threaded; the optional OpenMP loops below split
 * the same independent blocks the reference's ThreadPoolExecutor splits
 * (fft.py:278-295), so results are identical for any thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef uint32_t u32;
typedef unsigned __int128 u128;
typedef __int128 i128;

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ECONFIG 2
#define ORC_ENOMEM 3

/* ======================================================================== */
/* MT19937 with CPython's seeding (Modules/_randommodule.c)                  */

typedef struct {
    u32 mt[624];
    int mti;
} mt_state;

static void mt_init_genrand(mt_state *s, u32 seed)
{
    s->mt[0] = seed;
    for (int i = 1; i < 624; i++)
        s->mt[i] = 1812433253U * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (u32)i;
    s->mti = 624;
}

static void mt_init_by_array(mt_state *s, const u32 *key, size_t len)
{
    mt_init_genrand(s, 19650218U);
    size_t i = 1, j = 0;
    size_t k = 624 > len ? 624 : len;
    for (; k; k--) {
        s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1664525U))
                   + key[j] + (u32)j;
        i++;
        j++;
        if (i >= 624) {
            s->mt[0] = s->mt[623];
            i = 1;
        }
        if (j >= len)
            j = 0;
    }
    for (k = 623; k; k--) {
        s->mt[i] = (s->mt[i] ^ ((s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) * 1566083941U))
                   - (u32)i;
        i++;
        if (i >= 624) {
            s->mt[0] = s->mt[623];
            i = 1;
        }
    }
    s->mt[0] = 0x80000000U;
}

static u32 mt_next(mt_state *s)
{
    static const u32 mag01[2] = {0x0U, 0x9908b0dfU};
    u32 y;
    if (s->mti >= 624) {
        int kk;
        for (kk = 0; kk < 624 - 397; kk++) {
            y = (s->mt[kk] & 0x80000000U) | (s->mt[kk + 1] & 0x7fffffffU);
            s->mt[kk] = s->mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1U];
        }
        for (; kk < 623; kk++) {
            y = (s->mt[kk] & 0x80000000U) | (s->mt[kk + 1] & 0x7fffffffU);
            s->mt[kk] = s->mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1U];
        }
        y = (s->mt[623] & 0x80000000U) | (s->mt[0] & 0x7fffffffU);
        s->mt[623] = s->mt[396] ^ (y >> 1) ^ mag01[y & 1U];
        s->mti = 0;
    }
    y = s->mt[s->mti++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680U;
    y ^= (y << 15) & 0xefc60000U;
    y ^= (y >> 18);
    return y;
}

/* random.Random(seed) for a non-negative integer seed < 2^64 */
static void mt_seed_u64(mt_state *s, u64 seed)
{
    u32 key[2];
    size_t len;
    key[0] = (u32)seed;
    key[1] = (u32)(seed >> 32);
    len = key[1] ? 2 : 1;
    mt_init_by_array(s, key, len);
}

/* getrandbits(nbits) into little-endian u64 limbs (nl = ceil(nbits/64)) */
static void mt_getrandbits(mt_state *s, int nbits, u64 *out, int nl)
{
    memset(out, 0, sizeof(u64) * (size_t)nl);
    if (nbits <= 32) {
        out[0] = mt_next(s) >> (32 - nbits);
        return;
    }
    int words = (nbits - 1) / 32 + 1;
    int k = nbits;
    for (int i = 0; i < words; i++, k -= 32) {
        u32 r = mt_next(s);
        if (k < 32)
            r >>= (32 - k);
        out[i / 2] |= (u64)r << (32 * (i & 1));
    }
}

/* ======================================================================== */
/* small multi-limb helpers (little-endian u64 limbs)                        */

static int big_cmp(const u64 *a, const u64 *b, int n)
{
    for (int i = n - 1; i >= 0; i--) {
        if (a[i] != b[i])
            return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

static int big_bitlen(const u64 *a, int n)
{
    for (int i = n - 1; i >= 0; i--)
        if (a[i])
            return 64 * i + 64 - __builtin_clzll(a[i]);
    return 0;
}

/* a = a * m (+ add); returns carry limb */
static u64 big_mul_small(u64 *a, int n, u64 m, u64 add)
{
    u64 carry = add;
    for (int i = 0; i < n; i++) {
        u128 t = (u128)a[i] * m + carry;
        a[i] = (u64)t;
        carry = (u64)(t >> 64);
    }
    return carry;
}

/* a = a / d, returns remainder */
static u64 big_divmod_small(u64 *a, int n, u64 d)
{
    u128 rem = 0;
    for (int i = n - 1; i >= 0; i--) {
        u128 cur = (rem << 64) | a[i];
        a[i] = (u64)(cur / d);
        rem = cur % d;
    }
    return (u64)rem;
}

/* p - 1 = r^k as limbs, nl limbs (nl >= k + 1) */
static void big_r_pow_k(u64 *out, int nl, u64 r, int k)
{
    memset(out, 0, sizeof(u64) * (size_t)nl);
    out[0] = 1;
    for (int i = 0; i < k; i++)
        big_mul_small(out, nl, r, 0);
}

static inline int limbs_for(int k) { return k + 2; }

/* ======================================================================== */
/* GFP digit arithmetic (gfp_field.py)                                       */

/* gfp_encode (gfp_field.py:69-79) of n in [0, p), n given as limbs (destroyed) */
static void gfp_encode_big(u64 *n, int nl, const u64 *pm1, int k, u64 r, u64 *out)
{
    if (big_cmp(n, pm1, nl) == 0) {
        memset(out, 0, sizeof(u64) * (size_t)k);
        out[k - 1] = r;
        return;
    }
    for (int i = 0; i < k; i++)
        out[i] = big_divmod_small(n, nl, r);
}

static int is_canonical(const u64 *x, int k, u64 r)
{
    int all = 1;
    for (int i = 0; i < k; i++)
        if (x[i] >= r)
            all = 0;
    if (all)
        return 1;
    if (x[k - 1] != r)
        return 0;
    for (int i = 0; i < k - 1; i++)
        if (x[i])
            return 0;
    return 1;
}

/* gfp_add (gfp_field.py:82-109); z may alias x or y */
static void gfp_add(const u64 *x, const u64 *y, u64 *z, int k, u64 r)
{
    u64 t[256];
    int carry = 0;
    for (int i = 0; i < k; i++) {
        u128 s = (u128)x[i] + y[i] + (u64)carry;
        if (s >= r) {
            s -= r;
            carry = 1;
        } else {
            carry = 0;
        }
        t[i] = (u64)s;
    }
    if (carry) {
        int i0;
        for (i0 = 0; i0 < k; i0++) {
            if (t[i0]) {
                for (int j = 0; j < i0; j++)
                    t[j] = r - 1;
                t[i0] -= 1;
                break;
            }
        }
        if (i0 == k) {
            memset(z, 0, sizeof(u64) * (size_t)k);
            z[k - 1] = r;
            return;
        }
    }
    memcpy(z, t, sizeof(u64) * (size_t)k);
}

/* gfp_sub (gfp_field.py:112-135) */
static void gfp_sub(const u64 *x, const u64 *y, u64 *z, int k, u64 r)
{
    u64 t[256];
    int borrow = 0;
    for (int i = 0; i < k; i++) {
        i128 d = (i128)x[i] - (i128)y[i] - borrow;
        if (d < 0) {
            d += r;
            borrow = 1;
        } else {
            borrow = 0;
        }
        t[i] = (u64)d;
    }
    if (borrow) {
        int i;
        for (i = 0; i < k; i++) {
            if ((u128)t[i] + 1 < r) {
                t[i] += 1;
                break;
            }
            t[i] = 0;
        }
        if (i == k) {
            memset(z, 0, sizeof(u64) * (size_t)k);
            z[k - 1] = r;
            return;
        }
    }
    memcpy(z, t, sizeof(u64) * (size_t)k);
}

/* gfp_mul_pow_r (gfp_field.py:138-161); 0 <= i <= 2k */
static int gfp_mul_pow_r(const u64 *x_in, int i, u64 *z, int k, u64 r)
{
    u64 x[256], a[256], b[256];
    if (i < 0 || i > 2 * k)
        return ORC_EINVAL;
    i %= 2 * k;
    memcpy(x, x_in, sizeof(u64) * (size_t)k);
    if (i == 0) {
        memcpy(z, x, sizeof(u64) * (size_t)k);
        return ORC_OK;
    }
    if (i >= k) {
        u64 zero[256];
        memset(zero, 0, sizeof(u64) * (size_t)k);
        gfp_sub(zero, x, x, k, r);
        i -= k;
        if (i == 0) {
            memcpy(z, x, sizeof(u64) * (size_t)k);
            return ORC_OK;
        }
    }
    for (int j = 0; j < k; j++) {
        b[j] = j < i ? 0 : x[j - i];
        a[j] = j < i ? x[k - i + j] : 0;
    }
    if (x[k - 1] == r) {
        a[i - 1] -= r;
        a[i] += 1;
    }
    gfp_sub(b, a, z, k, r);
    return ORC_OK;
}

/* ======================================================================== */
/* word primes in Montgomery form (word_field.py)                            */

static const u64 ORC_P1 = 4179340454199820289ULL;
static const u64 ORC_P2 = 2485986994308513793ULL;

typedef struct {
    u64 q, q_neg_inv, r2, one_mont;
} word_prime;

static word_prime word_prime_make(u64 q)
{
    word_prime c;
    c.q = q;
    u64 inv = q; /* Newton: inv = q^{-1} mod 2^64 */
    for (int i = 0; i < 6; i++)
        inv *= 2 - q * inv;
    c.q_neg_inv = (u64)0 - inv;
    c.one_mont = (u64)(((u128)1 << 64) % q);
    c.r2 = (u64)(((u128)c.one_mont * c.one_mont) % q);
    return c;
}

static inline u64 mont_mul(const word_prime *c, u64 a, u64 b)
{
    u128 t = (u128)a * b;
    u64 d = (u64)t * c->q_neg_inv;
    t = (t + (u128)c->q * d) >> 64;
    u64 v = (u64)t;
    return v >= c->q ? v - c->q : v;
}

static u64 mont_in(const word_prime *c, u64 a) { return mont_mul(c, a, c->r2); }
static u64 mont_out(const word_prime *c, u64 a) { return mont_mul(c, a, 1); }

static u64 word_pow(const word_prime *c, u64 a, u64 e)
{
    u64 acc = c->one_mont, base = a;
    while (e) {
        if (e & 1)
            acc = mont_mul(c, base, acc);
        base = mont_mul(c, base, base);
        e >>= 1;
    }
    return acc;
}

static u64 mont_inv(const word_prime *c, u64 a) { return word_pow(c, a, c->q - 2); }

/* word_primitive_root(ctx, n, seed=0) (word_field.py:174-196) */
static u64 word_primitive_root(const word_prime *c, u64 n)
{
    if (n == 1)
        return c->one_mont;
    u64 minus_one = mont_in(c, c->q - 1);
    mt_state s;
    mt_seed_u64(&s, 0);
    u64 e = (c->q - 1) / n;
    u64 width = c->q - 1; /* randrange(1, q) = 1 + _randbelow(q - 1) */
    int nb = 64 - __builtin_clzll(width);
    for (;;) {
        u64 v[2];
        do {
            mt_getrandbits(&s, nb, v, 1);
        } while (v[0] >= width);
        u64 cand = v[0] + 1;
        u64 g = word_pow(c, mont_in(c, cand), e);
        if (word_pow(c, g, n / 2) == minus_one)
            return g;
    }
}

/* ======================================================================== */
/* base_case_ops (fft.py:114-168)                                            */

typedef struct {
    int kind; /* 0 dft2, 1 tw, 2 swap */
    int i, j;
} base_op;

/* _gen_layers: returns number of layers, fills layers[l] lists */
typedef struct {
    base_op *ops;
    int n;
} op_layer;

static int gen_layers(const int *pos, int s, int unit, op_layer *layers, int *order)
{
    /* layers must have room for 2*log2(s) entries; caller frees ops */
    if (s == 2) {
        layers[0].ops = (base_op *)malloc(sizeof(base_op));
        layers[0].ops[0].kind = 0;
        layers[0].ops[0].i = pos[0];
        layers[0].ops[0].j = pos[1];
        layers[0].n = 1;
        order[0] = pos[0];
        order[1] = pos[1];
        return 1;
    }
    int half = s / 2;
    int *pa = (int *)malloc(sizeof(int) * (size_t)half);
    int *pb = (int *)malloc(sizeof(int) * (size_t)half);
    int *oa = (int *)malloc(sizeof(int) * (size_t)half);
    int *ob = (int *)malloc(sizeof(int) * (size_t)half);
    for (int i = 0; i < half; i++) {
        pa[i] = pos[2 * i];
        pb[i] = pos[2 * i + 1];
    }
    op_layer la[64], lb[64];
    int na = gen_layers(pa, half, unit * 2, la, oa);
    int nb = gen_layers(pb, half, unit * 2, lb, ob);
    (void)nb;
    for (int l = 0; l < na; l++) {
        layers[l].n = la[l].n + lb[l].n;
        layers[l].ops = (base_op *)malloc(sizeof(base_op) * (size_t)layers[l].n);
        memcpy(layers[l].ops, la[l].ops, sizeof(base_op) * (size_t)la[l].n);
        memcpy(layers[l].ops + la[l].n, lb[l].ops, sizeof(base_op) * (size_t)lb[l].n);
        free(la[l].ops);
        free(lb[l].ops);
    }
    int nl = na;
    layers[nl].n = half - 1;
    layers[nl].ops = (base_op *)malloc(sizeof(base_op) * (size_t)(half > 1 ? half - 1 : 1));
    for (int t = 1; t < half; t++) {
        layers[nl].ops[t - 1].kind = 1;
        layers[nl].ops[t - 1].i = ob[t];
        layers[nl].ops[t - 1].j = t * unit;
    }
    nl++;
    int *merged = (int *)malloc(sizeof(int) * (size_t)s);
    for (int i = 0; i < half; i++) {
        merged[2 * i] = oa[i];
        merged[2 * i + 1] = ob[i];
    }
    layers[nl].n = half;
    layers[nl].ops = (base_op *)malloc(sizeof(base_op) * (size_t)half);
    for (int i = 0; i < half; i++) {
        layers[nl].ops[i].kind = 0;
        layers[nl].ops[i].i = merged[2 * i];
        layers[nl].ops[i].j = merged[2 * i + 1];
    }
    nl++;
    for (int i = 0; i < half; i++) {
        order[i] = merged[2 * i];
        order[half + i] = merged[2 * i + 1];
    }
    free(pa);
    free(pb);
    free(oa);
    free(ob);
    free(merged);
    return nl;
}

/* flat op list; returns count (or -1 on bad K); caller frees *out */
static int base_case_ops(int K, base_op **out)
{
    if (K != 8 && K != 16 && K != 32 && K != 64)
        return -1;
    int pos[64], order[64];
    for (int i = 0; i < K; i++)
        pos[i] = i;
    op_layer layers[64];
    int nl = gen_layers(pos, K, 1, layers, order);
    int total = 0;
    for (int l = 0; l < nl; l++)
        total += layers[l].n;
    base_op *ops = (base_op *)malloc(sizeof(base_op) * (size_t)(total + K));
    int n = 0;
    for (int l = 0; l < nl; l++) {
        memcpy(ops + n, layers[l].ops, sizeof(base_op) * (size_t)layers[l].n);
        n += layers[l].n;
        free(layers[l].ops);
    }
    int seen[64] = {0};
    for (int start = 0; start < K; start++) {
        if (seen[start] || order[start] == start)
            continue;
        int cycle[64], cl = 0;
        cycle[cl++] = start;
        seen[start] = 1;
        int t = order[start];
        while (t != start) {
            cycle[cl++] = t;
            seen[t] = 1;
            t = order[t];
        }
        int head = cycle[0];
        for (int c = 1; c < cl; c++) {
            ops[n].kind = 2;
            ops[n].i = head;
            ops[n].j = cycle[c];
            n++;
            head = cycle[c];
        }
    }
    *out = ops;
    return n;
}

/* ======================================================================== */
/* negacyclic convolution mod a word prime (gfp_mult.py:280-378)            */

typedef struct {
    word_prime ctx;
    int n;
    u64 in_table[128], out_table[128];
    u64 fwd_pows[128], inv_pows[128]; /* omega^t / omega^-t (mont) */
    base_op *ops;
    int nops;
} nega_plan;

static int transform_is_base(int n) { return n == 8 || n == 16 || n == 32 || n == 64; }

static void nega_plan_make(nega_plan *pl, u64 q, int k)
{
    word_prime c = word_prime_make(q);
    pl->ctx = c;
    pl->n = k;
    u64 theta = word_primitive_root(&c, 2 * (u64)k);
    u64 omega = mont_mul(&c, theta, theta);
    u64 tm = c.one_mont;
    for (int i = 0; i < k; i++) {
        pl->in_table[i] = mont_mul(&c, tm, c.r2);
        tm = mont_mul(&c, tm, theta);
    }
    u64 theta_inv = mont_inv(&c, theta);
    u64 acc = mont_inv(&c, mont_in(&c, (u64)k % q));
    for (int i = 0; i < k; i++) {
        pl->out_table[i] = mont_out(&c, acc);
        acc = mont_mul(&c, acc, theta_inv);
    }
    u64 omega_inv = mont_inv(&c, omega);
    pl->fwd_pows[0] = pl->inv_pows[0] = c.one_mont;
    for (int t = 1; t < k; t++) {
        pl->fwd_pows[t] = mont_mul(&c, pl->fwd_pows[t - 1], omega);
        pl->inv_pows[t] = mont_mul(&c, pl->inv_pows[t - 1], omega_inv);
    }
    pl->ops = NULL;
    pl->nops = 0;
    if (transform_is_base(k))
        pl->nops = base_case_ops(k, &pl->ops);
}

/* forward (inv=0) or unscaled inverse (inv=1) k-point DFT over Z/qZ, in place.
   dft_base over MontField (fft.py:186-193) for k in BASE_SIZES, the naive DFT
   of gfp_mult.py:323-332 otherwise. */
static void nega_transform(const nega_plan *pl, u64 *v, int inv)
{
    const word_prime *c = &pl->ctx;
    const u64 *pows = inv ? pl->inv_pows : pl->fwd_pows;
    int n = pl->n;
    u64 q = c->q;
    if (pl->ops) {
        for (int o = 0; o < pl->nops; o++) {
            const base_op *op = &pl->ops[o];
            if (op->kind == 0) {
                u64 a = v[op->i], b = v[op->j];
                u64 s = a + b;
                v[op->i] = s >= q ? s - q : s;
                v[op->j] = a >= b ? a - b : a + q - b;
            } else if (op->kind == 1) {
                v[op->i] = mont_mul(c, v[op->i], pows[op->j]);
            } else {
                u64 t = v[op->i];
                v[op->i] = v[op->j];
                v[op->j] = t;
            }
        }
    } else if (n > 1) {
        u64 out[128];
        for (int i = 0; i < n; i++) {
            u128 s = 0;
            for (int j = 0; j < n; j++)
                s += mont_mul(c, v[j], pows[(i * j) % n]);
            out[i] = (u64)(s % q);
        }
        memcpy(v, out, sizeof(u64) * (size_t)n);
    }
}

/* ======================================================================== */
/* CRT + LHC + gfp_mul_fft (gfp_mult.py:131-226, 396-501)                    */

typedef struct {
    nega_plan p1, p2;
    u64 m1_red, m2_red;
    u128 p1p2, half_range;
} crt_ctx;

static u64 inv_mod_u64(u64 a, u64 m)
{
    i128 t = 0, newt = 1, rr = m, newr = a % m;
    while (newr) {
        i128 qq = rr / newr, tmp;
        tmp = t - qq * newt;
        t = newt;
        newt = tmp;
        tmp = rr - qq * newr;
        rr = newr;
        newr = tmp;
    }
    if (t < 0)
        t += m;
    return (u64)t;
}

static void crt_make(crt_ctx *c, int k)
{
    nega_plan_make(&c->p1, ORC_P1, k);
    nega_plan_make(&c->p2, ORC_P2, k);
    u64 q1 = ORC_P1, q2 = ORC_P2;
    u64 m2 = inv_mod_u64(q2 % q1, q1);
    i128 m1 = ((i128)1 - (i128)q2 * m2) / (i128)q1;
    i128 m1r = m1 % (i128)q2;
    if (m1r < 0)
        m1r += q2;
    c->m1_red = (u64)m1r;
    c->m2_red = m2 % q1;
    c->p1p2 = (u128)q1 * q2;
    c->half_range = (c->p1p2 - 1) / 2;
}

/* crt_combine (gfp_mult.py:184-198): signed v with |v| <= half_range */
static void crt_combine(const crt_ctx *c, u64 a1, u64 a2, u128 *mag, int *neg)
{
    u64 q1 = ORC_P1, q2 = ORC_P2;
    u64 r1 = (u64)(((u128)a1 * c->m2_red) % q1);
    u64 r2 = (u64)(((u128)a2 * c->m1_red) % q2);
    u128 v = (u128)r1 * q2 + (u128)r2 * q1;
    if (v >= c->p1p2)
        v -= c->p1p2;
    if (v > c->half_range) {
        *mag = c->p1p2 - v;
        *neg = 1;
    } else {
        *mag = v;
        *neg = 0;
    }
}

/* lhc_decompose (gfp_mult.py:96-116): s = l + h r + c r^2, 0 <= l, h < r */
static void lhc_decompose(u128 s, u64 r, u64 *l, u64 *h, u64 *cc)
{
    u128 q0 = s / r;
    *l = (u64)(s % r);
    *h = (u64)(q0 % r);
    *cc = (u64)(q0 / r);
}

/* _carry_normalize (gfp_mult.py:405-413) */
static u64 carry_normalize(const u64 *d, u64 *out, int k, u64 r)
{
    u128 carry = 0;
    for (int i = 0; i < k; i++) {
        u128 t = (u128)d[i] + carry;
        out[i] = (u64)(t % r);
        carry = t / r;
    }
    return (u64)carry;
}

/* canonical element for w * r^2 mod p, w small (the wrap fixups at
   gfp_mult.py:496-500); built from digit-exact shifts */
static void encode_w_r2(u64 w, u64 *out, int k, u64 r)
{
    u64 acc[256], t[256], sh[256];
    memset(acc, 0, sizeof(u64) * (size_t)k);
    int pos = 0;
    while (w) {
        memset(t, 0, sizeof(u64) * (size_t)k);
        t[0] = w % r;
        w /= r;
        gfp_mul_pow_r(t, (pos + 2) % (2 * k), sh, k, r);
        gfp_add(acc, sh, acc, k, r);
        pos++;
    }
    memcpy(out, acc, sizeof(u64) * (size_t)k);
}

static int check_compat(int k, u64 r)
{
    u128 limit = ((u128)ORC_P1 * ORC_P2 - 1) / 2;
    u128 r2 = (u128)r * r;
    if (r2 > limit / (u64)k)
        return 0;
    if ((ORC_P1 - 1) % (2 * (u64)k) || (ORC_P2 - 1) % (2 * (u64)k))
        return 0;
    return 1;
}

/* gfp_mul_fft (gfp_mult.py:416-501) */
static void gfp_mul_fft(const crt_ctx *c, const u64 *x, const u64 *y, u64 *z, int k, u64 r)
{
    u64 a1[128], b1[128], a2[128], b2[128], z1[128], z2[128];
    const nega_plan *P1 = &c->p1, *P2 = &c->p2;
    u64 q1 = P1->ctx.q, q2 = P2->ctx.q;
    for (int i = 0; i < k; i++) {
        a1[i] = mont_mul(&P1->ctx, x[i] % q1, P1->in_table[i]);
        b1[i] = mont_mul(&P1->ctx, y[i] % q1, P1->in_table[i]);
        a2[i] = mont_mul(&P2->ctx, x[i] % q2, P2->in_table[i]);
        b2[i] = mont_mul(&P2->ctx, y[i] % q2, P2->in_table[i]);
    }
    nega_transform(P1, a1, 0);
    nega_transform(P1, b1, 0);
    for (int i = 0; i < k; i++)
        z1[i] = mont_mul(&P1->ctx, a1[i], b1[i]);
    nega_transform(P1, z1, 1);
    nega_transform(P2, a2, 0);
    nega_transform(P2, b2, 0);
    for (int i = 0; i < k; i++)
        z2[i] = mont_mul(&P2->ctx, a2[i], b2[i]);
    nega_transform(P2, z2, 1);
    for (int i = 0; i < k; i++) {
        z1[i] = mont_mul(&P1->ctx, z1[i], P1->out_table[i]);
        z2[i] = mont_mul(&P2->ctx, z2[i], P2->out_table[i]);
    }
    u64 lp[256] = {0}, hp[256] = {0}, cp[256] = {0};
    u64 ln[256] = {0}, hn[256] = {0}, cn[256] = {0};
    for (int i = 0; i < k; i++) {
        u128 mag;
        int neg;
        crt_combine(c, z1[i], z2[i], &mag, &neg);
        if (mag == 0)
            continue;
        u64 l, h, cc;
        lhc_decompose(mag, r, &l, &h, &cc);
        if (neg) {
            ln[i] = l;
            hn[i] = h;
            cn[i] = cc;
        } else {
            lp[i] = l;
            hp[i] = h;
            cp[i] = cc;
        }
    }
    u64 u[256], t[256], cv[256] = {0};
    memcpy(u, lp, sizeof(u64) * (size_t)k);
    gfp_mul_pow_r(hp, 1, t, k, r);
    gfp_add(u, t, u, k, r);
    u64 wrap_p = carry_normalize(cp, cv, k, r);
    gfp_mul_pow_r(cv, 2 % (2 * k), t, k, r);
    gfp_add(u, t, u, k, r);
    gfp_sub(u, ln, u, k, r);
    gfp_mul_pow_r(hn, 1, t, k, r);
    gfp_sub(u, t, u, k, r);
    u64 wrap_n = carry_normalize(cn, cv, k, r);
    gfp_mul_pow_r(cv, 2 % (2 * k), t, k, r);
    gfp_sub(u, t, u, k, r);
    if (wrap_p) {
        encode_w_r2(wrap_p, t, k, r);
        gfp_sub(u, t, u, k, r);
    }
    if (wrap_n) {
        encode_w_r2(wrap_n, t, k, r);
        gfp_add(u, t, u, k, r);
    }
    memcpy(z, u, sizeof(u64) * (size_t)k);
}

/* independent second opinion: exact schoolbook negacyclic product with a
   3-word signed accumulator, then carry normalisation and canonicalisation */
static void gfp_mul_school(const u64 *x, const u64 *y, u64 *z, int k, u64 r)
{
    /* column m = sum_{i+j=m} x_i y_j - sum_{i+j=m+k} x_i y_j; keep as
       (pos, neg) unsigned 192-bit via hi carry words */
    u64 pos_lo[128], pos_mid[128], pos_hi[128];
    u64 neg_lo[128], neg_mid[128], neg_hi[128];
    memset(pos_lo, 0, sizeof(pos_lo));
    memset(pos_mid, 0, sizeof(pos_mid));
    memset(pos_hi, 0, sizeof(pos_hi));
    memset(neg_lo, 0, sizeof(neg_lo));
    memset(neg_mid, 0, sizeof(neg_mid));
    memset(neg_hi, 0, sizeof(neg_hi));
    for (int i = 0; i < k; i++)
        for (int j = 0; j < k; j++) {
            u128 pr = (u128)x[i] * y[j];
            int m = i + j;
            u64 *lo, *mid, *hi;
            if (m < k) {
                lo = &pos_lo[m];
                mid = &pos_mid[m];
                hi = &pos_hi[m];
            } else {
                m -= k;
                lo = &neg_lo[m];
                mid = &neg_mid[m];
                hi = &neg_hi[m];
            }
            u128 t = (u128)*lo + (u64)pr;
            *lo = (u64)t;
            t = (u128)*mid + (u64)(pr >> 64) + (u64)(t >> 64);
            *mid = (u64)t;
            *hi += (u64)(t >> 64);
        }
    /* value = sum_m (P_m - N_m) r^m.  Normalise P and N separately into
       radix-r digit vectors with wrap carries, as canonical elements. */
    u64 acc[256], tmp[256];
    memset(acc, 0, sizeof(u64) * (size_t)k);
    for (int side = 0; side < 2; side++) {
        u64 *lo = side ? neg_lo : pos_lo, *mid = side ? neg_mid : pos_mid,
            *hi = side ? neg_hi : pos_hi;
        /* per column: 192-bit value -> digits at m, m+1, m+2, m+3 ... */
        for (int m = 0; m < k; m++) {
            u64 w[3] = {lo[m], mid[m], hi[m]};
            int d = 0;
            while (w[0] || w[1] || w[2]) {
                u64 dig = big_divmod_small(w, 3, r);
                if (dig) {
                    memset(tmp, 0, sizeof(u64) * (size_t)k);
                    tmp[0] = dig;
                    gfp_mul_pow_r(tmp, (m + d) % (2 * k), tmp, k, r);
                    if (side)
                        gfp_sub(acc, tmp, acc, k, r);
                    else
                        gfp_add(acc, tmp, acc, k, r);
                }
                d++;
            }
        }
    }
    memcpy(z, acc, sizeof(u64) * (size_t)k);
}

/* ======================================================================== */
/* field helpers for the transform                                           */

typedef struct {
    int k;
    u64 r;
    int backend; /* 0 = gfp_mul_fft restatement, 1 = schoolbook */
    crt_ctx *crt;
} gfp_field;

static void field_mul(const gfp_field *f, const u64 *x, const u64 *y, u64 *z)
{
    if (f->backend == 0 && f->crt)
        gfp_mul_fft(f->crt, x, y, z, f->k, f->r);
    else
        gfp_mul_school(x, y, z, f->k, f->r);
}

static void field_one(int k, u64 *z)
{
    memset(z, 0, sizeof(u64) * (size_t)k);
    z[0] = 1;
}

static void field_minus_one(int k, u64 r, u64 *z)
{
    memset(z, 0, sizeof(u64) * (size_t)k);
    z[k - 1] = r;
}

/* x^e for e given as little-endian limbs (gfp_pow, gfp_field.py:164-177) */
static void field_pow_big(const gfp_field *f, const u64 *x, const u64 *e, int el, u64 *z)
{
    int k = f->k;
    u64 acc[256], base[256];
    field_one(k, acc);
    memcpy(base, x, sizeof(u64) * (size_t)k);
    int nb = big_bitlen(e, el);
    for (int b = 0; b < nb; b++) {
        if ((e[b / 64] >> (b % 64)) & 1)
            field_mul(f, acc, base, acc);
        if (b + 1 < nb)
            field_mul(f, base, base, base);
    }
    memcpy(z, acc, sizeof(u64) * (size_t)k);
}

static void field_pow(const gfp_field *f, const u64 *x, u64 e, u64 *z)
{
    field_pow_big(f, x, &e, 1, z);
}

static int elem_eq(const u64 *a, const u64 *b, int k)
{
    return memcmp(a, b, sizeof(u64) * (size_t)k) == 0;
}

/* ======================================================================== */
/* the six-step transform (fft.py:199-370)                                   */

typedef struct orc_plan {
    gfp_field field;
    int K, e;
    int64_t N;
    u64 *omega;
    u64 *table; /* K^(e-1) entries, element-major */
    int64_t table_n;
    int shift_step;
    base_op *ops;
    int nops;
    struct orc_plan *inverse;
    u64 *n_inv;
} orc_plan;

static void plan_free(orc_plan *p)
{
    if (!p)
        return;
    free(p->omega);
    free(p->table);
    free(p->ops);
    free(p->n_inv);
    if (p->inverse)
        plan_free(p->inverse);
    free(p);
}

/* build_plan (fft.py:237-275) for the GFP field */
static orc_plan *plan_build(const gfp_field *f, int K, int e, const u64 *omega, int *err)
{
    int k = f->k;
    u64 r = f->r;
    *err = ORC_EINVAL;
    if (K != 8 && K != 16 && K != 32 && K != 64)
        return NULL;
    if (e < 1)
        return NULL;
    if (!is_canonical(omega, k, r))
        return NULL;
    int64_t N = 1;
    for (int i = 0; i < e; i++)
        N *= K;
    u64 one[256], mone[256], t[256];
    field_one(k, one);
    field_minus_one(k, r, mone);
    field_pow(f, omega, (u64)N, t);
    if (!elem_eq(t, one, k))
        return NULL;
    field_pow(f, omega, (u64)(N / 2), t);
    if (!elem_eq(t, mone, k))
        return NULL;
    if (K != 2 * k)
        return NULL;
    u64 shift_root[256], shift_root_inv[256];
    memset(shift_root, 0, sizeof(u64) * (size_t)k);
    if (k == 1) {
        /* encode(r) with p = r + 1: r == p - 1 -> form B (0,...,r) */
        shift_root[0] = r;
    } else {
        shift_root[1] = 1;
    }
    gfp_mul_pow_r(one, 2 * k - 1, shift_root_inv, k, r);
    field_pow(f, omega, (u64)(N / (2 * k)), t);
    int step;
    if (elem_eq(t, shift_root, k))
        step = 1;
    else if (elem_eq(t, shift_root_inv, k))
        step = -1;
    else
        return NULL;
    orc_plan *p = (orc_plan *)calloc(1, sizeof(orc_plan));
    if (!p) {
        *err = ORC_ENOMEM;
        return NULL;
    }
    p->field = *f;
    p->K = K;
    p->e = e;
    p->N = N;
    p->shift_step = step;
    p->omega = (u64 *)malloc(sizeof(u64) * (size_t)k);
    memcpy(p->omega, omega, sizeof(u64) * (size_t)k);
    p->table_n = N / K;
    p->table = (u64 *)malloc(sizeof(u64) * (size_t)k * (size_t)p->table_n);
    if (!p->table) {
        plan_free(p);
        *err = ORC_ENOMEM;
        return NULL;
    }
    field_one(k, p->table);
    for (int64_t i = 1; i < p->table_n; i++)
        field_mul(f, p->table + (i - 1) * k, omega, p->table + i * k);
    p->nops = base_case_ops(K, &p->ops);
    *err = ORC_OK;
    return p;
}

/* stride_permutation (fft.py:34-56): element j*m + i -> i*n + j */
static void stride_permutation(u64 *v, int64_t m, int64_t n, int64_t offset, int k, u64 *scratch)
{
    if (m == 1 || n == 1)
        return;
    size_t es = sizeof(u64) * (size_t)k;
    for (int64_t j = 0; j < n; j++)
        for (int64_t i = 0; i < m; i++)
            memcpy(scratch + (i * n + j) * k, v + (offset + j * m + i) * k, es);
    memcpy(v + offset * k, scratch, es * (size_t)(m * n));
}

/* _run_base (fft.py:171-183) with the shift multiplier of
   GfpFftField.root_power_mul_factory (gfp_mult.py:574-581) */
static void run_base(u64 *v, const orc_plan *p)
{
    int k = p->field.k;
    u64 r = p->field.r;
    u64 a[256], b[256];
    for (int o = 0; o < p->nops; o++) {
        const base_op *op = &p->ops[o];
        u64 *xi = v + (size_t)op->i * k, *xj = v + (size_t)op->j * k;
        if (op->kind == 0) {
            memcpy(a, xi, sizeof(u64) * (size_t)k);
            memcpy(b, xj, sizeof(u64) * (size_t)k);
            gfp_add(a, b, xi, k, r);
            gfp_sub(a, b, xj, k, r);
        } else if (op->kind == 1) {
            int t = op->j;
            if (p->shift_step < 0)
                t = (2 * k - t) % (2 * k);
            gfp_mul_pow_r(xi, t, xi, k, r);
        } else {
            memcpy(a, xi, sizeof(u64) * (size_t)k);
            memcpy(xi, xj, sizeof(u64) * (size_t)k);
            memcpy(xj, a, sizeof(u64) * (size_t)k);
        }
    }
}

static void base_pass(u64 *v, const orc_plan *p, int threads)
{
    int64_t nblocks = p->N / p->K;
    int k = p->field.k;
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
    for (int64_t j = 0; j < nblocks; j++)
        run_base(v + j * p->K * k, p);
}

/* _twiddle_level_cheap (fft.py:84-103), applied to every block of `size`
   elements at once so one parallel region covers the whole level */
static void twiddle_level(u64 *v, int64_t N, int64_t size, int64_t m, int64_t stride,
                          const orc_plan *p, int threads)
{
    int k = p->field.k;
    u64 r = p->field.r;
    int K = p->K;
    int forward = p->shift_step > 0;
    int64_t per_block = (int64_t)(K - 1) * (m - 1);
    int64_t total = (N / size) * per_block;
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
    for (int64_t w = 0; w < total; w++) {
        int64_t off = (w / per_block) * size;
        int64_t rem = w % per_block;
        int64_t j = 1 + rem / (m - 1), i = 1 + rem % (m - 1);
        u64 x[256];
        int64_t base = off + j * m;
        int64_t a = (i * j) / m, b = (i * j) % m;
        u64 *slot = v + (base + i) * k;
        memcpy(x, slot, sizeof(u64) * (size_t)k);
        if (a)
            gfp_mul_pow_r(x, (int)(forward ? a : 2 * k - a), x, k, r);
        if (b)
            field_mul(&p->field, x, p->table + (b * stride) * k, x);
        memcpy(slot, x, sizeof(u64) * (size_t)k);
    }
}

/* dft_general (fft.py:298-360) */
static int dft_general(u64 *v, const orc_plan *p, int threads)
{
    int K = p->K, e = p->e, k = p->field.k;
    int64_t N = p->N;
    u64 *scratch = (u64 *)malloc(sizeof(u64) * (size_t)k * (size_t)N);
    if (!scratch)
        return ORC_ENOMEM;
    for (int i = 0; i < e - 1; i++) {
        int64_t size = 1;
        for (int t = 0; t < e - i; t++)
            size *= K;
        int64_t sub = size / K;
        for (int64_t j = 0; j < N; j += size)
            stride_permutation(v, K, sub, j, k, scratch);
    }
    base_pass(v, p, threads);
    for (int i = e - 2; i >= 0; i--) {
        int64_t size = 1, m = 1, stride = 1;
        for (int t = 0; t < e - i; t++)
            size *= K;
        m = size / K;
        for (int t = 0; t < i; t++)
            stride *= K;
        twiddle_level(v, N, size, m, stride, p, threads);
        for (int64_t j = 0; j < N; j += size)
            stride_permutation(v, m, K, j, k, scratch);
        base_pass(v, p, threads);
        for (int64_t j = 0; j < N; j += size)
            stride_permutation(v, K, m, j, k, scratch);
    }
    free(scratch);
    return ORC_OK;
}

/* N^{-1} mod p as a canonical element: N | r^k = p - 1, so
   N^{-1} = -(r^k / N) mod p (the value of GfpFftField.inv_scalar,
   gfp_mult.py:562-563) */
static void n_inverse(int64_t N, int k, u64 r, u64 *out)
{
    int nl = limbs_for(k);
    u64 *v = (u64 *)calloc((size_t)nl, sizeof(u64));
    big_r_pow_k(v, nl, r, k);
    big_divmod_small(v, nl, (u64)N);
    u64 *pm1 = (u64 *)calloc((size_t)nl, sizeof(u64));
    big_r_pow_k(pm1, nl, r, k);
    u64 t[256], zero[256];
    gfp_encode_big(v, nl, pm1, k, r, t);
    memset(zero, 0, sizeof(u64) * (size_t)k);
    gfp_sub(zero, t, out, k, r);
    free(v);
    free(pm1);
}

static int plan_ensure_inverse(orc_plan *p)
{
    if (p->inverse)
        return ORC_OK;
    int k = p->field.k, err;
    u64 winv[256];
    field_pow(&p->field, p->omega, (u64)(p->N - 1), winv);
    p->inverse = plan_build(&p->field, p->K, p->e, winv, &err);
    if (!p->inverse)
        return err;
    p->n_inv = (u64 *)malloc(sizeof(u64) * (size_t)k);
    n_inverse(p->N, k, p->field.r, p->n_inv);
    return ORC_OK;
}

/* ======================================================================== */
/* root routine (gfp_field.py:185-237, bench_cli.py:398-402)                 */

static int find_nth_root(const gfp_field *f, int64_t N, u64 seed, u64 *g_out)
{
    int k = f->k;
    u64 r = f->r;
    int nl = limbs_for(k);
    u64 *pm1 = (u64 *)calloc((size_t)nl, sizeof(u64));
    u64 *ex = (u64 *)calloc((size_t)nl, sizeof(u64));
    u64 *cand = (u64 *)calloc((size_t)nl + 1, sizeof(u64));
    u64 *width = (u64 *)calloc((size_t)nl, sizeof(u64));
    big_r_pow_k(pm1, nl, r, k);
    memcpy(ex, pm1, sizeof(u64) * (size_t)nl);
    if (big_divmod_small(ex, nl, (u64)N) != 0) {
        free(pm1);
        free(ex);
        free(cand);
        free(width);
        return ORC_EINVAL;
    }
    /* randrange(1, p): width = p - 1 = r^k, value = 1 + randbelow(r^k) */
    memcpy(width, pm1, sizeof(u64) * (size_t)nl);
    int nb = big_bitlen(width, nl);
    mt_state s;
    mt_seed_u64(&s, seed);
    u64 mone[256], c[256], g[256], t[256];
    field_minus_one(k, r, mone);
    for (;;) {
        do {
            mt_getrandbits(&s, nb, cand, nl);
        } while (big_cmp(cand, width, nl) >= 0);
        /* cand + 1 < p always; encode */
        u64 carry = 1;
        for (int i = 0; i < nl && carry; i++) {
            cand[i] += carry;
            carry = cand[i] == 0;
        }
        gfp_encode_big(cand, nl, pm1, k, r, c);
        field_pow_big(f, c, ex, nl, g);
        field_pow(f, g, (u64)(N / 2), t);
        if (elem_eq(t, mone, k))
            break;
    }
    memcpy(g_out, g, sizeof(u64) * (size_t)k);
    free(pm1);
    free(ex);
    free(cand);
    free(width);
    return ORC_OK;
}

static int primitive_root(const gfp_field *f, int64_t N, const u64 *g, u64 *omega)
{
    int k = f->k;
    u64 r = f->r;
    if (N % (2 * k))
        return ORC_EINVAL;
    u64 r_elem[256], a[256], b[256], t[256], one[256], mone[256];
    memset(r_elem, 0, sizeof(u64) * (size_t)k);
    if (k == 1)
        r_elem[0] = r;
    else
        r_elem[1] = 1;
    field_pow(f, g, (u64)(N / (2 * k)), a);
    memcpy(b, a, sizeof(u64) * (size_t)k);
    int64_t j = 1;
    while (!elem_eq(b, r_elem, k)) {
        j++;
        if (j > 2 * k)
            return ORC_EINVAL;
        field_mul(f, a, b, b);
    }
    field_pow(f, g, (u64)j, omega);
    field_one(k, one);
    field_minus_one(k, r, mone);
    field_pow(f, omega, (u64)N, t);
    if (!elem_eq(t, one, k))
        return ORC_EINVAL;
    field_pow(f, omega, (u64)(N / 2), t);
    if (!elem_eq(t, mone, k))
        return ORC_EINVAL;
    return ORC_OK;
}

/* ======================================================================== */
/* exported C API (ctypes)                                                   */

#define ORC_API __attribute__((visibility("default")))

ORC_API int orc_version(void) { return 1; }

ORC_API int orc_random_elements(u64 seed, int k, u64 r, int64_t skip, int64_t n, u64 *out)
{
    /* the first (skip + n) draws of Random(seed).randrange(p), encoded;
       the first `skip` are discarded */
    int nl = limbs_for(k);
    u64 *pm1 = (u64 *)calloc((size_t)nl, sizeof(u64));
    u64 *p = (u64 *)calloc((size_t)nl, sizeof(u64));
    u64 *cand = (u64 *)calloc((size_t)nl + 1, sizeof(u64));
    if (!pm1 || !p || !cand)
        return ORC_ENOMEM;
    big_r_pow_k(pm1, nl, r, k);
    memcpy(p, pm1, sizeof(u64) * (size_t)nl);
    for (int i = 0; i < nl; i++) {
        p[i] += 1;
        if (p[i])
            break;
    }
    int nb = big_bitlen(p, nl);
    mt_state s;
    mt_seed_u64(&s, seed);
    for (int64_t i = 0; i < skip + n; i++) {
        do {
            mt_getrandbits(&s, nb, cand, nl);
        } while (big_cmp(cand, p, nl) >= 0);
        if (i >= skip)
            gfp_encode_big(cand, nl, pm1, k, r, out + (i - skip) * k);
    }
    free(pm1);
    free(p);
    free(cand);
    return ORC_OK;
}

ORC_API int orc_is_canonical(const u64 *x, int64_t n, int k, u64 r, uint8_t *out)
{
    for (int64_t i = 0; i < n; i++)
        out[i] = (uint8_t)is_canonical(x + i * k, k, r);
    return ORC_OK;
}

ORC_API int orc_gfp_add(const u64 *x, const u64 *y, u64 *z, int64_t n, int k, u64 r)
{
    if (k < 1 || k > 256)
        return ORC_EINVAL;
    for (int64_t i = 0; i < n; i++)
        gfp_add(x + i * k, y + i * k, z + i * k, k, r);
    return ORC_OK;
}

ORC_API int orc_gfp_sub(const u64 *x, const u64 *y, u64 *z, int64_t n, int k, u64 r)
{
    if (k < 1 || k > 256)
        return ORC_EINVAL;
    for (int64_t i = 0; i < n; i++)
        gfp_sub(x + i * k, y + i * k, z + i * k, k, r);
    return ORC_OK;
}

ORC_API int orc_gfp_mul_pow_r(const u64 *x, u64 *z, int64_t n, int k, u64 r, int i)
{
    if (k < 1 || k > 256 || i < 0 || i > 2 * k)
        return ORC_EINVAL;
    for (int64_t e = 0; e < n; e++)
        gfp_mul_pow_r(x + e * k, i, z + e * k, k, r);
    return ORC_OK;
}

ORC_API int orc_check_prime_compat(int k, u64 r) { return check_compat(k, r); }

/* backend 0: gfp_mul_fft restatement (needs compat), 1: schoolbook */
ORC_API int orc_gfp_mul(const u64 *x, const u64 *y, u64 *z, int64_t n, int k, u64 r,
                        int backend, int threads)
{
    if (k < 1 || k > 128)
        return ORC_EINVAL;
    crt_ctx *crt = NULL;
    if (backend == 0) {
        if (!check_compat(k, r))
            return ORC_ECONFIG;
        crt = (crt_ctx *)malloc(sizeof(crt_ctx));
        crt_make(crt, k);
    }
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
    for (int64_t i = 0; i < n; i++) {
        if (backend == 0)
            gfp_mul_fft(crt, x + i * k, y + i * k, z + i * k, k, r);
        else
            gfp_mul_school(x + i * k, y + i * k, z + i * k, k, r);
    }
    if (crt) {
        free(crt->p1.ops);
        free(crt->p2.ops);
        free(crt);
    }
    return ORC_OK;
}

ORC_API int orc_base_case_ops(int K, int32_t *out, int cap)
{
    base_op *ops;
    int n = base_case_ops(K, &ops);
    if (n < 0)
        return -1;
    if (n * 3 > cap) {
        free(ops);
        return -2;
    }
    for (int i = 0; i < n; i++) {
        out[3 * i] = ops[i].kind;
        out[3 * i + 1] = ops[i].i;
        out[3 * i + 2] = ops[i].j;
    }
    free(ops);
    return n;
}

static int make_field(gfp_field *f, int k, u64 r, int backend)
{
    f->k = k;
    f->r = r;
    f->backend = backend;
    f->crt = NULL;
    if (backend == 0) {
        if (!check_compat(k, r))
            return ORC_ECONFIG;
        f->crt = (crt_ctx *)malloc(sizeof(crt_ctx));
        crt_make(f->crt, k);
    }
    return ORC_OK;
}

ORC_API int orc_gfp_root(int k, u64 r, int64_t N, u64 *g_out, u64 *omega_out)
{
    gfp_field f;
    int err = make_field(&f, k, r, 1);
    if (err)
        return err;
    err = find_nth_root(&f, N, 0, g_out);
    if (err)
        return err;
    return primitive_root(&f, N, g_out, omega_out);
}

ORC_API void *orc_plan_create(int k, u64 r, int K, int e, const u64 *omega, int backend,
                              int *err)
{
    gfp_field f;
    *err = make_field(&f, k, r, backend);
    if (*err)
        return NULL;
    orc_plan *p = plan_build(&f, K, e, omega, err);
    return p;
}

ORC_API void orc_plan_destroy(void *h)
{
    orc_plan *p = (orc_plan *)h;
    if (!p)
        return;
    crt_ctx *crt = p->field.crt;
    plan_free(p);
    if (crt) {
        free(crt->p1.ops);
        free(crt->p2.ops);
        free(crt);
    }
}

ORC_API int orc_plan_prepare_inverse(void *h)
{
    return plan_ensure_inverse((orc_plan *)h);
}

ORC_API int orc_plan_table(void *h, u64 *out, int64_t n)
{
    orc_plan *p = (orc_plan *)h;
    if (n > p->table_n)
        return ORC_EINVAL;
    memcpy(out, p->table, sizeof(u64) * (size_t)n * (size_t)p->field.k);
    return ORC_OK;
}

/* dft_general (inverse=0) or dft_inverse (inverse=1), in place */
ORC_API int orc_plan_exec(void *h, u64 *v, int inverse, int threads)
{
    orc_plan *p = (orc_plan *)h;
    int k = p->field.k;
    if (!inverse)
        return dft_general(v, p, threads);
    int err = plan_ensure_inverse(p);
    if (err)
        return err;
    err = dft_general(v, p->inverse, threads);
    if (err)
        return err;
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
    for (int64_t i = 0; i < p->N; i++)
        field_mul(&p->field, v + i * k, p->n_inv, v + i * k);
    return ORC_OK;
}

/* poly multiply composition: out = IDFT(DFT(f) .* DFT(g)) */
ORC_API int orc_poly_mul(void *h, const u64 *f, const u64 *g, u64 *out, int threads)
{
    orc_plan *p = (orc_plan *)h;
    int k = p->field.k;
    size_t bytes = sizeof(u64) * (size_t)k * (size_t)p->N;
    u64 *F = (u64 *)malloc(bytes);
    if (!F)
        return ORC_ENOMEM;
    memcpy(F, f, bytes);
    memcpy(out, g, bytes);
    int err = dft_general(F, p, threads);
    if (!err)
        err = dft_general(out, p, threads);
    if (!err) {
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1)
        for (int64_t i = 0; i < p->N; i++)
            field_mul(&p->field, F + i * k, out + i * k, out + i * k);
        err = orc_plan_exec(h, out, 1, threads);
    }
    free(F);
    return err;
}

ORC_API int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
