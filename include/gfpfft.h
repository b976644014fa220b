/*
 * gfpfft.h -- C-ABI of the B200-native GF(p) FFT library (libgfpfft.so),
 * p = r^k + 1 a generalized Fermat prime, k a power of two, 2 <= r < 2^64.
 *
 * This is the drop-in boundary for the reference package `gfpfft`
 * (arxiv/paper_1811_01490).  The reference is pure Python; its "plugin"
 * surface is the field protocol consumed by fft.py (fft.py:13-17) and the
 * public functions re-exported by gfpfft/__init__.py:9-38.  Each entry point
 * below cites the reference function it replaces.  A reference-side binding
 * (ctypes) is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Device buffers are digit-major: a vector of n elements is
 *     uint64[k][n] (digit d of element i at ptr[d * n + i]); a batch of
 *     transforms is uint64[batch][k][N].  All device pointers must be
 *     8-byte aligned device memory.  Host entry points (*_host) take
 *     element-major uint64[n][k] (the reference's tuple order and the GFPV
 *     payload order, bench_cli.py:88-116).
 *   - Inputs must be canonical (gfp_field.py:1-8: every digit < r, or the
 *     form-B encoding (0,...,0,r) of p-1).  Outputs are canonical.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and asynchronous unless the name ends in _host.
 *   - Return codes: GFP_OK, or an error the Python layer maps to the
 *     reference's exception (ValueError / ConfigurationError).
 */
#ifndef GFPFFT_H
#define GFPFFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFP_OK 0
#define GFP_EINVAL 1      /* ValueError in the reference */
#define GFP_ECONFIG 2     /* gfp_mult.ConfigurationError (gfp_mult.py:35) */
#define GFP_ECUDA 3       /* CUDA runtime failure */
#define GFP_ENOMEM 4      /* device allocation failure */
#define GFP_EUNSUPPORTED 5 /* parameters outside the transform kernels' range */

typedef struct gfp_fft_plan gfp_fft_plan;

/* Human-readable message for a return code. */
const char *gfp_strerror(int code);

/* Library version (ABI revision). */
int gfp_version(void);

/* 1 if k*r^2 <= (P1*P2-1)/2 and 2k | P_i - 1 for the reference's default
   word primes: check_prime_compat (gfp_mult.py:207-226).  The device
   multiply does not need it (it is exact for every (k, r)); the Python
   layer uses it to keep gfp_mul_fft's ConfigurationError contract. */
int gfp_check_prime_compat(int k, uint64_t r);

/* 1 if the transform / fast-multiply kernels accept (k, r): k in
   {4, 8, 16, 32} and r large enough that the limb-split accumulation bounds
   hold.  Every configuration in BASELINE.json qualifies. */
int gfp_fast_path_ok(int k, uint64_t r);

/* ---- element-wise vectors (device, digit-major [k][n]) ------------------ */

/* z = x + y mod p.  Replaces gfp_add (gfp_field.py:82-109) per element. */
int gfp_vec_add(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k,
                uint64_t r, void *stream);

/* z = x - y mod p.  Replaces gfp_sub (gfp_field.py:112-135). */
int gfp_vec_sub(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k,
                uint64_t r, void *stream);

/* z = x * r^i mod p, 0 <= i <= 2k (GFP_EINVAL otherwise).  Replaces
   gfp_mul_pow_r (gfp_field.py:138-161). */
int gfp_vec_mul_pow_r(const uint64_t *x, uint64_t *z, int64_t n, int k, uint64_t r, int i,
                      void *stream);

/* z = x * y mod p, exact for every (k, r).  Replaces gfp_mul_fft
   (gfp_mult.py:416-501) / gfp_mul_bigint (gfp_mult.py:504-512); both compute
   the same canonical product.  y_inc = 1: element-wise; y_inc = 0: y is a
   single element ([k][1]) broadcast over x. */
int gfp_vec_mul(const uint64_t *x, const uint64_t *y, int64_t y_inc, uint64_t *z, int64_t n,
                int k, uint64_t r, void *stream);

/* One element operation on host digit tuples (k <= 128 canonical digits
   each): the reference's scalar functions in one synchronous call (one H2D
   through a persistent pinned staging buffer, one kernel, one D2H).
     op 0  z = x + y          gfp_add        (gfp_field.py:82-109)
     op 1  z = x - y          gfp_sub        (gfp_field.py:112-135)
     op 2  z = x r^arg        gfp_mul_pow_r  (gfp_field.py:138-161), 0 <= arg <= 2k
     op 3  z = x y            gfp_mul_bigint (gfp_mult.py:504-512), direct multiply
     op 4  z = x y            gfp_mul_fft    (gfp_mult.py:416-501), the mechanism
                              (GFP_ECONFIG when check_prime_compat fails)
     op 5  z = x^e            gfp_pow        (gfp_field.py:164-177), e = y[0..arg)
                              little-endian 64-bit limbs, arg <= 64 */
int gfp_scalar_op(int op, const uint64_t *x, const uint64_t *y, int64_t arg, uint64_t *z, int k,
                  uint64_t r, void *stream);

/* Host-buffer element-wise product: x, y, z are element-major host arrays
   uint64[n][k] (the reference's tuple order); H2D, layout conversion,
   gfp_vec_mul, back; synchronous.  The call a reference-side binding makes
   for a list of gfp_mul_fft / gfp_mul_bigint products (bench_cli bench-mul,
   bench_cli.py:282-324). */
int gfp_vec_mul_host(const uint64_t *x, const uint64_t *y, uint64_t *z, int64_t n, int k,
                     uint64_t r, void *stream);

/* z = x * y mod p through the reference's own mechanism (gfp_mul_fft,
   gfp_mult.py:416-501, paper Alg. 13): negacyclic convolutions of the digit
   vectors over the word primes P1, P2 (theta-weighted NTTs in Montgomery
   form), CRT to signed coefficients, LHC split, carry normalisation.  The
   same canonical product as gfp_vec_mul (which the transforms use);
   GFP_ECONFIG when check_prime_compat fails (gfp_mult.py:207-226),
   GFP_EUNSUPPORTED for k > 64.  y_inc as in gfp_vec_mul. */
int gfp_vec_mul_crt(const uint64_t *x, const uint64_t *y, int64_t y_inc, uint64_t *z, int64_t n,
                    int k, uint64_t r, void *stream);

/* gfp_vec_mul_crt with the reference's per-step profile (gfp_mul_fft's
   profile= keys, gfp_mult.py:428-500; bench_cli cmd_profile_mul,
   bench_cli.py:470-494): step_cycles[0..5] (host) receive the SM cycles the
   threads spent in convert_in, convolution, convert_out, crt, lhc and final
   (summed over threads), *ms the kernel's device time.  A separate
   instrumented kernel (clock64 around each step); same product.
   Synchronous. */
int gfp_vec_mul_crt_profile(const uint64_t *x, const uint64_t *y, int64_t y_inc, uint64_t *z,
                            int64_t n, int k, uint64_t r, uint64_t *step_cycles, float *ms,
                            void *stream);

/* z = x^e mod p, e given as little-endian host uint64 limbs shared by all
   elements.  Replaces gfp_pow (gfp_field.py:164-177) /
   GfpFftField.pow (gfp_mult.py:552-554). */
int gfp_vec_pow(const uint64_t *x, const uint64_t *e_limbs, int e_nlimbs, uint64_t *z,
                int64_t n, int k, uint64_t r, void *stream);

/* out[i] = 1 if element i is canonical.  Replaces is_canonical
   (gfp_field.py:49-56). */
int gfp_vec_is_canonical(const uint64_t *x, uint8_t *out, int64_t n, int k, uint64_t r,
                         void *stream);

/* Seeded synthetic canonical elements, digits uniform in [0, r). */
int gfp_vec_uniform(uint64_t *z, int64_t n, int k, uint64_t r, uint64_t seed, void *stream);

/* Layout conversion element-major [n][k] <-> digit-major [k][n] (device). */
int gfp_to_digit_major(const uint64_t *src, uint64_t *dst, int64_t n, int k, void *stream);
int gfp_to_element_major(const uint64_t *src, uint64_t *dst, int64_t n, int k, void *stream);

/* ---- transforms ----------------------------------------------------------- */

/* Plan for the DFT of N = K^e points at root omega (host array of k
   canonical digits).  Replaces build_plan (fft.py:237-275) for the GFP field
   (GfpFftField, gfp_mult.py:518-592): validates omega^N = 1,
   omega^(N/2) = -1, K = 2k and omega^(N/2k) in {r, 1/r} exactly like the
   reference (GFP_EINVAL otherwise), and builds the device twiddle tables
   (omega^j, j < N/K, and omega^j * N^-1) with the exact device multiply.
   Every r < 2^64 and k in {4, 8, 16, 32} is accepted: radices with the
   fast path's headroom (gfp_fast_path_ok) run the lazy-digit pass kernels,
   the others (e.g. r close to 2^64) radix-2 passes on canonical digits with
   the reference's element algorithms (gfp_fft_plan_caps = 0; exact, slower).
   Work is enqueued on `stream`; the call synchronises it before returning. */
int gfp_fft_plan_create(gfp_fft_plan **plan, int k, uint64_t r, int K, int e,
                        const uint64_t *omega, void *stream);

int gfp_fft_plan_destroy(gfp_fft_plan *plan);

/* N of a plan, and the number of uint64 words of device workspace
   gfp_fft_exec / gfp_poly_mul need for `batch` transforms. */
int64_t gfp_fft_plan_size(const gfp_fft_plan *plan);
int64_t gfp_fft_workspace_words(const gfp_fft_plan *plan, int64_t batch);

/* Forward (inverse = 0) or inverse (inverse = 1, includes the N^-1 scale)
   DFT of `batch` vectors, natural order in and out, digit-major
   [batch][k][N].  in may equal out.  Replaces dft_general (fft.py:298-360)
   and dft_inverse (fft.py:363-370). */
int gfp_fft_exec(const gfp_fft_plan *plan, const uint64_t *in, uint64_t *out, uint64_t *work,
                 int64_t batch, int inverse, void *stream);

/* gfp_fft_exec with the digit forms chosen by the caller and, optionally,
   the four-step inter-stage twiddle of an enclosing transform folded into
   the first pass: with ft != NULL, element (b, i) of the batch is first
   multiplied by w^((ft_row0 + b) i) (w^-(...) if ft_inverse), w the root of
   plan `ft` (same k; exponents mod ft's N) -- the D_{N1,N2} stage of the
   reference's tensor formula (fft.py:62-103) without a separate pass.
   in_canon = 0: the input is balanced lazy (the output of a call with
   out_canon = 0), required when ft is given.  GFP_EUNSUPPORTED if this k's
   pass kernel cannot fold the twiddle (then use gfp_fft_twiddle). */
int gfp_fft_exec_ex(const gfp_fft_plan *plan, const uint64_t *in, uint64_t *out, uint64_t *work,
                    int64_t batch, int inverse, int in_canon, int out_canon,
                    const gfp_fft_plan *ft, int64_t ft_row0, int ft_inverse, void *stream);

/* Cyclic product of length N: out = IDFT(DFT(f) .* DFT(g)), the polynomial
   product when deg f + deg g < N (the reference composes
   it from dft_general, GfpFftField.mul and dft_inverse). */
int gfp_poly_mul(const gfp_fft_plan *plan, const uint64_t *f, const uint64_t *g,
                 uint64_t *out, uint64_t *work, int64_t batch, void *stream);

/* Host-buffer entry points (element-major [batch][N][k] host arrays; H2D,
   transform, D2H; synchronous).  The call a reference-side binding makes
   in place of dft_general / dft_inverse / the poly-mul composition on a
   list of digit tuples. */
int gfp_fft_exec_host(gfp_fft_plan *plan, uint64_t *v, int64_t batch, int inverse,
                      void *stream);
int gfp_poly_mul_host(gfp_fft_plan *plan, const uint64_t *f, const uint64_t *g, uint64_t *out,
                      int64_t batch, void *stream);

/* Polynomial product from host coefficient arrays of their own lengths:
   f is [batch][nf][k], g is [batch][ng][k] (element-major, canonical,
   1 <= nf, ng <= N), out is [batch][n_out][k] with n_out = min(nf + ng - 1, N):
   the linear product when nf + ng - 1 <= N (the reference's composition,
   SURVEY §3.4: zero-pad to N, dft_general both, multiply, dft_inverse),
   otherwise the first N coefficients of the cyclic product.  Pinned host
   buffers (cudaHostAlloc / cudaHostRegister) are read by the first
   transform pass and written by the last one directly (zero-copy: only the
   nf + ng input and n_out output elements cross PCIe); pageable buffers are
   staged.  Synchronous. */
int gfp_poly_mul_host2(gfp_fft_plan *plan, const uint64_t *f, int64_t nf, const uint64_t *g,
                       int64_t ng, uint64_t *out, int64_t batch, void *stream);

/* Four-step inter-stage twiddle of the sharded transform: x is canonical
   digit-major [batch][k][n]; element (b, i) is multiplied by
   omega^((row0 + b) * i) (omega^-((row0 + b) * i) if inverse), omega the
   plan's N-th root (exponents taken mod N).  Canonical output; out may
   equal x.  (The reference has no distributed transform;
   this is the D_{N1,N2} stage of its tensor formula, fft.py:62-103.) */
int gfp_fft_twiddle(const gfp_fft_plan *plan, const uint64_t *x, uint64_t *out, int64_t batch,
                    int64_t n, int64_t row0, int inverse, void *stream);

/* The four-step transpose as direct stores into every rank's receive
   buffer (the reference has no distributed transform --
   this replaces the pack / all_to_all / unpack of the exchange that
   sharded.py otherwise does with torch.distributed.all_to_all_single).
   src is this rank's digit-major block [A][k][B]; dst[g] (g < world <= 16)
   is rank g's receive buffer [B/world][k][world * A] -- a peer pointer from
   gfp_ipc_open, or a local buffer -- and
       dst[g][bl][d][rank * A + a] = src[a][d][g * (B/world) + bl].
   One HBM/NVLink-bound kernel, stream-ordered; the caller separates it from
   the peers' use of their buffers with a barrier.  GFP_EINVAL on bad sizes
   (B % world != 0, world > 16, null pointers). */
int gfp_exchange_transpose(const uint64_t *src, uint64_t *const *dst, int world, int rank,
                           int64_t A, int k, int64_t B, void *stream);

/* gfp_fft_exec_ex (no four-step twiddle) whose LAST pass stores straight
   into the exchange's receive buffers instead of an output vector: the
   column DFTs of the sharded four-step fused with the transpose (SURVEY 8(e)
   steps 2-4).  in is this rank's batch [batch][k][N]; element (b, i) of the
   result lands in dst[g] (world ranks, g = i / (N/world)) at
   [(i mod N/world)][d][rank * batch + b] -- gfp_exchange_transpose's layout
   with A = batch, B = N.  scratch and work are two [batch][k][N] buffers.
   GFP_EUNSUPPORTED unless k = 8 (the radix-16 pass kernel), e >= 2,
   world <= 8 a power of two, batch % 8 == 0 (then use gfp_fft_exec_ex +
   gfp_exchange_transpose). */
int gfp_fft_exec_exchange(const gfp_fft_plan *plan, const uint64_t *in, uint64_t *scratch,
                          uint64_t *work, int64_t batch, int inverse, int in_canon, int out_canon,
                          uint64_t *const *dst, int world, int rank, void *stream);

/* Device-side completion flags of the peer exchange (replacing host
   barriers).  Each rank owns uint64 flags[slots][world] in device memory,
   shared with the peers like the receive buffers; flags[slot][g] is written
   only by rank g.  gfp_flag_signal stores `epoch` with system-scope release
   semantics into peer_flags[g][slot][rank] for every rank g (after the
   kernels queued before it on `stream`, whose stores it publishes);
   gfp_flag_wait spins with system-scope acquire loads until every
   my_flags[slot][g] >= epoch, so kernels queued after it see the peers'
   published stores.  A wait not satisfied within max_spins polls writes
   1 + slot * 256 + g into *err (device int) and returns -- a protocol error
   is reported, never a hung GPU.  Both are one tiny stream-ordered kernel;
   the host never blocks.  GFP_EINVAL for world > 16 or bad arguments. */
int gfp_flag_signal(uint64_t *const *peer_flags, int world, int slot, int rank, uint64_t epoch,
                    void *stream);
int gfp_flag_wait(const uint64_t *my_flags, int world, int slot, uint64_t epoch,
                  int64_t max_spins, int *err, void *stream);

/* CUDA IPC for the exchange's peer pointers (one process per GPU):
   gfp_ipc_get_handle writes the 64-byte handle of the allocation holding ptr
   and ptr's byte offset in it; gfp_ipc_open maps a peer's handle and returns
   the peer address (+ offset); gfp_ipc_close unmaps it. */
int gfp_ipc_get_handle(const void *ptr, unsigned char *handle64, int64_t *offset);
int gfp_ipc_open(const unsigned char *handle64, int64_t offset, void **ptr);
int gfp_ipc_close(void *ptr, int64_t offset);

/* Number of kernel launches issued by the last exec/poly_mul call on this
   plan (instrumentation for the benchmark's gpu_launches count). */
int64_t gfp_fft_plan_last_launches(const gfp_fft_plan *plan);

/* Capabilities of a plan's pass kernels (bit flags): GFP_CAP_EM_IO -- the
   first / last pass read / write element-major (host) buffers themselves
   (zero-copy host I/O); GFP_CAP_FT -- gfp_fft_exec_ex can fold a four-step
   twiddle into the first pass; GFP_CAP_XCH -- gfp_fft_exec_exchange can
   store the last pass into peer buffers.  Plans without a flag take the
   staged / separate-kernel route for that feature. */
#define GFP_CAP_EM_IO 1
#define GFP_CAP_FT 2
#define GFP_CAP_XCH 4
int gfp_fft_plan_caps(const gfp_fft_plan *plan);

/* Per-pass device timing.  With timing on, every later call on the plan
   records CUDA events on its stream around each pass launch (the reference's
   dft_general(profile=) phase accounting, fft.py:298-360, and the
   benchmark's per-pass roofline); gfp_fft_plan_pass_times synchronises on
   the last event and writes up to `max` per-launch durations (ms) with the
   pass index of each launch within its transform (0 = the multiply-free
   first pass of a forward transform), returning the count (negative
   GFP_E* on failure).  Off by default: no events, no overhead. */
int gfp_fft_plan_set_timing(gfp_fft_plan *plan, int on);
int gfp_fft_plan_pass_times(gfp_fft_plan *plan, float *ms, int *pass, int max);

/* Which arithmetic mode the transform / multiply kernels take for (k, r), as
   decided by the host-side bound proofs (make_consts: exact integer bounds on
   every sub-column, carry and lazy stage of the multiply and the butterflies):
   3 -- compile-time radix r = 2^a + 2^b (the paper's radices; shift quotients,
        sequential carry with the rounding column quotient);
   2 -- r = 2^a + 2^b at run time;  1 -- sparse r = 2^a + eps;  0 -- reciprocal
        quotient;  -1 -- no lazy-digit headroom (the generic canonical-digit
        path);  -2 for an invalid (k, r).  Host only: needs no GPU. */
int gfp_radix_mode(int k, uint64_t r);

/* Number of transform launches of this process that ran as one of the
   TMA-tile kernels (cp.async.bulk.tensor tile loads / stores): the k = 8 pass
   k_pass44t (gfp_pass44t.cuh), the k = 16 first pass k_first16t
   (gfp_pass16t.cuh), the fused middle of a poly-multiply k_pmid44t
   (gfp_pmid44t.cuh) -- lets a test or the benchmark confirm which kernel
   served a transform. */
int64_t gfp_tma_pass_launches(void);

/* 1 in the checked build (GFP_DEBUG: index guards + timing jitter in the
   pass / exchange kernels, the stand-in for compute-sanitizer), else 0.
   gfp_debug_selftest launches one kernel that performs a deliberately
   out-of-range guarded index, so a checked build prints its GFP_CHECK line
   (proving the guards are live); GFP_EUNSUPPORTED in the product build. */
int gfp_debug_build(void);
int gfp_debug_selftest(void *stream);

/* Instrumentation: run `iters` x 8 independent IMAD.WIDE (32x32 -> 64)
   product chains per thread on a blocks x threads grid and report the kernel time and the
   number of IMAD.WIDE executed -- the measured integer-pipe peak the
   benchmark's roofline divides by. */
int gfp_probe_imad_wide(int64_t iters, int blocks, int threads, float *ms_out, double *ops_out,
                        void *stream);

/* ------------------------------------------------------------------------
 * Word-prime transform: DFT over Z/qZ, q an odd prime < 2^63, on Montgomery
 * residues (R = 2^64), and the convolutions built on it.  Replaces the
 * reference's MontField transform (fft.py:376-421 with word_field.py:103-200)
 * and cyclic_convolution / negacyclic_convolution (gfp_mult.py:230-386).
 * Buffers are plain uint64[batch][n] device arrays of residues in [0, q).
 * ------------------------------------------------------------------------ */
typedef struct gfp_word_plan gfp_word_plan;

/* WordPrime.make constants (word_field.py:111-119): -q^-1 mod 2^64,
   2^128 mod q, 2^64 mod q.  GFP_EINVAL unless q is odd, 3 <= q < 2^63. */
int gfp_word_consts(uint64_t q, uint64_t *qinv, uint64_t *r2, uint64_t *one);

/* z[i] = mont_mul(a[i], b[i]) = a b 2^-64 mod q (word_field.py:133-140). */
int gfp_word_vec_mont_mul(uint64_t q, const uint64_t *a, const uint64_t *b, uint64_t *z,
                          int64_t n, void *stream);

/* Plan for n-point transforms (n a power of two dividing q - 1) at the
   Montgomery-form root omega: GFP_EINVAL unless omega^n = 1 and
   omega^(n/2) = -1 (build_plan's check, fft.py:250-254).  negacyclic != 0:
   theta is a primitive 2n-th root with theta^2 = omega and gfp_word_convolve
   computes the product mod (X^n + 1) (_nega_plan, gfp_mult.py:280-305);
   otherwise mod (X^n - 1) (_cyclic_plan, gfp_mult.py:308-322). */
int gfp_word_plan_create(gfp_word_plan **plan, uint64_t q, int64_t n, uint64_t omega,
                         int negacyclic, uint64_t theta, void *stream);
int gfp_word_plan_destroy(gfp_word_plan *plan);

/* Natural-order DFT of Montgomery residues (dft_general on a MontField plan,
   fft.py:298-360); inverse != 0: at omega^-1 with the n^-1 scale
   (dft_inverse, fft.py:363-370).  in may equal out. */
int gfp_word_ntt_exec(gfp_word_plan *plan, const uint64_t *in, uint64_t *out, int64_t batch,
                      int inverse, void *stream);

/* Convolution of standard-form inputs in [0, q) (GFP_EINVAL otherwise:
   _check_reduced, gfp_mult.py:361-366), standard-form output: _convolve
   (gfp_mult.py:351-358) -- weights, two forward transforms, pointwise
   product, inverse transform and the output weights with 1/n.  Synchronous
   (the input range check). */
int gfp_word_convolve(gfp_word_plan *plan, const uint64_t *x, const uint64_t *y, uint64_t *out,
                      int64_t batch, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* GFPFFT_H */
