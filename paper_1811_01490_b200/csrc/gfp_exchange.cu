// gfp_exchange.cu -- the four-step transpose as direct stores into the
// peers' receive buffers ("fuse it into ... stores via
// peer pointers"), replacing pack (permute + copy) -> NCCL all_to_all ->
// unpack (permute + copy) with ONE kernel that reads the local digit-major
// block once and writes every element straight to its owner over NVLink
// (peer pointers from CUDA IPC, gfp_ipc_*), or to local memory for the
// rank's own slice.
//
// Layout (the generic form of both directions of sharded.py):
//   src   [A][k][B]            this rank's block, B = G * b
//   dst_g [b][k][G * A]        rank g's receive buffer
//   dst_g[bl][d][rank * A + a] = src[a][d][g * b + bl]
// forward: A = N2/G local columns, B = N1 (k1), b = N1/G  (cols -> rows)
// inverse: A = N1/G local rows,    B = N2 (n2), b = N2/G  (rows -> cols)
//
// HBM/NVLink bound: 8 bytes read + 8 written per digit, nothing else.  A CTA
// moves a 32 (a) x 64 (B) tile of one digit row through shared memory so the
// reads (along B) and the writes (along a) are both 256-byte warp rows.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "gfp_internal.cuh"
#include "gfpfft.h"

namespace {

constexpr int XMAX = 16;  // ranks per exchange (one NVSwitch node is 8)
constexpr int TA = 32, TB = 64, TY = 8;

struct PeerPtrs {
    uint64_t *p[XMAX];
};

__global__ void __launch_bounds__(TA *TY) k_exchange(const uint64_t *__restrict__ src, PeerPtrs dst,
                                                     int rank, int G, int64_t A, int k, int64_t B,
                                                     int64_t b)
{
    __shared__ uint64_t tile[TA][TB + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t b0 = (int64_t)blockIdx.x * TB, a0 = (int64_t)blockIdx.y * TA;
    const int d = blockIdx.z;
    // read: rows a0 + ty + TY i, columns b0 + tx (+ 32)
#pragma unroll
    for (int i = 0; i < TA / TY; i++) {
        const int64_t a = a0 + ty + TY * i;
        if (a < A) {
#pragma unroll
            for (int h = 0; h < TB / 32; h++) {
                const int64_t bc = b0 + tx + 32 * h;
                if (bc < B)
                    tile[ty + TY * i][tx + 32 * h] =
                        __ldcs(src + GFP_IDX((a * k + d) * B + bc, A * k * B));
            }
        }
    }
    // destination bases in shared memory (compile-time parameter indices: a
    // dynamic index into the parameter struct would copy it to the stack)
    __shared__ uint64_t *sdst[XMAX];
    const int tid = ty * 32 + tx;
    if (tid < XMAX) {
        uint64_t *v = dst.p[0];
#pragma unroll
        for (int q = 1; q < XMAX; q++)
            v = tid == q ? dst.p[q] : v;
        sdst[tid] = v;
    }
    GFP_JITTER(1);
    __syncthreads();
    // write: for column bc = b0 + j (j = ty + TY i), 32 consecutive a; the
    // owner g and local index bl advance incrementally (one division per
    // thread, not per store)
    const int64_t GA = (int64_t)G * A;
    const int64_t a = a0 + tx;
    int g = (int)((b0 + ty) / b);
    int64_t bl = b0 + ty - (int64_t)g * b;
#pragma unroll
    for (int i = 0; i < TB / TY; i++) {
        const int j = ty + TY * i;
        if (i > 0) {
            bl += TY;
            while (bl >= b) {
                bl -= b;
                g++;
            }
        }
        if (b0 + j < B && a < A)
            __stcs(sdst[GFP_IDX(g, G)] + GFP_IDX((bl * k + d) * GA + (int64_t)rank * A + a,
                                                   b * k * GA),
                   tile[tx][j]);
    }
}

}  // namespace

extern "C" int gfp_exchange_transpose(const uint64_t *src, uint64_t *const *dst, int world,
                                      int rank, int64_t A, int k, int64_t B, void *stream)
{
    if (!src || !dst || world < 1 || world > XMAX || rank < 0 || rank >= world || A < 1 ||
        k < 1 || B < 1 || B % world)
        return GFP_EINVAL;
    PeerPtrs pp;
    memset(&pp, 0, sizeof(pp));
    for (int g = 0; g < world; g++) {
        if (!dst[g])
            return GFP_EINVAL;
        pp.p[g] = dst[g];
    }
    const int64_t gx = (B + TB - 1) / TB, gy = (A + TA - 1) / TA;
    if (gy > 65535 || k > 65535)
        return GFP_EINVAL;
    dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)k), block(32, TY);
    k_exchange<<<grid, block, 0, (cudaStream_t)stream>>>(src, pp, rank, world, A, k, B, B / world);
    return cuda_status();
}

// ---------------------------------------------------------------------------
// CUDA IPC: peer pointers for the exchange (one process per GPU).  The handle
// names the allocation that contains `ptr` (torch's caching allocator hands
// out sub-ranges of cudaMalloc segments), so the byte offset travels with it.

typedef int (*PFN_getAddressRange)(unsigned long long *, size_t *, unsigned long long);

extern "C" int gfp_ipc_get_handle(const void *ptr, unsigned char *handle64, int64_t *offset)
{
    if (!ptr || !handle64 || !offset)
        return GFP_EINVAL;
    static PFN_getAddressRange range_fn = nullptr;
    if (!range_fn) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return GFP_ECUDA;
        range_fn = (PFN_getAddressRange)fn;
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range_fn(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
        return GFP_ECUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base) != cudaSuccess) {
        cudaGetLastError();
        return GFP_ECUDA;
    }
    memcpy(handle64, &h, sizeof(h) < 64 ? sizeof(h) : 64);
    *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
    return GFP_OK;
}

extern "C" int gfp_ipc_open(const unsigned char *handle64, int64_t offset, void **ptr)
{
    if (!handle64 || !ptr || offset < 0)
        return GFP_EINVAL;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    void *base = nullptr;
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return GFP_ECUDA;
    }
    *ptr = (char *)base + offset;
    return GFP_OK;
}

extern "C" int gfp_ipc_close(void *ptr, int64_t offset)
{
    if (!ptr)
        return GFP_EINVAL;
    if (cudaIpcCloseMemHandle((char *)ptr - offset) != cudaSuccess) {
        cudaGetLastError();
        return GFP_ECUDA;
    }
    return GFP_OK;
}

// ---------------------------------------------------------------------------
// Device-side completion flags for the peer exchange (no host barriers).
// Every rank owns a flag array in its device memory, shared with the peers
// through the same IPC mappings as the receive buffers; flags[slot][g] is
// written only by rank g.  A signal is a system-scope release store of an
// epoch into every peer's flags[slot][rank] issued AFTER the kernels whose
// stores it publishes (stream order: those kernels happen-before it); a wait
// spins with system-scope acquire loads until every flags[slot][g] >= epoch,
// and the kernels queued after it (stream order) see everything the peers
// published -- the release/acquire pair carries the peers' NVLink stores.
// A wait that does not see its epoch within max_spins polls records the slot
// and rank in err[0] and returns instead of hanging the GPU.

__global__ void k_flag_signal(PeerPtrs flags, int world, int slot, int rank,
                              unsigned long long epoch)
{
    const int g = threadIdx.x;
    if (g >= world)
        return;
    unsigned long long *f = reinterpret_cast<unsigned long long *>(flags.p[0]);
#pragma unroll 1
    for (int q = 1; q < XMAX; q++)
        if (q == g)
            f = reinterpret_cast<unsigned long long *>(flags.p[q]);
    f += (int64_t)slot * world + rank;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
}

__global__ void k_flag_wait(const unsigned long long *flags, int world, int slot,
                            unsigned long long epoch, long long max_spins, int *err)
{
    const int g = threadIdx.x;
    if (g < world) {
        const unsigned long long *f = flags + (int64_t)slot * world + g;
        unsigned long long v = 0;
        long long spins = 0;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
            if (v >= epoch)
                break;
            if (++spins > max_spins) {
                atomicCAS(err, 0, 1 + slot * 256 + g);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
}

extern "C" int gfp_flag_signal(uint64_t *const *peer_flags, int world, int slot, int rank,
                               uint64_t epoch, void *stream)
{
    if (!peer_flags || world < 1 || world > XMAX || rank < 0 || rank >= world || slot < 0 ||
        slot > 255)
        return GFP_EINVAL;
    PeerPtrs pp;
    memset(&pp, 0, sizeof(pp));
    for (int g = 0; g < world; g++) {
        if (!peer_flags[g])
            return GFP_EINVAL;
        pp.p[g] = peer_flags[g];
    }
    k_flag_signal<<<1, 32, 0, (cudaStream_t)stream>>>(pp, world, slot, rank,
                                                      (unsigned long long)epoch);
    return cuda_status();
}

extern "C" int gfp_flag_wait(const uint64_t *my_flags, int world, int slot, uint64_t epoch,
                             int64_t max_spins, int *err, void *stream)
{
    if (!my_flags || !err || world < 1 || world > XMAX || slot < 0 || slot > 255 ||
        max_spins < 1)
        return GFP_EINVAL;
    k_flag_wait<<<1, 32, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const unsigned long long *>(my_flags), world, slot,
        (unsigned long long)epoch, (long long)max_spins, err);
    return cuda_status();
}
