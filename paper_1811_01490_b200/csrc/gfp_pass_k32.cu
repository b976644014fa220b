// instantiation of the pass kernel for k = 32 (one translation unit per k so
// the heavy template instantiations compile in parallel)
#include "gfp_pass.cuh"

template int launch_pass<32>(const gfp_fft_plan *, const u64 *, u64 *, const u64 *, u64 *,
                             const u64 *, int64_t, int64_t, int, int, int, int, const PassIO *,
                             cudaStream_t);
