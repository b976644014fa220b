// instantiation of the pass kernel for k = 8 (one translation unit per k so
// the heavy template instantiations compile in parallel)
#include "gfp_pass.cuh"
#include "gfp_pmid44t.cuh"

template int launch_pass<8>(const gfp_fft_plan *, const u64 *, u64 *, const u64 *, u64 *,
                             const u64 *, int64_t, int64_t, int, int, int, int, const PassIO *,
                             cudaStream_t);

bool em_io_supported(const gfp_fft_plan *p) { return pass44_enabled(p->k, p->rc); }


// the fused middle of a poly-multiply (gfp_pmid44t.cuh)
bool poly_mid_supported(const gfp_fft_plan *p) { return pmid_takes(p); }
int launch_poly_mid(const gfp_fft_plan *p, const u64 *f_in, const u64 *g_in, u64 *out,
                    int64_t batch, cudaStream_t st)
{
    if (!launch_pmid44t(p, f_in, g_in, out, batch, st))
        return GFP_EUNSUPPORTED;
    return cuda_status();
}
