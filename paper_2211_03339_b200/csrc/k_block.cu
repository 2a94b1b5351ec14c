// k_block.cu -- block Jacobi variant (placeholder until the DMMA block kernels land).
#include "mpj_device.cuh"
#include "mpj_internal.h"

namespace mpj {

template <typename R>
size_t block_scratch_bytes(int np, int b)
{
    (void)np; (void)b;
    return 256;
}

template <typename R>
mpj_status block_sweep(R *, int64_t, R *, int64_t, int, const DevSched &, R, int, unsigned long long *,
                       void *, cudaStream_t)
{
    set_error("block variant not available in this build");
    return MPJ_ERR_INVALID;
}

template size_t block_scratch_bytes<double>(int, int);
template size_t block_scratch_bytes<float>(int, int);
template mpj_status block_sweep<double>(double *, int64_t, double *, int64_t, int, const DevSched &, double,
                                        int, unsigned long long *, void *, cudaStream_t);
template mpj_status block_sweep<float>(float *, int64_t, float *, int64_t, int, const DevSched &, float, int,
                                       unsigned long long *, void *, cudaStream_t);

}  // namespace mpj
