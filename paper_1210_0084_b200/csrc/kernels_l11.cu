#define SLICQ_LOGN 11
// Instantiation of the per-slice spectrum kernels for N = 2^SLICQ_LOGN (one translation
// unit per size so that the sizes compile in parallel).
#include "kernels_dev.cuh"
#include "kernels_long_api.h"

namespace slicq {
namespace kern {

template <>
int set_attrs<SLICQ_LOGN>(size_t smem) {
  const void *fns[] = {(const void *)slicq_fwd_spec_kernel<SLICQ_LOGN, 0>,
                       (const void *)slicq_inv_spec_kernel<SLICQ_LOGN, 0>,
                       (const void *)slicq_fwd_spec_kernel<SLICQ_LOGN, 1>,
                       (const void *)slicq_inv_spec_kernel<SLICQ_LOGN, 1>};
  for (const void *f : fns) {
    (void)smem;
    const cudaError_t e = allow_max_dyn_smem(f);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

template <class K>
static cudaError_t launch_pdl(K kernel, const KArgs &a, dim3 grid, int threads, size_t smem,
                              cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

template <>
cudaError_t launch_fwd_spec<SLICQ_LOGN>(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s,
                                        bool pdl, int mode) {
  if (mode == 1)
    return launch_pdl(slicq_fwd_spec_kernel<SLICQ_LOGN, 1>, a, grid, Big<SLICQ_LOGN>::T, smem, s,
                      pdl);
  return launch_pdl(slicq_fwd_spec_kernel<SLICQ_LOGN, 0>, a, grid, Big<SLICQ_LOGN>::T, smem, s, pdl);
}

template <>
cudaError_t launch_inv_spec<SLICQ_LOGN>(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s,
                                        bool pdl, int mode) {
  if (mode == 1)
    return launch_pdl(slicq_inv_spec_kernel<SLICQ_LOGN, 1>, a, grid, Big<SLICQ_LOGN>::T, smem, s,
                      pdl);
  return launch_pdl(slicq_inv_spec_kernel<SLICQ_LOGN, 0>, a, grid, Big<SLICQ_LOGN>::T, smem, s, pdl);
}

template <>
int phase_times<SLICQ_LOGN>(unsigned long long *out32, int reset) {
#ifdef SLICQ_PHASE_TIMING
  if (cudaMemcpyFromSymbol(out32, g_phase_cycles, sizeof(g_phase_cycles)) != cudaSuccess) return -1;
  if (reset) {
    static const unsigned long long zero[2][16] = {};
    if (cudaMemcpyToSymbol(g_phase_cycles, zero, sizeof(zero)) != cudaSuccess) return -1;
  }
  return 0;
#else
  (void)out32;
  (void)reset;
  return -1;
#endif
}

}  // namespace kern
}  // namespace slicq
