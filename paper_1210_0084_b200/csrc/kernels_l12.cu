#define SLICQ_LOGN 12
// Instantiation of the sliCQ kernels for N = 2^SLICQ_LOGN (one translation unit per size
// so that the four sizes compile in parallel).
#include "kernels_dev.cuh"

namespace slicq {
namespace kern {

template <>
int set_attrs<SLICQ_LOGN>(size_t fwd_smem, size_t inv_smem) {
  cudaError_t e1 = cudaFuncSetAttribute(slicq_fwd_kernel<SLICQ_LOGN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem);
  cudaError_t e2 = cudaFuncSetAttribute(slicq_inv_kernel<SLICQ_LOGN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)inv_smem);
  if (e1 != cudaSuccess) return (int)e1;
  if (e2 != cudaSuccess) return (int)e2;
  return 0;
}

template <>
cudaError_t launch_fwd<SLICQ_LOGN>(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s) {
  slicq_fwd_kernel<SLICQ_LOGN><<<grid, Big<SLICQ_LOGN>::T, smem, s>>>(a);
  return cudaGetLastError();
}

template <>
cudaError_t launch_inv<SLICQ_LOGN>(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s) {
  slicq_inv_kernel<SLICQ_LOGN><<<grid, Big<SLICQ_LOGN>::T, smem, s>>>(a);
  return cudaGetLastError();
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
