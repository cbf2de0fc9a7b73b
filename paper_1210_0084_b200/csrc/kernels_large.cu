// Large-slice kernels (2N = 2^(SLICQ_LOGN+1) >= 65536), see kernels_large.cuh.  Compiled once
// per size (build.py: -DSLICQ_LOGN=15, 16).
#ifndef SLICQ_LOGN
#error "compile with -DSLICQ_LOGN=<15|16>"
#endif
#include "kernels_large.cuh"

namespace slicq {
namespace kern {

template <class K>
static cudaError_t lpdl(K kernel, const KArgs &a, dim3 grid, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(LT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

template <>
int large_set_attrs<SLICQ_LOGN>() {
  const int sm = (int)large_smem_bytes<SLICQ_LOGN>();
  cudaError_t e = cudaSuccess;
  for (const void *f : {(const void *)fwd_large_col<SLICQ_LOGN, 0>, (const void *)fwd_large_col<SLICQ_LOGN, 1>,
                        (const void *)fwd_large_row<SLICQ_LOGN>, (const void *)inv_large_pack<SLICQ_LOGN>,
                        (const void *)inv_large_col<SLICQ_LOGN>, (const void *)inv_large_row<SLICQ_LOGN, 0>,
                        (const void *)inv_large_row<SLICQ_LOGN, 1>}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

template <>
cudaError_t large_forward<SLICQ_LOGN>(const KArgs &a, cudaStream_t s, int mode) {
  using G = Large<SLICQ_LOGN>;
  const size_t sm = large_smem_bytes<SLICQ_LOGN>();
  const unsigned nu = (unsigned)a.nunits;
  cudaError_t e = mode == 1 ? lpdl(fwd_large_col<SLICQ_LOGN, 1>, a, dim3(nu, G::N2 / LB), sm, s)
                            : lpdl(fwd_large_col<SLICQ_LOGN, 0>, a, dim3(nu, G::N2 / LB), sm, s);
  if (e == cudaSuccess) e = lpdl(fwd_large_row<SLICQ_LOGN>, a, dim3(nu, (G::N1 / 2 + 1 + 7) / 8), sm, s);
  return e;
}

template <>
cudaError_t large_inverse_spec<SLICQ_LOGN>(const KArgs &a, cudaStream_t s, int mode) {
  using G = Large<SLICQ_LOGN>;
  const size_t sm = large_smem_bytes<SLICQ_LOGN>();
  const unsigned nu = (unsigned)a.nunits;
  cudaError_t e = lpdl(inv_large_pack<SLICQ_LOGN>, a, dim3(nu, (G::N / 2 + 1 + LT - 1) / LT), 0, s);
  if (e == cudaSuccess) e = lpdl(inv_large_col<SLICQ_LOGN>, a, dim3(nu, G::N2 / LB), sm, s);
  if (e == cudaSuccess)
    e = mode == 1 ? lpdl(inv_large_row<SLICQ_LOGN, 1>, a, dim3(nu, G::N1 / LB), sm, s)
                  : lpdl(inv_large_row<SLICQ_LOGN, 0>, a, dim3(nu, G::N1 / LB), sm, s);
  if (e == cudaSuccess && mode == 0)
    e = lpdl(inv_large_bnd<SLICQ_LOGN>, a, dim3(nu, (unsigned)((a.tr - 1 + LT - 1) / LT)), 0, s);
  return e;
}

}  // namespace kern
}  // namespace slicq
