// Large-slice kernels (2N = 2^(SLICQ_LOGN+1) >= 65536), see kernels_large.cuh.  Compiled once
// per size (build.py: -DSLICQ_LOGN=15, 16).
#ifndef SLICQ_LOGN
#error "compile with -DSLICQ_LOGN=<15|16>"
#endif
#include <algorithm>

#include "kernels_large_cluster.cuh"

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

// 16-CTA cluster launch (kernels_large_cluster.cuh): grid (units, 16), cluster
// (1, 16, 1), with programmatic dependent launch like the split kernels
template <class K>
static cudaError_t lcluster(K kernel, const KArgs &a, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.nunits, LCL);
  cfg.blockDim = dim3(LT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = LCL;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}
constexpr size_t kClusterSmem = cluster_smem_bytes<SLICQ_LOGN>();

template <>
bool large_cluster_ok<SLICQ_LOGN>() {
#if SLICQ_LOGN == 16
  for (const void *f : {(const void *)fwd_large_cluster<SLICQ_LOGN>, (const void *)inv_large_cluster<SLICQ_LOGN>}) {
    if (cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kClusterSmem) !=
            cudaSuccess)
      return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, LCL);
    cfg.blockDim = dim3(LT);
    cfg.dynamicSmemBytes = kClusterSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = LCL;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, f, &cfg) != cudaSuccess || n < 1) {
      (void)cudaGetLastError();
      return false;
    }
  }
  return true;
#else
  return false;
#endif
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
cudaError_t large_forward<SLICQ_LOGN>(const KArgs &a, cudaStream_t s, int mode, bool cluster) {
  using G = Large<SLICQ_LOGN>;
  const size_t sm = large_smem_bytes<SLICQ_LOGN>();
  const unsigned nu = (unsigned)a.nunits;
#if SLICQ_LOGN == 16
  if (cluster && mode == 0) return lcluster(fwd_large_cluster<SLICQ_LOGN>, a, kClusterSmem, s);
#else
  (void)cluster;
#endif
  cudaError_t e = mode == 1 ? lpdl(fwd_large_col<SLICQ_LOGN, 1>, a, dim3(nu, G::N2 / LB), sm, s)
                            : lpdl(fwd_large_col<SLICQ_LOGN, 0>, a, dim3(nu, G::N2 / LB), sm, s);
  if (e == cudaSuccess) e = lpdl(fwd_large_row<SLICQ_LOGN>, a, dim3(nu, (G::N1 / 2 + 1 + 7) / 8), sm, s);
  return e;
}

template <>
cudaError_t large_inverse_spec<SLICQ_LOGN>(const KArgs &a, cudaStream_t s, int mode, bool cluster) {
  using G = Large<SLICQ_LOGN>;
  const size_t sm = large_smem_bytes<SLICQ_LOGN>();
  const unsigned nu = (unsigned)a.nunits;
#if SLICQ_LOGN == 16
  if (cluster && mode == 0) {
    cudaError_t e = lcluster(inv_large_cluster<SLICQ_LOGN>, a, kClusterSmem, s);
    if (e == cudaSuccess)
      e = lpdl(inv_large_bnd<SLICQ_LOGN>, a, dim3(nu, (unsigned)((a.tr - 1 + LT - 1) / LT)), 0, s);
    return e;
  }
#else
  (void)cluster;
#endif
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
