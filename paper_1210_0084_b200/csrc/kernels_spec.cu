#include <cstdlib>
// Instantiation of the per-slice spectrum kernels and the fused kernels for N = 2^SLICQ_LOGN.
// Compiled once per size (build.py: -DSLICQ_LOGN=11..14, one object each, in parallel).
#ifndef SLICQ_LOGN
#error "compile with -DSLICQ_LOGN=<11..14>"
#endif
#include <algorithm>

#include "kernels_dev.cuh"
#include "kernels_fused.cuh"
#include "kernels_ring.cuh"
#include "kernels_long_api.h"

// dev override (SLICQ_SPEC_PER_SM): cap on the persistent spectrum kernels' CTAs per SM, so
// that a channel kernel of another chunk (another stream) can share the SMs (0: occupancy)
static int spec_per_sm() {
  static const int v = [] {
    const char *e = std::getenv("SLICQ_SPEC_PER_SM");
    return e && *e ? std::atoi(e) : 0;
  }();
  return v;
}

namespace slicq {
namespace kern {

template <>
int set_attrs<SLICQ_LOGN>(size_t smem) {
  const void *fns[] = {(const void *)slicq_fwd_spec_kernel<SLICQ_LOGN, 0>,
                       (const void *)slicq_inv_spec_kernel<SLICQ_LOGN, 0>,
                       (const void *)slicq_inv_spec_persist_kernel<SLICQ_LOGN>,
                       (const void *)slicq_fwd_spec_persist_kernel<SLICQ_LOGN>,
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
int fused_attrs<SLICQ_LOGN>() {
  const void *fns[] = {(const void *)slicq_fwd_fused_kernel<SLICQ_LOGN>,
                       (const void *)slicq_fwd_cluster_kernel<SLICQ_LOGN>};
  for (const void *f : fns) {
    const cudaError_t e = allow_max_dyn_smem(f);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

template <>
cudaError_t launch_fwd_fused<SLICQ_LOGN>(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s,
                                         bool pdl) {
  return launch_pdl(slicq_fwd_fused_kernel<SLICQ_LOGN>, a, grid, Big<SLICQ_LOGN>::T, smem, s, pdl);
}

// cluster-fused forward: grid = the units rounded up to G, clusters of G consecutive CTAs
template <>
cudaError_t launch_fwd_cluster<SLICQ_LOGN>(const KArgs &a, int G, size_t smem, cudaStream_t s,
                                           bool pdl) {
  if (G > 8) {
    const cudaError_t e = cudaFuncSetAttribute(slicq_fwd_cluster_kernel<SLICQ_LOGN>,
                                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(((int64_t)a.nunits + G - 1) / G * G));
  cfg.blockDim = dim3(Big<SLICQ_LOGN>::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, slicq_fwd_cluster_kernel<SLICQ_LOGN>, a);
}

#if SLICQ_LOGN == 12 || SLICQ_LOGN == 13
template <>
int ring_attrs<SLICQ_LOGN>() {
  int rc = (int)allow_max_dyn_smem((const void *)slicq_fwd_ring_kernel<SLICQ_LOGN>);
  if (rc == 0) rc = (int)allow_max_dyn_smem((const void *)slicq_fwd_band_kernel<SLICQ_LOGN>);
  return rc;
}
template <>
cudaError_t launch_fwd_band<SLICQ_LOGN>(const KArgs &a, const RArgs &r, size_t smem, int grid,
                                        cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(RING_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, slicq_fwd_band_kernel<SLICQ_LOGN>, a, r);
}
template <>
cudaError_t launch_fwd_ring<SLICQ_LOGN>(const KArgs &a, const RArgs &r, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)r.ngrid);
  cfg.blockDim = dim3(RING_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the roles wait on each other
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, slicq_fwd_ring_kernel<SLICQ_LOGN>, a, r);
}
#endif

template <>
cudaError_t launch_inv_spec_persist<SLICQ_LOGN>(const KArgs &a, size_t smem, cudaStream_t s,
                                                bool pdl, int *grid_out) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occ, slicq_inv_spec_persist_kernel<SLICQ_LOGN>, Big<SLICQ_LOGN>::T, smem);
  if (e != cudaSuccess) return e;
  if (spec_per_sm() > 0) occ = std::min(std::max(occ, 1), spec_per_sm());
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(occ, 1) * nsm, a.nunits));
  if (grid_out) *grid_out = grid;
  return launch_pdl(slicq_inv_spec_persist_kernel<SLICQ_LOGN>, a, dim3((unsigned)grid),
                    Big<SLICQ_LOGN>::T, smem, s, pdl);
}

template <>
cudaError_t launch_fwd_spec_persist<SLICQ_LOGN>(const KArgs &a, size_t smem, cudaStream_t s,
                                                bool pdl) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occ, slicq_fwd_spec_persist_kernel<SLICQ_LOGN>, Big<SLICQ_LOGN>::T, smem);
  if (e != cudaSuccess) return e;
  if (spec_per_sm() > 0) occ = std::min(std::max(occ, 1), spec_per_sm());
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(occ, 1) * nsm, a.nunits));
  return launch_pdl(slicq_fwd_spec_persist_kernel<SLICQ_LOGN>, a, dim3((unsigned)grid),
                    Big<SLICQ_LOGN>::T, smem, s, pdl);
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
