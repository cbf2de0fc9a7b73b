// Full-length CQ-NSGT of long signals (L = 2^18 .. 2^22), see kernels_long.cuh.
#include "kernels_long.cuh"

#include <algorithm>

namespace slicq {
namespace kern {

template <class K>
static cudaError_t pdl_launch(K kernel, const KArgs &a, dim3 grid, int threads, size_t smem,
                              cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

template <int LOGN>
static int set_attrs_logn() {
  const int cs = (int)long_col_smem<LOGN>(), rs = (int)large_smem_bytes<LOGN>();
  cudaError_t e = cudaFuncSetAttribute(long_fwd_col<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(long_inv_col<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fwd_large_row<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, rs);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(inv_large_row<LOGN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, rs);
  return (int)e;
}

static void (*chan_kernel(bool fwd, int c))(const KArgs) {
  if (c == kLongClasses - 1) return fwd ? long_chan_fwd_big : long_chan_inv_big;
  switch (c) {
    case 0: return fwd ? long_chan_fwd<long_class_threads(0)> : long_chan_inv<long_class_threads(0)>;
    case 1: return fwd ? long_chan_fwd<long_class_threads(1)> : long_chan_inv<long_class_threads(1)>;
  }
  return fwd ? long_chan_fwd<512> : long_chan_inv<512>;
}

// the channel kernels of one direction, one launch per non-empty size class
static cudaError_t launch_classes(bool fwd, KArgs a, const LongClasses &cls, cudaStream_t s) {
  const int32_t *list = a.pchans;
  for (int c = 0; c < kLongClasses; ++c) {
    const int n = cls.off[c + 1] - cls.off[c];
    if (!n) continue;
    a.pchans = list + cls.off[c];
    const cudaError_t e = pdl_launch(chan_kernel(fwd, c), a, dim3((unsigned)n, (unsigned)a.nunits),
                                     long_class_threads(c), cls.smem[c], s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int long_set_attrs(int logN, const LongClasses &cls) {
  int rc = 0;
  switch (logN) {
    case 17: rc = set_attrs_logn<17>(); break;
    case 18: rc = set_attrs_logn<18>(); break;
    case 19: rc = set_attrs_logn<19>(); break;
    case 20: rc = set_attrs_logn<20>(); break;
    case 21: rc = set_attrs_logn<21>(); break;
    default: return (int)cudaErrorInvalidValue;
  }
  if (rc) return rc;
  cudaError_t e = cudaSuccess;
  for (int c = 0; c < kLongClasses && e == cudaSuccess; ++c)
    for (int f = 0; f < 2 && e == cudaSuccess; ++f)
      e = allow_max_dyn_smem((const void *)chan_kernel(f == 0, c));  // not the plan's size
  return (int)e;
}

template <int LOGN>
static cudaError_t fwd_logn(const KArgs &a, const LongClasses &cls, cudaStream_t s) {
  using G = Large<LOGN>;
  const unsigned nu = (unsigned)a.nunits;
  cudaError_t e = pdl_launch(long_fwd_col<LOGN>, a, dim3(nu, G::N2 / LongCol<LOGN>::NB), LCT,
                             long_col_smem<LOGN>(), s);
  if (e == cudaSuccess)
    e = pdl_launch(fwd_large_row<LOGN>, a, dim3(nu, (G::N1 / 2 + 1 + 7) / 8), LT,
                   large_smem_bytes<LOGN>(), s);
  if (e == cudaSuccess) e = launch_classes(true, a, cls, s);
  return e;
}

template <int LOGN>
static cudaError_t inv_logn(const KArgs &a, const LongClasses &cls, cudaStream_t s) {
  using G = Large<LOGN>;
  const unsigned nu = (unsigned)a.nunits;
  cudaError_t e = launch_classes(false, a, cls, s);
  if (e == cudaSuccess)
    e = pdl_launch(long_inv_pack, a, dim3(nu, (G::N / 2 + 1 + LT - 1) / LT), LT, 0, s);
  if (e == cudaSuccess)
    e = pdl_launch(long_inv_col<LOGN>, a, dim3(nu, G::N2 / LongCol<LOGN>::NB), LCT,
                   long_col_smem<LOGN>(), s);
  if (e == cudaSuccess)
    e = pdl_launch(inv_large_row<LOGN, 1>, a, dim3(nu, G::N1 / LB), LT, large_smem_bytes<LOGN>(), s);
  return e;
}

static void (*big_kernel(bool fwd, int c))(const KArgs) {
  switch (c) {
    case 0: return fwd ? long_chan_fwd<long_class_threads(0)> : long_chan_inv_slots<long_class_threads(0)>;
    case 1: return fwd ? long_chan_fwd<long_class_threads(1)> : long_chan_inv_slots<long_class_threads(1)>;
  }
  return fwd ? long_chan_fwd<512> : long_chan_inv_slots<512>;
}

int slice_big_attrs() {
  cudaError_t e = cudaSuccess;
  for (int c = 0; c < kLongClasses - 1 && e == cudaSuccess; ++c)
    for (int f = 0; f < 2 && e == cudaSuccess; ++f)
      e = allow_max_dyn_smem((const void *)big_kernel(f == 0, c));
  return (int)e;
}

cudaError_t slice_big_launch(bool fwd, KArgs a, const int32_t *list, const LongClasses &cls,
                             cudaStream_t s) {
  a.L = 2 * (int64_t)a.Nh;  // long_chan_fwd reads 2N from L
  for (int c = 0; c < kLongClasses - 1; ++c) {
    const int n = cls.off[c + 1] - cls.off[c];
    if (!n) continue;
    a.pchans = list + cls.off[c];
    const cudaError_t e = pdl_launch(big_kernel(fwd, c), a, dim3((unsigned)n, (unsigned)a.nunits),
                                     long_class_threads(c), cls.smem[c], s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t long_forward(int logN, const KArgs &a, const LongClasses &cls, cudaStream_t s) {
  switch (logN) {
    case 17: return fwd_logn<17>(a, cls, s);
    case 18: return fwd_logn<18>(a, cls, s);
    case 19: return fwd_logn<19>(a, cls, s);
    case 20: return fwd_logn<20>(a, cls, s);
    case 21: return fwd_logn<21>(a, cls, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t long_inverse(int logN, const KArgs &a, const LongClasses &cls, cudaStream_t s) {
  switch (logN) {
    case 17: return inv_logn<17>(a, cls, s);
    case 18: return inv_logn<18>(a, cls, s);
    case 19: return inv_logn<19>(a, cls, s);
    case 20: return inv_logn<20>(a, cls, s);
    case 21: return inv_logn<21>(a, cls, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace kern
}  // namespace slicq
