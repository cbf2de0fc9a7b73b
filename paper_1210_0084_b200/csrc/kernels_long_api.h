// Host interface of the long full-length CQ-NSGT kernels (kernels_long.cuh / .cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace slicq {
namespace kern {
struct KArgs;

// Allow a kernel the device's whole opt-in shared memory (minus its static shared memory).
// The dynamic shared-memory limit is a per-function attribute shared by every plan in the
// process; each launch passes its own size, so a later plan with a smaller configuration
// cannot invalidate an earlier plan's launches.
inline cudaError_t allow_max_dyn_smem(const void *f) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, f);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes);
  return e;
}

// channel-kernel size classes: CTA threads and the largest M_k of each (shared memory is
// sized per class, so the many short channels do not pay for the longest one's buffer)
// class 4 (kLongClasses - 1): M_k > 26000, a four-step M1 x M2 through the row's staging
// scratch with M2 <= 26000 in shared memory
constexpr int kLongClasses = 5;
constexpr int kLongSmemMax = 26000;  // largest shared-memory DFT
__host__ __device__ constexpr int long_class_threads(int c) { return c == 0 ? 128 : c == 1 ? 256 : 512; }
__host__ __device__ constexpr int long_class_maxm(int c) {
  return c == 0 ? 1536 : c == 1 ? 6144 : c == 2 ? 12288 : c == 3 ? kLongSmemMax : 16 * kLongSmemMax;
}

// largest stage count of a channel DFT (radices >= 2: log2(26000) < 15)
constexpr int kDifMaxStages = 16;
// shared bytes of the per-CTA stage plan (kernels_long.cuh DifPlan), rounded to float2
constexpr int kDifPlanEntries = (4 + 5 * 4 * kDifMaxStages + 7) / 8;

// shared two-level twiddle table entries of a channel of length M (kernels_long.cuh)
__host__ __device__ constexpr int long_twiddle_entries(int M) { return 64 + ((M + 63) >> 6); }

// per size class c: channels [off[c], off[c+1]) of the device channel list (KArgs::pchans)
// and the class's dynamic shared-memory bytes
struct LongClasses {
  int off[kLongClasses + 1];
  size_t smem[kLongClasses];
};
int long_set_attrs(int logN, const LongClasses &cls);
cudaError_t long_forward(int logN, const KArgs &a, const LongClasses &cls, cudaStream_t s);
cudaError_t long_inverse(int logN, const KArgs &a, const LongClasses &cls, cudaStream_t s);
// sliCQ channels with M_k > 1024 (split design): one CTA per (channel, unit), size classes 0..3
// (M_k <= 26000); forward reads the staged X, inverse writes the slot staging (a.bent)
int slice_big_attrs();
cudaError_t slice_big_launch(bool fwd, KArgs a, const int32_t *list, const LongClasses &cls,
                             cudaStream_t s);
}  // namespace kern
}  // namespace slicq
