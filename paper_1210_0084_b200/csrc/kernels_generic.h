// Host interface of the generic-length spectrum kernels (kernels_generic.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <vector_types.h>

namespace slicq {
namespace kern {
struct KArgs;

constexpr int kGenericMaxPasses = 24;
constexpr int kGenericMaxN = 26624;  // complex points: N * 8 bytes of shared memory per CTA

// an in-place mixed-radix DIT pass: r sub-DFTs of size S combined (elements S apart)
struct GPass {
  int r, S;
};
struct GArgs {
  int N, np;
  GPass pass[kGenericMaxPasses];  // execution order
  const float2 *twN;              // e^{-2 pi i t / N}, t < N
  const int *perm;                // input n -> position (mixed-radix digit reversal)
};

size_t generic_smem_bytes(int N);
int generic_set_attrs();
cudaError_t launch_generic(bool fwd, const KArgs &a, const GArgs &g, int nunits, cudaStream_t s,
                           bool pdl, int mode);
}  // namespace kern
}  // namespace slicq
