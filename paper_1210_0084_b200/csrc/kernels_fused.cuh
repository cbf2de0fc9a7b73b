// Fused sliCQ kernels for sm_100a: one CTA per (row, slice) unit does the whole slice with the
// spectrum resident in shared memory, so the only HBM traffic is the signal read and the
// coefficient write (forward) or the coefficient read and the signal write (inverse).
// DESIGN.md "Fused kernels" describes the design; step names follow SURVEY.md §8(a).
//
//   forward  slicq_fwd_fused_kernel<LOGN>
//     F1 + F2   fwd_spectrum<LOGN, 0, true> (kernels_dev.cuh): windowed frame -> X[0..N] in
//               shared memory
//     F3 - F5   warp tasks over the plan's channel groups: y[d] = X(lo + d) g_k[d] / sqrt(M_k)
//               read contiguously (no fold table), c[n] = sum_d y[d] w^{(d + lo) n},
//               w = e^{+2 pi i / M_k}: a whole DFT_M per lane (small M) or a four-step
//               M1 x M2 whose twiddles and second-step input index absorb the rotation by lo
//               (the fold j mod M_k, C5); coefficients stored once
//
// The warps of a CTA take the tasks in plan order (sorted by code shape), so at any time the
// CTA's warps run one or two shapes' code (instruction-cache locality).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_dev.cuh"

namespace slicq {
namespace kern {

__device__ __forceinline__ FChan ld_fchan(const FChan *p) {
  const int4 *q = reinterpret_cast<const int4 *>(p);
  const int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  FChan f;
  f.lo = a.x; f.len = a.y; f.M = a.z; f.goff = a.w;
  f.off = b.x; f.twoff = b.y; f.lo_mod = b.z; f.lom2 = b.w;
  f.d0 = c.x; f.d1 = c.y; f.ovoff = c.z; f.flags = c.w;
  return f;
}

// X(j) for an unwrapped bin j in (-2N, 2N) of a real signal's spectrum, from X[0..N] in
// shared memory: X[j mod 2N], or conj X[2N - (j mod 2N)] above N (C15)
template <int N>
__device__ __forceinline__ float2 x_at(const float2 *X, int j) {
  const int jj = j < 0 ? j + 2 * N : j;
  const bool up = jj > N;
  const float2 v = X[padi(up ? 2 * N - jj : jj)];
  return make_float2(v.x, up ? -v.y : v.y);
}

// ---- forward, small task: lane c owns channel c; buf[p] = y[(p - lo) mod M] (the fold of
// P:193), DFT_M (sign +) in registers, coefficients stored as 16-byte pairs
template <int M, int N>
__device__ __forceinline__ void ff_small(const KArgs &a, const FTask &tk, const float2 *X,
                                         float2 *out_row, int lane, bool inter) {
  if (lane >= tk.nch) return;
  const FChan ch = ld_fchan(a.fch + tk.coff + lane);
  const float *g = a.gw + ch.goff;
  float2 v[M];
#pragma unroll
  for (int p = 0; p < M; ++p) {
    int d = p - ch.lo_mod;
    d += d < 0 ? M : 0;
    const bool in = d < ch.len;
    const float w = in ? __ldg(g + d) : 0.f;
    float2 x = make_float2(0.f, 0.f);
    if (in) x = inter ? X[padi(ch.lo + d)] : x_at<N>(X, ch.lo + d);
    v[p] = make_float2(x.x * w, x.y * w);
  }
  dft<M, +1>(v);
  float2 *o = out_row + ch.off;
  if (a.vec16) {
    float4 *o4 = reinterpret_cast<float4 *>(o);
#pragma unroll
    for (int n = 0; n < M / 2; ++n)
      __stcs(o4 + n, make_float4(v[2 * n].x, v[2 * n].y, v[2 * n + 1].x, v[2 * n + 1].y));
  } else {
#pragma unroll
    for (int n = 0; n < M; ++n) __stcs(o + n, v[n]);
  }
}

// ---- forward, two-step task, step 1: item (c, d2): the column d = M2 d1 + d2 of channel c's
// contiguous support, DFT_M1 (sign +) over d1, twiddle w^{(d2 + lo) n1}; stored to the warp
// scratch at A[c][n1][(d2 + lo) mod M2] (stride S2 = M2 | 1, conflict-free both ways)
template <int M1, int N>
__device__ __forceinline__ void ff_s1(const KArgs &a, const FTask &tk, int m2, const float2 *X,
                                      float2 *scr, int lane, bool inter) {
  const int items = tk.nch * m2;
  const int S2 = m2 | 1;
  const unsigned mag2 = tk.mags & 0xffffu;
  for (int i = lane; i < items; i += 32) {
    const int c = (int)((i * mag2) >> 16), d2 = i - c * m2;
    const FChan ch = ld_fchan(a.fch + tk.coff + c);
    const float *g = a.gw + ch.goff;
    float2 v[M1];
#pragma unroll
    for (int d1 = 0; d1 < M1; ++d1) {
      const int d = d1 * m2 + d2;
      const bool in = d < ch.len;
      const float w = in ? __ldg(g + d) : 0.f;
      float2 x = make_float2(0.f, 0.f);
      if (in) x = inter ? X[padi(ch.lo + d)] : x_at<N>(X, ch.lo + d);
      v[d1] = make_float2(x.x * w, x.y * w);
    }
    dft<M1, +1>(v);
    int e = d2 + ch.lo_mod;
    e -= e >= ch.M ? ch.M : 0;
    chan_twiddle<M1, +1>(v, e, ch.M, a.twM + ch.twoff);
    int e2 = d2 + ch.lom2;
    e2 -= e2 >= m2 ? m2 : 0;
    float2 *A = scr + c * M1 * S2 + e2;
#pragma unroll
    for (int n1 = 0; n1 < M1; ++n1) A[n1 * S2] = v[n1];
  }
}

// ---- forward, two-step task, step 2: item (c, n1): DFT_M2 (sign +) over the rotated column
// -> c[n1 + M1 n2], coalesced over n1
template <int M2>
__device__ __forceinline__ void ff_s2(const KArgs &a, const FTask &tk, int m1, const float2 *scr,
                                      float2 *out_row, int lane) {
  const int items = tk.nch * m1;
  constexpr int S2 = M2 | 1;
  const unsigned mag1 = tk.mags >> 16;
  for (int i = lane; i < items; i += 32) {
    const int c = (int)((i * mag1) >> 16), n1 = i - c * m1;
    const int off = __ldg(&a.fch[tk.coff + c].off);
    const float2 *A = scr + (c * m1 + n1) * S2;
    float2 v[M2];
#pragma unroll
    for (int e2 = 0; e2 < M2; ++e2) v[e2] = A[e2];
    dft<M2, +1>(v);
    float2 *o = out_row + off + n1;
#pragma unroll
    for (int n2 = 0; n2 < M2; ++n2) __stcs(o + m1 * n2, v[n2]);
  }
}

#define SLICQ_FSMALL(X) X(4) X(6) X(8) X(10) X(12) X(16) X(18) X(20) X(24) X(30) X(32)
#define SLICQ_FSIZES(X) \
  X(2) X(3) X(4) X(5) X(6) X(8) X(9) X(10) X(12) X(15) X(16) X(18) X(20) X(24) X(25) X(27) X(30) X(32)

// F3 - F5 of forward task t for the unit whose spectrum X[0..N] (padded) is at X -- in this
// CTA's shared memory, or (cluster kernel) another CTA's, through a generic DSMEM address
template <int N>
__device__ __forceinline__ void fwd_task(const KArgs &a, int t, const float2 *X, float2 *scr,
                                         float2 *out_row, int lane) {
  const int4 tv = __ldg(reinterpret_cast<const int4 *>(a.ftask + t));
  FTask tk;
  tk.code = tv.x; tk.nch = tv.y; tk.coff = tv.z; tk.mags = (uint32_t)tv.w;
  const int m1 = tk.code & 255, m2 = (tk.code >> 8) & 255;
  const bool small = (tk.code >> 16) & 1, inter = (tk.code >> 17) & 1;
  if (small) {
    switch (m1) {
#define X_(S) case S: ff_small<S, N>(a, tk, X, out_row, lane, inter); break;
      SLICQ_FSMALL(X_)
#undef X_
    }
    return;
  }
  switch (m1) {
#define X_(S) case S: ff_s1<S, N>(a, tk, m2, X, scr, lane, inter); break;
    SLICQ_FSIZES(X_)
#undef X_
  }
  __syncwarp();
  switch (m2) {
#define X_(S) case S: ff_s2<S>(a, tk, m1, scr, out_row, lane); break;
    SLICQ_FSIZES(X_)
#undef X_
  }
  __syncwarp();
}

// F3 - F5 for one unit: the warps of the CTA take the plan's forward tasks round robin
template <int N, int T>
__device__ __forceinline__ void fwd_channel_stage(const KArgs &a, const float2 *X, float2 *scr_all,
                                                  float2 *out_row) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2 *scr = scr_all + warp * a.fscr;
  for (int t = warp; t < a.nftask; t += T / 32) fwd_task<N>(a, t, X, scr, out_row, lane);
}

// shared memory of the fused forward kernel: X (padded) | FFT twiddles | max(window
// transitions, per-warp channel scratch)
template <int LOGN>
constexpr size_t fused_fwd_smem(int tr, int fscr) {
  const size_t r1 = sizeof(float) * (size_t)((tr + 3) & ~3);
  const size_t r2 = sizeof(float2) * (size_t)fscr * (Big<LOGN>::T / 32);
  return sizeof(float2) * (size_t)(spec_entries<LOGN>() + tw_entries<LOGN>()) + (r1 > r2 ? r1 : r2);
}

template <int LOGN>
__global__ void __launch_bounds__(Big<LOGN>::T, Big<LOGN>::MINB) slicq_fwd_fused_kernel(const KArgs a) {
  using CF = Big<LOGN>;
  extern __shared__ float4 smem4[];
  float2 *spec = reinterpret_cast<float2 *>(smem4);
  float2 *tw = spec + spec_entries<LOGN>();
  float2 *region = tw + tw_entries<LOGN>();
  // F1 + F2: X[0..N] in shared memory (the window-transition table lives in the scratch region)
  fwd_spectrum<LOGN, 0, true>(a, spec, tw, reinterpret_cast<float *>(region),
                              a.unit0 + blockIdx.x, nullptr);
  __syncthreads();
  float2 *out_row = a.coef_out + (a.unit0 + blockIdx.x) * a.C;
  fwd_channel_stage<CF::N, CF::T>(a, spec, region, out_row);
  pdl_trigger();
}

// ---- cluster-fused forward: a thread-block cluster of G CTAs
// owns G consecutive units.  CTA r transforms unit r (F1 + F2) into its own shared memory;
// after one cluster barrier the cluster's warps claim (task, unit) items in task-major order
// from one counter in CTA 0's shared memory (atom.shared::cluster) and read each unit's
// spectrum through DSMEM (mapa: the generic address of the same buffer in CTA g).  No
// staging: the only HBM traffic is the frame read and the coefficient write.  Claiming in
// task order keeps the cluster's warps on one or two code shapes at a time, and each CTA
// walks the task list once per G slices instead of once per slice (the fused per-slice
// kernel's instruction-cache starvation); the dynamic claim balances the CTAs.
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");  // (.release)
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");    // (.acquire)
}
template <class P>
__device__ __forceinline__ const P *cl_map(const P *p, unsigned rank) {  // generic -> CTA rank's copy
  uint64_t r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<const P *>(r);
}
__device__ __forceinline__ unsigned cl_claim(unsigned *ctr_local, unsigned rank) {
  uint32_t sa = (uint32_t)__cvta_generic_to_shared(ctr_local), ra, old;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(sa), "r"(rank));
  asm volatile("atom.shared::cluster.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(ra) : "memory");
  return old;
}

template <int LOGN>
__global__ void __launch_bounds__(Big<LOGN>::T, Big<LOGN>::MINB) slicq_fwd_cluster_kernel(const KArgs a) {
  using CF = Big<LOGN>;
  extern __shared__ float4 smem4[];
  __shared__ unsigned s_next;  // CTA 0's copy: the cluster's item counter
  float2 *spec = reinterpret_cast<float2 *>(smem4);
  float2 *tw = spec + spec_entries<LOGN>();
  float2 *region = tw + tw_entries<LOGN>();
  const unsigned rank = cl_rank(), G = cl_size();
  const int64_t cu0 = (int64_t)blockIdx.x - rank;  // the cluster's first unit (chunk-local)
  const int64_t rem_u = a.nunits - cu0;
  const int nu = rem_u < (int64_t)G ? (int)rem_u : (int)G;
  if (threadIdx.x == 0) s_next = 0;
  if ((int)rank < nu)
    fwd_spectrum<LOGN, 0, true>(a, spec, tw, reinterpret_cast<float *>(region), a.unit0 + cu0 + rank,
                                nullptr);
  cl_sync();  // every spectrum of the cluster complete and visible; the counter is 0
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2 *scr = region + warp * a.fscr;
  const int nitems = a.nftask * nu;
  for (;;) {
    unsigned i = 0;
    if (lane == 0) i = cl_claim(&s_next, 0);
    i = __shfl_sync(FULL, i, 0);
    if ((int)i >= nitems) break;
    const int t = (int)i / nu, g = (int)i - t * nu;
    fwd_task<CF::N>(a, t, cl_map(spec, (unsigned)g), scr, a.coef_out + (a.unit0 + cu0 + g) * a.C, lane);
  }
  cl_sync();  // no CTA leaves while another still reads its spectrum
  pdl_trigger();
}

// Per-size entry points (kernels_spec.cu, one object per LOGN)
template <int LOGN>
int fused_attrs();
template <int LOGN>
cudaError_t launch_fwd_fused(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s, bool pdl);
template <int LOGN>
cudaError_t launch_fwd_cluster(const KArgs &a, int G, size_t smem, cudaStream_t s, bool pdl);

}  // namespace kern
}  // namespace slicq
