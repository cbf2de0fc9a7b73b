// Forward channel kernel v2 (split design, F3 - F5; included by kernels_host.cu only).
//
// The same persistent packet-major structure as slicq_fwd_chan_kernel (a work item is
// (packet, tile of units); the warps of a CTA split the tile's units into warp tasks of nu
// units; every SM runs one packet's code at a time), with two changes measured against it
// (DESIGN.md "Forward channel kernel v2"):
//  * no fold table: a channel's support is read contiguously from the staged spectrum,
//    y[d] = X(lo + d) g_k[d] / sqrt(M_k), and the fold's rotation by lo (j mod M_k, C5) moves
//    into the four-step twiddle w^{(d2 + lo) n1} and the second step's input index;
//  * multi-round warp tasks: a step's lane items (virtual channel, column) may exceed 32 and
//    are processed in rounds, so the plan can pick packet shapes that fill the lanes
//    (round 1's shapes left ~27 % of the lanes idle on cfg4).
#pragma once
#include "kernels_dev.cuh"
#include "kernels_fused.cuh"

namespace slicq {
namespace kern {

// (P2Dev: slicq_internal.h)
struct C2Args {
  const P2Dev *pk;
  int npk;
  const FChan *fch;
};

// X(j) for an unwrapped bin j in (-2N, 2N) from a staged half spectrum X[0..N] (C15)
__device__ __forceinline__ float2 x_at_g(const float2 *Xu, int j, int N) {
  const int jj = j < 0 ? j + 2 * N : j;
  const bool up = jj > N;
  const float2 v = __ldg(Xu + (up ? 2 * N - jj : jj));
  return make_float2(v.x, up ? -v.y : v.y);
}

template <int M, int V>
__device__ __forceinline__ void f2_small(const KArgs &a, const C2Args &c2, const P2Dev &P, int nvc,
                                         const float2 *X, float2 *out, int lane, bool inter) {
  if (lane >= nvc) return;
  const int u = (int)(((unsigned)lane * P.magC) >> 16), c = lane - u * P.nch;
  const FChan ch = ld_fchan(c2.fch + P.coff + c);
  const float2 *Xu = X + (int64_t)u * a.xs;
  const float *g = a.gw + ch.goff;
  float2 v[M];
#pragma unroll
  for (int p = 0; p < M; ++p) {
    int d = p - ch.lo_mod;
    d += d < 0 ? M : 0;
    const bool in = d < ch.len;
    const float w = in ? __ldg(g + d) : 0.f;
    float2 x = make_float2(0.f, 0.f);
    if (in) x = inter ? __ldg(Xu + ch.lo + d) : x_at_g(Xu, ch.lo + d, a.Nh);
    v[p] = make_float2(x.x * w, x.y * w);
  }
  dft<M, +1>(v);
  float2 *o = out + (int64_t)u * a.C + ch.off;
  if (a.vec16) {
    float4 *o4 = reinterpret_cast<float4 *>(o);
#pragma unroll
    for (int n = 0; n < M / 2; ++n)
      SLICQ_CSTORE(o4 + n, make_float4(v[2 * n].x, v[2 * n].y, v[2 * n + 1].x, v[2 * n + 1].y));
  } else {
#pragma unroll
    for (int n = 0; n < M; ++n) SLICQ_CSTORE(o + n, v[n]);
  }
}

template <int M1, int V>
__device__ __forceinline__ void f2_s1(const KArgs &a, const C2Args &c2, const P2Dev &P, int m2,
                                      int nvc, const float2 *X, float2 *scr, int lane, bool inter) {
  const int items = nvc * m2;
  const int S2 = m2 | 1;
  for (int i = lane; i < items; i += 32) {
    const int ci = (int)(((unsigned)i * P.magA) >> 16), d2 = i - ci * m2;
    const int u = (int)(((unsigned)ci * P.magC) >> 16), c = ci - u * P.nch;
    const FChan ch = ld_fchan(c2.fch + P.coff + c);
    const float2 *Xu = X + (int64_t)u * a.xs;
    const float *g = a.gw + ch.goff + d2;
    const int lim = ch.len - d2;
    float2 v[M1];
    if (inter) {
      const float2 *xp = Xu + ch.lo + d2;
#pragma unroll
      for (int d1 = 0; d1 < M1; ++d1) {
        const bool in = d1 * m2 < lim;
        const float w = in ? __ldg(g + d1 * m2) : 0.f;
        const float2 x = in ? __ldg(xp + d1 * m2) : make_float2(0.f, 0.f);
        v[d1] = make_float2(x.x * w, x.y * w);
      }
    } else {
#pragma unroll
      for (int d1 = 0; d1 < M1; ++d1) {
        const bool in = d1 * m2 < lim;
        const float w = in ? __ldg(g + d1 * m2) : 0.f;
        const float2 x = in ? x_at_g(Xu, ch.lo + d2 + d1 * m2, a.Nh) : make_float2(0.f, 0.f);
        v[d1] = make_float2(x.x * w, x.y * w);
      }
    }
    dft<M1, +1>(v);
    int e = d2 + ch.lo_mod;
    e -= e >= ch.M ? ch.M : 0;
    chan_twiddle<M1, +1>(v, e, ch.M, a.twM + ch.twoff);
    int e2 = d2 + ch.lom2;
    e2 -= e2 >= m2 ? m2 : 0;
    float2 *A = scr + ci * M1 * S2 + e2;
#pragma unroll
    for (int n1 = 0; n1 < M1; ++n1) A[n1 * S2] = v[n1];
  }
}

template <int M2, int V>
__device__ __forceinline__ void f2_s2(const KArgs &a, const C2Args &c2, const P2Dev &P, int m1,
                                      int nvc, const float2 *scr, float2 *out, int lane) {
  const int items = nvc * m1;
  constexpr int S2 = M2 | 1;
  for (int i = lane; i < items; i += 32) {
    const int ci = (int)(((unsigned)i * P.magB) >> 16), n1 = i - ci * m1;
    const int u = (int)(((unsigned)ci * P.magC) >> 16), c = ci - u * P.nch;
    const int off = __ldg(&c2.fch[P.coff + c].off);
    const float2 *A = scr + (ci * m1 + n1) * S2;
    float2 v[M2];
#pragma unroll
    for (int e2 = 0; e2 < M2; ++e2) v[e2] = A[e2];
    dft<M2, +1>(v);
    float2 *o = out + (int64_t)u * a.C + off + n1;
#pragma unroll
    for (int n2 = 0; n2 < M2; ++n2) SLICQ_CSTORE(o + m1 * n2, v[n2]);
  }
}

template <int MAXS, int MINB>
__global__ void __launch_bounds__(CHAN_T, MINB) slicq_fwd_chan2_kernel(const KArgs a, const C2Args c2) {
  extern __shared__ float4 smem4[];
  constexpr int NW = CHAN_T / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();
  const int ntiles = (a.nunits + a.tile - 1) / a.tile;
  const int nitems = c2.npk * ntiles;
  float2 *scr = reinterpret_cast<float2 *>(smem4) + warp * a.scr;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int pkx = item / ntiles, tile = item - pkx * ntiles;
    const int4 q0 = __ldg(reinterpret_cast<const int4 *>(c2.pk + pkx));
    const int4 q1 = __ldg(reinterpret_cast<const int4 *>(c2.pk + pkx) + 1);
    P2Dev P;
    P.code = q0.x; P.nch = q0.y; P.coff = q0.z; P.nu = q0.w;
    P.magA = (uint32_t)q1.x; P.magB = (uint32_t)q1.y; P.magC = (uint32_t)q1.z;
    const int m1 = P.code & 255, m2 = (P.code >> 8) & 255;
    const bool small = (P.code >> 16) & 1, inter = (P.code >> 17) & 1;
    const int u_lo = tile * a.tile, u_hi = min(a.nunits, u_lo + a.tile);
    const int ntask = (u_hi - u_lo + P.nu - 1) / P.nu;
    for (int t = warp; t < ntask; t += NW) {
      const int g0 = u_lo + t * P.nu;
      const int nvc = min(P.nu, u_hi - g0) * P.nch;
      const float2 *X = a.stage + (int64_t)g0 * a.xs;
      float2 *out = a.coef_out + (a.unit0 + g0) * a.C;
      if (small) {
        switch (m1) {
#define X_(S) case S: if constexpr (S <= MAXS) f2_small<S, MAXS>(a, c2, P, nvc, X, out, lane, inter); break;
          SLICQ_SMALL(X_)
#undef X_
        }
        continue;
      }
      switch (m1) {
#define X_(S) case S: if constexpr (S <= MAXS) f2_s1<S, MAXS>(a, c2, P, m2, nvc, X, scr, lane, inter); break;
        SLICQ_SIZES(X_)
#undef X_
      }
      __syncwarp();
      switch (m2) {
#define X_(S) case S: if constexpr (S <= MAXS) f2_s2<S, MAXS>(a, c2, P, m1, nvc, scr, out, lane); break;
        SLICQ_SIZES(X_)
#undef X_
      }
      __syncwarp();
    }
  }
  pdl_trigger();
}

}  // namespace kern
}  // namespace slicq
