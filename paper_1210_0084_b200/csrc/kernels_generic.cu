// Generic-length spectrum kernels: slices of any 2/3/5-smooth 2N that fit one CTA's shared
// memory (N <= kGenericMaxN complex points), in particular the non-power-of-two lengths the
// power-of-two kernels (kernels_spec.cu) cannot run, e.g. 2N = 12288, 24000, 50000.
//
// The N-point complex FFT of z[p] = f[2p] + i f[2p+1] (real-input packing, as for 2^k) runs in
// place in shared memory as a mixed-radix decimation-in-time plan chosen at plan time
// (radices 16/8/4/2/3/5): the frame is loaded into digit-reversed positions, each pass combines
// r sub-DFTs of size S with twiddles e^{-+2 pi i j k / (r S)} from an N-entry table, and the
// output comes out in natural order.  Then the r2c packing (forward) or, before the
// FFT, the slot sum and c2r packing (inverse); the inverse ends with the dual
// window and the overlap-add of round 1's spectrum kernel (cross-CTA pairing through the
// workspace).  The channel kernels are the power-of-two path's (they read X[0..N]).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_dev.cuh"
#include "kernels_generic.h"

namespace slicq {
namespace kern {

namespace {

constexpr int GT = 512;  // threads per CTA

template <int R, int SIGN>
__device__ __forceinline__ void gpass(float2 *z, int N, int S, const float2 *twN) {
  const int tasks = N / R;
  const int step = N / (R * S);  // e^{-2 pi i / (R S)} = e^{-2 pi i step / N}
  for (int t = threadIdx.x; t < tasks; t += GT) {
    const int blk = t / S, k = t - blk * S;
    float2 *b = z + blk * R * S + k;
    float2 v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = b[j * S];
    if (S > 1) {
#pragma unroll
      for (int j = 1; j < R; ++j) {
        float2 w = __ldg(twN + j * k * step);
        if (SIGN > 0) w = cconj(w);
        v[j] = cmul(v[j], w);
      }
    }
    dft<R, SIGN>(v);
#pragma unroll
    for (int j = 0; j < R; ++j) b[j * S] = v[j];
  }
}

template <int SIGN>
__device__ __forceinline__ void gfft(float2 *z, const GArgs &g) {
  for (int i = 0; i < g.np; ++i) {
    const int r = g.pass[i].r, S = g.pass[i].S;
    switch (r) {
      case 2: gpass<2, SIGN>(z, g.N, S, g.twN); break;
      case 3: gpass<3, SIGN>(z, g.N, S, g.twN); break;
      case 4: gpass<4, SIGN>(z, g.N, S, g.twN); break;
      case 5: gpass<5, SIGN>(z, g.N, S, g.twN); break;
      case 8: gpass<8, SIGN>(z, g.N, S, g.twN); break;
      case 16: gpass<16, SIGN>(z, g.N, S, g.twN); break;
    }
    __syncthreads();
  }
}

// e^{-i pi k / N} from the two-level table (64 + 2N/64 entries; any N)
__device__ __forceinline__ float2 tw2(const float2 *t, int k) {
  return cmul(__ldg(t + 64 + (k >> 6)), __ldg(t + (k & 63)));
}

}  // namespace

// F1 + F2 of one unit per CTA (MODE 0: windowed slice, MODE 1: the whole signal as the frame)
template <int MODE>
__global__ void __launch_bounds__(GT, 1) slicq_fwd_spec_generic(const KArgs a, const GArgs g) {
  extern __shared__ float4 smem4[];
  float2 *z = reinterpret_cast<float2 *>(smem4);
  const int N = g.N, tid = threadIdx.x;
  const int64_t ul = blockIdx.x, u = a.unit0 + ul;
  const int64_t row = unit_row(u, a.nslices), mloc = u - row * a.nslices;
  const int64_t mg = a.slice0 + mloc;
  const float *xr = a.x + row * a.x_stride;
  const int64_t s0 = MODE ? -a.base_off : (mg - 1) * N - a.base_off;  // frame sample 0
  const int Bw = MODE ? N + 1 : (N + a.tr) / 2;  // |t| < Bw: nonzero window
  pdl_wait();
  auto sample = [&](int i) -> float {  // windowed frame sample i (t = i - N)
    const int t = i - N;
    if (!MODE && (t <= -Bw || t >= Bw)) return 0.f;
    int64_t xi = s0 + i;
    if (a.wrap && xi < 0) xi += a.L;
    const float xv = (xi >= 0 && xi < a.x_len) ? __ldg(xr + xi) : 0.f;
    return MODE ? xv : xv * __ldg(a.h0 + i);
  };
  for (int p = tid; p < N; p += GT) z[__ldg(g.perm + p)] = make_float2(sample(2 * p), sample(2 * p + 1));
  __syncthreads();
  gfft<-1>(z, g);
  // r2c packing: X[k] = E[k] + e^{-i pi k / N} O[k], k = 0..N (Z[N] := Z[0])
  for (int k = tid; k <= N / 2; k += GT) {
    const float2 zk = z[k], zn = z[k == 0 ? 0 : N - k];
    if (k == 0) {
      z[0] = make_float2(zk.x + zk.y, 0.f);
      // X[N] goes straight to the staging row below (z has N entries)
    } else {
      const float2 E = cscale(cadd(zk, cconj(zn)), 0.5f);
      const float2 O = cscale(mul_si<-1>(csub(zk, cconj(zn))), 0.5f);
      const float2 wO = cmul(tw2(a.tw2n, k), O);
      z[k] = cadd(E, wO);
      if (k != N - k) z[N - k] = csub(cconj(E), cconj(wO));
    }
    if (k == 0) a.stage[ul * a.xs + N] = make_float2(zk.x - zk.y, 0.f);
  }
  __syncthreads();
  float2 *Xo = a.stage + ul * a.xs;
  for (int k = tid; k < N; k += GT) Xo[k] = z[k];
  pdl_trigger();
}

// I3b + I4 + I5 of one unit per CTA (MODE 0: dual window + paired overlap-add; MODE 1: the
// frame is the signal)
template <int MODE>
__global__ void __launch_bounds__(GT, 1) slicq_inv_spec_generic(const KArgs a, const GArgs g) {
  extern __shared__ float4 smem4[];
  float2 *z = reinterpret_cast<float2 *>(smem4);
  const int N = g.N, tid = threadIdx.x;
  const int64_t ul = blockIdx.x, u = a.unit0 + ul;
  const int64_t row = unit_row(u, a.nslices);
  const int mloc = (int)(u - row * a.nslices);
  const int64_t mg = a.slice0 + mloc;
  pdl_wait();
  // half-spectrum bin b: slot0 + slot1 (+ its overflow run in plan order)
  const float2 *Z0 = a.stage + ul * a.zs, *Z1 = Z0 + a.zso, *Zo = Z0 + 2 * a.zso;
  auto H = [&](int b) {
    float2 h = cadd(__ldcg(Z0 + b), __ldcg(Z1 + b));
    const uint32_t d = __ldg(a.dpos + b);
    for (int e = 0; e < (int)(d >> 20); ++e) h = cadd(h, __ldcg(Zo + (d & 0xfffff) + e));
    return h;
  };
  // c2r packing Z[k] = E + iO, E = (H[k] + conj H[N-k])/2, O = (H[k] - conj H[N-k]) e^{+i pi k/N}/2,
  // written to the digit-reversed positions of the in-place DIT
  for (int k = tid; k <= N / 2; k += GT) {
    const float2 hk = H(k), hn = H(N - k);
    const float2 E = cscale(cadd(hk, cconj(hn)), 0.5f);
    const float2 D = cscale(csub(hk, cconj(hn)), 0.5f);
    const float2 w = cconj(tw2(a.tw2n, k));
    const float2 O = cmul(D, w);
    z[__ldg(g.perm + k)] = cadd(E, mul_si<+1>(O));
    if (k != 0 && k != N - k) {
      z[__ldg(g.perm + (N - k))] = cadd(cconj(E), make_float2(O.y, O.x));  // (conj D)(conj w) = conj O
    }
  }
  __syncthreads();
  gfft<+1>(z, g);
  const float invN = 1.0f / (float)N;
  auto fr = [&](int i) {  // frame sample i
    const float2 v = z[i >> 1];
    return ((i & 1) ? v.y : v.x) * invN;
  };
  float *yrow = a.y + row * a.y_stride;
  if constexpr (MODE == 1) {
    const int cnt = (int)min((int64_t)(2 * N), a.y_len);
    for (int i = tid; i < cnt; i += GT) yrow[i] = fr(i);
    pdl_trigger();
    return;
  }
  const int A = (N - a.tr) / 2, Bw = (N + a.tr) / 2;
  const int S = a.nslices;
  const bool left_paired = a.circular || mloc > 0;
  const bool right_paired = a.circular || mloc + 1 < S;
  const int bl = mloc > 0 ? mloc - 1 : S - 1, br = mloc;
  const int trp = a.tr;
  float *bnd_row = a.bnd + (int64_t)row * S * 2 * trp;
  const int64_t sbase = (mg - 1) * N;
  const float *hd = a.h0dual;  // h~_0[t + N]
  // exclusive part |t| <= A: h~_0 = 1
  for (int i = N - A + tid; i <= N + A; i += GT) {
    const float val = fr(i);
    const int64_t sg = sbase + i;
    if (a.circular) {
      const int64_t sw = sg < 0 ? sg + a.L : (sg >= a.L ? sg - a.L : sg);
      if (sw < a.y_len) yrow[sw] = val;
    } else {
      const int64_t li = sg - a.y_base;
      if (li >= 0) yrow[li] = val;
      else a.spill[row * a.halo + (li + a.halo)] = val;
    }
  }
  // transitions, u = 0 .. tr-2
  for (int u2 = tid; u2 < trp - 1; u2 += GT) {
    const int il = N - Bw + 1 + u2;
    const float vl = fr(il) * __ldg(hd + il);
    const int64_t sl = sbase + il;
    if (left_paired) bnd_row[((int64_t)bl * 2 + 1) * trp + u2] = vl;
    else a.spill[row * a.halo + (sl - a.y_base + a.halo)] = vl;
    const int ir = N + A + 1 + u2;
    const float vr = fr(ir) * __ldg(hd + ir);
    if (right_paired) bnd_row[((int64_t)br * 2 + 0) * trp + u2] = vr;
    else yrow[sbase + ir - a.y_base] = vr;
  }
  if (!a.circular && mloc + 1 == S)
    for (int u2 = tid; u2 < A; u2 += GT) yrow[(mg + 1) * N - A + u2 - a.y_base] = 0.f;
  if (!a.circular && mloc == 0)
    for (int u2 = tid; u2 < a.halo - (Bw - 1); u2 += GT) a.spill[row * a.halo + u2] = 0.f;
  // pairing: the second CTA to finish a boundary adds both halves (as slicq_inv_spec_kernel)
  __syncthreads();
  __shared__ int sflag[2];
  if (tid == 0) {
    __threadfence();
    int second_l = 0, second_r = 0;
    if (left_paired) second_l = (atomicAdd(a.cnt + row * S + bl, 1u) & 1u) ? 1 : 0;
    if (right_paired) second_r = (atomicAdd(a.cnt + row * S + br, 1u) & 1u) ? 1 : 0;
    __threadfence();
    sflag[0] = second_l;
    sflag[1] = second_r;
  }
  __syncthreads();
  const bool f0 = sflag[0], f1 = sflag[1];
  if (f0 || f1) {
    const float *hp0 = bnd_row + ((int64_t)bl * 2 + 0) * trp;
    const float *hp1 = bnd_row + ((int64_t)br * 2 + 1) * trp;
    const int64_t t0 = (a.slice0 + bl) * N + A + 1, t1 = (a.slice0 + br) * N + A + 1;
    auto put = [&](int64_t s, float val) {
      if (a.circular) {
        const int64_t sw = s >= a.L ? s - a.L : s;
        if (sw < a.y_len) yrow[sw] = val;
      } else {
        yrow[s - a.y_base] = val;
      }
    };
    for (int u2 = tid; u2 < trp - 1; u2 += GT) {
      const float p0 = f0 ? __ldcg(hp0 + u2) : 0.f, p1 = f1 ? __ldcg(hp1 + u2) : 0.f;
      const int il = N - Bw + 1 + u2, ir = N + A + 1 + u2;
      if (f0) put(t0 + u2, p0 + __fmul_rn(fr(il), __ldg(hd + il)));
      if (f1) put(t1 + u2, p1 + __fmul_rn(fr(ir), __ldg(hd + ir)));
    }
  }
  pdl_trigger();
}

size_t generic_smem_bytes(int N) { return sizeof(float2) * (size_t)N; }

int generic_set_attrs() {
  const void *fns[] = {(const void *)slicq_fwd_spec_generic<0>, (const void *)slicq_fwd_spec_generic<1>,
                       (const void *)slicq_inv_spec_generic<0>, (const void *)slicq_inv_spec_generic<1>};
  for (const void *f : fns) {
    const cudaError_t e = allow_max_dyn_smem(f);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

cudaError_t launch_generic(bool fwd, const KArgs &a, const GArgs &g, int nunits, cudaStream_t s,
                           bool pdl, int mode) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nunits);
  cfg.blockDim = dim3(GT);
  cfg.dynamicSmemBytes = generic_smem_bytes(g.N);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (fwd)
    return mode ? cudaLaunchKernelEx(&cfg, slicq_fwd_spec_generic<1>, a, g)
                : cudaLaunchKernelEx(&cfg, slicq_fwd_spec_generic<0>, a, g);
  return mode ? cudaLaunchKernelEx(&cfg, slicq_inv_spec_generic<1>, a, g)
              : cudaLaunchKernelEx(&cfg, slicq_inv_spec_generic<0>, a, g);
}

}  // namespace kern
}  // namespace slicq
