// Large slices (2N >= 65536: the spectrum of one slice exceeds a CTA's shared memory).
// The N-point complex FFT of the r2c / c2r step is split four-step style, N = N1 * N2
// (N2 = 256), through the workspace staging buffer:
//
//   z index p = N2 p1 + p2, spectrum index k = k1 + N1 k2
//   Z[k1 + N1 k2] = sum_p2 w_N2^{p2 k2} w_N^{p2 k1} sum_p1 z[N2 p1 + p2] w_N1^{p1 k1}
//
// forward:  fwd_large_col  (16 columns p2 per CTA: window F1, DFT_N1, twiddle) -> T[k1][p2]
//           fwd_large_row  (rows k1 and N1-k1: DFT_N2, r2c packing) -> X[0..N]
// inverse:  inv_large_pack (per-bin gather of the channel contributions + c2r packing) -> W
//           inv_large_col  (DFT_N1 over p1 per column, twiddle, in place)
//           inv_large_row  (16 rows n1 per CTA: DFT_N2, dual window, overlap-add; slice
//                           boundary halves to the workspace)
//           inv_large_bnd  (side0 + side1 for every paired boundary)
// Same arithmetic as the single-CTA kernels (kernels_dev.cuh), only the data movement of the
// FFT differs.
#pragma once
#include "kernels_dev.cuh"

namespace slicq {
namespace kern {

template <int LOGN>
struct Large;
template <>
struct Large<15> {
  static constexpr int N = 32768, N1 = 128, N2 = 256;
  static constexpr int C1 = 16, C2 = 8;  // column DFT radices (N1)
};
template <>
struct Large<16> {
  static constexpr int N = 65536, N1 = 256, N2 = 256;
  static constexpr int C1 = 16, C2 = 16;
};
constexpr int LT = 256;        // threads per CTA
constexpr int LB = 16;         // columns / rows per CTA
constexpr int R_ROW = 16;      // row DFT radices (N2 = 256 = 16 * 16)

template <int P>
constexpr int colstride() {
  return padi(P) + 2;
}

// B = LB independent P-point Stockham passes in shared memory (column c at c * CS)
template <int NTAB, int P, int R, int NS, int SIGN, class TW>
__device__ __forceinline__ void bpass(float2 *buf, TW tw) {
  constexpr int TPC = P / R, TASKS = LB * TPC, PER = (TASKS + LT - 1) / LT;
  constexpr int CS = colstride<P>();
  float2 v[PER][R];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int t = threadIdx.x + q * LT;
    if (TASKS % LT == 0 || t < TASKS) {
      const int c = t / TPC, j = t - c * TPC;
      const float2 *col = buf + c * CS;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = col[padi(j + r * TPC)];
      pass_twiddle<NTAB, R, NS, SIGN>(v[q], j, tw);
      dft<R, SIGN>(v[q]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int t = threadIdx.x + q * LT;
    if (TASKS % LT == 0 || t < TASKS) {
      const int c = t / TPC, j = t - c * TPC;
      float2 *col = buf + c * CS;
      const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
      for (int r = 0; r < R; ++r) col[padi(base + r * NS)] = v[q][r];
    }
  }
  __syncthreads();
}

// e^{-i pi e/N}, e any integer (reduced mod 2N)
template <int N, class TW>
__device__ __forceinline__ float2 tw_any(TW tw, int64_t e) {
  return tw_lookup(tw, (int)(e & (2 * N - 1)));
}

__device__ __forceinline__ void unit_coords(const KArgs &a, int64_t ul, int64_t &row,
                                            int64_t &mloc, int64_t &mg) {
  const int64_t u = a.unit0 + ul;
  row = unit_row(u, a.nslices);
  mloc = u - row * a.nslices;
  mg = a.slice0 + mloc;
}

// ------------------------------------------------------------------ forward
template <int LOGN, int MODE = 0>  // MODE 1: full-length CQ-NSGT frame (no window)
__global__ void __launch_bounds__(LT) fwd_large_col(const KArgs a) {
  using G = Large<LOGN>;
  constexpr int N = G::N, N1 = G::N1, N2 = G::N2, CS = colstride<N1>();
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const GlobalTw tw{a.tw2n};  // two-level twiddle table, read through L1 (17 KB at N = 65536)
  const int tid = threadIdx.x;
  const int64_t ul = blockIdx.x;
  int64_t row, mloc, mg;
  unit_coords(a, ul, row, mloc, mg);
  const int p2_0 = blockIdx.y * LB;
  pdl_wait();
  // F1: windowed z[N2 p1 + p2] = (f[2p], f[2p+1]) * h_0, 16 consecutive p2 per row p1
  {
    const float *xr = a.x + row * a.x_stride;
    const bool vec = ((reinterpret_cast<uintptr_t>(xr) & 7) == 0);
    const int64_t s0 = (mg - 1) * N - a.base_off;
    const int A = (N - a.tr) / 2, Bw = (N + a.tr) / 2;
    for (int idx = tid; idx < LB * N1; idx += LT) {
      const int c = idx % LB, p1 = idx / LB;
      const int i0 = 2 * (N2 * p1 + p2_0 + c);
      const int t0 = i0 - N;
      const int at0 = t0 < 0 ? -t0 : t0;
      const int at1 = (t0 + 1) < 0 ? -(t0 + 1) : (t0 + 1);
      float x0 = 0.f, x1 = 0.f;
      if (MODE == 1 || at0 < Bw || at1 < Bw) {
        int64_t xi = s0 + i0;
        if (a.wrap && xi < 0) xi += a.L;
        if (vec && xi >= 0 && xi + 1 < a.x_len) {
          const float2 xv = __ldcs(reinterpret_cast<const float2 *>(xr + xi));
          x0 = xv.x;
          x1 = xv.y;
        } else {
          if (xi >= 0 && xi < a.x_len) x0 = __ldg(xr + xi);
          if (xi + 1 >= 0 && xi + 1 < a.x_len) x1 = __ldg(xr + xi + 1);
        }
        if constexpr (MODE == 0) {
          const float ha = at0 <= A ? 1.f : (at0 < Bw ? __ldg(a.h0 + i0) : 0.f);
          const float hb = at1 <= A ? 1.f : (at1 < Bw ? __ldg(a.h0 + i0 + 1) : 0.f);
          x0 *= ha;
          x1 *= hb;
        }
      }
      buf[c * CS + padi(p1)] = make_float2(x0, x1);
    }
  }
  __syncthreads();
  bpass<N, N1, G::C1, 1, -1>(buf, tw);
  bpass<N, N1, G::C2, G::C1, -1>(buf, tw);
  // twiddle w_N^{p2 k1} and store T[k1][p2]
  float2 *T = a.stage + ul * a.xs + a.toff;
  for (int idx = tid; idx < LB * N1; idx += LT) {
    const int c = idx % LB, k1 = idx / LB;
    const int p2 = p2_0 + c;
    const float2 v = cmul(buf[c * CS + padi(k1)], tw_any<N>(tw, 2 * (int64_t)p2 * k1));
    T[(int64_t)k1 * N2 + p2] = v;
  }
  pdl_trigger();
}

template <int LOGN>
__global__ void __launch_bounds__(LT) fwd_large_row(const KArgs a) {
  using G = Large<LOGN>;
  constexpr int N = G::N, N1 = G::N1, N2 = G::N2, CS = colstride<N2>();
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const GlobalTw tw{a.tw2n};  // two-level twiddle table, read through L1 (17 KB at N = 65536)
  const int tid = threadIdx.x;
  const int64_t ul = blockIdx.x;
  const int kb = blockIdx.y * 8;  // rows kb..kb+7 (<= N1/2) and their partners N1 - k1
  pdl_wait();
  const float2 *T = a.stage + ul * a.xs + a.toff;
  auto slot_row = [&](int s) -> int {  // -1: empty slot
    if (s < 8) return kb + s <= N1 / 2 ? kb + s : -1;
    const int k1 = kb + s - 8;
    return (k1 > 0 && k1 < N1 / 2) ? N1 - k1 : -1;
  };
  {  // all of a thread's row loads in flight together (streaming, L2 only)
    constexpr int PERL = LB * N2 / LT;
    float2 v[PERL];
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LT, s = idx / N2, k2 = idx % N2;
      const int r = slot_row(s);
      v[q] = r >= 0 ? __ldcs(T + (int64_t)r * N2 + k2) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LT;
      buf[(idx / N2) * CS + padi(idx % N2)] = v[q];
    }
  }
  __syncthreads();
  bpass<N, N2, R_ROW, 1, -1>(buf, tw);
  bpass<N, N2, R_ROW, R_ROW, -1>(buf, tw);
  // buf[slot][k2] = Z[k1 + N1 k2].  r2c packing (as in slicq_fwd_spec_kernel):
  // X[k] = E + w O, X[N-k] = conj(E) - conj(w O), w = e^{-i pi k/N}
  float2 *Xo = a.stage + ul * a.xs;
  // consecutive threads take consecutive rows k1 of one column k2: the outputs
  // X[k1 + N1 k2] (and their mirrors) are stored as 8-entry contiguous runs
  for (int idx = tid; idx < 8 * N2; idx += LT) {
    const int s = idx % 8, k2 = idx / 8;
    const int k1 = kb + s;
    if (k1 > N1 / 2) continue;
    int ps, pk2;  // partner slot / column of Z[N - k]
    if (k1 == 0) {
      if (k2 > N2 / 2) continue;
      ps = s;
      pk2 = (N2 - k2) & (N2 - 1);
    } else if (k1 == N1 / 2) {
      if (k2 >= N2 / 2) continue;
      ps = s;
      pk2 = N2 - 1 - k2;
    } else {
      ps = s + 8;
      pk2 = N2 - 1 - k2;
    }
    const int k = k1 + N1 * k2;
    const float2 zk = buf[s * CS + padi(k2)];
    const float2 zn = buf[ps * CS + padi(pk2)];
    if (k == 0) {
      Xo[0] = make_float2(zk.x + zk.y, 0.f);
      Xo[N] = make_float2(zk.x - zk.y, 0.f);
      continue;
    }
    const float2 E = cscale(cadd(zk, cconj(zn)), 0.5f);
    const float2 O = cscale(mul_si<-1>(csub(zk, cconj(zn))), 0.5f);
    const float2 wO = cmul(tw_lookup(tw, k), O);
    Xo[k] = cadd(E, wO);
    if (k != N / 2) Xo[N - k] = csub(cconj(E), cconj(wO));
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ inverse
// c2r packing of the gathered half spectrum H (see slicq_inv_spec_kernel):
// Z[k] = E + iO, Z[N-k] = conj(E) + i conj(D) e^{-i pi k/N}, E = (H[k] + conj H[N-k])/2,
// D = (H[k] - conj H[N-k])/2, O = D e^{+i pi k/N}.
template <int N>
__device__ __forceinline__ float2 gather_bin(const KArgs &a, const float2 *Z, int b) {
  float2 acc = cadd(__ldcg(Z + b), __ldcg(Z + a.zso + b));
  const uint32_t dp = __ldg(a.dpos + b);
  if (dp) {  // deep-overlap bin: overflow terms in order
    const float2 *Zo = Z + 2 * a.zso + (dp & 0xfffff);
    const int cnt = dp >> 20;
    for (int i = 0; i < cnt; ++i) acc = cadd(acc, __ldcg(Zo + i));
  }
  return acc;
}

template <int LOGN>
__global__ void __launch_bounds__(LT) inv_large_pack(const KArgs a) {
  using G = Large<LOGN>;
  constexpr int N = G::N;
  const GlobalTw tw{a.tw2n};  // two-level twiddle table, read through L1
  pdl_wait();
  const int64_t ul = blockIdx.x;
  const float2 *Z = a.stage + ul * a.zs;
  float2 *W = a.stage + ul * a.zs + a.toff;
  const int k = blockIdx.y * LT + threadIdx.x;
  if (k <= N / 2) {
    const float2 hk = gather_bin<N>(a, Z, k);
    const float2 hn = gather_bin<N>(a, Z, N - k);
    const float2 E = cscale(cadd(hk, cconj(hn)), 0.5f);
    const float2 D = cscale(csub(hk, cconj(hn)), 0.5f);
    const float2 w = cconj(tw_lookup(tw, k));  // e^{+i pi k/N}
    const float2 O = cmul(D, w);
    W[k] = cadd(E, mul_si<+1>(O));
    if (k != 0 && k != N / 2) {
      W[N - k] = cadd(cconj(E), make_float2(O.y, O.x));  // (conj D)(conj w) = conj O
    }
  }
  pdl_trigger();
}

template <int LOGN>
__global__ void __launch_bounds__(LT) inv_large_col(const KArgs a) {
  using G = Large<LOGN>;
  constexpr int N = G::N, N1 = G::N1, N2 = G::N2, CS = colstride<N1>();
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const GlobalTw tw{a.tw2n};  // two-level twiddle table, read through L1 (17 KB at N = 65536)
  const int tid = threadIdx.x;
  const int64_t ul = blockIdx.x;
  const int p2_0 = blockIdx.y * LB;
  pdl_wait();
  float2 *W = a.stage + ul * a.zs + a.toff;
  {  // all of a thread's column loads in flight together (streaming, L2 only)
    constexpr int PERL = LB * N1 / LT;
    float2 v[PERL];
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LT;
      v[q] = __ldcs(W + (int64_t)N2 * (idx / LB) + p2_0 + idx % LB);
    }
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LT;
      buf[(idx % LB) * CS + padi(idx / LB)] = v[q];
    }
  }
  __syncthreads();
  bpass<N, N1, G::C1, 1, +1>(buf, tw);
  bpass<N, N1, G::C2, G::C1, +1>(buf, tw);
  for (int idx = tid; idx < LB * N1; idx += LT) {
    const int c = idx % LB, n1 = idx / LB;
    const int p2 = p2_0 + c;
    const float2 v = cmul(buf[c * CS + padi(n1)], cconj(tw_any<N>(tw, 2 * (int64_t)p2 * n1)));
    W[(int64_t)n1 * N2 + p2] = v;  // same columns as read: in place per CTA
  }
  pdl_trigger();
}

// rows n1 in [16 b, 16 b + 16): z[n1 + N1 n2] -> samples 2n, 2n+1, times h~_0 / N.
// Exclusive samples go to y; transition samples of a paired boundary to the workspace
// (combined by inv_large_bnd); unpaired ones (slice-range edges) straight to y / the spill.
template <int LOGN, int MODE = 0>  // MODE 1: full-length CQ-NSGT synthesis (frame -> y)
__global__ void __launch_bounds__(LT) inv_large_row(const KArgs a) {
  using G = Large<LOGN>;
  constexpr int N = G::N, N1 = G::N1, N2 = G::N2, CS = colstride<N2>();
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const GlobalTw tw{a.tw2n};  // two-level twiddle table, read through L1 (17 KB at N = 65536)
  const int tid = threadIdx.x;
  const int64_t ul = blockIdx.x;
  int64_t row, mloc, mg;
  unit_coords(a, ul, row, mloc, mg);
  const int n1_0 = blockIdx.y * LB;
  pdl_wait();
  const float2 *W = a.stage + ul * a.zs + a.toff;
  {  // all of a thread's row loads in flight together (streaming, L2 only)
    constexpr int PERL = LB * N2 / LT;
    float2 v[PERL];
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LT;
      v[q] = __ldcs(W + (int64_t)(n1_0 + idx / N2) * N2 + idx % N2);
    }
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LT;
      buf[(idx / N2) * CS + padi(idx % N2)] = v[q];
    }
  }
  __syncthreads();
  bpass<N, N2, R_ROW, 1, +1>(buf, tw);
  bpass<N, N2, R_ROW, R_ROW, +1>(buf, tw);
  const int A = (N - a.tr) / 2, Bw = (N + a.tr) / 2;
  const float invN = 1.0f / (float)N;
  const int S = a.nslices;
  const bool left_paired = a.circular || mloc > 0;
  const bool right_paired = a.circular || mloc + 1 < S;
  const int64_t bl = mloc > 0 ? mloc - 1 : S - 1, br = mloc;
  const int trp = a.tr;
  float *yrow = a.y + row * a.y_stride;
  float *bnd_row = a.bnd + row * (int64_t)S * 2 * trp;
  if constexpr (MODE == 1) {  // the frame is the signal: samples 2p, 2p+1 -> y (p < N)
    for (int idx = tid; idx < LB * N2; idx += LT) {
      const int s = idx % LB, n2 = idx / LB;
      const float2 z = buf[s * CS + padi(n2)];
      const int64_t i = 2 * (int64_t)(n1_0 + s + N1 * n2);
      if (i < a.y_len) yrow[i] = z.x * invN;
      if (i + 1 < a.y_len) yrow[i + 1] = z.y * invN;
    }
    (void)A; (void)Bw; (void)left_paired; (void)right_paired; (void)bl; (void)br; (void)trp;
    (void)bnd_row; (void)S;
  } else {
  // consecutive threads take consecutive n1 (16 rows) of one n2: 32 consecutive samples
  for (int idx = tid; idx < LB * N2; idx += LT) {
    const int s = idx % LB, n2 = idx / LB;
    const float2 z = buf[s * CS + padi(n2)];
    const int p = n1_0 + s + N1 * n2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * p + h;
      const int t = i - N;
      const int at = t < 0 ? -t : t;
      const int64_t sg = (mg - 1) * N + i;
      if (at >= Bw) {
        // range mode, last local slice: zero the samples no local slice reaches
        if (!a.circular && mloc + 1 == S && t >= Bw) yrow[sg - a.y_base] = 0.f;
        continue;
      }
      const float hd = at <= A ? 1.f : __ldg(a.h0dual + i);
      const float val = (h ? z.y : z.x) * invN * hd;
      if (at <= A) {
        if (a.circular) {
          const int64_t sw = sg < 0 ? sg + a.L : (sg >= a.L ? sg - a.L : sg);
          if (sw < a.y_len) yrow[sw] = val;
        } else {
          const int64_t li = sg - a.y_base;
          if (li >= 0) yrow[li] = val;
          else a.spill[row * a.halo + (li + a.halo)] = val;
        }
      } else if (t < 0) {
        const int u = t + Bw - 1;
        if (left_paired) bnd_row[(bl * 2 + 1) * trp + u] = val;
        else a.spill[row * a.halo + (sg - a.y_base + a.halo)] = val;
      } else {
        const int u = t - A - 1;
        if (right_paired) bnd_row[(br * 2 + 0) * trp + u] = val;
        else yrow[sg - a.y_base] = val;
      }
    }
  }
  if (!a.circular && mloc == 0 && blockIdx.y == 0)
    for (int u = tid; u < a.halo - (Bw - 1); u += LT) a.spill[row * a.halo + u] = 0.f;
  }  // MODE 0
  pdl_trigger();
}

// y = side0 + side1 on the tr-1 samples of every paired boundary (right boundary of each unit)
template <int LOGN>
__global__ void __launch_bounds__(LT) inv_large_bnd(const KArgs a) {
  constexpr int N = Large<LOGN>::N;
  pdl_wait();
  const int64_t ul = blockIdx.x;
  int64_t row, mloc, mg;
  unit_coords(a, ul, row, mloc, mg);
  const int S = a.nslices;
  if (!(a.circular || mloc + 1 < S)) return;
  const int A = (N - a.tr) / 2;
  const int trp = a.tr;
  const float *h0p = a.bnd + row * (int64_t)S * 2 * trp + mloc * 2 * trp;
  const float *h1p = h0p + trp;
  float *yrow = a.y + row * a.y_stride;
  for (int u = blockIdx.y * LT + threadIdx.x; u < a.tr - 1; u += gridDim.y * LT) {
    const float val = __ldcg(h0p + u) + __ldcg(h1p + u);
    const int64_t sg = mg * N + A + 1 + u;
    if (a.circular) {
      const int64_t sw = sg >= a.L ? sg - a.L : sg;
      if (sw < a.y_len) yrow[sw] = val;
    } else {
      yrow[sg - a.y_base] = val;
    }
  }
  pdl_trigger();
}

template <int LOGN>
constexpr size_t large_smem_bytes() {
  return sizeof(float2) * (size_t)(LB * colstride<256>());
}

// entry points (kernels_large.cu)
template <int LOGN>
int large_set_attrs();
template <int LOGN>
cudaError_t large_forward(const KArgs &a, cudaStream_t s, int mode = 0, bool cluster = false);
template <int LOGN>
cudaError_t large_inverse_spec(const KArgs &a, cudaStream_t s, int mode = 0, bool cluster = false);
template <int LOGN>
bool large_cluster_ok();  // the 16-CTA cluster kernels can be resident (2N = 131072)

}  // namespace kern
}  // namespace slicq
