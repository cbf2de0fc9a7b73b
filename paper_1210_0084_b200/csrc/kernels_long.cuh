// Full-length CQ-NSGT for long signals, L = 2N = 2^18 .. 2^22:
// Alg. 1 / Alg. 2 on the whole signal, one "unit" per batch row.  The sliCQ
// path's per-slice machinery (packet tables, 14/17-bit element encodings, one-CTA spectra)
// is sized for slices <= 2^17; a whole signal needs the same steps at larger sizes:
//
//   FFT_L (r2c)   four-step N = N1 * 256 through the staging buffer: long_fwd_col (NB
//                 columns of N1 points per CTA, three Stockham passes in shared memory,
//                 twiddle) -> fwd_large_row (256-point rows + r2c packing, kernels_large.cuh)
//   channels      long_chan_fwd: one CTA per (channel, row): fold X(j) g_k[j]/sqrt(M_k) into
//                 a shared-memory vector of M_k (painless: one term per position, M_k >= L_k),
//                 in-place mixed-radix (2/3/4/5/8/9/16/25) decimation-in-frequency IFFT_{M_k}
//                 (runtime radix sequence, table twiddles e^{2 pi i t/M_k}), coefficients
//                 stored from the digit-reversed positions
//   synthesis     long_chan_inv: FFT_{M_k} of c_k, term F_k[j mod M_k] g~_k[j]/sqrt(M_k) per
//                 support bin to the row's term array (channel k at goff_k);
//                 long_inv_pack: per half-spectrum bin the sum of its terms in plan order
//                 (CSR: term index | conj << 31, Hermitian rule C15) + c2r packing;
//                 long_inv_col + inv_large_row<LOGN, 1> (c2r IFFT_L, 1/N, y)
//
// Deterministic (no atomics).  M_k is limited by shared memory (M_k <= 27 000, checked at
// plan time); the radix sequence is the greedy rule long_radix() on both sides (the
// butterflies and the digit reversal of the output).
#pragma once
#include "kernels_large.cuh"
#include "kernels_long_api.h"

namespace slicq {
namespace kern {

template <>
struct Large<17> {
  static constexpr int N = 1 << 17, N1 = 512, N2 = 256;
};
template <>
struct Large<18> {
  static constexpr int N = 1 << 18, N1 = 1024, N2 = 256;
};
template <>
struct Large<19> {
  static constexpr int N = 1 << 19, N1 = 2048, N2 = 256;
};
template <>
struct Large<20> {
  static constexpr int N = 1 << 20, N1 = 4096, N2 = 256;
};
template <>
struct Large<21> {
  static constexpr int N = 1 << 21, N1 = 8192, N2 = 256;
};

// column FFTs of the four-step: P = N1 points, NB columns per CTA (NB * P = 8192 points,
// 16 per thread), radices R1 R2 R3 (R3 = 1: two passes)
template <int LOGN>
struct LongCol;
template <>
struct LongCol<17> {
  static constexpr int P = 512, NB = 16, R1 = 16, R2 = 32, R3 = 1;
};
template <>
struct LongCol<18> {
  static constexpr int P = 1024, NB = 8, R1 = 32, R2 = 32, R3 = 1;
};
template <>
struct LongCol<19> {
  static constexpr int P = 2048, NB = 4, R1 = 16, R2 = 16, R3 = 8;
};
template <>
struct LongCol<20> {
  static constexpr int P = 4096, NB = 2, R1 = 16, R2 = 16, R3 = 16;
};
template <>
struct LongCol<21> {
  static constexpr int P = 8192, NB = 1, R1 = 16, R2 = 16, R3 = 32;
};
constexpr int LCT = 512;  // column-kernel threads

template <int LOGN>
constexpr size_t long_col_smem() {
  return sizeof(float2) * (size_t)(LongCol<LOGN>::NB * colstride<LongCol<LOGN>::P>());
}

// NB independent P-point Stockham passes in shared memory (column c at c * CS), LCT threads
template <int NTAB, int P, int NB, int R, int NS, int SIGN, class TW>
__device__ __forceinline__ void cpass(float2 *buf, TW tw) {
  if constexpr (R > 1) {
    constexpr int TPC = P / R, TASKS = NB * TPC, PER = (TASKS + LCT - 1) / LCT;
    constexpr int CS = colstride<P>();
    float2 v[PER][R];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int t = threadIdx.x + q * LCT;
      if (TASKS % LCT == 0 || t < TASKS) {
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
      const int t = threadIdx.x + q * LCT;
      if (TASKS % LCT == 0 || t < TASKS) {
        const int c = t / TPC, j = t - c * TPC;
        float2 *col = buf + c * CS;
        const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
        for (int r = 0; r < R; ++r) col[padi(base + r * NS)] = v[q][r];
      }
    }
    __syncthreads();
  }
}

// forward four-step, first half: z[N2 p1 + p2] = (x[2p], x[2p+1]) (zero past n), DFT_N1 over
// p1 for NB consecutive columns p2, twiddle w_N^{p2 k1}, T[k1][p2] to the staging buffer
template <int LOGN>
__global__ void __launch_bounds__(LCT) long_fwd_col(const KArgs a) {
  using G = LongCol<LOGN>;
  constexpr int N = 1 << LOGN, P = G::P, NB = G::NB, N2 = 256, CS = colstride<P>();
  static_assert(P * N2 == N, "four-step split");
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const GlobalTw tw{a.tw2n};
  const int tid = threadIdx.x;
  const int64_t ul = blockIdx.x;
  const int64_t row = a.unit0 + ul;
  const int p2_0 = blockIdx.y * NB;
  pdl_wait();
  const float *xr = a.x + row * a.x_stride;
  const bool vec = ((reinterpret_cast<uintptr_t>(xr) & 7) == 0);
  for (int idx = tid; idx < NB * P; idx += LCT) {
    const int c = idx % NB, p1 = idx / NB;
    const int64_t i0 = 2 * (int64_t)(N2 * p1 + p2_0 + c);
    float x0 = 0.f, x1 = 0.f;
    if (vec && i0 + 1 < a.x_len) {
      const float2 xv = __ldcs(reinterpret_cast<const float2 *>(xr + i0));
      x0 = xv.x;
      x1 = xv.y;
    } else {
      if (i0 < a.x_len) x0 = __ldg(xr + i0);
      if (i0 + 1 < a.x_len) x1 = __ldg(xr + i0 + 1);
    }
    buf[c * CS + padi(p1)] = make_float2(x0, x1);
  }
  __syncthreads();
  cpass<N, P, NB, G::R1, 1, -1>(buf, tw);
  cpass<N, P, NB, G::R2, G::R1, -1>(buf, tw);
  cpass<N, P, NB, G::R3, G::R1 * G::R2, -1>(buf, tw);
  float2 *T = a.stage + ul * a.xs + a.toff;
  for (int idx = tid; idx < NB * P; idx += LCT) {
    const int c = idx % NB, k1 = idx / NB;
    const int p2 = p2_0 + c;
    T[(int64_t)k1 * N2 + p2] = cmul(buf[c * CS + padi(k1)], tw_any<N>(tw, 2 * (int64_t)p2 * k1));
  }
  pdl_trigger();
}

// inverse four-step, first half (in place): DFT_N1 (sign +) over n1 of W[N2 n1 + p2] for NB
// columns, twiddle conj(w_N^{p2 n1}); inv_large_row<LOGN, 1> finishes the rows
template <int LOGN>
__global__ void __launch_bounds__(LCT) long_inv_col(const KArgs a) {
  using G = LongCol<LOGN>;
  constexpr int N = 1 << LOGN, P = G::P, NB = G::NB, N2 = 256, CS = colstride<P>();
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const GlobalTw tw{a.tw2n};
  const int tid = threadIdx.x;
  const int64_t ul = blockIdx.x;
  const int p2_0 = blockIdx.y * NB;
  pdl_wait();
  float2 *W = a.stage + ul * a.zs + a.toff;
  {
    constexpr int PERL = NB * P / LCT;
    float2 v[PERL];
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LCT;
      v[q] = __ldcs(W + (int64_t)N2 * (idx / NB) + p2_0 + idx % NB);
    }
#pragma unroll
    for (int q = 0; q < PERL; ++q) {
      const int idx = tid + q * LCT;
      buf[(idx % NB) * CS + padi(idx / NB)] = v[q];
    }
  }
  __syncthreads();
  cpass<N, P, NB, G::R1, 1, +1>(buf, tw);
  cpass<N, P, NB, G::R2, G::R1, +1>(buf, tw);
  cpass<N, P, NB, G::R3, G::R1 * G::R2, +1>(buf, tw);
  for (int idx = tid; idx < NB * P; idx += LCT) {
    const int c = idx % NB, n1 = idx / NB;
    const int p2 = p2_0 + c;
    W[(int64_t)n1 * N2 + p2] =
        cmul(buf[c * CS + padi(n1)], cconj(tw_any<N>(tw, 2 * (int64_t)p2 * n1)));
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ channel FFTs
// greedy radix of a remaining (2/3/5-smooth) transform size m; the same rule orders the
// butterflies and the output digits
__device__ __forceinline__ int long_radix(int m) {
  return (m & 15) == 0 ? 16
         : (m & 7) == 0 ? 8
         : (m & 3) == 0 ? 4
         : (m & 1) == 0 ? 2
         : m % 9 == 0   ? 9
         : m % 3 == 0   ? 3
                        : 5;
}

// The stage plan of DFT_M (built once per CTA in shared memory): stage s has radix R[s] and
// span Q[s] = Ms / R[s] (Ms: the block size the stage splits), twiddle stride M / Ms, and
// exact reciprocals for the index arithmetic: x / d = umulhi(x, ceil(2^32 / d)) for
// x, d < 2^16 (M_k <= 26000).
struct DifPlan {
  int ns;
  int R[kDifMaxStages], Q[kDifMaxStages], tstep[kDifMaxStages];
  unsigned magR[kDifMaxStages], magQ[kDifMaxStages];
};
__device__ __forceinline__ unsigned recip32(int d) {  // d >= 2 (d = 1 is special-cased)
  return (unsigned)((0x100000000ull + (unsigned)d - 1) / (unsigned)d);
}
__device__ __forceinline__ void build_dif_plan(DifPlan &pl, int M) {  // one thread
  int Ms = M, s = 0;
  while (Ms > 1) {
    const int R = long_radix(Ms);
    pl.R[s] = R;
    pl.Q[s] = Ms / R;
    pl.tstep[s] = M / Ms;
    pl.magR[s] = recip32(R);
    pl.magQ[s] = recip32(Ms / R);
    Ms /= R;
    ++s;
  }
  pl.ns = s;
}

// one decimation-in-frequency stage over all M/Ms blocks of size Ms = R Q (in place):
// y_k1[n'] = w_Ms^{SIGN n' k1} sum_r x[n' + r Q] w_R^{SIGN r k1} -> position n' + k1 Q
template <int R, int SIGN, int T>
__device__ __forceinline__ void dif_stage(float2 *buf, int M, int Q, int tstep, unsigned magQ,
                                          const float2 *tw) {
  const int tasks = M / R;
  for (int t = threadIdx.x; t < tasks; t += T) {
    const int blk = Q == 1 ? t : (int)__umulhi((unsigned)t, magQ), np = t - blk * Q;
    const int base = blk * (R * Q) + np;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = buf[padi(base + r * Q)];
    dft<R, SIGN>(v);
    if (np) {
      const int e1 = np * tstep;  // e^{2 pi i n' k1 / Ms} = table[n' k1 M/Ms], index < M
      int e = 0;
#pragma unroll
      for (int k = 1; k < R; ++k) {
        e += e1;
        float2 w = cmul(tw[e & 63], tw[64 + (e >> 6)]);  // shared two-level table
        if (SIGN < 0) w = cconj(w);
        v[k] = cmul(v[k], w);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) buf[padi(base + r * Q)] = v[r];
  }
}

// shared-memory two-level twiddle table of e^{2 pi i t/M}: tw[l] (l < 64), tw[64 + h] = t = 64 h,
// from the plan's full table twM (global)
// (stride s: the table of M / s from the table of M, e^{2 pi i t/(M/s)} = twM[s t])
template <int T>
__device__ __forceinline__ void load_twiddles(float2 *tw, const float2 *twM, int M, int s = 1) {
  const int nh = (M + 63) >> 6;
  for (int i = threadIdx.x; i < 64 + nh; i += T) {
    const int t = i < 64 ? i : 64 * (i - 64);
    tw[i] = t < M ? __ldg(twM + (int64_t)t * s) : make_float2(1.f, 0.f);
  }
}

// DFT_M (unnormalised, sign SIGN) of buf[padi(0..M)) in place; X[k] ends at dif_pos(k)
// (tw: the shared table of load_twiddles; pl: the shared stage plan)
template <int SIGN, int T>
__device__ __noinline__ void dif_fft(float2 *buf, int M, const float2 *tw, const DifPlan &pl) {
  for (int s = 0; s < pl.ns; ++s) {
    const int Q = pl.Q[s], ts = pl.tstep[s];
    const unsigned mq = pl.magQ[s];
    switch (pl.R[s]) {
      case 16: dif_stage<16, SIGN, T>(buf, M, Q, ts, mq, tw); break;
      case 8: dif_stage<8, SIGN, T>(buf, M, Q, ts, mq, tw); break;
      case 4: dif_stage<4, SIGN, T>(buf, M, Q, ts, mq, tw); break;
      case 2: dif_stage<2, SIGN, T>(buf, M, Q, ts, mq, tw); break;
      case 9: dif_stage<9, SIGN, T>(buf, M, Q, ts, mq, tw); break;
      case 3: dif_stage<3, SIGN, T>(buf, M, Q, ts, mq, tw); break;
      default: dif_stage<5, SIGN, T>(buf, M, Q, ts, mq, tw); break;
    }
    __syncthreads();
  }
}

// position of output k: k = d1 + R1 d2 + R1 R2 d3 + ... sits at d1 Q1 + d2 Q2 + ...
__device__ __forceinline__ int dif_pos(int k, const DifPlan &pl) {
  int pos = 0;
  for (int s = 0; s < pl.ns; ++s) {
    const int q = (int)__umulhi((unsigned)k, pl.magR[s]);
    pos += (k - q * pl.R[s]) * pl.Q[s];
    k = q;
  }
  return pos;
}

// shared-memory layout of a channel CTA: buf [padi(M) + 1], twiddles, stage plan
__device__ __forceinline__ float2 *long_tw_ptr(float2 *buf, int M) { return buf + padi(M) + 1; }
__device__ __forceinline__ DifPlan *long_plan_ptr(float2 *buf, int M) {
  return reinterpret_cast<DifPlan *>(long_tw_ptr(buf, M) + long_twiddle_entries(M));
}

// fold position q of channel k: sum over the support bins j = lo + dd, dd = q - lo (mod M),
// of X(j) g_k[j]/sqrt(M_k) (one term for a painless system; the aliases dd + M, dd + 2M ...
// of a sampled_from system, reading C21); real input: X(j) = conj X(2N - j), j in (-2N, 2N)
__device__ __forceinline__ float2 long_fold(const KArgs &a, const ChanDev &ch, const float2 *X,
                                            int q, int N2x, int N) {
  int dd = q - ch.lo_mod;
  if (dd < 0) dd += ch.M;
  float2 v = make_float2(0.f, 0.f);
  for (; dd < ch.len; dd += ch.M) {
    int jj = ch.lo + dd;
    if (jj < 0) jj += N2x;
    else if (jj >= N2x) jj -= N2x;
    const bool cj = jj > N;
    const float2 xv = __ldcg(X + (cj ? N2x - jj : jj));
    const float w = __ldg(a.gw + ch.goff + dd);
    v.x = fmaf(xv.x, w, v.x);
    v.y = fmaf(cj ? -xv.y : xv.y, w, v.y);
  }
  return v;
}

// Alg. 1 per channel: c_k = sqrt(M_k) IFFT_{M_k}(fold of X g_k)  (C1, C5, C15)
// (grid x: the channels of one size class, listed in a.pchans; 64 registers per thread)
template <int T>
__global__ void __launch_bounds__(T, 65536 / (64 * T)) long_chan_fwd(const KArgs a) {
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const ChanDev ch = a.chan[a.pchans[blockIdx.x]];
  const int64_t ul = blockIdx.y, row = a.unit0 + ul;
  const int N2x = (int)a.L, N = N2x / 2;
  const int M = ch.M;
  pdl_wait();
  const float2 *X = a.stage + ul * a.xs;
  float2 *tws = long_tw_ptr(buf, M);
  DifPlan &pl = *long_plan_ptr(buf, M);
  if (threadIdx.x == 0) build_dif_plan(pl, M);
  load_twiddles<T>(tws, a.twM + ch.twoff, M);
  for (int q = threadIdx.x; q < M; q += T) buf[padi(q)] = long_fold(a, ch, X, q, N2x, N);
  __syncthreads();
  dif_fft<+1, T>(buf, M, tws, pl);
  float2 *out = a.coef_out + row * a.C + ch.off;
  for (int m = threadIdx.x; m < M; m += T) __stcs(out + m, buf[padi(dif_pos(m, pl))]);
  pdl_trigger();
}

// Alg. 2 per channel: terms FFT_{M_k}(c_k)[j mod M_k] g~_k[j] / sqrt(M_k)
template <int T>
__global__ void __launch_bounds__(T, 65536 / (64 * T)) long_chan_inv(const KArgs a) {
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const ChanDev ch = a.chan[a.pchans[blockIdx.x]];
  const int64_t ul = blockIdx.y, row = a.unit0 + ul;
  const int M = ch.M;
  pdl_wait();
  const float2 *in = a.coef_in + row * a.C + ch.off;
  float2 *tws = long_tw_ptr(buf, M);
  DifPlan &pl = *long_plan_ptr(buf, M);
  if (threadIdx.x == 0) build_dif_plan(pl, M);
  load_twiddles<T>(tws, a.twM + ch.twoff, M);
  for (int m = threadIdx.x; m < M; m += T) buf[padi(m)] = __ldcs(in + m);
  __syncthreads();
  dif_fft<-1, T>(buf, M, tws, pl);
  float2 *terms = a.stage + ul * a.zs + ch.goff;
  for (int dd = threadIdx.x; dd < ch.len; dd += T) {
    int q = ch.lo_mod + dd;
    if (q >= M) q -= M;
    const float2 F = buf[padi(dif_pos(q, pl))];
    const float w = __ldg(a.gdw + ch.goff + dd);
    __stcg(terms + dd, make_float2(F.x * w, F.y * w));
  }
  pdl_trigger();
}

// sliCQ channels too long for the register-DFT packets (M_k > 1024; split design): Alg. 2 per
// channel as long_chan_inv, the terms going to their slots of the unit's half-spectrum staging
// (slot arrays / overflow, the destinations the plan assigned to every (channel, d) term with the
// Hermitian rule C15) -- entries a.bent[ch.soff .. + ch.m1): (dst | conj << 31, d | zero << 31)
template <int T>
__global__ void __launch_bounds__(T, 65536 / (64 * T)) long_chan_inv_slots(const KArgs a) {
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const ChanDev ch = a.chan[a.pchans[blockIdx.x]];
  const int64_t ul = blockIdx.y, row = a.unit0 + ul;
  const int M = ch.M;
  pdl_wait();
  const float2 *in = a.coef_in + row * a.C + ch.off;
  float2 *tws = long_tw_ptr(buf, M);
  DifPlan &pl = *long_plan_ptr(buf, M);
  if (threadIdx.x == 0) build_dif_plan(pl, M);
  load_twiddles<T>(tws, a.twM + ch.twoff, M);
  for (int m = threadIdx.x; m < M; m += T) buf[padi(m)] = __ldcs(in + m);
  __syncthreads();
  dif_fft<-1, T>(buf, M, tws, pl);
  float2 *Z = a.stage + ul * a.zs;
  for (int e = threadIdx.x; e < ch.m1; e += T) {
    const uint2 en = __ldg(a.bent + ch.soff + e);
    const int dd = (int)(en.y & 0x7fffffffu);
    int q = ch.lo_mod + dd;
    if (q >= M) q -= M;
    const float2 F = buf[padi(dif_pos(q, pl))];
    const float w = (en.y >> 31) ? 0.f : __ldg(a.gdw + ch.goff + dd);
    const bool cj = en.x >> 31;
    __stcs(Z + (en.x & 0x7fffffffu), make_float2(F.x * w, cj ? -F.y * w : F.y * w));
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ M_k > 26000
// Four-step M = M1 M2 (M2 <= 26000): q = M2 n1 + n2, k = k1 + M1 k2,
//   Y[k1 + M1 k2] = sum_n2 w_M2^{n2 k2} w_M^{n2 k1} sum_n1 y[M2 n1 + n2] w_M1^{n1 k1}
// (w = e^{SIGN 2 pi i / .}).  Step 1 (register DFT_M1 per n2, twiddle) writes the rows
// A[k1][n2] to the channel's staging scratch; step 2 runs each row's DFT_M2 in shared memory.
template <int M1, int SIGN, class LD>
__device__ __forceinline__ void big_step1(float2 *A, int M, int M2, const float2 *twM, LD load) {
  for (int n2 = threadIdx.x; n2 < M2; n2 += 512) {
    float2 v[M1];
#pragma unroll
    for (int n1 = 0; n1 < M1; ++n1) v[n1] = load(M2 * n1 + n2);
    dft<M1, SIGN>(v);
#pragma unroll
    for (int k1 = 0; k1 < M1; ++k1) {
      float2 w = __ldg(twM + n2 * k1);  // e^{2 pi i n2 k1 / M}, index < M
      if (SIGN < 0) w = cconj(w);
      __stcg(A + (int64_t)k1 * M2 + n2, k1 ? cmul(v[k1], w) : v[k1]);
    }
  }
}
template <int SIGN, class LD>
__device__ __forceinline__ void big_step1_any(int M1, float2 *A, int M, int M2, const float2 *twM,
                                              LD load) {
  switch (M1) {
    case 2: big_step1<2, SIGN>(A, M, M2, twM, load); break;
    case 3: big_step1<3, SIGN>(A, M, M2, twM, load); break;
    case 4: big_step1<4, SIGN>(A, M, M2, twM, load); break;
    case 5: big_step1<5, SIGN>(A, M, M2, twM, load); break;
    case 6: big_step1<6, SIGN>(A, M, M2, twM, load); break;
    case 8: big_step1<8, SIGN>(A, M, M2, twM, load); break;
    case 9: big_step1<9, SIGN>(A, M, M2, twM, load); break;
    case 10: big_step1<10, SIGN>(A, M, M2, twM, load); break;
    case 12: big_step1<12, SIGN>(A, M, M2, twM, load); break;
    case 15: big_step1<15, SIGN>(A, M, M2, twM, load); break;
    default: big_step1<16, SIGN>(A, M, M2, twM, load); break;
  }
}

__global__ void __launch_bounds__(512, 1) long_chan_fwd_big(const KArgs a) {
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const ChanDev ch = a.chan[a.pchans[blockIdx.x]];
  const int64_t ul = blockIdx.y, row = a.unit0 + ul;
  const int N2x = (int)a.L, N = N2x / 2;
  const int M = ch.M, M1 = ch.m1, M2 = M / M1;
  const float2 *twM = a.twM + ch.twoff;
  float2 *tws = long_tw_ptr(buf, M2);
  DifPlan &pl = *long_plan_ptr(buf, M2);
  if (threadIdx.x == 0) build_dif_plan(pl, M2);
  load_twiddles<512>(tws, twM, M2, M1);
  pdl_wait();
  const float2 *X = a.stage + ul * a.xs;
  float2 *A = a.stage + ul * a.xs + ch.soff;
  big_step1_any<+1>(M1, A, M, M2, twM, [&](int q) { return long_fold(a, ch, X, q, N2x, N); });
  __syncthreads();
  float2 *out = a.coef_out + row * a.C + ch.off;
  for (int k1 = 0; k1 < M1; ++k1) {
    for (int n2 = threadIdx.x; n2 < M2; n2 += 512) buf[padi(n2)] = __ldcg(A + (int64_t)k1 * M2 + n2);
    __syncthreads();
    dif_fft<+1, 512>(buf, M2, tws, pl);
    for (int k2 = threadIdx.x; k2 < M2; k2 += 512) __stcs(out + k1 + M1 * k2, buf[padi(dif_pos(k2, pl))]);
    __syncthreads();
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(512, 1) long_chan_inv_big(const KArgs a) {
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);
  const ChanDev ch = a.chan[a.pchans[blockIdx.x]];
  const int64_t ul = blockIdx.y, row = a.unit0 + ul;
  const int M = ch.M, M1 = ch.m1, M2 = M / M1;
  const float2 *twM = a.twM + ch.twoff;
  float2 *tws = long_tw_ptr(buf, M2);
  DifPlan &pl = *long_plan_ptr(buf, M2);
  if (threadIdx.x == 0) build_dif_plan(pl, M2);
  load_twiddles<512>(tws, twM, M2, M1);
  pdl_wait();
  const float2 *in = a.coef_in + row * a.C + ch.off;
  float2 *A = a.stage + ul * a.zs + ch.soff;
  big_step1_any<-1>(M1, A, M, M2, twM, [&](int q) { return __ldcs(in + q); });
  __syncthreads();
  float2 *terms = a.stage + ul * a.zs + ch.goff;
  for (int k1 = 0; k1 < M1; ++k1) {
    for (int n2 = threadIdx.x; n2 < M2; n2 += 512) buf[padi(n2)] = __ldcg(A + (int64_t)k1 * M2 + n2);
    __syncthreads();
    dif_fft<-1, 512>(buf, M2, tws, pl);
    // F[q], q = k1 + M1 k2 -> the support bins dd = q - lo_mod (mod M) < L_k
    for (int k2 = threadIdx.x; k2 < M2; k2 += 512) {
      int dd = k1 + M1 * k2 - ch.lo_mod;
      if (dd < 0) dd += M;
      if (dd >= ch.len) continue;
      const float2 F = buf[padi(dif_pos(k2, pl))];
      const float w = __ldg(a.gdw + ch.goff + dd);
      __stcg(terms + dd, make_float2(F.x * w, F.y * w));
    }
    __syncthreads();
  }
  pdl_trigger();
}

// half-spectrum bin b: sum of its channel terms in plan order (conjugated where C15 mirrors)
__device__ __forceinline__ float2 long_gather(const KArgs &a, const float2 *Tm, int b) {
  float2 acc = make_float2(0.f, 0.f);
  const uint32_t e0 = __ldg(a.lrow + b), e1 = __ldg(a.lrow + b + 1);
  for (uint32_t i = e0; i < e1; ++i) {
    const uint32_t e = __ldg(a.lent + i);
    float2 t = __ldcg(Tm + (e & 0x7fffffffu));
    if (e >> 31) t.y = -t.y;
    acc = cadd(acc, t);
  }
  return acc;
}

// H -> c2r-packed W (as inv_large_pack, kernels_large.cuh)
__global__ void __launch_bounds__(LT) long_inv_pack(const KArgs a) {
  const GlobalTw tw{a.tw2n};
  const int N = (int)(a.L / 2);
  pdl_wait();
  const int64_t ul = blockIdx.x;
  const float2 *Tm = a.stage + ul * a.zs;
  float2 *W = a.stage + ul * a.zs + a.toff;
  const int k = blockIdx.y * LT + threadIdx.x;
  if (k <= N / 2) {
    const float2 hk = long_gather(a, Tm, k);
    const float2 hn = long_gather(a, Tm, N - k);
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

// entry points (kernels_long.cu)

}  // namespace kern
}  // namespace slicq
