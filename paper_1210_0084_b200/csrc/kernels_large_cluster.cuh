// 2N = 131072 (N1 = N2 = 256): the four-step FFT of one slice on a 16-CTA thread-block
// cluster (included by kernels_large.cu only).  The transpose between the column and the
// row step goes through distributed shared memory instead of the staging buffer in HBM
// (VERDICT round 1, item 5): CTA r of the cluster of unit u runs the column step of its 16
// columns exactly as the split kernels do, stores every twiddled value straight into the
// shared memory of the CTA that owns its row (mapa + st.shared::cluster), one cluster
// barrier, then runs the row step of its 16 rows, again exactly as the split kernels.  Same
// arithmetic in the same order: the output is bit-identical to fwd_large_col + fwd_large_row
// (inv_large_pack + inv_large_col + inv_large_row).  Per slice this removes one write and one
// read of the N-point intermediate (2 x 512 KB) and two kernel boundaries per direction.
#pragma once
#include "kernels_large.cuh"

namespace slicq {
namespace kern {

__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");  // (.release)
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // (.acquire)
}
// store v to the shared-memory location `off` bytes into `base` (this CTA's buffer) of
// CTA `rank` of the cluster
__device__ __forceinline__ void st_remote(uint32_t base, uint32_t off, unsigned rank, float2 v) {
  uint32_t dst;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(base + off), "r"(rank));
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(dst), "f"(v.x), "f"(v.y)
               : "memory");
}
#ifndef SLICQ_LCL_SINGLE
#define SLICQ_LCL_SINGLE 1  // 1: one buffer (rows overwrite columns after an extra cluster barrier)
#endif
#ifndef SLICQ_LCL_MINB
#define SLICQ_LCL_MINB 5  // __launch_bounds__ min CTAs per SM (measured on cfg5: 5 beats 3, 4 and 6)
#endif
#ifndef SLICQ_LCL_QB
#define SLICQ_LCL_QB 4  // inverse gather: bins per thread with their loads in flight together (packed code: 4 beats 8 -- 64 vs 120 B of spills at 48 registers; cfg5 inverse 1.85 -> 1.79 ms)
#endif
constexpr int LCL = 16;  // CTAs per cluster (non-portable: cudaFuncAttributeNonPortableClusterSizeAllowed)

template <int LOGN>
constexpr size_t cluster_smem_bytes() {  // column buffer + row buffer (or one shared buffer)
  return (SLICQ_LCL_SINGLE ? 1 : 2) * large_smem_bytes<LOGN>();
}

// forward: column step (fwd_large_col) -> DSMEM -> row step (fwd_large_row).  Rows: CTA r owns
// k1 = 8 r + s (slot s < 8) and their partners N1 - k1 (slot 8 + s, k1 > 0); CTA 0's slot 8
// (k1 = 0 has no partner) holds the self-paired row N1/2.
template <int LOGN>
__global__ void __launch_bounds__(LT, SLICQ_LCL_MINB) fwd_large_cluster(const KArgs a) {
  using G = Large<LOGN>;
  constexpr int N = G::N, N1 = G::N1, N2 = G::N2, CS1 = colstride<N1>(), CS2 = colstride<N2>();
  static_assert(N1 == 256 && N2 == 256 && N2 / LB == LCL, "cluster path: 2N = 131072");
  constexpr int HR = N1 / (2 * LCL);  // 8 rows (+ partners) per CTA
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);  // columns [LB][CS1]
  float2 *rbuf = SLICQ_LCL_SINGLE ? buf : buf + LB * CS1;  // rows [2 HR][CS2], written by the cluster
  cluster_arrive_relaxed();  // (every CTA has started before the first remote store)
  const GlobalTw tw{a.tw2n};
  const int tid = threadIdx.x;
  const unsigned rank = blockIdx.y;  // cluster dims (1, LCL, 1)
  const int64_t ul = blockIdx.x;
  int64_t row, mloc, mg;
  unit_coords(a, ul, row, mloc, mg);
  const int p2_0 = (int)rank * LB;
  pdl_wait();
  {  // F1 (as fwd_large_col): windowed z[N2 p1 + p2] = (f[2p], f[2p+1]) * h_0
    const float *xr = a.x + row * a.x_stride;
    const bool vec = ((reinterpret_cast<uintptr_t>(xr) & 7) == 0);
    const int64_t s0 = (mg - 1) * N - a.base_off;
    const int A = (N - a.tr) / 2, Bw = (N + a.tr) / 2;
    constexpr int PERL = LB * N1 / LT;
    // interior frame (no wrap, inside the row, 8-byte aligned): every pair load of the
    // thread in flight together, window values after
    if (vec && s0 >= 0 && s0 + 2 * N <= a.x_len) {
      float2 v[PERL];
#pragma unroll
      for (int q = 0; q < PERL; ++q) {
        const int idx = tid + q * LT, c = idx % LB, p1 = idx / LB;
        const int i0 = 2 * (N2 * p1 + p2_0 + c), t0 = i0 - N;
        const int at0 = t0 < 0 ? -t0 : t0, at1 = (t0 + 1) < 0 ? -(t0 + 1) : (t0 + 1);
        v[q] = (at0 < Bw || at1 < Bw) ? __ldcs(reinterpret_cast<const float2 *>(xr + s0 + i0))
                                      : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < PERL; ++q) {
        const int idx = tid + q * LT, c = idx % LB, p1 = idx / LB;
        const int i0 = 2 * (N2 * p1 + p2_0 + c), t0 = i0 - N;
        const int at0 = t0 < 0 ? -t0 : t0, at1 = (t0 + 1) < 0 ? -(t0 + 1) : (t0 + 1);
        if (at0 > A || at1 > A) {
          const float ha = at0 <= A ? 1.f : (at0 < Bw ? __ldg(a.h0 + i0) : 0.f);
          const float hb = at1 <= A ? 1.f : (at1 < Bw ? __ldg(a.h0 + i0 + 1) : 0.f);
          v[q].x *= ha;
          v[q].y *= hb;
        }
        buf[c * CS1 + padi(p1)] = v[q];
      }
    } else {
      for (int idx = tid; idx < LB * N1; idx += LT) {
        const int c = idx % LB, p1 = idx / LB;
        const int i0 = 2 * (N2 * p1 + p2_0 + c);
        const int t0 = i0 - N;
        const int at0 = t0 < 0 ? -t0 : t0;
        const int at1 = (t0 + 1) < 0 ? -(t0 + 1) : (t0 + 1);
        float x0 = 0.f, x1 = 0.f;
        if (at0 < Bw || at1 < Bw) {
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
          const float ha = at0 <= A ? 1.f : (at0 < Bw ? __ldg(a.h0 + i0) : 0.f);
          const float hb = at1 <= A ? 1.f : (at1 < Bw ? __ldg(a.h0 + i0 + 1) : 0.f);
          x0 *= ha;
          x1 *= hb;
        }
        buf[c * CS1 + padi(p1)] = make_float2(x0, x1);
      }
    }
  }
  __syncthreads();
  bpass<N, N1, G::C1, 1, -1>(buf, tw);
  bpass<N, N1, G::C2, G::C1, -1>(buf, tw);
  cluster_wait();
  // twiddle w_N^{p2 k1}; T[k1][p2] -> the slot of row k1 in its owner CTA
  const uint32_t rb = (uint32_t)__cvta_generic_to_shared(rbuf);
  constexpr int PERX = LB * N1 / LT;
#if SLICQ_LCL_SINGLE
  float2 vx[PERX];
#pragma unroll
  for (int q = 0; q < PERX; ++q) {
    const int idx = tid + q * LT, c = idx % LB, k1 = idx / LB;
    vx[q] = cmul(buf[c * CS1 + padi(k1)], tw_any<N>(tw, 2 * (int64_t)(p2_0 + c) * k1));
  }
  cluster_arrive();  // every CTA has read its columns: the buffer takes rows
  cluster_wait();
#endif
#pragma unroll
  for (int q = 0; q < PERX; ++q) {
    const int idx = tid + q * LT, c = idx % LB, k1 = idx / LB;
    const int p2 = p2_0 + c;
#if SLICQ_LCL_SINGLE
    const float2 v = vx[q];
#else
    const float2 v = cmul(buf[c * CS1 + padi(k1)], tw_any<N>(tw, 2 * (int64_t)p2 * k1));
#endif
    int own, slot;
    if (k1 < N1 / 2) {
      own = k1 / HR;
      slot = k1 % HR;
    } else if (k1 == N1 / 2) {
      own = 0;
      slot = HR;
    } else {
      own = (N1 - k1) / HR;
      slot = HR + (N1 - k1) % HR;
    }
    st_remote(rb, (uint32_t)(sizeof(float2) * (slot * CS2 + padi(p2))), (unsigned)own, v);
  }
  cluster_arrive();
  cluster_wait();  // every row complete; no remote store into this CTA follows
  bpass<N, N2, R_ROW, 1, -1>(rbuf, tw);
  bpass<N, N2, R_ROW, R_ROW, -1>(rbuf, tw);
  // r2c packing (as fwd_large_row): X[k] = E + w O, X[N-k] = conj(E) - conj(w O)
  float2 *Xo = a.stage + ul * a.xs;
  const int kb = (int)rank * HR;
  auto pack = [&](int s, int ps, int pk2, int k2, int k1) {
    const int k = k1 + N1 * k2;
    const float2 zk = rbuf[s * CS2 + padi(k2)];
    const float2 zn = rbuf[ps * CS2 + padi(pk2)];
    if (k == 0) {
      Xo[0] = make_float2(zk.x + zk.y, 0.f);
      Xo[N] = make_float2(zk.x - zk.y, 0.f);
      return;
    }
    const float2 E = cscale(cadd(zk, cconj(zn)), 0.5f);
    const float2 O = cscale(mul_si<-1>(csub(zk, cconj(zn))), 0.5f);
    const float2 wO = cmul(tw_lookup(tw, k), O);
    Xo[k] = cadd(E, wO);
    if (k != N / 2) Xo[N - k] = csub(cconj(E), cconj(wO));
  };
  for (int idx = tid; idx < HR * N2; idx += LT) {
    const int s = idx % HR, k2 = idx / HR;
    const int k1 = kb + s;
    if (k1 == 0) {
      if (k2 <= N2 / 2) pack(s, s, (N2 - k2) & (N2 - 1), k2, k1);
    } else {
      pack(s, s + HR, N2 - 1 - k2, k2, k1);
    }
  }
  if (rank == 0)  // row N1/2 (slot HR): self-paired
    for (int k2 = tid; k2 < N2 / 2; k2 += LT) pack(HR, HR, N2 - 1 - k2, k2, N1 / 2);
  pdl_trigger();
}

// inverse: per-bin gather + c2r packing of the CTA's 16 columns (inv_large_pack), column step
// (inv_large_col) -> DSMEM -> row step with dual window and overlap-add (inv_large_row,
// MODE 0).  Columns: CTA r owns p2 = 8 r + s (slot s < 8) and N2 - p2 (slot 8 + s, p2 > 0),
// CTA 0's slot 8 the self-paired column N2/2, so that both bins of every c2r pair (k, N - k)
// lie in one CTA; rows: CTA r owns n1 = 16 r + s.
template <int LOGN>
__global__ void __launch_bounds__(LT, SLICQ_LCL_MINB) inv_large_cluster(const KArgs a) {
  using G = Large<LOGN>;
  constexpr int N = G::N, N1 = G::N1, N2 = G::N2, CS1 = colstride<N1>(), CS2 = colstride<N2>();
  static_assert(N1 == 256 && N2 == 256 && N2 / LB == LCL, "cluster path: 2N = 131072");
  constexpr int HC = N2 / (2 * LCL);  // 8 columns (+ partners) per CTA
  extern __shared__ float4 smem4[];
  float2 *buf = reinterpret_cast<float2 *>(smem4);  // columns [LB][CS1]
  float2 *rbuf = SLICQ_LCL_SINGLE ? buf : buf + LB * CS1;  // rows [LB][CS2], written by the cluster
  cluster_arrive_relaxed();
  const GlobalTw tw{a.tw2n};
  const int tid = threadIdx.x;
  const unsigned rank = blockIdx.y;
  const int64_t ul = blockIdx.x;
  int64_t row, mloc, mg;
  unit_coords(a, ul, row, mloc, mg);
  pdl_wait();
  const float2 *Z = a.stage + ul * a.zs;
  const int pb = (int)rank * HC;
  auto slot_col = [&](int s) {  // column p2 of slot s
    if (s < HC) return pb + s;
    if (s == HC && rank == 0) return N2 / 2;
    return N2 - (pb + s - HC);
  };
  // I3b gather, one bin per item: H[k] of the CTA's 16 columns x N1 rows -> buf (bin N, the
  // partner of bin 0, in a spare entry of column slot 0); all slot and dpos loads of a batch
  // in flight before any overflow branch
  constexpr int PERB = LB * N1 / LT, QB = SLICQ_LCL_QB;
  float2 *hN = buf + padi(N1);
#pragma unroll
  for (int q0 = 0; q0 < PERB; q0 += QB) {
    float2 h[QB];
    uint32_t d[QB];
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      const int idx = tid + (q0 + q) * LT, c = idx % LB, p1 = idx / LB;
      const int k = N2 * p1 + slot_col(c);
      h[q] = cadd(__ldcg(Z + k), __ldcg(Z + a.zso + k));
      d[q] = __ldg(a.dpos + k);
    }
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      const int idx = tid + (q0 + q) * LT, c = idx % LB, p1 = idx / LB;
      for (int i = 0; i < (int)(d[q] >> 20); ++i)  // deep-overlap bins: overflow terms in order
        h[q] = cadd(h[q], __ldcg(Z + 2 * a.zso + (d[q] & 0xfffff) + i));
      buf[c * CS1 + padi(p1)] = h[q];
    }
  }
  if (rank == 0 && tid == 0) *hN = gather_bin<N>(a, Z, N);
  __syncthreads();
  // c2r packing in place, pair (k, N - k) with k <= N/2 (as inv_large_pack): Z[k] = E + iO,
  // Z[N-k] = conj(E) + i conj(D) conj(w).  H[k] at (sa, ia), H[N-k] at (sb, ib); sb < 0:
  // k = 0 (H[N] in hN) or k = N/2 (its own partner), Z[k] only
  auto pack = [&](int k, int sa, int ia, int sb, int ib) {
    const float2 hk = buf[sa * CS1 + padi(ia)];
    const float2 hn = sb >= 0 ? buf[sb * CS1 + padi(ib)] : (k == 0 ? *hN : hk);
    const float2 E = cscale(cadd(hk, cconj(hn)), 0.5f);
    const float2 D = cscale(csub(hk, cconj(hn)), 0.5f);
    const float2 w = cconj(tw_lookup(tw, k));  // e^{+i pi k/N}
    const float2 O = cmul(D, w);
    buf[sa * CS1 + padi(ia)] = cadd(E, mul_si<+1>(O));
    if (sb >= 0) {
      buf[sb * CS1 + padi(ib)] = cadd(cconj(E), make_float2(O.y, O.x));  // (conj D)(conj w) = conj O
    }
  };
  for (int idx = tid; idx < HC * N1; idx += LT) {
    const int s = idx % HC, p1 = idx / HC, p2 = pb + s;
    if (p2 == 0) {  // column 0: pairs (p1, N1 - p1); p1 = 0 pairs bin 0 with bin N
      if (p1 <= N1 / 2) pack(N2 * p1, 0, p1, (p1 == 0 || p1 == N1 / 2) ? -1 : 0, N1 - p1);
    } else {  // N - k = N2 (N1 - 1 - p1) + (N2 - p2): slot s + HC
      const int k = N2 * p1 + p2;
      if (k <= N / 2) pack(k, s, p1, s + HC, N1 - 1 - p1);
      else pack(N - k, s + HC, N1 - 1 - p1, s, p1);
    }
  }
  if (rank == 0 && tid < N1 / 2)  // column N2/2 (slot HC): k = N2 p1 + N2/2, p1' = N1 - 1 - p1
    pack(N2 * tid + N2 / 2, HC, tid, HC, N1 - 1 - tid);
  __syncthreads();
  bpass<N, N1, G::C1, 1, +1>(buf, tw);
  bpass<N, N1, G::C2, G::C1, +1>(buf, tw);
  cluster_wait();
  // twiddle conj(w_N^{p2 n1}); W[n1][p2] -> row n1 of CTA n1 / LB
  const uint32_t rb = (uint32_t)__cvta_generic_to_shared(rbuf);
  constexpr int PERX = LB * N1 / LT;
#if SLICQ_LCL_SINGLE
  float2 vx[PERX];
#pragma unroll
  for (int q = 0; q < PERX; ++q) {
    const int idx = tid + q * LT, c = idx % LB, n1 = idx / LB;
    vx[q] = cmul(buf[c * CS1 + padi(n1)], cconj(tw_any<N>(tw, 2 * (int64_t)slot_col(c) * n1)));
  }
  cluster_arrive();  // every CTA has read its columns: the buffer takes rows
  cluster_wait();
#endif
#pragma unroll
  for (int q = 0; q < PERX; ++q) {
    const int idx = tid + q * LT, c = idx % LB, n1 = idx / LB;
    const int p2 = slot_col(c);
#if SLICQ_LCL_SINGLE
    const float2 v = vx[q];
#else
    const float2 v = cmul(buf[c * CS1 + padi(n1)], cconj(tw_any<N>(tw, 2 * (int64_t)p2 * n1)));
#endif
    st_remote(rb, (uint32_t)(sizeof(float2) * ((n1 % LB) * CS2 + padi(p2))), (unsigned)(n1 / LB), v);
  }
  cluster_arrive();
  cluster_wait();
  bpass<N, N2, R_ROW, 1, +1>(rbuf, tw);
  bpass<N, N2, R_ROW, R_ROW, +1>(rbuf, tw);
  // dual window and overlap-add of rows n1 in [16 r, 16 r + 16) (as inv_large_row, MODE 0)
  const int n1_0 = (int)rank * LB;
  const int A = (N - a.tr) / 2, Bw = (N + a.tr) / 2;
  const float invN = 1.0f / (float)N;
  const int S = a.nslices;
  const bool left_paired = a.circular || mloc > 0;
  const bool right_paired = a.circular || mloc + 1 < S;
  const int64_t bl = mloc > 0 ? mloc - 1 : S - 1, br = mloc;
  const int trp = a.tr;
  float *yrow = a.y + row * a.y_stride;
  float *bnd_row = a.bnd + row * (int64_t)S * 2 * trp;
  const int64_t sbase = (mg - 1) * N;  // global sample of frame index 0
  // interior slice (both boundaries paired, the frame inside the row: no wrap, no trim, no
  // spill): 32-bit frame indices, exclusive sample pairs as one 8-byte store; the same
  // products as the general path below (h~_0 = 1 on the exclusive part), so bit-identical
  const bool fast = left_paired && right_paired &&
                    (a.circular ? (sbase >= 0 && sbase + 2 * N <= a.L && sbase + 2 * N <= a.y_len)
                                : (sbase + N - A - a.y_base >= 0)) &&
                    !(reinterpret_cast<uintptr_t>(yrow + (a.circular ? sbase : sbase - a.y_base)) & 7);
  if (fast) {
    float *yb = yrow + (a.circular ? sbase : sbase - a.y_base);  // frame index i -> yb[i]
    float *lh = bnd_row + (bl * 2 + 1) * trp + (Bw - 1 - N);      // left half: t + Bw - 1
    float *rh = bnd_row + (br * 2 + 0) * trp + (-A - 1 - N);      // right half: t - A - 1
    for (int idx = tid; idx < LB * N2; idx += LT) {
      const int s = idx % LB, n2 = idx / LB;
      const float2 z = rbuf[s * CS2 + padi(n2)];
      const int i0 = 2 * (n1_0 + s + N1 * n2), t0 = i0 - N;
      if (t0 >= -A && t0 < A) {  // both samples exclusive
        *reinterpret_cast<float2 *>(yb + i0) = make_float2(z.x * invN, z.y * invN);
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + h, t = i - N, at = t < 0 ? -t : t;
        if (at >= Bw) continue;
        const float hd = at <= A ? 1.f : __ldg(a.h0dual + i);
        const float val = (h ? z.y : z.x) * invN * hd;
        if (at <= A) yb[i] = val;
        else if (t < 0) lh[i] = val;
        else rh[i] = val;
      }
    }
    pdl_trigger();
    return;
  }
  for (int idx = tid; idx < LB * N2; idx += LT) {
    const int s = idx % LB, n2 = idx / LB;
    const float2 z = rbuf[s * CS2 + padi(n2)];
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
  if (!a.circular && mloc == 0 && rank == 0)
    for (int u = tid; u < a.halo - (Bw - 1); u += LT) a.spill[row * a.halo + u] = 0.f;
  pdl_trigger();
}

}  // namespace kern
}  // namespace slicq
