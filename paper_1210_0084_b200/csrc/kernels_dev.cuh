// sm_100a kernels of the sliCQ hot path (device code).  DESIGN.md "Kernels" describes the
// design; step names follow SURVEY.md §8(a).  Per direction a spectrum kernel and one or two
// channel kernels (lite / full register variants), over (row, slice) units whose
// intermediate goes through the workspace staging buffer:
//
//   forward
//     slicq_fwd_spec_kernel<LOGN>   one CTA per unit:
//       F1  first radix pass straight from HBM: Tukey-windowed frame pairs
//       F2  r2c FFT_{2N}: complex N-point Stockham FFT in shared memory; the last pass, the
//           packing step and the store of X[0..N] to the staging buffer fused in registers
//           (mirror-paired tasks; the two self-mirrored tasks of thread 0 are packed by
//           warp 0 cooperatively, one bin per lane)
//     slicq_fwd_chan_kernel<MAXS,MINB>  one warp task = (packet, nu units) of a tile:
//       F3  fold: buf[p] = X(j) g_k[j]/sqrt(M_k), j = p mod M_k, from a plan-time element
//           table (bin | scratch position, weight with the conjugation flag as its sign)
//                                                                  (C5)
//       F4  IFFT_{M_k} as a four-step M1 x M2 register DFT (M_k > 32) or a whole DFT_M per
//           lane (M_k <= 32), compile-time twiddles
//       F5  store c^m_k                                            (P:320-323 layout view)
//   inverse
//     slicq_inv_chan_kernel<MAXS,MINB>  one warp task = (packet, nu units) of a tile:
//       I1/I2  load c^m_k, FFT_{M_k} (four-step / per lane)
//       I3a    term F_k[j mod M_k] g~_k[j]/sqrt(M_k) (conjugated where C15 mirrors it) into
//              its bin-major slot of the unit's half spectrum
//     slicq_inv_spec_kernel<LOGN>   one CTA per unit:
//       I3b H[b] = slot0[b] + slot1[b] (+ the bin's overflow run, plan order) -- no index
//           tables, no atomics, deterministic; fused with the c2r packing and the first
//           radix pass in registers
//       I4  c2r IFFT_{2N} (N-point Stockham)
//       I5  multiply by h~_0 and overlap-add; slice-boundary samples are paired across CTAs
//           through the workspace with a parity counter (no spinning, deterministic a+b)
//
// The channel kernels amortise their per-shape code (I-cache) and plan tables over a tile of
// slices: the plan is identical for every slice.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "fft_dev.cuh"
#include "slicq_internal.h"

namespace slicq {
namespace kern {

using namespace slicq::dev;

constexpr unsigned FULL = 0xffffffffu;

// Opt-in phase timing (debug library only: -DSLICQ_PHASE_TIMING).  Thread 0 of every CTA
// accumulates clock64 deltas between phase marks; read with slicq_debug_phase_times().
#ifdef SLICQ_PHASE_TIMING
static __device__ unsigned long long g_phase_cycles[2][16];
#define PHASE_INIT() long long _t_prev = clock64()
#define PHASE_MARK(dir, i)                                             \
  do {                                                                 \
    __syncthreads();                                                   \
    if (threadIdx.x == 0) {                                            \
      const long long _t = clock64();                                  \
      atomicAdd(&g_phase_cycles[dir][i], (unsigned long long)(_t - _t_prev)); \
      _t_prev = _t;                                                    \
    }                                                                  \
  } while (0)
#else
#define PHASE_INIT() \
  do {               \
  } while (0)
#define PHASE_MARK(dir, i) \
  do {                     \
  } while (0)
#endif

// one pad entry per 16 complex: radix-16 strided stores and contiguous loads are
// bank-conflict free for 8-byte accesses
__host__ __device__ constexpr int padi(int i) { return i + (i >> 4); }

// unit u = row * S + local slice: 32-bit division when u fits (the 64-bit one is a
// software routine of ~70 instructions, executed by every thread of a spectrum CTA)
__device__ __forceinline__ int64_t unit_row(int64_t u, int S) {
  return (u >> 32) == 0 ? (int64_t)((uint32_t)u / (uint32_t)S) : u / S;
}

// Big-FFT plans: N = 2^LOGN complex points, T threads, radix sequences per direction.
template <int LOGN>
struct Big;
// store flavours (tunable): coefficients are streamed out, staged terms are re-read by the
// spectrum kernel
__device__ __forceinline__ void st_plain(float2 *p, float2 v) { *p = v; }
#ifndef SLICQ_XSTORE
#define SLICQ_XSTORE st_plain
#endif
#ifndef SLICQ_ZLOAD
#define SLICQ_ZLOAD __ldcg
#endif
#ifndef SLICQ_CSTORE
#define SLICQ_CSTORE __stcs
#endif
#ifndef SLICQ_ZSTORE
#define SLICQ_ZSTORE __stcs  // (measured: evict-first beats .cg by ~1 % on cfg4)
#endif
#ifndef SLICQ_INV_PF2
#define SLICQ_INV_PF2 1  // inverse spectrum: bulk L2 prefetch of the second load batch's bins
#endif
#ifndef SLICQ_OVP
#define SLICQ_OVP 1  // persistent inverse spectrum kernel: overflow-bin sums in a CTA-wide pre-pass
#endif
#ifndef SLICQ_OV_ASYNC
#define SLICQ_OV_ASYNC 0  // (opt-in) the next unit's overflow terms fetched by cp.async one unit ahead: measured slower (cfg4 inverse 2.61 vs 2.575 ms)
#endif
#ifndef SLICQ_IA_GROUP
#define SLICQ_IA_GROUP 4  // inverse spectrum: r-values of slot loads per batch (packed code: 4
#endif                    // beats 8, cfg4 inverse 2.575 -> 2.52 ms; the scalar code preferred 8)
#ifndef SLICQ_T13
#define SLICQ_T13 256
#endif
#ifndef SLICQ_MINB13
#define SLICQ_MINB13 2
#endif
#ifndef SLICQ_MINB13F
#define SLICQ_MINB13F SLICQ_MINB13  // forward spectrum kernels' CTAs per SM (register cap)
#endif
// MINB = CTAs per SM the shared-memory budget is sized for (two slices in flight per SM
// overlap one CTA's HBM loads / barriers with the other's arithmetic).
template <>
struct Big<11> {
  static constexpr int N = 2048, T = 128, MINB = 2, MINBF = 2;
  static constexpr int F1 = 16, F2 = 16, F3 = 8;   // forward pass radices
  static constexpr int I1 = 16, I2 = 8, I3 = 16;   // inverse pass radices
};
template <>
struct Big<12> {
  static constexpr int N = 4096, T = 256, MINB = 2, MINBF = 2;
  static constexpr int F1 = 16, F2 = 16, F3 = 16;
  static constexpr int I1 = 16, I2 = 16, I3 = 16;
};
// radix sequences (tunable at build time: SLICQ_F13A/B/C, SLICQ_I13A/B/C)
#ifndef SLICQ_F13A
#define SLICQ_F13A 16
#define SLICQ_F13B 32
#define SLICQ_F13C 16
#endif
#ifndef SLICQ_I13A
#define SLICQ_I13A 16
#define SLICQ_I13B 32
#define SLICQ_I13C 16
#endif
template <>
struct Big<13> {
  static constexpr int N = 8192, T = SLICQ_T13, MINB = SLICQ_MINB13, MINBF = SLICQ_MINB13F;
  static constexpr int F1 = SLICQ_F13A, F2 = SLICQ_F13B, F3 = SLICQ_F13C;
  static constexpr int I1 = SLICQ_I13A, I2 = SLICQ_I13B, I3 = SLICQ_I13C;
};
template <>
struct Big<14> {
  static constexpr int N = 16384, T = 512, MINB = 1, MINBF = 1;
  static constexpr int F1 = 32, F2 = 32, F3 = 16;
  static constexpr int I1 = 16, I2 = 32, I3 = 32;
};

template <int LOGN>
constexpr int spec_entries() {
  return padi(Big<LOGN>::N) + 2;  // X[0..N-1] padded, X[N] at padi(N), one spare
}
template <int N>
constexpr int tw_entries_n() {
  return 64 + 2 * N / 64;
}
template <int LOGN>
constexpr int tw_entries() {
  return tw_entries_n<Big<LOGN>::N>();
}

struct KArgs {
  // signal side
  const float *x;
  float *y;
  float *spill;
  int64_t x_len, x_stride, base_off, L;
  int64_t y_len, y_stride, y_base, halo;
  int wrap;       // forward: negative sample indices wrap by L (circular)
  int circular;   // inverse: slice S-1 pairs with slice 0
  int64_t slice0; // global index of local slice 0
  int nslices;    // slices per row (S, or the local range)
  int tr;
  // chunk of units (unit u = row * nslices + local slice)
  int64_t unit0;
  int nunits;
  int tile;       // units per channel-kernel tile
  int stiles;     // channel kernels: tiles per super-tile (0: the whole chunk)
  int pf;         // persistent inverse spectrum kernel: L2 prefetch of the next unit (0 off)
  int Nh;         // N (half the slice length)
  const uint2 *bent;  // sliCQ channels with M_k > 1024: inverse term destinations (kernels_long.cuh)
  // coefficients
  int64_t C;
  float2 *coef_out;
  const float2 *coef_in;
  const float *mask;     // inverse: optional real mask [batch][S][C] fused into the loads
  int mask_db;           // 1: dB-scaled mask, amplitude 10^(-5 (1 - m))
  // staging (workspace): X spectra [unit][xs], contributions [unit][zs]
  float2 *stage;
  int64_t xs, zs;
  int64_t toff;   // large slices: offset of the four-step intermediate inside a unit's staging
  // plan tables
  const ChanDev *chan;
  const PacketDev *packets;
  const int32_t *pchans;
  int npackets;
  int scr;                  // channel kernels: per-warp scratch entries
  const uint2 *fent;        // forward element table (enc, weight bits)
  const uint2 *ient;        // inverse element table (scratch pos, weight bits)
  const uint32_t *dpos;     // inverse overflow run per bin: start | count << 20 (0: none)
  const uint2 *ovbins;      // inverse: per overflow bin (first term, term count) in ovterm
  const uint32_t *dord;     // inverse: per bin 1 + its index in ovbins (0: none)
  int novbins;
  const uint32_t *ovterm;   // inverse: the overflow bins' terms, staging-row offsets, in
  int novterm;              //   summation order (slot 0, slot 1, overflow run)
  int64_t zso;              // inverse staging: slot 1 at zso, overflow at 2 zso
  const float *h0;
  const float *h0dual;
  const float2 *tw2n;
  const float2 *twM;
  unsigned *cnt;  // inverse workspace: [batch][nslices] pairing counters
  float *bnd;     // inverse workspace: [batch][nslices][2][tr] boundary halves
  // long full-length CQ-NSGT (kernels_long.cuh): fp32 g_k / sqrt(M_k), g~_k / sqrt(M_k)
  // (x 1/2 on the plateaus, C15) at the filter offsets goff_k; per-bin term lists (CSR)
  const float *gw, *gdw;
  const uint32_t *lrow, *lent;
  // fused kernels (kernels_fused.cuh)
  const FChan *fch;     // channel descriptors in task order
  const FTask *ftask;   // warp tasks (inverse: phase A first)
  int nftask, nphase_a;
  int fscr;             // per-warp scratch entries
  const int2 *ovb;      // inverse: overflow bins (bin, first | count << 20)
  int novb;
  const int32_t *ovl;   // inverse: overflow slot lists
  int nov;              // inverse: overflow slots per unit
  int vec16;            // coefficient rows are 16-byte aligned (vector stores / loads)
  int tbe;              // TMA-staged channel kernels: per-warp buffer entries (kernels_tb.cuh)
};


// e^{-i pi e / N} for e in [0, 2N): two-level table, 2 shared loads + 1 complex multiply
__device__ __forceinline__ float2 tw_lookup(const float2 *tw, int e) {
  return cmul(tw[64 + (e >> 6)], tw[e & 63]);
}
// the same table read from global memory through the read-only (L1) path
struct GlobalTw {
  const float2 *p;
};
__device__ __forceinline__ float2 tw_lookup(GlobalTw tw, int e) {
  return cmul(__ldg(tw.p + 64 + (e >> 6)), __ldg(tw.p + (e & 63)));
}

// Stockham twiddles for task j of a radix-R pass with span NS (applied before the
// butterfly): w^r for r = 1..R-1, w = e^{SIGN 2 pi i (j mod NS)/(NS R)}.  w^{4q} comes
// from the table, w^{4q+s} = w^{4q} * w^s (s = 1..3): at most two roundings deep.
template <int N, int R, int NS, int SIGN, class TW>
__device__ __forceinline__ void pass_twiddle(float2 (&v)[R], int j, TW tw) {
  if constexpr (NS > 1) {
    static_assert(R % 4 == 0, "big-FFT radices are multiples of 4");
    constexpr int STEP = 2 * (N / (NS * R));  // units of e^{-i pi/N}
    const int base = (j & (NS - 1)) * STEP;
    float2 w1 = tw_lookup(tw, base);
    if (SIGN > 0) w1 = cconj(w1);
    const float2 w2 = cmul(w1, w1);
    const float2 w3 = cmul(w2, w1);
    float2 w4q = make_float2(1.f, 0.f);
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const int s = r & 3;
      if (s == 0) {
        w4q = tw_lookup(tw, (base * r) & (2 * N - 1));
        if (SIGN > 0) w4q = cconj(w4q);
      }
      const float2 ws = s == 1 ? w1 : (s == 2 ? w2 : w3);
      const float2 w = s == 0 ? w4q : (r < 4 ? ws : cmul(w4q, ws));
      v[r] = cmul(v[r], w);
    }
  }
}

// One in-place Stockham pass over the padded shared-memory array.
template <int N, int R, int NS, int SIGN, int T>
__device__ __forceinline__ void pass_smem(float2 *spec, const float2 *tw) {
  constexpr int TASKS = N / R;
  constexpr int PER = (TASKS + T - 1) / T;
  float2 v[PER][R];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = threadIdx.x + q * T;
    if (TASKS % T == 0 || j < TASKS) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = spec[padi(j + r * TASKS)];
      pass_twiddle<N, R, NS, SIGN>(v[q], j, tw);
      dft<R, SIGN>(v[q]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = threadIdx.x + q * T;
    if (TASKS % T == 0 || j < TASKS) {
      const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
      for (int r = 0; r < R; ++r) spec[padi(base + r * NS)] = v[q][r];
    }
  }
  __syncthreads();
}

// X(j) for an unwrapped bin j in (-2N, 2N) from the half spectrum X[0..N] (real input).
template <int N>
__device__ __forceinline__ float2 spec_at(const float2 *spec, int j) {
  const int jj = j < 0 ? j + 2 * N : j;
  const bool up = jj > N;
  const float2 v = spec[padi(up ? 2 * N - jj : jj)];
  return make_float2(v.x, up ? -v.y : v.y);
}

// v[n1] *= e^{SIGN 2 pi i p2 n1 / M}, n1 = 1..M1-1, from the per-M table e^{+2 pi i t/M}:
// table loads at n1 = 1 and n1 = 4q, products for the rest.
template <int M1, int SIGN>
__device__ __forceinline__ void chan_twiddle(float2 (&v)[M1], int p2, int M, const float2 *tab) {
  if constexpr (M1 > 1) {
    float2 w1 = __ldg(tab + p2);
    if (SIGN < 0) w1 = cconj(w1);
    const float2 w2 = cmul(w1, w1);
    const float2 w3 = cmul(w2, w1);
    float2 w4q = make_float2(1.f, 0.f);
    int step4 = 4 * p2;
    while (step4 >= M) step4 -= M;
    int e4 = 0;
#pragma unroll
    for (int n1 = 1; n1 < M1; ++n1) {
      const int s = n1 & 3;
      if (s == 0) {
        e4 += step4;
        if (e4 >= M) e4 -= M;
        w4q = __ldg(tab + e4);
        if (SIGN < 0) w4q = cconj(w4q);
      }
      const float2 ws = s == 1 ? w1 : (s == 2 ? w2 : w3);
      const float2 w = s == 0 ? w4q : (n1 < 4 ? ws : cmul(w4q, ws));
      v[n1] = cmul(v[n1], w);
    }
  }
}

// ------------------------------------------------------------------ PDL helpers
// Programmatic dependent launch: kernels of a call are launched back to back; each waits for
// its predecessor's memory before touching shared buffers and lets the next one launch
// when its CTA is done (hides launch gaps, keeps stream order).
// hide a pointer's derivation from the optimiser so that element accesses p[i] with a
// 32-bit i compile to one IMAD.WIDE instead of re-associated 64-bit index arithmetic
// plain global load (default caching), for pointers the compiler cannot classify
__device__ __forceinline__ float2 ld_global(const float2 *p) {
  float2 v;
  asm volatile("ld.global.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
template <class P>
__device__ __forceinline__ P *opaque(P *p) {
  asm("" : "+l"(p));
  return p;
}
#ifndef SLICQ_FWD_OPAQUE
#define SLICQ_FWD_OPAQUE 1  // forward fold: per-lane spectrum base opaque (32-bit bin indexing);
#endif                      // bit 0: four-step packets (full variant), bit 1: small packets
                            // (measured neutral on cfg4: off)
#if SLICQ_FWD_OPAQUE & 1
#define SLICQ_FWD_OPQ1(p) opaque(p)
#else
#define SLICQ_FWD_OPQ1(p) (p)
#endif
#if SLICQ_FWD_OPAQUE & 2
#define SLICQ_FWD_OPQ2(p) opaque(p)
#else
#define SLICQ_FWD_OPQ2(p) (p)
#endif

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// bring [p, p + bytes) into L2 (one prefetch per 128-byte line, spread over the warp)
__device__ __forceinline__ void prefetch_l2(const void *p, int64_t bytes, int idx, int nthr = 32) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(127);
  const int nl = (int)(((reinterpret_cast<uintptr_t>(p) + bytes - 1) >> 7) - (a0 >> 7)) + 1;
  for (int l = idx; l < nl; l += nthr)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a0 + ((uintptr_t)l << 7)));
}
// the same with one TMA bulk prefetch (cp.async.bulk.prefetch.L2, one instruction for the
// whole 16-byte-aligned envelope of the range; the caller issues it from one lane)
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, int64_t bytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((unsigned)(a1 - a0))
               : "memory");
}
#ifndef SLICQ_BULK_PF
#define SLICQ_BULK_PF 1
#endif
// channel-kernel step codelets, per direction: inlined into the size switch (measured: the
// forward gains 6 % -- no call/return, no spills around the calls, uniform addressing) or
// out of line (one copy per DFT size: smaller instruction-cache footprint)
#ifndef SLICQ_FWD_STEP_INLINE
#define SLICQ_FWD_STEP_INLINE __forceinline__
#endif
#ifndef SLICQ_FWDS_INLINE
#define SLICQ_FWDS_INLINE SLICQ_FWD_STEP_INLINE
#endif
#ifndef SLICQ_FWD2_INLINE
#define SLICQ_FWD2_INLINE SLICQ_FWD_STEP_INLINE
#endif
#ifndef SLICQ_IB_PF_AHEAD
#define SLICQ_IB_PF_AHEAD 1
#endif
#ifndef SLICQ_INV_STEP_INLINE
#define SLICQ_INV_STEP_INLINE __noinline__
#endif
#ifndef SLICQ_INV1_INLINE_MAXS
#define SLICQ_INV1_INLINE_MAXS 16
#endif
#ifndef SLICQ_INV2_INLINE
#define SLICQ_INV2_INLINE SLICQ_INV_STEP_INLINE
#endif
#ifndef SLICQ_INVS_INLINE
#define SLICQ_INVS_INLINE SLICQ_INV_STEP_INLINE
#endif
// ------------------------------------------------------------------ channel packets
// A packet = channels of one length M.  Big packets (M > 32) are a four-step M1 x M2 DFT
// with one task per lane and step; channel ci owns the region ci*M1*S2 (S2 = M2 | 1) of the
// warp scratch: first the length-M vector (fold / F), in between A[n1][p2].  Small packets
// (M <= 32) give each lane a whole channel.

// F3 fold fused into F4 step 1: task (ci, p2) reads its column q = M2 p1 + p2, p1 < M1, of
// the folded vector straight from the element table (entry c M + q: bin | ..., weight with
// the conjugation flag as its sign) and the unit's staged spectrum -- M1 independent loads
// in flight per lane, no shared-memory round trip; DFT_{M1} (sign +), twiddle, stores
// A[n1 S2 + p2].  Virtual channel ci = u * r + c (unit u of the task, channel c).
template <int M1, int V>  // V: channel-kernel variant (separate register budgets)
__device__ SLICQ_FWD_STEP_INLINE void fwd_step1f(const uint2 *ent, const float2 *X, int64_t xs, int r,
                                           unsigned magc, const float2 *twM, float2 *reg, int m2,
                                           int nch, unsigned mag2, int twoff_lane, int lane) {
  const int nt = nch * m2;
  const bool act = lane < nt;
  const int ci = act ? (lane * (int)mag2) >> 16 : 0;
  const int p2 = act ? lane - ci * m2 : 0;
  const int twoff = __shfl_sync(FULL, twoff_lane, ci);
  if (!act) return;
  const int u = (ci * (int)magc) >> 16, c = ci - u * r;
  const int M = M1 * m2;
  const uint2 *e0 = ent + c * M + p2;
  // full variant: the per-lane base made opaque (32-bit bin index, one IMAD.WIDE per load:
  // cfg3 forward -1.6 %); the lite variant keeps the compiler's 64-bit index arithmetic
  // (opaque there: +2.5 % on cfg4 -- more spills at 80 registers)
  const float2 *Xu = V > 16 ? SLICQ_FWD_OPQ1(X + u * xs) : X + u * xs;
  float2 v[M1];
#pragma unroll
  for (int p1 = 0; p1 < M1; ++p1) {
    const uint2 en = __ldg(e0 + m2 * p1);
    const float2 xv = __ldg(Xu + (en.x & 0x3ffff));
    const float gv = __uint_as_float(en.y);  // sign bit: conjugate X (g >= 0)
    v[p1] = make_float2(xv.x * fabsf(gv), xv.y * gv);
  }
  dft<M1, +1>(v);
  chan_twiddle<M1, +1>(v, p2, M, twM + twoff);
  const int S2 = m2 | 1;
  float2 *base = reg + ci * M1 * S2;
#pragma unroll
  for (int n1 = 0; n1 < M1; ++n1) base[n1 * S2 + p2] = v[n1];
}

// F4 step 2 + F5: task (ci, n1): DFT_{M2} over p2 -> c[n1 + M1 n2] (coalesced over n1).
template <int M2, int V>  // V: channel-kernel variant (separate register budgets)
__device__ SLICQ_FWD2_INLINE void fwd_step2(const float2 *reg, float2 *out_row, int m1, int nch,
                                          unsigned mag1, int off_lane, int lane) {
  const int nt = nch * m1;
  constexpr int S2 = M2 | 1;
  const int ci = lane < nt ? (lane * (int)mag1) >> 16 : 0;
  const int n1 = lane - ci * m1;
  const int off = __shfl_sync(FULL, off_lane, ci);
  if (lane >= nt) return;
  float2 v[M2];
  const float2 *A = reg + ci * m1 * S2 + n1 * S2;
#pragma unroll
  for (int p2 = 0; p2 < M2; ++p2) v[p2] = A[p2];
  dft<M2, +1>(v);
  float2 *o = out_row + off + n1;
#pragma unroll
  for (int n2 = 0; n2 < M2; ++n2) SLICQ_CSTORE(o + m1 * n2, v[n2]);
}

// Small forward packet: lane vc = u * nch + c (u < nu) owns channel c of unit u; element p
// of its fold comes from the table entry p*32 + c (bin, weight with the conjugation flag
// as its sign; weight 0 for
// zero padding) -- ent and X arrive offset by c and u.
template <int M, int V>  // V: channel-kernel variant (separate register budgets)
__device__ SLICQ_FWDS_INLINE void fwd_small(const uint2 *ent, const float2 *X, float2 *out_row,
                                          bool act, int off_lane) {
  if (!act) return;
  float2 v[M];
#pragma unroll
  for (int p = 0; p < M; ++p) {
    const uint2 e = __ldg(ent + p * 32);
#if SLICQ_FWD_OPAQUE & 2
    const float2 xv = ld_global(X + e.x);  // (X opaque: global load, 32-bit index)
#else
    const float2 xv = X[e.x];
#endif
    const float gv = __uint_as_float(e.y);  // sign bit: conjugate X (g >= 0)
    v[p] = make_float2(xv.x * fabsf(gv), xv.y * gv);
  }
  dft<M, +1>(v);
  float2 *o = out_row + off_lane;
#pragma unroll
  for (int n = 0; n < M; ++n) SLICQ_CSTORE(o + n, v[n]);
}

// NEXT-4 coefficient mask fused into the inverse's coefficient loads (paper §VI):
// MK = 0 none, 1 linear amplitude m, 2 dB-scaled amplitude 10^(-5 (1 - m))
template <int MK>
__device__ __forceinline__ float2 mask_coef(float2 c, const float *m) {
  if constexpr (MK == 0) {
    return c;
  } else {
    const float mv = __ldcs(m);
    const float amp = MK == 1 ? mv : exp10f(-5.0f * (1.0f - mv));
    return make_float2(c.x * amp, c.y * amp);
  }
}

// I2 step 1: task (ci, p2) loads c[M2 p1 + p2]; DFT_{M1} (sign -); twiddle.
template <int M1, int V, int MK = 0>  // V: channel-kernel variant; MK: fused mask mode
__device__ __forceinline__ void inv_step1_body(const float2 *twM, const float2 *in_row, float2 *reg,
                                          int m2, int nch, unsigned mag2, int off_lane,
                                          int twoff_lane, int lane, const float *mrow = nullptr) {
  const int nt = nch * m2;
  const int ci = lane < nt ? (lane * (int)mag2) >> 16 : 0;
  const int p2 = lane - ci * m2;
  const int off = __shfl_sync(FULL, off_lane, ci), twoff = __shfl_sync(FULL, twoff_lane, ci);
  if (lane >= nt) return;
  float2 v[M1];
  const float2 *src = in_row + off + p2;
#pragma unroll
  for (int p1 = 0; p1 < M1; ++p1) v[p1] = __ldcs(src + p1 * m2);
  if constexpr (MK != 0) {
#pragma unroll
    for (int p1 = 0; p1 < M1; ++p1) v[p1] = mask_coef<MK>(v[p1], mrow + off + p2 + p1 * m2);
  }
  dft<M1, -1>(v);
  chan_twiddle<M1, -1>(v, p2, M1 * m2, twM + twoff);
  const int S2 = m2 | 1;
  float2 *A = reg + ci * M1 * S2 + p2;
#pragma unroll
  for (int n1 = 0; n1 < M1; ++n1) A[n1 * S2] = v[n1];
}
template <int M1, int V, int MK = 0>  // V: channel-kernel variant; MK: fused mask mode
__device__ __noinline__ void inv_step1_ool(const float2 *twM, const float2 *in_row, float2 *reg,
                                          int m2, int nch, unsigned mag2, int off_lane,
                                          int twoff_lane, int lane, const float *mrow) {
  inv_step1_body<M1, V, MK>(twM, in_row, reg, m2, nch, mag2, off_lane, twoff_lane, lane, mrow);
}
// inlined in the variants with DFT sizes <= SLICQ_INV1_INLINE_MAXS (the lite variant: -1.6 %
// on cfg4), out of line in the full variant (instruction-cache footprint: cfg3 +1 % inlined)
template <int M1, int V, int MK = 0>  // V: channel-kernel variant; MK: fused mask mode
__device__ __forceinline__ void inv_step1(const float2 *twM, const float2 *in_row, float2 *reg,
                                          int m2, int nch, unsigned mag2, int off_lane,
                                          int twoff_lane, int lane, const float *mrow = nullptr) {
  if constexpr (V <= SLICQ_INV1_INLINE_MAXS)
    inv_step1_body<M1, V, MK>(twM, in_row, reg, m2, nch, mag2, off_lane, twoff_lane, lane, mrow);
  else
    inv_step1_ool<M1, V, MK>(twM, in_row, reg, m2, nch, mag2, off_lane, twoff_lane, lane, mrow);
}

// I2 step 2, in place: F[n1 + M1 n2] = (unnormalised FFT_M of c) overwrites the region.
template <int M2, int V>  // V: channel-kernel variant (separate register budgets)
__device__ SLICQ_INV2_INLINE void inv_step2(float2 *reg, int m1, int nch, unsigned mag1, int lane) {
  const int nt = nch * m1;
  constexpr int S2 = M2 | 1;
  const bool act = lane < nt;
  const int ci = act ? (lane * (int)mag1) >> 16 : 0;
  const int n1 = act ? lane - ci * m1 : 0;
  float2 v[M2];
  float2 *base = reg + ci * m1 * S2;
  // idle lanes read row 0 too (valid memory) so that v is defined on every path
#pragma unroll
  for (int p2 = 0; p2 < M2; ++p2) v[p2] = base[n1 * S2 + p2];
  dft<M2, -1>(v);
  __syncwarp();
  if (act) {
#pragma unroll
    for (int n2 = 0; n2 < M2; ++n2) base[n1 + m1 * n2] = v[n2];
  }
}

// Small inverse packet: lane vc loads virtual channel vc, FFT_M, F[q] -> scratch q*nv + vc
// (nv odd: the term scatter's reads of consecutive q are bank-conflict free).
template <int M, int V, int MK = 0>  // V: channel-kernel variant; MK: fused mask mode
__device__ SLICQ_INVS_INLINE void inv_small(const float2 *in_row, float2 *reg, int nvc, int nv,
                                          int off_lane, int lane, const float *mrow = nullptr) {
  if (lane >= nvc) return;
  const float2 *src = in_row + off_lane;
  float2 v[M];
#pragma unroll
  for (int n = 0; n < M; ++n) v[n] = __ldcs(src + n);
  if constexpr (MK != 0) {
#pragma unroll
    for (int n = 0; n < M; ++n) v[n] = mask_coef<MK>(v[n], mrow + off_lane + n);
  }
  dft<M, -1>(v);
#pragma unroll
  for (int q = 0; q < M; ++q) reg[q * nv + lane] = v[q];
}

#define SLICQ_SMALL(X) X(4) X(6) X(8) X(10) X(12) X(16) X(18) X(20) X(24) X(30) X(32)
#define SLICQ_SIZES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(8) X(9) X(10) X(12) X(15) X(16) X(18) X(20) X(24) X(25) X(27) X(30) X(32)

#define SLICQ_PRAGMA_(x) _Pragma(#x)
#define SLICQ_UNROLL(n) SLICQ_PRAGMA_(unroll n)
#ifndef SLICQ_XLOAD
#define SLICQ_XLOAD __ldg  // fold reads of the staged spectra (prefetched to L2)
#endif
#ifndef SLICQ_FB_PREFETCH
#define SLICQ_FB_PREFETCH 0
#endif
#ifndef SLICQ_FOLD_UNROLL
#define SLICQ_FOLD_UNROLL 4  // element loops of the channel kernels: loads in flight per lane
#endif

// ------------------------------------------------------------------ channel kernels
// Persistent grid; a work item is (packet, tile of units), the CTA's warps split the units.
// Defined in one translation unit only (kernels_host.cu).
constexpr int CHAN_T = 256;
#ifndef SLICQ_CHAN_MINB
#define SLICQ_CHAN_MINB 2
#endif
#ifdef SLICQ_DEFINE_CHAN_KERNELS

template <int MAXS, int MINB>
__global__ void __launch_bounds__(CHAN_T, MINB) slicq_fwd_chan_kernel(const KArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int NW = CHAN_T / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();
  // persistent: a work item is (packet, tile of units), items in packet-major order, the
  // warps of a CTA split the tile's units: every warp of every SM runs the same packet
  // code at the same time (instruction-cache locality) and the packet's tables stay hot
  const int ntiles = (a.nunits + a.tile - 1) / a.tile;
  const int nitems = a.npackets * ntiles;
  const int sts = a.stiles > 0 ? a.stiles : ntiles;  // tiles per super-tile
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    // packet-major inside super-tiles of sts tiles: a super-tile's staged spectra stay in L2
    // while its packets pass over them (each packet's code still runs sts tiles in a row)
    const int per_st = a.npackets * sts;
    const int st = item / per_st, rem = item - st * per_st;
    const int st_n = min(sts, ntiles - st * sts);  // tiles in this (possibly last) super-tile
    const int pk = rem / st_n;
    const int tile = st * sts + (rem - pk * st_n);
    float2 *scr = reinterpret_cast<float2 *>(smem4) + warp * a.scr;
    const PacketDev P = a.packets[pk];
    const int m1 = P.m1m2 & 255, m2 = (P.m1m2 >> 8) & 255;
    const bool small = (P.m1m2 >> 17) & 1;
    const int r = P.nch, nu = P.nu;
    // this lane's virtual channel vc = u_l * r + c_l (a channel of one of the task's units)
    const int vcl = lane < nu * r ? lane : 0;
    const int u_l = (vcl * (int)P.magc) >> 16, c_l = vcl - u_l * r;
    const int ck = __ldg(a.pchans + P.chan_off + c_l);
    const int c_off = __ldg(&a.chan[ck].off) + u_l * (int)a.C;
    const int c_twoff = __ldg(&a.chan[ck].twoff);
    const uint2 *ent = a.fent + P.fent_off;
    const int ne = small ? 0 : r * m1 * m2;
    const int u_lo = tile * a.tile;
    const int u_hi = min(a.nunits, u_lo + a.tile);
    const int ntask = (u_hi - u_lo + nu - 1) / nu;
    for (int t = warp; t < ntask; t += NW) {
      const int g0 = u_lo + t * nu;          // the task's first unit
      const int nuu = min(nu, u_hi - g0);    // units in this task
      const int nvc = nuu * r;
      const float2 *X = a.stage + (int64_t)g0 * a.xs;
      float2 *out_row = a.coef_out + (a.unit0 + g0) * a.C;
#if SLICQ_FB_PREFETCH == 1  // (measured: no gain on cfg4; the fold's loads are L2-latency bound)
      if (t + NW < ntask) {  // this warp's next task: its spectrum bins -> L2 (staging in DRAM)
        const int g1 = g0 + NW * nu, n1u = min(nu, u_hi - g1);
        for (int u = 0; u < n1u; ++u)
          prefetch_l2(X + (int64_t)(NW * nu + u) * a.xs + P.xlo, (int64_t)(P.xhi - P.xlo + 1) * 8,
                      lane);
      }
#elif SLICQ_FB_PREFETCH == 2  // one TMA bulk prefetch per unit (lane u: unit u's band)
      if (t + NW < ntask) {
        const int g1 = g0 + NW * nu, n1u = min(nu, u_hi - g1);
        if (lane < n1u)
          prefetch_l2_bulk(X + (int64_t)(NW * nu + lane) * a.xs + P.xlo,
                           (int64_t)(P.xhi - P.xlo + 1) * 8);
      }
#endif
      if (small) {
        switch (m1) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) fwd_small<S, MAXS>(ent + c_l, SLICQ_FWD_OPQ2(X + (int64_t)u_l * a.xs), out_row, lane < nvc, c_off); break;
          SLICQ_SMALL(X_)
#undef X_
        }
        continue;
      }
      // F3 fold fused into step 1 (loads straight from the element table and the spectrum)
      (void)ne;
      switch (m1) {
#define X_(S)                                                                               \
  case S:                                                                                   \
    if constexpr (S <= MAXS)                                                                \
      fwd_step1f<S, MAXS>(ent, X, a.xs, r, P.magc, a.twM, scr, m2, nvc, P.mag2, c_twoff, lane); \
    break;
        SLICQ_SIZES(X_)
#undef X_
      }
      __syncwarp();
      switch (m2) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) fwd_step2<S, MAXS>(scr, out_row, m1, nvc, P.mag1, c_off, lane); break;
        SLICQ_SIZES(X_)
#undef X_
      }
      __syncwarp();
    }
  }
  pdl_trigger();
}

template <int MAXS, int MINB, int MK = 0>
__global__ void __launch_bounds__(CHAN_T, MINB) slicq_inv_chan_kernel(const KArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int NW = CHAN_T / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();
  // persistent: a work item is (packet, tile of units), items in packet-major order, the
  // warps of a CTA split the tile's units: every warp of every SM runs the same packet
  // code at the same time (instruction-cache locality) and the packet's tables stay hot
  const int ntiles = (a.nunits + a.tile - 1) / a.tile;
  const int nitems = a.npackets * ntiles;
  const int sts = a.stiles > 0 ? a.stiles : ntiles;  // tiles per super-tile
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    // packet-major inside super-tiles of sts tiles: a super-tile's staged spectra stay in L2
    // while its packets pass over them (each packet's code still runs sts tiles in a row)
    const int per_st = a.npackets * sts;
    const int st = item / per_st, rem = item - st * per_st;
    const int st_n = min(sts, ntiles - st * sts);  // tiles in this (possibly last) super-tile
    const int pk = rem / st_n;
    const int tile = st * sts + (rem - pk * st_n);
    float2 *scr = reinterpret_cast<float2 *>(smem4) + warp * a.scr;
    const PacketDev P = a.packets[pk];
    const int m1 = P.m1m2 & 255, m2 = (P.m1m2 >> 8) & 255;
    const bool small = (P.m1m2 >> 17) & 1;
    const int r = P.nch, nu = P.nu;
    const int vcl = lane < nu * r ? lane : 0;
    const int u_l = (vcl * (int)P.magc) >> 16, c_l = vcl - u_l * r;
    const int ck = __ldg(a.pchans + P.chan_off + c_l);
    const int c_off0 = __ldg(&a.chan[ck].off);
    const int c_off = c_off0 + u_l * (int)a.C;
    const int c_twoff = __ldg(&a.chan[ck].twoff);
    const uint2 *ent = a.ient + P.ient_off;
    const int ne = P.nz;  // entries (channel term -> staging slot) of the packet
    const int u_lo = tile * a.tile;
    const int u_hi = min(a.nunits, u_lo + a.tile);
    const int cbase = __shfl_sync(FULL, c_off0, 0);
    const int clen = __shfl_sync(FULL, c_off0, r - 1) - cbase + m1 * m2;
    const int ntask = (u_hi - u_lo + nu - 1) / nu;
    for (int t = warp; t < ntask; t += NW) {
      const int g0 = u_lo + t * nu;
      const int nuu = min(nu, u_hi - g0);
      const int nvc = nuu * r;
      const float2 *in_row = a.coef_in + (a.unit0 + g0) * a.C;
      const float *mrow = MK ? a.mask + (a.unit0 + g0) * a.C : nullptr;
      // L2 prefetch of the coefficient rows SLICQ_IB_PF_AHEAD tasks of this warp ahead: one
      // TMA bulk prefetch per unit (lane u issues unit u's run), not one prefetch per line
      if (t + SLICQ_IB_PF_AHEAD * NW < ntask) {
        const int g1 = g0 + SLICQ_IB_PF_AHEAD * NW * nu, n1u = min(nu, u_hi - g1);
        // (16-byte aligned rows: the envelope stays inside the coefficient row)
        if (SLICQ_BULK_PF && a.vec16) {
          if (lane < n1u)
            prefetch_l2_bulk(in_row + (int64_t)(SLICQ_IB_PF_AHEAD * NW * nu + lane) * a.C + cbase,
                             (int64_t)clen * 8);
        } else {
          for (int u = 0; u < n1u; ++u)
            prefetch_l2(in_row + (int64_t)(SLICQ_IB_PF_AHEAD * NW * nu + u) * a.C + cbase,
                        (int64_t)clen * 8, lane);
        }
      }
      if (small) {
        switch (m1) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) inv_small<S, MAXS, MK>(in_row, scr, nvc, (nu * r) | 1, c_off, lane, mrow); break;
          SLICQ_SMALL(X_)
#undef X_
        }
      } else {
        switch (m1) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) inv_step1<S, MAXS, MK>(a.twM, in_row, scr, m2, nvc, P.mag2, c_off, c_twoff, lane, mrow); break;
          SLICQ_SIZES(X_)
#undef X_
        }
        __syncwarp();
        switch (m2) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) inv_step2<S, MAXS>(scr, m1, nvc, P.mag1, lane); break;
          SLICQ_SIZES(X_)
#undef X_
        }
      }
      __syncwarp();
      // I3a terms F[q] * g~_k[j]/sqrt(M_k) (conjugated for mirrored bins) -> their slot of
      // the unit's half-spectrum staging (I3b sums the slots)
      for (int u = 0; u < nuu; ++u) {
        float2 *Zb = opaque(a.stage + (int64_t)(g0 + u) * a.zs);  // 32-bit indexing
        const float2 *su = scr + u * P.ustride;
        SLICQ_UNROLL(SLICQ_FOLD_UNROLL)
        for (int e = lane; e < ne; e += 32) {
          const uint2 en = __ldg(ent + e);
          const float2 f = su[en.x & 0x3fff];
          const float w = __uint_as_float(en.y);  // sign bit: conjugate the term (g~ >= 0)
          SLICQ_ZSTORE(Zb + (en.x >> 14), make_float2(f.x * fabsf(w), f.y * w));
        }
      }
      __syncwarp();
    }
  }
  pdl_trigger();
}

#endif  // SLICQ_DEFINE_CHAN_KERNELS

// ------------------------------------------------------------------ forward spectrum kernel
// MODE 0: sliCQ slice m (Tukey window, hop N, circular indices).  MODE 1: full-length
// CQ-NSGT (Alg. 1): the frame is the whole signal x[0..2N) (zeros past
// x_len), no window; one unit per row.
// F1 + F2 of unit u (row * nslices + local slice) into X[0..N].  TOSMEM = false: X goes to
// Xo[0..N] in global memory (the staging row of the split design, or a ring slot);
// TOSMEM = true: X stays in shared memory, spec[padi(k)] for k = 0..N.  htab: tr - 1 floats
// of shared scratch.  LOADTW: stage the twiddle table (persistent callers do it once).
// Bit qq * R + r of the result: this warp's 32 frame pairs q = j + r TASKS (first pass, task
// slot qq) touch a window transition, i.e. need the multiply by h_0 -- not all on the flat top
// (h_0 = 1) and not all outside the window support (zeros, not loaded).  Depends on (N, tr)
// and the warp only: the persistent kernel computes it once per CTA.
template <int LOGN, int MODE>
__device__ __forceinline__ uint32_t fwd_window_mask(const KArgs &a) {
  using CF = Big<LOGN>;
  constexpr int N = CF::N, T = CF::T, R = CF::F1, TASKS = N / R, PER = (TASKS + T - 1) / T;
  static_assert(PER * R <= 32, "window mask bits");
  if constexpr (MODE == 1) return 0u;  // no window
  const int A = (N - a.tr) / 2, Bw = (N + a.tr) / 2;
  const int q_lo = (N - Bw + 1) >> 1, q_hi = (N + Bw - 1) >> 1;
  const int qa = (N - A + 1) >> 1, qb = (N + A - 1) >> 1;  // pairs with |t| <= A for both
  uint32_t m = 0;
#pragma unroll
  for (int qq = 0; qq < PER; ++qq) {
    const int jw = ((int)threadIdx.x & ~31) + qq * T;  // this warp's first task
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int w0 = jw + r * TASKS, w1 = w0 + 31;
      if (!((w0 >= qa && w1 <= qb) || w1 < q_lo || w0 > q_hi)) m |= 1u << (qq * R + r);
    }
  }
  return m;
}

template <int LOGN, int MODE, bool TOSMEM, bool LOADTW = true, bool LOADH = true>
__device__ __forceinline__ void fwd_spectrum(const KArgs &a, float2 *spec, float2 *tw, float *htab,
                                             int64_t u, float2 *Xo, uint32_t wmask = 0,
                                             bool have_wmask = false) {
  using CF = Big<LOGN>;
  constexpr int N = CF::N, T = CF::T;
  const int tid = threadIdx.x;
  const int64_t row = unit_row(u, a.nslices);
  const int64_t mloc = u - row * a.nslices;
  const int64_t mg = a.slice0 + mloc;

  PHASE_INIT();
  if constexpr (LOADTW)
    for (int i = tid; i < tw_entries<LOGN>(); i += T) tw[i] = a.tw2n[i];
  pdl_wait();  // the staging buffer may still be read by the previous chunk's kernel

  // ---- F1 + first radix pass straight from HBM: task j takes the frame pairs
  // z[q] = (f[2q], f[2q+1]), q = j + r N/R, of the Tukey-windowed frame f^m[i] = x[s0 + i]
  // h_0[i - N] (wrapped by L for slice 0).  Zero-window pairs are not loaded; all of
  // a thread's loads are issued before any is used (HBM latency overlapped with the window
  // table staging); the window multiplies only the transitions (h_0 = 1 on the flat top).
  {
    constexpr int R = CF::F1, TASKS = N / R, PER = (TASKS + T - 1) / T;
    const float *xr = a.x + row * a.x_stride;
    const int64_t s0 = (mg - 1) * N - a.base_off;  // local x index of frame sample 0
    const bool vec = ((reinterpret_cast<uintptr_t>(xr + s0) & 7) == 0);  // 8-byte pairs
    const int A = MODE ? N : (N - a.tr) / 2, Bw = MODE ? N + 1 : (N + a.tr) / 2;
    if constexpr (MODE == 0 && LOADH)
      for (int u = tid; u < a.tr - 1; u += T) htab[u] = __ldg(a.h0 + N + A + 1 + u);
    // window support: pairs q_lo..q_hi hold at least one nonzero-window sample
    const int q_lo = MODE ? 0 : (N - Bw + 1) >> 1, q_hi = MODE ? N - 1 : (N + Bw - 1) >> 1;
    // interior frames (no wrap, no signal edge, 8-byte aligned row): unchecked pair loads
    const bool fast = vec && s0 + 2 * q_lo >= 0 && s0 + 2 * q_hi + 1 < a.x_len;
    const float2 *xp = reinterpret_cast<const float2 *>(xr + (fast ? s0 : 0));
    float2 v[PER][R];
    if (fast) {  // unswitched: predicated pair loads, no divergent branches
#pragma unroll
      for (int qq = 0; qq < PER; ++qq) {
        const int j = tid + qq * T;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int q = j + r * TASKS;
          const bool in = (TASKS % T == 0 || j < TASKS) && (unsigned)(q - q_lo) <= (unsigned)(q_hi - q_lo);
          v[qq][r] = in ? __ldcs(xp + q) : make_float2(0.f, 0.f);
        }
      }
    } else {
#pragma unroll
    for (int qq = 0; qq < PER; ++qq) {
      const int j = tid + qq * T;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int q = j + r * TASKS;
        float x0 = 0.f, x1 = 0.f;
        if ((TASKS % T == 0 || j < TASKS) && q >= q_lo && q <= q_hi) {
          {
            int64_t xi = s0 + 2 * q;
            if (a.wrap && xi < 0) xi += a.L;
            if (vec && xi >= 0 && xi + 1 < a.x_len) {
              const float2 t2 = __ldcs(reinterpret_cast<const float2 *>(xr + xi));
              x0 = t2.x;
              x1 = t2.y;
            } else {
              if (xi >= 0 && xi < a.x_len) x0 = __ldg(xr + xi);
              if (xi + 1 >= 0 && xi + 1 < a.x_len) x1 = __ldg(xr + xi + 1);
            }
          }
        }
        v[qq][r] = make_float2(x0, x1);
      }
    }
    }
    __syncthreads();  // window table staged (and twiddles)
    // warp-uniform skip mask (see fwd_window_mask; the persistent kernel passes it in)
    const uint32_t wm = have_wmask ? wmask : fwd_window_mask<LOGN, MODE>(a);
#pragma unroll
    for (int qq = 0; qq < PER; ++qq) {
      const int j = tid + qq * T;
      if (TASKS % T == 0 || j < TASKS) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int q = j + r * TASKS;
          // warp-uniform skip: the warp's 32 pairs all on the flat top (h_0 = 1), or all
          // outside the window support (not loaded: zeros)
          if constexpr (MODE == 1) continue;  // no window
          if (!((wm >> (qq * R + r)) & 1u)) continue;
          // |t| of the two samples (t = 2q - N and 2q + 1 - N); h_0 = 1 for |t| <= A, the
          // staged transition for A < |t| < Bw, 0 beyond (selects, no divergent branches)
          const int t0 = abs(2 * q - N), t1 = abs(2 * q + 1 - N);
          const float h0a = t0 <= A ? 1.f : (t0 < Bw ? htab[t0 - A - 1] : 0.f);
          const float h0b = t1 <= A ? 1.f : (t1 < Bw ? htab[t1 - A - 1] : 0.f);
          v[qq][r].x *= h0a;
          v[qq][r].y *= h0b;
        }
        dft<R, -1>(v[qq]);
#pragma unroll
        for (int r = 0; r < R; ++r) spec[padi(j * R + r)] = v[qq][r];
      }
    }
    __syncthreads();
  }
  PHASE_MARK(0, 0);
  pass_smem<N, CF::F2, CF::F1, -1, T>(spec, tw);
  PHASE_MARK(0, 1);
  constexpr int R3 = CF::F3, TASKS3 = N / R3;
  if constexpr (R3 == 16 && TASKS3 == 2 * T) {
    // ---- last radix-16 pass + r2c packing + store, fused in registers: thread t owns the
    // tasks jA = t and jB = TASKS3 - t (t = 0: 0 and TASKS3/2); their outputs Z[k],
    // k = j + TASKS3 r, pair up as mirrors N - (jA + TASKS3 r) = jB + TASKS3 (15 - r), so
    // X[k] = E + e^{-i pi k/N} O and X[N-k] = conj(E) - conj(e^{-i pi k/N} O),
    // E = (Z[k] + conj Z[N-k])/2, O = (Z[k] - conj Z[N-k])/(2i), come out of registers
    // and go straight to the staging buffer (coalesced across the warp).
    const int jA = tid, jB = tid == 0 ? TASKS3 / 2 : TASKS3 - tid;
    float2 vA[16], vB[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      vA[r] = spec[padi(jA + r * TASKS3)];
      vB[r] = spec[padi(jB + r * TASKS3)];
    }
    pass_twiddle<N, 16, TASKS3, -1>(vA, jA, tw);
    pass_twiddle<N, 16, TASKS3, -1>(vB, jB, tw);
    dft<16, -1>(vA);
    dft<16, -1>(vB);
    auto xst = [&](int k, float2 v) {
      if constexpr (TOSMEM) spec[padi(k)] = v;
      else SLICQ_XSTORE(Xo + k, v);
    };
    if constexpr (TOSMEM) __syncthreads();  // every pass-3 input read before X overwrites it
    auto r2c_w = [&](float2 zk, float2 zn, float2 w, int k, bool mirror) {
      const float2 E = cscale(cadd(zk, cconj(zn)), 0.5f);
      const float2 O = cscale(mul_si<-1>(csub(zk, cconj(zn))), 0.5f);
      const float2 wO = cmul(w, O);  // e^{-i pi k/N} O
      xst(k, cadd(E, wO));
      if (mirror) xst(N - k, csub(cconj(E), cconj(wO)));
    };
    auto r2c = [&](float2 zk, float2 zn, int k, bool mirror) {
      r2c_w(zk, zn, tw_lookup(tw, k), k, mirror);
    };
    // thread 0's tasks 0 and TASKS3/2 are their own mirrors: warp 0 packs their 32 bins
    // cooperatively, one bin per lane (X[k] = E + e^{-i pi k/N} O at each k; k = 0 also
    // gives X[N]), instead of a divergent special path
    __shared__ float2 svz[32];
    if (tid < 32) {  // warp 0 (warp-uniform branch)
      if (tid == 0) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          svz[r] = vA[r];
          svz[16 + r] = vB[r];
        }
      }
      __syncwarp();
      const int L = tid;
      const int ib = L == 0 ? 0 : (L < 16 ? 16 - L : 16 + 15 - (L - 16));  // Z[N - k]
      const int kk = L < 16 ? TASKS3 * L : TASKS3 / 2 + TASKS3 * (L - 16);
      const float2 zk = svz[L], zn = svz[ib];
      if (L == 0) {  // X[0], X[N] from Z[0]
        xst(0, make_float2(zk.x + zk.y, 0.f));
        xst(N, make_float2(zk.x - zk.y, 0.f));
      } else {
        r2c(zk, zn, kk, false);
      }
    }
    if (tid != 0) {
      // e^{-i pi (jA + TASKS3 r)/N} = e^{-i pi jA/N} e^{-2 pi i r/32}: one table lookup per
      // thread, the 16 rotations are compile-time twiddles (FMUL2/FFMA2 immediates)
      const float2 wb = tw_lookup(tw, jA);
      static_for<0, 16>([&](auto Rc) {
        constexpr int r = decltype(Rc)::value;
        r2c_w(vA[r], vB[15 - r], twiddle_c<r, 32, -1>(wb), jA + TASKS3 * r, true);
      });
    }
  } else {
    pass_smem<N, CF::F3, CF::F1 * CF::F2, -1, T>(spec, tw);
    PHASE_MARK(0, 2);

    // ---- r2c packing: X[k] = E[k] + e^{-i pi k/N} O[k], k = 0..N  (Z[N] := Z[0])
    for (int k = tid; k <= N / 2; k += T) {
      const float2 zk = spec[padi(k)];
      const float2 zn = spec[padi((N - k) & (N - 1))];
      if (k == 0) {
        spec[padi(0)] = make_float2(zk.x + zk.y, 0.f);
        spec[padi(N)] = make_float2(zk.x - zk.y, 0.f);
      } else {
        // E = (Zk + conj Zn)/2, O = (Zk - conj Zn)/(2i)
        const float2 E = cscale(cadd(zk, cconj(zn)), 0.5f);
        const float2 O = cscale(mul_si<-1>(csub(zk, cconj(zn))), 0.5f);
        const float2 wO = cmul(tw_lookup(tw, k), O);  // e^{-i pi k/N} O
        spec[padi(k)] = cadd(E, wO);
        // X[N-k] = conj(E) + e^{-i pi (N-k)/N} conj(O) = conj(E) - conj(wO)
        if (k != N / 2) spec[padi(N - k)] = csub(cconj(E), cconj(wO));
      }
    }
    __syncthreads();
    PHASE_MARK(0, 3);

    // ---- X[0..N] -> staging (coalesced)
    if constexpr (!TOSMEM) {
      for (int k = tid; k <= N; k += T) Xo[k] = spec[padi(k)];
    }
  }
  PHASE_MARK(0, 4);
}

template <int LOGN, int MODE = 0>
__global__ void __launch_bounds__(Big<LOGN>::T, Big<LOGN>::MINBF) slicq_fwd_spec_kernel(const KArgs a) {
  extern __shared__ float4 smem4[];
  float2 *spec = reinterpret_cast<float2 *>(smem4);
  float2 *tw = spec + spec_entries<LOGN>();
  float *htab = reinterpret_cast<float *>(tw + tw_entries<LOGN>());  // window transitions
  fwd_spectrum<LOGN, MODE, false>(a, spec, tw, htab, a.unit0 + blockIdx.x,
                                  a.stage + (int64_t)blockIdx.x * a.xs);
  pdl_trigger();
}

// Persistent variant (MODE 0): CTA c transforms the contiguous units [c U / G, (c+1) U / G) of
// the chunk; the twiddle table is staged once and the next unit's frame is prefetched to L2
// while this one is transformed (consecutive frames of a row also share tr - 1 samples).
template <int LOGN>
__global__ void __launch_bounds__(Big<LOGN>::T, Big<LOGN>::MINBF) slicq_fwd_spec_persist_kernel(const KArgs a) {
  using CF = Big<LOGN>;
  constexpr int N = CF::N, T = CF::T;
  extern __shared__ float4 smem4[];
  float2 *spec = reinterpret_cast<float2 *>(smem4);
  float2 *tw = spec + spec_entries<LOGN>();
  float *htab = reinterpret_cast<float *>(tw + tw_entries<LOGN>());
  const int tid = threadIdx.x;
  for (int i = tid; i < tw_entries<LOGN>(); i += T) tw[i] = a.tw2n[i];
  {  // the window's transition table, once per CTA
    const int A = (N - a.tr) / 2;
    for (int u = tid; u < a.tr - 1; u += T) htab[u] = __ldg(a.h0 + N + A + 1 + u);
  }
  const int64_t G = gridDim.x;
  const int64_t ub = blockIdx.x * (int64_t)a.nunits / G, ue = (blockIdx.x + 1) * (int64_t)a.nunits / G;
  const uint32_t wmask = fwd_window_mask<LOGN, 0>(a);  // once per CTA
  for (int64_t ul = ub; ul < ue; ++ul) {
    if (ul + 1 < ue && tid == 0) {  // the next frame's window support -> L2 (one bulk prefetch)
      const int64_t u = a.unit0 + ul + 1, row = unit_row(u, a.nslices);
      const int64_t s0 = (a.slice0 + (u - row * a.nslices) - 1) * N - a.base_off + (N - a.tr) / 2;
      const float *p0 = a.x + row * a.x_stride + s0;
      // (inside the row and 16-byte aligned at the row start: the envelope stays in x)
      if (s0 >= 4 && s0 + N + a.tr + 4 <= a.x_len)
        prefetch_l2_bulk(p0, (int64_t)(N + a.tr) * 4);
    }
    fwd_spectrum<LOGN, 0, false, false, false>(a, spec, tw, htab, a.unit0 + ul, a.stage + ul * a.xs,
                                               wmask, true);
    __syncthreads();  // (spec reused by the next unit)
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ inverse spectrum kernel
// MODE 0: sliCQ (dual window, overlap-add, paired boundaries).  MODE 1: full-length CQ-NSGT
// synthesis (Alg. 2): y[row][i] = the frame sample i for i < y_len, nothing else.
// I3b + I4 + I5 of unit ul of the chunk: the slot sum, c2r FFT, dual window and overlap-add.
// The caller has staged tw and htab (and waited for the channel kernel).  ll / rl: the left /
// right overlap with the neighbouring slice of the same row is resolved locally (persistent
// kernel: the neighbour is this CTA's previous / next unit), through carry[0 .. tr-1) in
// shared memory instead of the cross-CTA pairing through the workspace; the sums are the
// same (a + b, each half rounded as stored), so both kernels give bit-identical output.
// OVP (persistent kernel): the deep-overlap bins' sums slot0 + slot1 + overflow run (plan
// order) are formed in a pre-pass spread over all threads of the CTA into `ovs` (shared),
// instead of by the thread that owns the bin: the overflow bins crowd the low bins, i.e.
// the first warps, whose serial overflow loops the other warps waited for at the next
// barrier.  Same additions in the same order: bit-identical.
template <int LOGN, int MODE, bool OVP = false>
__device__ __forceinline__ void inv_unit(const KArgs &a, float2 *spec, float2 *tw, float *htab,
                                         float *carry, int64_t ul, bool ll, bool rl,
                                         float2 *ovs = nullptr, bool ovpre = false,
                                         bool ovnext = false) {
  using CF = Big<LOGN>;
  constexpr int N = CF::N, T = CF::T;
  const int tid = threadIdx.x;
  const int64_t u = a.unit0 + ul;
  const int64_t row = unit_row(u, a.nslices);
  const int mloc = (int)(u - row * a.nslices);
  const int64_t mg = a.slice0 + mloc;

  PHASE_INIT();
  constexpr bool hsm = true;

  constexpr int R1 = CF::I1, TASKS1 = N / R1;
  if constexpr (R1 == 16 && TASKS1 == 2 * T) {
    // ---- I3b + I4a + first radix-16 pass, fused in registers: thread t owns the pass-1
    // tasks jA = t and jB = TASKS1 - t (t = 0: tasks 0 and TASKS1/2), whose inputs
    // Z[k], k = j + TASKS1 r, pair up as mirrors: N - (jA + TASKS1 r) = jB + TASKS1 (15 - r),
    // so every half-spectrum bin H[b] = slot0[b] + slot1[b] (+ overflow) is loaded once
    // and the c2r packing Z[k] = E + iO, E = (H[k] + conj H[N-k])/2,
    // O = (H[k] - conj H[N-k]) e^{+i pi k/N} / 2, happens in registers.
    const float2 *Z0 = a.stage + ul * a.zs;
    const float2 *Z1 = Z0 + a.zso, *Zo = Z0 + 2 * a.zso;
    const int jA = tid, jB = tid == 0 ? TASKS1 / 2 : TASKS1 - tid;
#if SLICQ_INV_PF2
    // the second load batch's bins (r >= IG: k >= TASKS1 IG) of both slots -> L2 now, two bulk
    // prefetches, so that batch's loads hit L2 when they are issued after the first batch
    if (tid == 0) {
      constexpr int K2 = TASKS1 * SLICQ_IA_GROUP;
      prefetch_l2_bulk(Z0 + K2, (int64_t)(N + 1 - K2) * 8);
      prefetch_l2_bulk(Z1 + K2, (int64_t)(N + 1 - K2) * 8);
    }
#endif
    // e^{+i pi k / N} from the global two-level table (no wait for the shared copy)
    auto wk = [&](int k) {
      return cconj(cmul(__ldg(a.tw2n + 64 + (k >> 6)), __ldg(a.tw2n + (k & 63))));
    };
    // c2r packing of the pair (k, N - k): Z[k] = E + iO, Z[N-k] = conj(E) + i conj(D) conj(w)
    auto pack_w = [&](float2 &hk, float2 &hn, float2 w) {
      const float2 E = cscale(cadd(hk, cconj(hn)), 0.5f);
      const float2 D = cscale(csub(hk, cconj(hn)), 0.5f);
      const float2 O = cmul(D, w);  // (conj D)(conj w) = conj O, exactly
      hk = cadd(E, mul_si<+1>(O));                       // E + iO
      hn = cadd(cconj(E), make_float2(O.y, O.x));        // conj(E) + i conj(O)
    };
    // H at the thread's 32 bins jA + TASKS1 r (vA) and jB + TASKS1 r (vB): 4 r per batch,
    // all 16 slot loads and 8 overflow descriptors of a batch in flight together
    float2 vA[16], vB[16];
    // bin N (thread 0's self-mirrored task 0 pairs bin 0 with it): loads issued first, in
    // flight with the slot loads below (warp 0 must not wait on them alone)
    float2 hN = make_float2(0.f, 0.f);
    uint32_t dN = 0;
    if (tid == 0) {
      hN = cadd(__ldcg(Z0 + N), __ldcg(Z1 + N));
      dN = OVP ? __ldg(a.dord + N) : __ldg(a.dpos + N);
    }
    // warp 0's cooperative packing of the self-mirrored bins (below): lane L's bin and its
    // twiddle, loaded now
    const int ksp = tid < 16 ? TASKS1 * tid : TASKS1 / 2 + TASKS1 * (tid - 16);
    const float2 wsp = tid < 32 ? wk(ksp) : make_float2(1.f, 0.f);
    // e^{+i pi (jA + TASKS1 r)/N} = e^{+i pi jA/N} e^{+2 pi i r/32}: one table lookup per
    // thread (issued here, ahead of the slot loads), the 16 rotations are compile-time twiddles
    const float2 wb = wk(jA);
    constexpr int IG = SLICQ_IA_GROUP;  // r values per load batch
#pragma unroll
    for (int r0 = 0; r0 < 16; r0 += IG) {
      float2 a0[IG], a1[IG], b0[IG], b1[IG];
      uint32_t da[IG], db[IG];
#pragma unroll
      for (int q = 0; q < IG; ++q) {
        const int ka = jA + TASKS1 * (r0 + q), kb = jB + TASKS1 * (r0 + q);
        a0[q] = SLICQ_ZLOAD(Z0 + ka);
        a1[q] = SLICQ_ZLOAD(Z1 + ka);
        b0[q] = SLICQ_ZLOAD(Z0 + kb);
        b1[q] = SLICQ_ZLOAD(Z1 + kb);
        da[q] = OVP ? __ldg(a.dord + ka) : __ldg(a.dpos + ka);
        db[q] = OVP ? __ldg(a.dord + kb) : __ldg(a.dpos + kb);
      }
      if constexpr (OVP) {
        if (r0 == 0) {  // pre-pass, in flight with the first batch's loads
          // (a) every term of every overflow bin -> shared memory, all loads in flight at once
          // (persistent kernel: the previous unit issued them as cp.async copies -- ovpre --
          // so only the first unit of a CTA waits a full gather here)
          float2 *ovt = ovs + a.novbins;
          if (ovpre) {
            asm volatile("cp.async.wait_all;" ::: "memory");
          } else {
            for (int i = tid; i < a.novterm; i += T) ovt[i] = __ldcg(Z0 + __ldg(a.ovterm + i));
          }
          __syncthreads();
          // (b) each bin's sum in plan order, from shared memory
          for (int i = tid; i < a.novbins; i += T) {
            const uint2 e = __ldg(a.ovbins + i);
            float2 h = cadd(ovt[e.x], ovt[e.x + 1]);
            for (int k = 2; k < (int)e.y; ++k) h = cadd(h, ovt[e.x + k]);
            ovs[i] = h;
          }
          __syncthreads();
          if (ovnext) {  // the next unit's overflow terms -> ovt, asynchronously (ovt is free now)
            const float2 *Zn = Z0 + a.zs;
            for (int i = tid; i < a.novterm; i += T) {
              const unsigned dst = (unsigned)__cvta_generic_to_shared(ovt + i);
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst),
                           "l"(Zn + __ldg(a.ovterm + i))
                           : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
          }
        }
#pragma unroll
        for (int q = 0; q < IG; ++q) {
          vA[r0 + q] = da[q] ? ovs[da[q] - 1] : cadd(a0[q], a1[q]);
          vB[r0 + q] = db[q] ? ovs[db[q] - 1] : cadd(b0[q], b1[q]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < IG; ++q) {
          vA[r0 + q] = cadd(a0[q], a1[q]);
          vB[r0 + q] = cadd(b0[q], b1[q]);
          if (da[q] | db[q]) {  // deep-overlap bins: overflow terms in order
            for (int e = 0; e < (int)(da[q] >> 20); ++e)
              vA[r0 + q] = cadd(vA[r0 + q], __ldcg(Zo + (da[q] & 0xfffff) + e));
            for (int e = 0; e < (int)(db[q] >> 20); ++e)
              vB[r0 + q] = cadd(vB[r0 + q], __ldcg(Zo + (db[q] & 0xfffff) + e));
          }
        }
      }
    }
    // Thread 0's tasks 0 and TASKS1/2 are their own mirrors (bins TASKS1 r pair as
    // (r, 16 - r) with r = 0 pairing bin N, bins TASKS1/2 + TASKS1 r as (r, 15 - r)).  Rather
    // than a divergent special path in warp 0, the warp packs those 32 bins cooperatively,
    // one bin per lane, with the same formula: Z[k] = F(H[k], H[N-k], k) (the second output
    // of a pair is F at N - k).  Every lane also runs the regular pairing (lane 0's result is
    // replaced).
    __shared__ float2 sv[33], sz[32];
    if (tid < 32) {  // warp 0 (warp-uniform branch)
      if (tid == 0) {
        if constexpr (OVP) {
          if (dN) hN = ovs[dN - 1];
        } else {
          for (int e = 0; e < (int)(dN >> 20); ++e) hN = cadd(hN, __ldcg(Zo + (dN & 0xfffff) + e));
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          sv[r] = vA[r];
          sv[16 + r] = vB[r];
        }
        sv[32] = hN;
      }
      __syncwarp();
      const int L = tid;
      const int ia = L < 16 ? L : L;                                    // H[k]
      const int ib = L == 0 ? 32 : (L < 16 ? 16 - L : 16 + 15 - (L - 16));  // H[N - k]
      float2 hk = sv[ia], hn = sv[ib];
      pack_w(hk, hn, wsp);  // twiddle of bin ksp = TASKS1 L (L < 16), TASKS1/2 + TASKS1 (L-16)
      sz[L] = hk;
      __syncwarp();
    }
    // N - (jA + TASKS1 r) = jB + TASKS1 (15 - r)
    static_for<0, 16>([&](auto Rc) {
      constexpr int r = decltype(Rc)::value;
      pack_w(vA[r], vB[15 - r], twiddle_c<r, 32, +1>(wb));
    });
    if (tid == 0) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        vA[r] = sz[r];
        vB[r] = sz[16 + r];
      }
    }
    dft<16, +1>(vA);
    dft<16, +1>(vB);
#pragma unroll
    for (int r = 0; r < 16; ++r) {  // first Stockham pass (span 1): outputs 16 j + r
      spec[padi(16 * jA + r)] = vA[r];
      spec[padi(16 * jB + r)] = vB[r];
    }
    __syncthreads();  // (the shared twiddle table is also staged by now)
  } else {
    // ---- I3b: half-spectrum bin b = slot0[b] + slot1[b] (+ its overflow run, rare); two
    // bins per thread and load (16-byte), 4 pairs in flight
    {
      const float4 *Z0 = reinterpret_cast<const float4 *>(a.stage + ul * a.zs);
      const float4 *Z1 = reinterpret_cast<const float4 *>(a.stage + ul * a.zs + a.zso);
      const float2 *Zo = a.stage + ul * a.zs + 2 * a.zso;
      const uint2 *dpos2 = reinterpret_cast<const uint2 *>(a.dpos);
      constexpr int G = 4, NP = N / 2 + 1;  // bin pairs (2i, 2i+1); the pair (N, N+1) is padded
      for (int i0 = tid; i0 < NP; i0 += G * T) {
        float4 z0[G], z1[G];
        uint2 dp[G];
  #pragma unroll
        for (int q = 0; q < G; ++q) {
          const int i = min(i0 + q * T, NP - 1);
          z0[q] = __ldcg(Z0 + i);
          z1[q] = __ldcg(Z1 + i);
          dp[q] = __ldg(dpos2 + i);
        }
  #pragma unroll
        for (int q = 0; q < G; ++q) {
          const int i = i0 + q * T;
          if (i >= NP) continue;
          float2 acc0 = make_float2(z0[q].x + z1[q].x, z0[q].y + z1[q].y);
          float2 acc1 = make_float2(z0[q].z + z1[q].z, z0[q].w + z1[q].w);
          if (dp[q].x | dp[q].y) {  // deep-overlap bins: overflow terms in order
            for (int e = 0; e < (int)(dp[q].x >> 20); ++e)
              acc0 = cadd(acc0, __ldcg(Zo + (dp[q].x & 0xfffff) + e));
            for (int e = 0; e < (int)(dp[q].y >> 20); ++e)
              acc1 = cadd(acc1, __ldcg(Zo + (dp[q].y & 0xfffff) + e));
          }
          spec[padi(2 * i)] = acc0;
          if (2 * i + 1 <= N) spec[padi(2 * i + 1)] = acc1;
        }
      }
    }
    __syncthreads();
    PHASE_MARK(1, 0);

    // ---- I4a: c2r packing  Z[k] = E[k] + i O[k],
    //   E = (H[k] + conj H[N-k])/2,  O = (H[k] - conj H[N-k]) e^{+i pi k/N} / 2
    for (int k = tid; k <= N / 2; k += T) {
      const float2 hk = spec[padi(k)];
      const float2 hn = spec[padi(N - k)];
      const float2 E = cscale(cadd(hk, cconj(hn)), 0.5f);
      const float2 D = cscale(csub(hk, cconj(hn)), 0.5f);
      const float2 w = cconj(tw_lookup(tw, k));  // e^{+i pi k/N}
      const float2 O = cmul(D, w);
      spec[padi(k)] = cadd(E, mul_si<+1>(O));  // E + iO
      if (k != 0 && k != N / 2) {
        // pair N-k: E' = conj(E), O' = conj(D) e^{-i pi k/N} = conj(O), exactly
        spec[padi(N - k)] = cadd(cconj(E), make_float2(O.y, O.x));  // conj(E) + i O'
      }
    }
    __syncthreads();

    PHASE_MARK(1, 1);
    // ---- I4b: inverse N-point FFT (unnormalised), first passes in shared memory
    pass_smem<N, CF::I1, 1, +1, T>(spec, tw);
  }
  PHASE_MARK(1, 2);
  pass_smem<N, CF::I2, CF::I1, +1, T>(spec, tw);
  PHASE_MARK(1, 3);

  // ---- last pass + I5 epilogue: z[p] -> samples 2p, 2p+1, times h~_0 / N, overlap-add
  {
    constexpr int R = CF::I3, NS = CF::I1 * CF::I2, TASKS = N / R;
    constexpr int PER = (TASKS + T - 1) / T;
    static_assert(NS * R == N, "pass plan");
    const int A = (N - a.tr) / 2, Bw = (N + a.tr) / 2;
    const float invN = 1.0f / (float)N;
    const int S = a.nslices;
    // ll / rl: resolved locally (carry); otherwise paired across CTAs through the workspace
    const bool left_paired = (a.circular || mloc > 0) && !ll;
    const bool right_paired = (a.circular || mloc + 1 < S) && !rl;
    const int bl = mloc > 0 ? mloc - 1 : S - 1;  // boundary ids (local)
    const int br = mloc;
    const int trp = a.tr;
    float *yrow = a.y + row * a.y_stride;
    float *bnd_row = a.bnd + (int64_t)row * S * 2 * trp;
    float2 v[PER][R];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = tid + q * T;
      if (TASKS % T == 0 || j < TASKS) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[q][r] = spec[padi(j + r * TASKS)];
        pass_twiddle<N, R, NS, +1>(v[q], j, tw);
        dft<R, +1>(v[q]);
      }
    }
    // stage the output frame z[p] = (f[2p], f[2p+1]) in place: the last pass's outputs
    // j + r NS are exactly the padded entries its task read (NS = N / R), so no barrier is
    // needed between the reads and the writes; then write the exclusive part and the two
    // transitions as contiguous, coalesced runs
    static_assert(NS == TASKS, "the last Stockham pass is in place");
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = tid + q * T;
      if (TASKS % T == 0 || j < TASKS) {
#pragma unroll
        for (int r = 0; r < R; ++r) spec[padi(j + r * NS)] = cscale(v[q][r], invN);
      }
    }
    __syncthreads();
    auto fr = [&](int i) {  // frame sample i
      const float2 z = spec[padi(i >> 1)];
      return (i & 1) ? z.y : z.x;
    };
    if constexpr (MODE == 1) {  // full-length synthesis: the frame is the signal
      const int cnt = (int)min((int64_t)(2 * N), a.y_len);
      for (int i = tid; i < cnt; i += T) yrow[i] = fr(i);
      (void)A; (void)Bw; (void)left_paired; (void)right_paired; (void)bl; (void)br; (void)bnd_row;
      (void)carry;
      return;
    }
    const int64_t sbase = (mg - 1) * N;  // global sample of frame index 0
    // exclusive part |t| <= A: h~_0 = 1.  Interior frames (no wrap, no trim, no spill): a
    // plain coalesced copy; the others take the per-sample index logic.
    const bool excl_direct =
        a.circular ? (sbase + N - A >= 0 && sbase + N + A < a.L && sbase + N + A < a.y_len)
                   : (sbase + N - A - a.y_base >= 0);
    if (excl_direct) {
      float *yo = yrow + (a.circular ? sbase : sbase - a.y_base);
      const int i0 = N - A;
      if (!(i0 & 1) && !(reinterpret_cast<uintptr_t>(yo + i0) & 15)) {
        // four samples per step: frame pairs z[p], z[p+1] -> one 16-byte store
        const int n4 = (2 * A + 1) >> 2;
        for (int q = tid; q < n4; q += T) {
          const int p = (i0 >> 1) + 2 * q;
          const float2 z0 = spec[padi(p)], z1 = spec[padi(p + 1)];
          *reinterpret_cast<float4 *>(yo + i0 + 4 * q) = make_float4(z0.x, z0.y, z1.x, z1.y);
        }
        for (int i = i0 + 4 * n4 + tid; i <= N + A; i += T) yo[i] = fr(i);
      } else {
        for (int i = i0 + tid; i <= N + A; i += T) yo[i] = fr(i);
      }
    } else {
      for (int i = N - A + tid; i <= N + A; i += T) {
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
    }
    // transitions, u = 0 .. tr-2 (|t| = A + 1 + u on the right, Bw - 1 - u on the left)
    for (int u = tid; u < a.tr - 1; u += T) {
      const int il = N - Bw + 1 + u;  // left: t = u - Bw + 1
      const int64_t sl = sbase + il;
      if (ll) {  // previous slice's right half (same samples: index u) + this left half
        const float v = carry[u] + __fmul_rn(fr(il), htab[Bw - 2 - u - A]);
        if (!a.circular) yrow[sl - a.y_base] = v;
        else if (sl < a.y_len) yrow[sl] = v;  // (sl in [0, L) since mloc > 0; padding dropped)
      } else {
        const float vl = fr(il) * htab[Bw - 2 - u - A];
        if (left_paired) bnd_row[((int64_t)bl * 2 + 1) * trp + u] = vl;
        else a.spill[row * a.halo + (sl - a.y_base + a.halo)] = vl;
      }
      const int ir = N + A + 1 + u;   // right: t = A + 1 + u
      const float vr = fr(ir) * htab[u];
      if (rl) carry[u] = vr;
      else if (right_paired) bnd_row[((int64_t)br * 2 + 0) * trp + u] = vr;
      else yrow[sbase + ir - a.y_base] = vr;
    }
    (void)hsm;
    // range mode, last local slice: samples [(mg+1)N - A, (mg+1)N) get no local
    // contribution; store zeros so the neighbour's spill can be added in place.
    if (!a.circular && mloc + 1 == S) {
      for (int u = tid; u < A; u += T) yrow[(mg + 1) * N - A + u - a.y_base] = 0.f;
    }
    if (!a.circular && mloc == 0) {  // spill entries no slice reaches
      for (int u = tid; u < a.halo - (Bw - 1); u += T) a.spill[row * a.halo + u] = 0.f;
    }
    PHASE_MARK(1, 4);
    if (!left_paired && !right_paired) return;  // (both sides local or unpaired)
    // ---- pairing: the second CTA to finish a boundary adds both halves (side0 + side1).
    // Release: barrier, then one thread fences (cumulative, gpu scope) and counts; acquire:
    // that thread fences after the count, then the barrier (the cooperative-groups pattern).
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
    // the partner's half from the workspace, this CTA's own half recomputed from the frame
    // (a + b is commutative in IEEE arithmetic: the sum does not depend on who is second);
    // both sides in one loop so that all partner loads of a thread are in flight together
    const bool f0 = sflag[0], f1 = sflag[1];
    if (f0 || f1) {
      const float *hp0 = bnd_row + ((int64_t)bl * 2 + 0) * trp;  // left partner's right half
      const float *hp1 = bnd_row + ((int64_t)br * 2 + 1) * trp;  // right partner's left half
      const int64_t s0 = (a.slice0 + bl) * N + A + 1, s1 = (a.slice0 + br) * N + A + 1;
      auto put = [&](int64_t s, float val) {
        if (a.circular) {
          const int64_t sw = s >= a.L ? s - a.L : s;
          if (sw < a.y_len) yrow[sw] = val;
        } else {
          yrow[s - a.y_base] = val;
        }
      };
#pragma unroll 4
      for (int u = tid; u < a.tr - 1; u += T) {
        const float p0 = f0 ? __ldcg(hp0 + u) : 0.f, p1 = f1 ? __ldcg(hp1 + u) : 0.f;
        // __fmul_rn: no contraction into an FMA with the add (the half must round as stored)
        if (f0) put(s0 + u, p0 + __fmul_rn(fr(N - Bw + 1 + u), htab[Bw - 2 - u - A]));
        if (f1) put(s1 + u, p1 + __fmul_rn(fr(N + A + 1 + u), htab[u]));
      }
    }
  }
  PHASE_MARK(1, 5);
}

template <int LOGN, int MODE = 0>
__global__ void __launch_bounds__(Big<LOGN>::T, Big<LOGN>::MINB) slicq_inv_spec_kernel(const KArgs a) {
  using CF = Big<LOGN>;
  constexpr int N = CF::N, T = CF::T;
  extern __shared__ float4 smem4[];
  float2 *spec = reinterpret_cast<float2 *>(smem4);
  float2 *tw = spec + spec_entries<LOGN>();
  float *htab = reinterpret_cast<float *>(tw + tw_entries<LOGN>());
  const int tid = threadIdx.x;
  for (int i = tid; i < tw_entries<LOGN>(); i += T) tw[i] = a.tw2n[i];
  if constexpr (MODE == 0)
    for (int u2 = tid; u2 < a.tr - 1; u2 += T)
      htab[u2] = __ldg(a.h0dual + N + (N - a.tr) / 2 + 1 + u2);
  pdl_wait();  // contributions of this chunk come from the channel kernel
  prefetch_l2(a.stage + (int64_t)blockIdx.x * a.zs, a.zs * 8, tid, T);
  inv_unit<LOGN, MODE>(a, spec, tw, htab, nullptr, blockIdx.x, false, false);
  pdl_trigger();
}

// Persistent variant (MODE 0): CTA c handles the contiguous units [c U / G, (c+1) U / G) of the
// chunk; tw and htab are staged once, the next unit's slots are prefetched to L2 while this one
// is synthesised, and the overlap of consecutive slices of one row handled by the same CTA is
// added on chip (carry) instead of through the workspace pairing.
template <int LOGN>
__global__ void __launch_bounds__(Big<LOGN>::T, Big<LOGN>::MINB) slicq_inv_spec_persist_kernel(const KArgs a) {
  using CF = Big<LOGN>;
  constexpr int N = CF::N, T = CF::T;
  extern __shared__ float4 smem4[];
  float2 *spec = reinterpret_cast<float2 *>(smem4);
  float2 *tw = spec + spec_entries<LOGN>();
  float *htab = reinterpret_cast<float *>(tw + tw_entries<LOGN>());
  float *carry = htab + ((a.tr + 3) & ~3);
  float2 *ovs = reinterpret_cast<float2 *>(carry + ((a.tr + 3) & ~3));  // overflow-bin sums
  const int tid = threadIdx.x;
  for (int i = tid; i < tw_entries<LOGN>(); i += T) tw[i] = a.tw2n[i];
  for (int u2 = tid; u2 < a.tr - 1; u2 += T) htab[u2] = __ldg(a.h0dual + N + (N - a.tr) / 2 + 1 + u2);
  pdl_wait();  // contributions of this chunk come from the channel kernel
  const int64_t G = gridDim.x;
  const int64_t ub = blockIdx.x * (int64_t)a.nunits / G, ue = (blockIdx.x + 1) * (int64_t)a.nunits / G;
  if (a.pf && ub < ue) prefetch_l2(a.stage + ub * a.zs, a.zs * 8, tid, T);
  __syncthreads();
  for (int64_t ul = ub; ul < ue; ++ul) {
    const int64_t u = a.unit0 + ul;
    const int mloc = (int)(u - unit_row(u, a.nslices) * a.nslices);
    const bool ll = ul > ub && mloc > 0;                    // unit ul - 1 is slice mloc - 1
    const bool rl = ul + 1 < ue && mloc + 1 < a.nslices;  // unit ul + 1 is slice mloc + 1
    if (a.pf && ul + 1 < ue) {  // 1: per-line prefetches by all threads; 2: one bulk prefetch
      if (a.pf == 2) {
        if (tid == 0) prefetch_l2_bulk(a.stage + (ul + 1) * a.zs, a.zs * 8);
      } else {
        prefetch_l2(a.stage + (ul + 1) * a.zs, a.zs * 8, tid, T);
      }
    }
    constexpr bool fused1 = CF::I1 == 16 && N / 16 == 2 * T;  // (the pre-pass needs it)
    inv_unit<LOGN, 0, fused1 && SLICQ_OVP>(a, spec, tw, htab, carry, ul, ll, rl, ovs,
                                           SLICQ_OV_ASYNC && ul > ub, SLICQ_OV_ASYNC && ul + 1 < ue);
    __syncthreads();  // (spec, carry and ovs reused by the next unit)
  }
  pdl_trigger();
}

template <int LOGN>
constexpr size_t spec_smem_bytes(int tr) {
  return sizeof(float2) * (size_t)(spec_entries<LOGN>() + tw_entries<LOGN>()) +
         sizeof(float) * (size_t)((tr + 3) & ~3);
}
// the persistent inverse spectrum kernel adds the overlap carry (tr floats)
template <int LOGN>
constexpr size_t spec_persist_smem_bytes(int tr) {
  return spec_smem_bytes<LOGN>(tr) + sizeof(float) * (size_t)((tr + 3) & ~3);
}

// Per-size entry points (defined in kernels_l<LOGN>.cu)
template <int LOGN>
int phase_times(unsigned long long *out32, int reset);
template <int LOGN>
int set_attrs(size_t smem);
template <int LOGN>
cudaError_t launch_fwd_spec(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s, bool pdl,
                            int mode = 0);
template <int LOGN>
cudaError_t launch_inv_spec(const KArgs &a, dim3 grid, size_t smem, cudaStream_t s, bool pdl,
                            int mode = 0);
template <int LOGN>
cudaError_t launch_inv_spec_persist(const KArgs &a, size_t smem, cudaStream_t s, bool pdl,
                                    int *grid_out);
template <int LOGN>
cudaError_t launch_fwd_spec_persist(const KArgs &a, size_t smem, cudaStream_t s, bool pdl);

}  // namespace kern
}  // namespace slicq
