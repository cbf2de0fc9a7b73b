// Channel kernels with TMA staging of their HBM operands (round 2).
//
// The split design's channel kernels (kernels_dev.cuh) spend most of their stall cycles on
// the first use of a task's global loads (ncu source view, cfg4: 45 % of the forward
// kernel's samples are the fold's gathers from the staged spectrum X, 71 % of the inverse
// kernel's are long_scoreboard on the coefficient loads).  A warp's loads are issued only
// when its task starts, and the arithmetic of the task cannot begin before they land.
//
// Here every warp owns a shared-memory buffer and an mbarrier.  The operand block of a task
// is contiguous per unit -- forward: the bins [xlo, xhi] of X that the packet's channels
// read (the band of the channels), inverse: the coefficient columns of the
// packet's channels c^m_k -- so lane 0 moves it with one TMA bulk copy per unit
// (cp.async.bulk global -> shared, completion counted in the mbarrier's transaction bytes).
// The copy of the warp's NEXT task is issued as soon as the current task's operands are in
// registers, so it is in flight during the current task's DFTs, twiddles and stores; the
// fold / coefficient loads then read shared memory (no index-dependent HBM latency).  The
// arithmetic, the element tables and the output layout are those of kernels_dev.cuh: the
// results are bit-identical (tests/test_gpu_parity.py compares both builds).
#pragma once
#include "kernels_dev.cuh"

namespace slicq {
namespace kern {

__device__ __forceinline__ uint32_t tb_smem(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tb_bar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tb_smem(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// the single arrival of a phase, announcing the bytes its copies will deliver
__device__ __forceinline__ void tb_expect(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tb_smem(bar)),
               "r"(bytes)
               : "memory");
}
// bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void tb_copy(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tb_smem(dst)),
      "l"(src), "r"(bytes), "r"(tb_smem(bar))
      : "memory");
}
__device__ __forceinline__ void tb_wait(uint64_t *bar, unsigned parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(tb_smem(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// A persistent channel-kernel work item (packet, tile of units), in the order of
// kernels_dev.cuh (packet-major inside super-tiles of tiles).
struct ChanItem {
  int pk, u_lo, u_hi, nu;
};
__device__ __forceinline__ ChanItem chan_item(const KArgs &a, int item, int ntiles) {
  const int sts = a.stiles > 0 ? a.stiles : ntiles;
  const int per_st = a.npackets * sts;
  const int st = item / per_st, rem = item - st * per_st;
  const int st_n = min(sts, ntiles - st * sts);
  ChanItem it;
  it.pk = rem / st_n;
  const int tile = st * sts + (rem - it.pk * st_n);
  it.u_lo = tile * a.tile;
  it.u_hi = min(a.nunits, it.u_lo + a.tile);
  it.nu = __ldg(&a.packets[it.pk].nu);
  return it;
}
// The warp's task sequence: items blockIdx.x + i gridDim.x, tasks warp, warp + NW, ... of each
// (task t covers units u_lo + t nu ..).  Advance (item, t) to the warp's next task
// (item >= nitems: none left).
template <int NW>
__device__ __forceinline__ void chan_next(const KArgs &a, int nitems, int ntiles, int warp,
                                          int &item, int &t, ChanItem &it) {
  t += NW;
  while (item < nitems && t * it.nu >= it.u_hi - it.u_lo) {
    item += gridDim.x;
    t = warp;
    if (item < nitems) it = chan_item(a, item, ntiles);
  }
}

// Forward operand block of a task: bins [b0, b0 + W) of each unit's staged X, b0 = xlo & ~1,
// W = ((xhi + 2) & ~1) - b0 (16-byte granules), unit u at buf[u W].
__device__ __forceinline__ void fwd_tb_band(const PacketDev *P, int &b0, int &W) {
  b0 = __ldg(&P->xlo) & ~1;
  W = ((__ldg(&P->xhi) + 2) & ~1) - b0;
}
// (plain pointer / scalar arguments: a lambda holding a reference to the kernel parameter
// block would force a local copy of it)
__device__ __forceinline__ void fwd_tb_issue(const PacketDev *packets, const float2 *stage, int64_t xs,
                                             const ChanItem &it, int t, float2 *buf, uint64_t *bar) {
  int b0, W;
  fwd_tb_band(packets + it.pk, b0, W);
  const int g0 = it.u_lo + t * it.nu, nuu = min(it.nu, it.u_hi - g0);
  tb_expect(bar, (unsigned)(nuu * W * 8));
  for (int u = 0; u < nuu; ++u)
    tb_copy(buf + u * W, stage + (int64_t)(g0 + u) * xs + b0, (unsigned)(W * 8), bar);
}
// Inverse operand block: coefficient columns [c0, c0 + W) of each unit's row (the packet's
// channels are consecutive columns), c0 = off_first & ~1, W = ((off_last + M + 1) & ~1) - c0.
__device__ __forceinline__ void inv_tb_cols(const ChanDev *chan, const int32_t *pchans,
                                            const PacketDev *P, int &c0, int &W) {
  const int nch = __ldg(&P->nch), co = __ldg(&P->chan_off), mm = __ldg(&P->m1m2);
  const int M = (mm & 255) * ((mm >> 8) & 255);
  const int first = __ldg(&chan[__ldg(pchans + co)].off);
  const int last = __ldg(&chan[__ldg(pchans + co + nch - 1)].off);
  c0 = first & ~1;
  W = ((last + M + 1) & ~1) - c0;
}
__device__ __forceinline__ void inv_tb_issue(const ChanDev *chan, const int32_t *pchans,
                                             const PacketDev *packets, const float2 *coef_row0,
                                             int64_t C, const ChanItem &it, int t, float2 *buf,
                                             uint64_t *bar) {
  int c0, W;
  inv_tb_cols(chan, pchans, packets + it.pk, c0, W);
  const int g0 = it.u_lo + t * it.nu, nuu = min(it.nu, it.u_hi - g0);
  tb_expect(bar, (unsigned)(nuu * W * 8));
  for (int u = 0; u < nuu; ++u)
    tb_copy(buf + u * W, coef_row0 + (g0 + u) * C + c0, (unsigned)(W * 8), bar);
}

// ---- forward codelets reading the fold's bins from the warp's buffer (Xs[u W + bin - b0]);
// `after` runs once every lane holds its operands (it issues the next task's copy).
template <int M1, int V, class F>
__device__ __forceinline__ void fwd_step1f_tb(const uint2 *ent, const float2 *Xs, int W, int r,
                                              unsigned magc, const float2 *twM, float2 *reg, int m2,
                                              int nch, unsigned mag2, int twoff_lane, int lane,
                                              const F &after) {
  const int nt = nch * m2;
  const bool act = lane < nt;
  const int ci = act ? (lane * (int)mag2) >> 16 : 0;
  const int p2 = act ? lane - ci * m2 : 0;
  const int twoff = __shfl_sync(FULL, twoff_lane, ci);
  const int u = (ci * (int)magc) >> 16, c = ci - u * r;
  const int M = M1 * m2;
  const uint2 *e0 = ent + c * M + p2;
  const float2 *Xu = Xs + u * W;
  // every lane loads (inactive lanes: valid entries of task 0, results unused): a load under
  // `if (act)` ahead of the warp-synchronous issue measured 1.1 KB of register spills
  float2 v[M1];
  {
#pragma unroll
    for (int p1 = 0; p1 < M1; ++p1) {
      const uint2 en = __ldg(e0 + m2 * p1);
      const float2 xv = Xu[en.x & 0x3ffff];
      const float gv = __uint_as_float(en.y);  // sign bit: conjugate X (g >= 0)
      v[p1] = make_float2(xv.x * fabsf(gv), xv.y * gv);
    }
  }
  after();
  if (!act) return;
  dft<M1, +1>(v);
  chan_twiddle<M1, +1>(v, p2, M, twM + twoff);
  const int S2 = m2 | 1;
  float2 *base = reg + ci * M1 * S2;
#pragma unroll
  for (int n1 = 0; n1 < M1; ++n1) base[n1 * S2 + p2] = v[n1];
}
template <int M, int V, class F>
__device__ __forceinline__ void fwd_small_tb(const uint2 *ent, const float2 *Xs, float2 *out_row,
                                             bool act, int off_lane, const F &after) {
  float2 v[M];
  {  // every lane loads (inactive lanes read valid buffer entries; results unused)
#pragma unroll
    for (int p = 0; p < M; ++p) {
      const uint2 e = __ldg(ent + p * 32);
      const float2 xv = Xs[e.x];
      const float gv = __uint_as_float(e.y);  // sign bit: conjugate X (g >= 0)
      v[p] = make_float2(xv.x * fabsf(gv), xv.y * gv);
    }
  }
  after();
  if (!act) return;
  dft<M, +1>(v);
  float2 *o = out_row + off_lane;
#pragma unroll
  for (int n = 0; n < M; ++n) SLICQ_CSTORE(o + n, v[n]);
}

// ---- inverse codelets reading the coefficients from the warp's buffer
template <int M1, int V, class F>
__device__ __forceinline__ void inv_step1_tb(const float2 *twM, const float2 *in_s, float2 *reg,
                                             int m2, int nch, unsigned mag2, int off_lane,
                                             int twoff_lane, int lane, const F &after) {
  const int nt = nch * m2;
  const bool act = lane < nt;
  const int ci = act ? (lane * (int)mag2) >> 16 : 0;
  const int p2 = act ? lane - ci * m2 : 0;
  const int off = __shfl_sync(FULL, off_lane, ci), twoff = __shfl_sync(FULL, twoff_lane, ci);
  float2 v[M1];
  {  // every lane loads (inactive lanes: channel 0's column 0; results unused)
    const float2 *src = in_s + off + p2;
#pragma unroll
    for (int p1 = 0; p1 < M1; ++p1) v[p1] = src[p1 * m2];
  }
  after();
  if (!act) return;
  dft<M1, -1>(v);
  chan_twiddle<M1, -1>(v, p2, M1 * m2, twM + twoff);
  const int S2 = m2 | 1;
  float2 *A = reg + ci * M1 * S2 + p2;
#pragma unroll
  for (int n1 = 0; n1 < M1; ++n1) A[n1 * S2] = v[n1];
}
template <int M, int V, class F>
__device__ __forceinline__ void inv_small_tb(const float2 *in_s, float2 *reg, int nvc, int nv,
                                             int off_lane, int lane, const F &after) {
  float2 v[M];
  const bool act = lane < nvc;
  {  // every lane loads (inactive lanes read valid buffer entries; results unused)
    const float2 *src = in_s + off_lane;
#pragma unroll
    for (int n = 0; n < M; ++n) v[n] = src[n];
  }
  after();
  if (!act) return;
  dft<M, -1>(v);
#pragma unroll
  for (int q = 0; q < M; ++q) reg[q * nv + lane] = v[q];
}

#ifdef SLICQ_DEFINE_CHAN_KERNELS
// The warp's task cursor lives in shared memory (lane 0 advances it; warp-uniform values
// would otherwise stay live in registers across the inlined codelets): cur = the task being
// computed, nxt = the task whose operands are being copied.
struct TbCursor {
  int item, t;
  ChanItem it;
};
template <int NW>
__device__ __forceinline__ void tb_cursor_first(const KArgs &a, int nitems, int ntiles, int warp,
                                                TbCursor &c) {
  c.item = blockIdx.x;
  c.t = warp - NW;
  if (c.item < nitems) c.it = chan_item(a, c.item, ntiles);
  chan_next<NW>(a, nitems, ntiles, warp, c.item, c.t, c.it);
}

// `after` of the codelets: once the warp's operands are in registers, lane 0 issues the copy
// of the next task into the buffer (a functor with a force-inlined call operator: an
// out-of-line call would spill the codelet's live registers around it)
struct FwdTbNext {
  int lane, nitems;
  const TbCursor *nxt;
  float2 *buf;
  uint64_t *bar;
  const PacketDev *packets;
  const float2 *stage;
  int64_t xs;
  __device__ __forceinline__ void operator()() const {
    __syncwarp();
    if (lane == 0 && nxt->item < nitems) fwd_tb_issue(packets, stage, xs, nxt->it, nxt->t, buf, bar);
  }
};
struct InvTbNext {
  int lane, nitems;
  const TbCursor *nxt;
  float2 *buf;
  uint64_t *bar;
  const ChanDev *chan;
  const int32_t *pchans;
  const PacketDev *packets;
  const float2 *crow0;
  int64_t C;
  __device__ __forceinline__ void operator()() const {
    __syncwarp();
    if (lane == 0 && nxt->item < nitems)
      inv_tb_issue(chan, pchans, packets, crow0, C, nxt->it, nxt->t, buf, bar);
  }
};

// Shared memory: [NW warps x scr scratch][NW warps x tbe buffer][NW mbarriers][NW x 2 cursors].
template <int MAXS, int MINB>
__global__ void __launch_bounds__(CHAN_T, MINB) slicq_fwd_chan_tb_kernel(const KArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int NW = CHAN_T / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2 *sm = reinterpret_cast<float2 *>(smem4);
  float2 *scr = sm + warp * a.scr;
  float2 *buf = sm + NW * a.scr + warp * a.tbe;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + NW * (a.scr + a.tbe)) + warp;
  TbCursor *cur = reinterpret_cast<TbCursor *>(sm + NW * (a.scr + a.tbe + 1)) + 2 * warp;
  TbCursor *nxt = cur + 1;
  const int ntiles = (a.nunits + a.tile - 1) / a.tile;
  const int nitems = a.npackets * ntiles;
  if (lane == 0) tb_bar_init(bar);
  pdl_wait();
  if (lane == 0) {
    tb_cursor_first<NW>(a, nitems, ntiles, warp, *cur);
    if (cur->item < nitems) fwd_tb_issue(a.packets, a.stage, a.xs, cur->it, cur->t, buf, bar);
  }
  __syncwarp();
  unsigned ph = 0;
  int pk_cur = -1;
  int c_l = 0, u_l = 0, c_off = 0, c_twoff = 0, b0 = 0, W = 0;
  int m1 = 0, m2 = 0, r = 0;
  bool small = false;
  unsigned magc = 0, mag1 = 0, mag2 = 0;
  const uint2 *ent = nullptr;
  while (cur->item < nitems) {
    const int pk = cur->it.pk;
    if (pk != pk_cur) {  // the packet's lane mapping (as kernels_dev.cuh)
      pk_cur = pk;
      const PacketDev *P = a.packets + pk;
      const int mm = __ldg(&P->m1m2), nu = __ldg(&P->nu);
      m1 = mm & 255;
      m2 = (mm >> 8) & 255;
      small = (mm >> 17) & 1;
      r = __ldg(&P->nch);
      magc = __ldg(&P->magc);
      mag1 = __ldg(&P->mag1);
      mag2 = __ldg(&P->mag2);
      const int vcl = lane < nu * r ? lane : 0;
      u_l = (vcl * (int)magc) >> 16;
      c_l = vcl - u_l * r;
      const int ck = __ldg(a.pchans + __ldg(&P->chan_off) + c_l);
      c_off = __ldg(&a.chan[ck].off) + u_l * (int)a.C;
      c_twoff = __ldg(&a.chan[ck].twoff);
      ent = a.fent + __ldg(&P->fent_off);
      fwd_tb_band(P, b0, W);
    }
    const int g0 = cur->it.u_lo + cur->t * cur->it.nu;
    const int nvc = min(cur->it.nu, cur->it.u_hi - g0) * r;
    float2 *out_row = a.coef_out + (a.unit0 + g0) * a.C;
    if (lane == 0) {
      *nxt = *cur;
      chan_next<NW>(a, nitems, ntiles, warp, nxt->item, nxt->t, nxt->it);
    }
    tb_wait(bar, ph);
    ph ^= 1;
    const float2 *Xs = buf - b0;
    const PacketDev *packets = a.packets;
    const float2 *stage = a.stage;
    const int64_t xs = a.xs;
    const FwdTbNext after{lane, nitems, nxt, buf, bar, packets, stage, xs};
    if (small) {
      switch (m1) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) fwd_small_tb<S, MAXS>(ent + c_l, Xs + u_l * W, out_row, lane < nvc, c_off, after); break;
        SLICQ_SMALL(X_)
#undef X_
      }
    } else {
      switch (m1) {
#define X_(S)                                                                                    \
  case S:                                                                                        \
    if constexpr (S <= MAXS)                                                                     \
      fwd_step1f_tb<S, MAXS>(ent, Xs, W, r, magc, a.twM, scr, m2, nvc, mag2, c_twoff, lane, after); \
    break;
        SLICQ_SIZES(X_)
#undef X_
      }
      __syncwarp();
      switch (m2) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) fwd_step2<S, MAXS>(scr, out_row, m1, nvc, mag1, c_off, lane); break;
        SLICQ_SIZES(X_)
#undef X_
      }
    }
    __syncwarp();
    if (lane == 0) *cur = *nxt;
    __syncwarp();
  }
  pdl_trigger();
}

template <int MAXS, int MINB>
__global__ void __launch_bounds__(CHAN_T, MINB) slicq_inv_chan_tb_kernel(const KArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int NW = CHAN_T / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2 *sm = reinterpret_cast<float2 *>(smem4);
  float2 *scr = sm + warp * a.scr;
  float2 *buf = sm + NW * a.scr + warp * a.tbe;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + NW * (a.scr + a.tbe)) + warp;
  TbCursor *cur = reinterpret_cast<TbCursor *>(sm + NW * (a.scr + a.tbe + 1)) + 2 * warp;
  TbCursor *nxt = cur + 1;
  const int ntiles = (a.nunits + a.tile - 1) / a.tile;
  const int nitems = a.npackets * ntiles;
  if (lane == 0) tb_bar_init(bar);
  pdl_wait();
  if (lane == 0) {
    tb_cursor_first<NW>(a, nitems, ntiles, warp, *cur);
    if (cur->item < nitems)
      inv_tb_issue(a.chan, a.pchans, a.packets, a.coef_in + a.unit0 * a.C, a.C, cur->it, cur->t, buf, bar);
  }
  __syncwarp();
  unsigned ph = 0;
  int pk_cur = -1;
  int s_off = 0, c_twoff = 0, m1 = 0, m2 = 0, r = 0, nu = 0, ne = 0, ustride = 0;
  bool small = false;
  unsigned mag1 = 0, mag2 = 0;
  const uint2 *ent = nullptr;
  while (cur->item < nitems) {
    const int pk = cur->it.pk;
    if (pk != pk_cur) {  // the packet's lane mapping (as kernels_dev.cuh)
      pk_cur = pk;
      const PacketDev *P = a.packets + pk;
      const int mm = __ldg(&P->m1m2);
      m1 = mm & 255;
      m2 = (mm >> 8) & 255;
      small = (mm >> 17) & 1;
      r = __ldg(&P->nch);
      nu = __ldg(&P->nu);
      ne = __ldg(&P->nz);
      ustride = __ldg(&P->ustride);
      mag1 = __ldg(&P->mag1);
      mag2 = __ldg(&P->mag2);
      const unsigned magc = __ldg(&P->magc);
      const int vcl = lane < nu * r ? lane : 0;
      const int u_l = (vcl * (int)magc) >> 16, c_l = vcl - u_l * r;
      const int ck = __ldg(a.pchans + __ldg(&P->chan_off) + c_l);
      int c0, W;
      inv_tb_cols(a.chan, a.pchans, P, c0, W);
      s_off = u_l * W + __ldg(&a.chan[ck].off) - c0;  // the lane's channel in the buffer
      c_twoff = __ldg(&a.chan[ck].twoff);
      ent = a.ient + __ldg(&P->ient_off);
    }
    const int g0 = cur->it.u_lo + cur->t * nu;
    const int nuu = min(nu, cur->it.u_hi - g0);
    const int nvc = nuu * r;
    if (lane == 0) {
      *nxt = *cur;
      chan_next<NW>(a, nitems, ntiles, warp, nxt->item, nxt->t, nxt->it);
    }
    tb_wait(bar, ph);
    ph ^= 1;
    const ChanDev *chan = a.chan;
    const int32_t *pchans = a.pchans;
    const PacketDev *packets = a.packets;
    const float2 *crow0 = a.coef_in + a.unit0 * a.C;
    const int64_t C = a.C;
    const InvTbNext after{lane, nitems, nxt, buf, bar, chan, pchans, packets, crow0, C};
    if (small) {
      switch (m1) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) inv_small_tb<S, MAXS>(buf, scr, nvc, (nu * r) | 1, s_off, lane, after); break;
        SLICQ_SMALL(X_)
#undef X_
      }
    } else {
      switch (m1) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) inv_step1_tb<S, MAXS>(a.twM, buf, scr, m2, nvc, mag2, s_off, c_twoff, lane, after); break;
        SLICQ_SIZES(X_)
#undef X_
      }
      __syncwarp();
      switch (m2) {
#define X_(S) \
  case S: if constexpr (S <= MAXS) inv_step2<S, MAXS>(scr, m1, nvc, mag1, lane); break;
        SLICQ_SIZES(X_)
#undef X_
      }
    }
    __syncwarp();
    // I3a terms -> their slots of the unit's half-spectrum staging (as kernels_dev.cuh)
    for (int u = 0; u < nuu; ++u) {
      float2 *Zb = opaque(a.stage + (int64_t)(g0 + u) * a.zs);  // 32-bit indexing
      const float2 *su = scr + u * ustride;
      SLICQ_UNROLL(SLICQ_FOLD_UNROLL)
      for (int e = lane; e < ne; e += 32) {
        const uint2 en = __ldg(ent + e);
        const float2 f = su[en.x & 0x3fff];
        const float w = __uint_as_float(en.y);  // sign bit: conjugate the term (g~ >= 0)
        SLICQ_ZSTORE(Zb + (en.x >> 14), make_float2(f.x * fabsf(w), f.y * w));
      }
    }
    __syncwarp();
    if (lane == 0) *cur = *nxt;
    __syncwarp();
  }
  pdl_trigger();
}
#endif  // SLICQ_DEFINE_CHAN_KERNELS

}  // namespace kern
}  // namespace slicq
