// Ring kernels for sm_100a: one persistent cooperative launch per call with two CTA roles
// sharing every SM, joined by an L2-resident ring of slice spectra (no HBM staging).
// DESIGN.md "Ring kernels" describes the design; step names follow SURVEY.md §8(a).
//
//   forward  slicq_fwd_ring_kernel<LOGN>
//     spectrum CTAs   unit u (row, slice), in order: F1 + F2 (fwd_spectrum, kernels_dev.cuh)
//                     -> X[0..N] into ring slot u mod R, then publish ready[slot] = u + 1
//
//     channel CTAs    one frequency band (a contiguous run of channels) each; a loader warp
//                     pulls the band's bins of bt consecutive units from the ring into shared
//                     memory with TMA bulk copies (double-buffered, mbarrier-tracked) and
//                     releases the slots; the compute warps run the band's warp tasks:
//                     F3 band x g_k read contiguously, F4 IFFT_{M_k} (whole DFT per lane, or
//                     a four-step M1 x M2 whose twiddles / second-step index absorb the
//                     rotation by lo_k, C5), F5 coefficients stored once
//
// A band runs only its own channels' code (a few shapes: instruction-cache locality), keeps
// its filter weights and twiddles in shared memory, and amortises every table over bt units.
// The ring holds at most R spectra (R * (N + 2) * 8 bytes, sized to stay in L2): a spectrum
// CTA reuses slot u mod R only after every band has released unit u - R.  All waits are
// bounded (about 2 s, then __trap: a launch error instead of a hang).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_dev.cuh"
#include "kernels_fused.cuh"

namespace slicq {
namespace kern {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add_u32(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr uint64_t kRingTimeoutNs = 2000000000ull;  // 2 s
// spin (one thread) until *p >= want; bounded
__device__ __forceinline__ void ring_wait_ge(const unsigned *p, unsigned want, unsigned *err,
                                             unsigned code) {
  if (ld_acquire_u32(p) >= want) return;
  const uint64_t t0 = globaltimer_ns();
  unsigned ns = 32;
  while (ld_acquire_u32(p) < want) {
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : ns;
    if (globaltimer_ns() - t0 > kRingTimeoutNs) {
      atomicExch(err, code);
      __trap();
    }
  }
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity, unsigned *err, unsigned code) {
  if (mbar_try(bar, parity)) return;
  const uint64_t t0 = globaltimer_ns();
  while (!mbar_try(bar, parity)) {
    if (globaltimer_ns() - t0 > kRingTimeoutNs) {
      atomicExch(err, code);
      __trap();
    }
  }
}
// TMA bulk copy global -> shared (bytes % 16 == 0, both addresses 16-byte aligned), completion
// counted on the mbarrier's transaction bytes
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------ ring tables
// (RBand, RTask: slicq_internal.h)
// v[n1] *= e^{SIGN 2 pi i p2 n1 / M}, n1 = 1..M1-1, from a shared-memory table e^{+2 pi i t/M}
// (chan_twiddle with plain shared loads)
template <int M1, int SIGN>
__device__ __forceinline__ void chan_twiddle_s(float2 (&v)[M1], int p2, int M, const float2 *tab) {
  if constexpr (M1 > 1) {
    float2 w1 = tab[p2];
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
        w4q = tab[e4];
        if (SIGN < 0) w4q = cconj(w4q);
      }
      const float2 ws = s == 1 ? w1 : (s == 2 ? w2 : w3);
      const float2 w = s == 0 ? w4q : (n1 < 4 ? ws : cmul(w4q, ws));
      v[n1] = cmul(v[n1], w);
    }
  }
}

struct RArgs {
  float2 *ring;            // R slots of slot_entries float2
  int grp;                 // batches per channel item
  int meta;                // bytes of the largest band metadata block
  int64_t slot_entries;
  unsigned *ready;         // [R] forward: u + 1 once slot u mod R holds unit u
  unsigned *done;          // [R] cumulative band releases of the slot
  unsigned *err;           // timeout code (then __trap)
  int R;
  int nb, bt, la;          // bands, units per channel item, work-queue lookahead (batches)
  const RBand *band;
  const RTask *task;
  const FChan *fch;        // goff / twoff relative to the band's shared copies
  const float2 *btw;       // per-band twiddle tables e^{+2 pi i t / M}
  const int32_t *round;    // per-band round lists
  int xstride;             // float2 entries per unit in a band buffer (>= every bspan)
  int wmax, twmax;         // largest band weight / twiddle count (16-byte padded)
  int iscr;                // item scratch (float2)
  unsigned long long *qctr;   // work-queue claim counter
  unsigned long long *stats;  // optional (dev): per CTA [spectrum ns, channel ns, wait ns, -]
  int ngrid;               // CTAs of the launch
};

constexpr int RING_T = 256;              // threads per CTA
constexpr int RING_W = RING_T / 32;      // warps

// channel-item shared memory inside the union region: the band's metadata (tasks, channel
// descriptors, rounds), weights and twiddles, two X buffer sets (bins of bt units each: one
// batch computes while the next lands), then the item scratch
struct ChanSmem {
  size_t meta, w, tw, set[2], scr, total;
};
__host__ __device__ inline ChanSmem chan_smem_layout(int bt, int xstride, int wmax, int twmax,
                                                     int iscr, int meta) {
  ChanSmem s{};
  s.meta = 0;
  s.w = (size_t)((meta + 15) & ~15);
  s.tw = s.w + sizeof(float) * (size_t)((wmax + 3) & ~3);
  s.set[0] = (s.tw + sizeof(float2) * (size_t)((twmax + 1) & ~1) + 15) & ~size_t(15);
  s.set[1] = s.set[0] + sizeof(float2) * (size_t)bt * xstride;
  s.scr = s.set[1] + sizeof(float2) * (size_t)bt * xstride;
  s.total = s.scr + sizeof(float2) * (size_t)iscr;
  return s;
}

// a channel descriptor from shared memory
__device__ __forceinline__ FChan ld_fchan_s(const FChan *p) {
  const int4 *q = reinterpret_cast<const int4 *>(p);
  const int4 a = q[0], b = q[1], c = q[2];
  FChan f;
  f.lo = a.x; f.len = a.y; f.M = a.z; f.goff = a.w;
  f.off = b.x; f.twoff = b.y; f.lo_mod = b.z; f.lom2 = b.w;
  f.d0 = c.x; f.d1 = c.y; f.ovoff = c.z; f.flags = c.w;
  return f;
}

// ------------------------------------------------------------------ channel-item codelets
// (one lane item each; the phases distribute 32-lane rounds over the warps)
// X(j) of unit buffer Xu (bins blo ..): contiguous for interior channels, else the real-input
// mirror (C15)
template <int N, bool INTER>
__device__ __forceinline__ float2 xb_at(const float2 *Xu, int j, int blo) {
  if constexpr (INTER) {
    return Xu[j - blo];
  } else {
    const int jj = j < 0 ? j + 2 * N : j;
    const bool up = jj > N;
    const float2 v = Xu[(up ? 2 * N - jj : jj) - blo];
    return make_float2(v.x, up ? -v.y : v.y);
  }
}

// small task, lane item i = (unit sp, channel c): buf[p] = y[(p - lo) mod M] (the fold of
// P:193), DFT_M (sign +), 16-byte coefficient stores                    (F3 - F5)
template <int M, int N, bool INTER>
__device__ __forceinline__ void rf_small(const KArgs &a, const RArgs &r, const RTask &tk, int i,
                                         int nsb, int64_t ubase, const float2 *Xb, int blo,
                                         const float *wsm, const FChan *fchs) {
  if (i >= r.bt * tk.nch) return;
  const int sp = (int)(((unsigned)i * tk.magPa) >> 16), c = i - sp * tk.nch;
  if (sp >= nsb) return;
  const FChan ch = ld_fchan_s(fchs + tk.coff + c);
  const float2 *Xu = Xb + sp * r.xstride;
  const float *g = wsm + ch.goff;
  float2 v[M];
#pragma unroll
  for (int p = 0; p < M; ++p) {
    int d = p - ch.lo_mod;
    d += d < 0 ? M : 0;
    const bool in = d < ch.len;
    const float w = in ? g[d] : 0.f;
    const float2 x = in ? xb_at<N, INTER>(Xu, ch.lo + d, blo) : make_float2(0.f, 0.f);
    v[p] = make_float2(x.x * w, x.y * w);
  }
  dft<M, +1>(v);
  float2 *o = a.coef_out + (ubase + sp) * a.C + ch.off;
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

// two-step task, step 1, lane item i = (unit sp, channel c, column d2): y[M2 d1 + d2] of the
// contiguous support, DFT_M1 (sign +), twiddle w^{(d2 + lo) n1}, stored at
// A[sp][c][n1][(d2 + lo) mod M2] (stride S2 = M2 | 1: conflict-free both ways)   (F3, F4)
template <int M1, int N, bool INTER>
__device__ __forceinline__ void rf_s1(const RArgs &r, const RTask &tk, int i, int nsb,
                                      const float2 *Xb, int blo, const float *wsm,
                                      const float2 *twsm, float2 *scr, const FChan *fchs) {
  const int m2 = (tk.code >> 8) & 255;
  const int per = tk.nch * m2;
  if (i >= r.bt * per) return;
  const int sp = (int)(((unsigned)i * tk.magPa) >> 16), rem = i - sp * per;
  const int c = (int)(((unsigned)rem * tk.magM2) >> 16), d2 = rem - c * m2;
  if (sp >= nsb) return;
  const FChan ch = ld_fchan_s(fchs + tk.coff + c);
  const float2 *Xu = Xb + sp * r.xstride;
  const float *g = wsm + ch.goff + d2;
  float2 v[M1];
#pragma unroll
  for (int d1 = 0; d1 < M1; ++d1) {
    const int d = d1 * m2 + d2;
    const bool in = d < ch.len;
    const float w = in ? g[d1 * m2] : 0.f;
    const float2 x = in ? xb_at<N, INTER>(Xu, ch.lo + d, blo) : make_float2(0.f, 0.f);
    v[d1] = make_float2(x.x * w, x.y * w);
  }
  dft<M1, +1>(v);
  int e = d2 + ch.lo_mod;
  e -= e >= ch.M ? ch.M : 0;
  chan_twiddle_s<M1, +1>(v, e, ch.M, twsm + ch.twoff);
  int e2 = d2 + ch.lom2;
  e2 -= e2 >= m2 ? m2 : 0;
  const int S2 = m2 | 1;
  float2 *A = scr + tk.soff + (sp * tk.nch + c) * M1 * S2 + e2;
#pragma unroll
  for (int n1 = 0; n1 < M1; ++n1) A[n1 * S2] = v[n1];
}

// two-step task, step 2, lane item i = (unit sp, channel c, row n1): DFT_M2 (sign +) over the
// rotated column -> c[n1 + M1 n2], coalesced over n1                     (F4, F5)
template <int M2>
__device__ __forceinline__ void rf_s2(const KArgs &a, const RArgs &r, const RTask &tk, int i,
                                      int nsb, int64_t ubase, const float2 *scr, const FChan *fchs) {
  const int m1 = tk.code & 255;
  const int per = tk.nch * m1;
  if (i >= r.bt * per) return;
  const int sp = (int)(((unsigned)i * tk.magPb) >> 16), rem = i - sp * per;
  const int c = (int)(((unsigned)rem * tk.magM1) >> 16), n1 = rem - c * m1;
  if (sp >= nsb) return;
  constexpr int S2 = M2 | 1;
  const int off = fchs[tk.coff + c].off;
  const float2 *A = scr + tk.soff + ((sp * tk.nch + c) * m1 + n1) * S2;
  float2 v[M2];
#pragma unroll
  for (int e2 = 0; e2 < M2; ++e2) v[e2] = A[e2];
  dft<M2, +1>(v);
  float2 *o = a.coef_out + (ubase + sp) * a.C + off + n1;
#pragma unroll
  for (int n2 = 0; n2 < M2; ++n2) __stcs(o + m1 * n2, v[n2]);
}

__device__ __forceinline__ RTask ld_rtask(const RTask *p) {  // (shared memory)
  const int4 t0 = reinterpret_cast<const int4 *>(p)[0];
  const int4 t1 = reinterpret_cast<const int4 *>(p)[1];
  RTask tk;
  tk.code = t0.x; tk.nch = t0.y; tk.coff = t0.z; tk.soff = t0.w;
  tk.magPa = (uint32_t)t1.x; tk.magM2 = (uint32_t)t1.y; tk.magPb = (uint32_t)t1.z; tk.magM1 = (uint32_t)t1.w;
  return tk;
}

// ------------------------------------------------------------------ work queue
// Items in dependency order: batch s's spectrum items precede the channel items of batch
// s - la, so every item depends only on items with smaller indices; items are claimed in
// index order by co-resident CTAs, hence no deadlock.  type 0: spectrum (unit p0); 1: channel
// (batch p0, band p1); 2: nothing (a padding unit of the last batch).
__device__ __forceinline__ int ring_decode(int i, int U, int bt, int nb, int la, int &p0, int &p1) {
  const int T = (U + bt - 1) / bt;
  const int A = min(la, T);
  if (i < A * bt) {
    p0 = i;
    return p0 < U ? 0 : 2;
  }
  i -= A * bt;
  const int mid = T > la ? T - la : 0, seg = bt + nb;
  if (i < mid * seg) {
    const int q = i / seg, rr = i - q * seg, sg = la + q;
    if (rr < bt) {
      p0 = sg * bt + rr;
      return p0 < U ? 0 : 2;
    }
    p0 = sg - la;
    p1 = rr - bt;
    return 1;
  }
  i -= mid * seg;
  const int q = i / nb;
  p0 = (T > la ? T - la : 0) + q;
  p1 = i - q * nb;
  return 1;
}
__host__ __device__ inline int64_t ring_items(int64_t U, int bt, int nb, int la) {
  const int64_t T = (U + bt - 1) / bt;
  const int64_t A = T < la ? T : la;
  const int64_t mid = T > la ? T - la : 0;
  return A * bt + mid * (bt + nb) + A * nb;
}

// (warp 0, lane 0) the band's metadata, weights and twiddles into the channel region
__device__ __forceinline__ void band_load(const KArgs &a, const RArgs &r, const RBand &B, char *uni,
                                          const ChanSmem &L, uint64_t *bar) {
  const unsigned tb = (unsigned)(sizeof(RTask) * B.ntask), fb = (unsigned)(sizeof(FChan) * B.nf);
  const unsigned rb = 4u * (unsigned)((B.r2off + ((B.nr2 + 3) & ~3)) - B.r1off);
  const int g0a = B.g0 & ~3;
  const unsigned wbytes = (unsigned)(((B.g0 + B.ng + 3) & ~3) - g0a) * 4u;
  const unsigned tbytes = (unsigned)((B.ntw + 1) & ~1) * 8u;
  mbar_arrive_tx(bar, tb + fb + rb + wbytes + tbytes);
  bulk_g2s(uni + L.meta, r.task + B.task0, tb, bar);
  bulk_g2s(uni + L.meta + tb, r.fch + B.f0, fb, bar);
  if (rb) bulk_g2s(uni + L.meta + tb + fb, r.round + B.r1off, rb, bar);
  bulk_g2s(uni + L.w, a.gw + g0a, wbytes, bar);
  bulk_g2s(uni + L.tw, r.btw + B.tw0, tbytes, bar);
}
// (warp 0) the band's X bins of the units of batch t into buffer set xb
__device__ __forceinline__ void x_load(const KArgs &a, const RArgs &r, const RBand &B, int t,
                                       float2 *xb, uint64_t *bar, int lane) {
  const int64_t u0 = (int64_t)t * r.bt;
  const int nsb = (int)min((int64_t)r.bt, (int64_t)a.nunits - u0);
  const unsigned xbytes = (unsigned)B.bspan * 8u;
  if (lane == 0) mbar_arrive_tx(bar, xbytes * (unsigned)nsb);
  __syncwarp();
  for (int i = lane; i < nsb; i += 32) {
    const int64_t u = u0 + i;
    const int slot = (int)(u % r.R);
    ring_wait_ge(r.ready + slot, (unsigned)(u + 1), r.err, 3u);
    fence_proxy_async();
    bulk_g2s(xb + (int64_t)i * r.xstride, r.ring + slot * r.slot_entries + B.blo, xbytes, bar);
  }
}

// (warp 0) the band's X bins of batch t from the split design's staging (unit u of the chunk
// at a.stage + u * a.xs; the spectrum kernel has completed: no flags)
__device__ __forceinline__ void x_load_staged(const KArgs &a, const RArgs &r, const RBand &B, int t,
                                              float2 *xb, uint64_t *bar, int lane) {
  const int64_t u0 = (int64_t)t * r.bt;
  const int nsb = (int)min((int64_t)r.bt, (int64_t)a.nunits - u0);
  const unsigned xbytes = (unsigned)B.bspan * 8u;
  if (lane == 0) mbar_arrive_tx(bar, xbytes * (unsigned)nsb);
  __syncwarp();
  for (int i = lane; i < nsb; i += 32)
    bulk_g2s(xb + (int64_t)i * r.xstride, a.stage + (u0 + i) * a.xs + B.blo, xbytes, bar);
}

// One channel item: band p1 for batches [p0 grp, p0 grp + grp) of bt units (F3 - F5).  The
// band's tables land once; the X bins of batch t + 1 land while batch t computes.  STAGED:
// X comes from the split design's staging buffer, else from the ring (ready flags; the slots
// are released once a batch has landed).
template <int LOGN, bool STAGED>
__device__ __forceinline__ void chan_item(const KArgs &a, const RArgs &r, int p0, int p1, char *uni,
                                          const ChanSmem &L, uint64_t *bar, unsigned *uses,
                                          int *s_round, uint64_t &t_wait) {
  constexpr int N = Big<LOGN>::N;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int U = a.nunits;
  const int NB = (U + r.bt - 1) / r.bt;
  float2 *scr = reinterpret_cast<float2 *>(uni + L.scr);
  const RBand B = r.band[p1];
  const int tb0 = p0 * r.grp, tb1 = min(NB, tb0 + r.grp);
  if (warp == 0) {
    if (lane == 0) band_load(a, r, B, uni, L, &bar[2]);
    if (STAGED) x_load_staged(a, r, B, tb0, reinterpret_cast<float2 *>(uni + L.set[0]), &bar[0], lane);
    else x_load(a, r, B, tb0, reinterpret_cast<float2 *>(uni + L.set[0]), &bar[0], lane);
  }
  mbar_wait(&bar[2], uses[2] & 1, r.err, 6u);
  ++uses[2];
  const RTask *tks = reinterpret_cast<const RTask *>(uni + L.meta);
  const FChan *fchs = reinterpret_cast<const FChan *>(uni + L.meta + sizeof(RTask) * B.ntask) - B.f0;
  const int32_t *rnd = reinterpret_cast<const int32_t *>(uni + L.meta + sizeof(RTask) * B.ntask +
                                                         sizeof(FChan) * B.nf);
  const int32_t *rnd2 = rnd + (B.r2off - B.r1off);
  const float *wb = reinterpret_cast<const float *>(uni + L.w) + (B.g0 & 3);
  const float2 *twsm = reinterpret_cast<const float2 *>(uni + L.tw);
  for (int t = tb0; t < tb1; ++t) {
    const int set = (t - tb0) & 1;
    const int64_t u0 = (int64_t)t * r.bt;
    const int nsb = (int)min((int64_t)r.bt, (int64_t)U - u0);
    const uint64_t tw0 = r.stats ? globaltimer_ns() : 0;
    if (tid == 0) *s_round = 0;
    mbar_wait(&bar[set], uses[set] & 1, r.err, 4u);
    ++uses[set];
    if (r.stats) t_wait += globaltimer_ns() - tw0;
    __syncthreads();  // (s_round; every warp past the previous batch's phase 2)
    if (warp == 0) {
      if (!STAGED)  // this batch's slots are free for the spectrum items of units u + R
        for (int i = lane; i < nsb; i += 32) red_release_add_u32(r.done + (int)((u0 + i) % r.R), 1u);
      if (t + 1 < tb1) {
        float2 *nx = reinterpret_cast<float2 *>(uni + L.set[set ^ 1]);
        if (STAGED) x_load_staged(a, r, B, t + 1, nx, &bar[set ^ 1], lane);
        else x_load(a, r, B, t + 1, nx, &bar[set ^ 1], lane);
      }
    }
    const float2 *Xb = reinterpret_cast<const float2 *>(uni + L.set[set]);
    const int64_t ub = a.unit0 + u0;
    // phase 1: small tasks and two-step step 1, rounds claimed dynamically
    for (;;) {
      int ri = 0;
      if (lane == 0) ri = atomicAdd(s_round, 1);
      ri = __shfl_sync(0xffffffffu, ri, 0);
      if (ri >= B.nr1) break;
      const int e = rnd[ri];
      const RTask tk = ld_rtask(tks + (e >> 16));
      const int i = (e & 0xffff) * 32 + lane;
      const int m1 = tk.code & 255;
      const bool small = (tk.code >> 16) & 1, inter = (tk.code >> 17) & 1;
      if (small) {
        switch (m1) {
#define X_(S) case S: if (inter) rf_small<S, N, true>(a, r, tk, i, nsb, ub, Xb, B.blo, wb, fchs); \
                      else rf_small<S, N, false>(a, r, tk, i, nsb, ub, Xb, B.blo, wb, fchs); break;
          SLICQ_FSMALL(X_)
#undef X_
        }
      } else {
        switch (m1) {
#define X_(S) case S: if (inter) rf_s1<S, N, true>(r, tk, i, nsb, Xb, B.blo, wb, twsm, scr, fchs); \
                      else rf_s1<S, N, false>(r, tk, i, nsb, Xb, B.blo, wb, twsm, scr, fchs); break;
          SLICQ_FSIZES(X_)
#undef X_
        }
      }
    }
    __syncthreads();
    if (tid == 0) *s_round = 0;
    __syncthreads();
    // phase 2: two-step step 2
    for (;;) {
      int ri = 0;
      if (lane == 0) ri = atomicAdd(s_round, 1);
      ri = __shfl_sync(0xffffffffu, ri, 0);
      if (ri >= B.nr2) break;
      const int e = rnd2[ri];
      const RTask tk = ld_rtask(tks + (e >> 16));
      const int i = (e & 0xffff) * 32 + lane;
      switch ((tk.code >> 8) & 255) {
#define X_(S) case S: rf_s2<S>(a, r, tk, i, nsb, ub, scr, fchs); break;
        SLICQ_FSIZES(X_)
#undef X_
      }
    }
    __syncthreads();  // (the scratch and this set are free)
  }
}

// ------------------------------------------------------------------ band-major channel kernel
// The split design's forward channel stage as band items: a persistent grid claims (group of
// grp batches, band) items in group-major order from a counter (zeroed by the launcher) and
// reads the staged spectra with TMA bulk copies.
template <int LOGN>
__global__ void __launch_bounds__(RING_T, 2) slicq_fwd_band_kernel(const KArgs a, const RArgs r) {
  extern __shared__ float4 smem4[];
  char *uni = reinterpret_cast<char *>(smem4);
  __shared__ uint64_t bar[3];
  __shared__ int s_item, s_round;
  const int tid = threadIdx.x;
  const ChanSmem L = chan_smem_layout(r.bt, r.xstride, r.wmax, r.twmax, r.iscr, r.meta);
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned uses[3] = {0u, 0u, 0u};
  uint64_t t_wait = 0;
  const int NBt = (a.nunits + r.bt - 1) / r.bt;
  const int ngroups = (NBt + r.grp - 1) / r.grp;
  const int nitems = ngroups * r.nb;
  pdl_wait();  // the staged spectra come from the spectrum kernel
  __syncthreads();
  for (;;) {
    if (tid == 0) s_item = (int)atomicAdd(r.qctr, 1ull);
    __syncthreads();
    const int item = s_item;
    if (item >= nitems) break;
    const int g = item / r.nb, b = item - g * r.nb;
    chan_item<LOGN, true>(a, r, g, b, uni, L, bar, uses, &s_round, t_wait);
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ forward kernel
// Every CTA runs both kinds of items.  Dynamic shared memory: [FFT twiddles (persistent)]
// [union: FFT frame + window table | channel region (chan_smem_layout)].  A channel item is
// one band for grp consecutive batches of bt units: the band's tables land once, the X bins
// of batch g + 1 land while batch g computes.
template <int LOGN>
__global__ void __launch_bounds__(RING_T, 2) slicq_fwd_ring_kernel(const KArgs a, const RArgs r) {
  using CF = Big<LOGN>;
  constexpr int N = CF::N;
  static_assert(CF::T == RING_T, "spectrum items run the 256-thread FFT");
  extern __shared__ float4 smem4[];
  float2 *tw = reinterpret_cast<float2 *>(smem4);
  char *uni = reinterpret_cast<char *>(tw + tw_entries<LOGN>());
  __shared__ uint64_t bar[3];  // X set 0, X set 1, band tables
  __shared__ long long s_next;
  __shared__ int s_round;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < tw_entries<LOGN>(); i += RING_T) tw[i] = a.tw2n[i];
  const ChanSmem L = chan_smem_layout(r.bt, r.xstride, r.wmax, r.twmax, r.iscr, r.meta);
  const int U = a.nunits;
  const int UG = r.bt * r.grp;                   // units per channel item
  const int64_t nitems = ring_items(U, UG, r.nb, r.la);
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_next = (long long)atomicAdd(r.qctr, 1ull);
  }
  unsigned uses[3] = {0u, 0u, 0u};  // completed phases of each barrier
  uint64_t t_spec = 0, t_chan = 0, t_wait = 0;
  __syncthreads();
  for (;;) {
    const int64_t item = s_next;
    if (item >= nitems) break;
    unsigned long long claim = 0;
    if (tid == 0) claim = atomicAdd(r.qctr, 1ull);  // (its latency hides behind this item)
    int p0 = 0, p1 = 0;
    const int type = ring_decode((int)item, U, UG, r.nb, r.la, p0, p1);
    const uint64_t t0 = r.stats ? globaltimer_ns() : 0;
    if (type == 0) {
      // ---- spectrum item: unit p0 -> ring slot p0 mod R (F1 + F2)
      const int slot = p0 % r.R;
      const unsigned gen = (unsigned)(p0 / r.R);
      if (tid == 0 && gen > 0) ring_wait_ge(r.done + slot, gen * (unsigned)r.nb, r.err, 1u);
      __syncthreads();
      float2 *spec = reinterpret_cast<float2 *>(uni);
      float *htab = reinterpret_cast<float *>(spec + spec_entries<LOGN>());
      fwd_spectrum<LOGN, 0, false, false>(a, spec, tw, htab, a.unit0 + p0,
                                          r.ring + slot * r.slot_entries);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release_u32(r.ready + slot, (unsigned)(p0 + 1));
      }
      if (r.stats) t_spec += globaltimer_ns() - t0;
    } else if (type == 1) {
      chan_item<LOGN, false>(a, r, p0, p1, uni, L, bar, uses, &s_round, t_wait);
      if (r.stats) t_chan += globaltimer_ns() - t0;
    }
    if (tid == 0) s_next = (long long)claim;
    __syncthreads();  // shared memory (and the claim) ready for the next item
  }
  if (r.stats && tid == 0) {
    r.stats[blockIdx.x * 4 + 0] = t_spec;
    r.stats[blockIdx.x * 4 + 1] = t_chan;
    r.stats[blockIdx.x * 4 + 2] = t_wait;
  }
}

// dynamic shared memory of the ring kernel: persistent FFT twiddles + the larger of a spectrum
// item's (padded frame, window table) and a channel item's (chan_smem_layout) needs
template <int LOGN>
constexpr size_t ring_smem(int tr, size_t chan_bytes) {
  const size_t spec = sizeof(float2) * (size_t)spec_entries<LOGN>() + sizeof(float) * (size_t)((tr + 3) & ~3);
  return sizeof(float2) * (size_t)tw_entries<LOGN>() + (spec > chan_bytes ? spec : chan_bytes);
}

template <int LOGN>
int ring_attrs();
template <int LOGN>
cudaError_t launch_fwd_band(const KArgs &a, const RArgs &r, size_t smem, int grid, cudaStream_t s,
                            bool pdl);
template <int LOGN>
cudaError_t launch_fwd_ring(const KArgs &a, const RArgs &r, size_t smem, cudaStream_t s);

}  // namespace kern
}  // namespace slicq
