// Internal structures shared by the host plan (plan.cpp) and the kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector_types.h>
#include <vector>

#include "../../include/slicq.h"
#include "kernels_long_api.h"
#include "kernels_generic.h"

namespace slicq {

// Per stored channel, as the kernels read it (32 bytes, one __ldg of two int4).
struct ChanDev {
  int32_t lo;      // first bin of the unwrapped support J_k (C5)
  int32_t len;     // L_k
  int32_t M;       // M_k
  int32_t goff;    // offset of g_k / dual_k in the filter tables
  int32_t off;     // column offset of channel k in a coefficient row
  int32_t twoff;   // offset of the e^{+2 pi i t / M_k} table
  float scale;     // 1/sqrt(M_k)  (Alg. 1 sqrt(M)*IFFT incl. 1/M, Alg. 2 FFT/sqrt(M); C1)
  int32_t lo_mod;  // lo_k mod M_k in [0, M_k)
  int32_t m1 = 0;   // long mode, M_k > 26000: four-step factor M1 (M_k = M1 * M2)
  int32_t soff = 0; // long mode, M_k > 26000: offset of the channel's staging scratch
};

// A packet = consecutive channels of one length M, processed for nu consecutive units at
// once: virtual channel vc = u * nch + c (u < nu, c < nch).  Big packets (M > 32): four-step
// M1 x M2 DFT, one task per lane and step (nu*nch*M1, nu*nch*M2 <= 32).  Small packets
// (M <= 32, flag bit 17): one lane per virtual channel, whole DFT_M in registers.
struct PacketDev {
  int32_t m1m2;     // M1 | (M2 << 8) | SMALL << 17  (small: M1 = M, M2 = 1)
  int32_t nch;      // channels in the packet
  int32_t chan_off; // offset into the packet channel list
  int32_t fent_off; // forward element table offset
  int32_t ient_off; // inverse element table offset
  int32_t nz;       // inverse contributions (sum of the channels' L_k)
  uint32_t mag1;    // ceil(2^16 / M1): q / M1 = (q * mag1) >> 16 for q < 64
  uint32_t mag2;    // ceil(2^16 / M2)
  int32_t xlo, xhi; // forward: spectrum bins [xlo, xhi] the fold reads (L2 prefetch)
  int32_t nu;       // units per warp task
  uint32_t magc;    // ceil(2^16 / nch): vc / nch = (vc * magc) >> 16
  int32_t ustride;  // scratch entries per unit (small: nch, big: nch * M1 * (M2 | 1))
};

// Fused kernels (kernels_fused.cuh): a channel as one warp task reads it (48 bytes, three
// int4).  Coefficient n of channel k is sum_d y[d] w^{(d + lo) n}, y[d] = X(lo + d) g_k[d]
// (d < L_k), w = e^{2 pi i / M_k}: the support is read contiguously and the rotation by lo
// (the fold's j mod M_k, C5) becomes a shift of the four-step twiddle and of the second
// step's input index.
struct FChan {
  int32_t lo;      // first bin of J_k (unwrapped, C5)
  int32_t len;     // L_k
  int32_t M;       // M_k
  int32_t goff;    // offset of the channel's weights in gw / gdw
  int32_t off;     // column offset in a coefficient row
  int32_t twoff;   // offset of the e^{+2 pi i t / M_k} table
  int32_t lo_mod;  // lo mod M_k in [0, M_k)
  int32_t lom2;    // lo mod M2 (two-step tasks), else 0
  int32_t d0, d1;  // synthesis: core terms d in [d0, d1) are added to the bin lo + d in place
  int32_t ovoff;   // synthesis: overflow slot of the channel's first non-core term
  int32_t flags;   // bit 0: support inside [0, N] (no mirrored bins)
};
// A warp task: nch channels of one length M = M1 * M2 (two-step) or M (small: one lane per
// channel).  code = M1 | M2 << 8 | small << 16 | interior << 17.
struct FTask {
  int32_t code;
  int32_t nch;
  int32_t coff;    // first FChan of the task
  uint32_t mags;   // ceil(2^16 / M2) | ceil(2^16 / M1) << 16: exact q / M for the task's q
};

// Ring kernels (kernels_ring.cuh).  A band: channels forming a contiguous run, the X bins
// [blo, blo + bspan) they read, its tasks [task0, task0 + ntask), its weights (gw / gdw
// [g0, g0 + ng)), twiddles (btw [tw0, tw0 + ntw)) and its two lists of 32-lane rounds
// (phase 1: small tasks and two-step step 1; phase 2: two-step step 2).
struct RBand {
  int32_t blo, bspan;
  int32_t task0, ntask;
  int32_t g0, ng;
  int32_t tw0, ntw;
  int32_t r1off, nr1;   // rounds: [r1off, r1off + nr1) phase 1, [r2off, r2off + nr2) phase 2
  int32_t r2off, nr2;   // (r1off, r2off multiples of 4; r2off = r1off + nr1 rounded up to 4)
  int32_t f0, nf;       // the band's channel descriptors [f0, f0 + nf) of rfch
  int32_t pad0, pad1;
};
// A task of a band: nch channels of one length, for all bt units of an item.
// code = M1 | M2 << 8 | small << 16 | interior << 17 (small: M1 = M, M2 = 1); soff: the
// task's offset (float2) in the item scratch.
struct RTask {
  int32_t code, nch, coff, soff;
  // exact q / d = (q * mag) >> 16 for the task's q (mag = ceil(2^16 / d) <= 2^16):
  uint32_t magPa;  // d = nch * M2 (small: nch)
  uint32_t magM2;  // d = M2
  uint32_t magPb;  // d = nch * M1
  uint32_t magM1;  // d = M1
};

// Forward channel kernel v2 (kernels_chan2.cuh): a packet of nch channels of one length
// (two-step M1 x M2, or small: M1 = M, a whole DFT per lane), nu units per warp task;
// code = M1 | M2 << 8 | small << 16 | interior << 17.  Exact q / d = (q * mag) >> 16.
struct P2Dev {
  int32_t code, nch, coff, nu;
  uint32_t magA;  // d = M2: step-1 item -> virtual channel
  uint32_t magB;  // d = M1: step-2 item -> virtual channel
  uint32_t magC;  // d = nch: virtual channel -> unit
  int32_t pad;
};

struct DeviceTables {
  ChanDev *chan = nullptr;
  PacketDev *packets = nullptr;
  int32_t *pchans = nullptr;
  uint2 *fent = nullptr;     // forward element table
  uint2 *ient = nullptr;     // inverse element table
  uint32_t *dpos = nullptr;  // inverse overflow run per bin: start | count << 20 (0: none)
  uint2 *ovbins = nullptr;   // inverse: per overflow bin (first term, term count) in ovterm
  uint32_t *dord = nullptr;  // inverse: per bin, 1 + its index in ovbins (0: none)
  uint32_t *ovterm = nullptr;  // inverse: the overflow bins' terms (staging-row offsets)
  float *h0 = nullptr;      // fp32 h_0[t+N], t in [-N, N)
  float *h0dual = nullptr;  // fp32 h~_0[t+N]
  float *tw2n = nullptr;    // float2: [64] e^{-i pi t/N} for t < 64, then [2N/64] for t = 64 h
  float *twM = nullptr;     // float2 tables e^{+2 pi i t / M}
  float *gw = nullptr;      // long mode: g_k / sqrt(M_k) (fp32, at goff_k)
  float *gdw = nullptr;     // long mode: g~_k / sqrt(M_k) (x 1/2 on the plateaus)
  uint32_t *lrow = nullptr; // long mode: per-bin term list start [N + 2]
  uint32_t *lent = nullptr; // long mode: term index | conj << 31
  uint2 *cxf = nullptr;     // complex input, per full-layout column: source column, twiddle
  uint2 *cxs = nullptr;     // complex input, per stored column: mirror column, twiddle
  FChan *fchf = nullptr, *fchi = nullptr;  // fused kernels: channels in forward / inverse task order
  FTask *ftf = nullptr, *fti = nullptr;    // fused kernels: forward / inverse warp tasks
  int2 *ovb = nullptr;      // fused inverse: bins with overflow terms (bin, first entry | count << 20)
  int32_t *ovl = nullptr;   // fused inverse: overflow slots per such bin, plan order
  RBand *rband = nullptr;   // ring kernels: bands
  RTask *rtask = nullptr;   // ring kernels: band warp tasks
  FChan *rfch = nullptr;    // ring kernels: channels (band-local weight / twiddle offsets)
  float2 *rbtw = nullptr;   // ring kernels: per-band twiddle tables
  int32_t *rround = nullptr; // ring kernels: per-band round lists (task << 16 | round)
  int32_t *pbig = nullptr;   // sliCQ channels with M_k > 1024, by size class
  uint2 *bent = nullptr;     // their inverse term destinations
  P2Dev *f2pk = nullptr;     // forward channel kernel v2: packets
  FChan *f2ch = nullptr;     // forward channel kernel v2: channels in packet order
  void *block = nullptr;    // single allocation holding all of the above
  cudaStream_t pipe[2] = {nullptr, nullptr};  // chunk pipelining (kc.pipe): two streams
  cudaEvent_t pev[3] = {nullptr, nullptr, nullptr};
  size_t bytes = 0;
};

struct KernelConfig {
  int logN = 0;          // N = 2^logN complex points in the r2c FFT of a 2N slice
  int threads = 0;       // spectrum-kernel CTA size
  size_t spec_smem = 0;  // spectrum kernels: dynamic shared memory bytes
  size_t spec_smem_p = 0;  // persistent inverse spectrum kernel (+ overlap carry)
  bool inv_persist = false;  // inverse spectrum stage runs persistent (on-chip overlap carry)
  bool fwd_persist = false;  // forward spectrum stage runs persistent
  int scr = 0;           // channel kernels: per-warp scratch (float2 entries)
  size_t chan_smem = 0;
  // TMA-staged channel kernels (kernels_tb.cuh): per-warp operand buffer (float2 entries)
  bool tb = false;
  int scr_f = 0;              // forward scratch (big packets only; small ones use none)
  int tbe_f = 0, tbe_i = 0;   // buffer entries: forward band, inverse coefficient columns
  size_t tb_smem_f = 0, tb_smem_i = 0;
  int npackets = 0;
  int nlite = 0;              // packets [0, nlite) run in the micro / lite variants
  int voff[4] = {0, 0, 0, 0}; // packets [voff[v], voff[v+1]) run in variant v (micro, lite, full)
  int64_t xs = 0, zs = 0;     // staging row strides (float2): X spectra, contributions
  int64_t zso = 0, nover = 0; // inverse staging: slot-1 offset, overflow entries
  bool large = false;         // 2N >= 65536: four-step FFT through the staging buffer
  int64_t toff_f = 0, toff_i = 0;  // offsets of the four-step intermediate in a unit
  int64_t chunk_units = 0;    // units per chunk (staging is sized for one chunk)
  int tile = 16;              // units per channel-kernel tile
  int stiles = 0;             // channel kernels: tiles per super-tile (0: the whole chunk)
  int lcluster = 0;           // 2N = 131072 slice FFT on 16-CTA clusters: bit 0 fwd, 1 inv
  int pf = 0;                 // persistent inverse spectrum kernel: L2 prefetch of the next unit
                              // (SLICQ_INV_PF; measured: off is 2 % faster on cfg4, the prefetched
                              // slots were evicted before use -- 1.6 GB of re-reads per call)
  int chan_per_sm = 0;        // channel-kernel CTAs per SM cap (0: occupancy)
  bool pipe = false;          // chunks alternate between two streams, ping-pong staging
  bool pdl = true;            // launch with programmatic stream serialization
  int64_t pipe_min = 8192;    // ... for calls of at least this many units
  int64_t pipe_parts = 4;     // ... split into this many chunks
  bool longmode = false;      // sl_len 2^18..2^22: full-length CQ-NSGT only (kernels_long.cuh)
  kern::LongClasses lcls{};   // long mode: channel size classes (kernels_long_api.h)
  // fused kernels (kernels_fused.cuh): one CTA per unit, no staging
  bool ftables = false;       // fused / ring tables built (fused_host.cu)
  bool fused = false;         // forward runs the fused per-slice kernel (opt-in)
  int cluster = 0;            // forward runs the cluster-fused kernel with clusters of this many CTAs (0: off)
  bool band = false;          // forward channel stage runs the band-major kernel (split design)
  int nftf = 0, nfti = 0;     // forward / inverse warp tasks
  int nphase_a = 0;           // inverse: tasks [0, nphase_a) are phase A (even channels)
  int fscr = 0;               // per-warp scratch (float2 entries)
  int nov = 0, novb = 0;      // inverse overflow slots per unit, bins with overflow terms
  size_t fsmem_f = 0, fsmem_i = 0;  // dynamic shared memory of the fused kernels
  // ring kernels (kernels_ring.cuh): one persistent cooperative launch per call
  bool ring = false;
  int rR = 0, rnspec = 0, rnchan = 0, rnb = 0, rq = 0, rbt = 0, rla = 0;
  int rxstride = 0, rwmax = 0, rtwmax = 0, rfscr = 0;  // rfscr: item scratch (float2)
  int rgroup = 1, rmeta = 0;  // batches per channel item; largest band metadata (bytes)
  // sliCQ channels with M_k > 1024 (kernels_long.cuh, one CTA per channel and unit)
  int nbig = 0;
  kern::LongClasses bcls{};
  // generic-length spectrum kernels (kernels_generic.cu): any 2/3/5-smooth N that fits
  bool generic = false;
  kern::GArgs gargs{};        // radix plan; device pointers set by upload()
  // forward channel kernel v2 (kernels_chan2.cuh)
  bool fwd2 = false;
  int f2voff[3] = {0, 0, 0};  // packets [f2voff[v], f2voff[v+1]) run in variant v (lite, full)
  int f2scr = 0;              // per-warp scratch (float2)
  int64_t rslot = 0;          // float2 entries per ring slot
  size_t rsmem = 0;           // dynamic shared memory of the ring kernel
  size_t rchsmem = 0;         // dynamic shared memory of the band-major channel kernel
};

}  // namespace slicq

struct slicq_plan {
  // parameters
  double fs, fmin, fmax;
  int B;
  int64_t sl_len, N, tr;
  int raster;
  int window = 0;              // SLICQ_WINDOW_*
  double min_width = 4.0;      // C7 lower bound on the filter width (bins)
  int64_t sampled_from = 0;    // Prop. 4: 2N' whose filters this system samples (0: none)
  bool painless = true;        // M_k >= L_k for all k (false only with sampled_from)
  // serialises the fork / launch / join sequence of pipelined calls (the plan's two
  // streams and three events are shared by all calls on the plan)
  mutable std::mutex pipe_mu;
  // Table 1 layout
  int K;
  double Q;
  std::vector<double> xi;  // xi_1..xi_K
  // stored channels 0..K+1
  std::vector<int32_t> lo, len, M;
  std::vector<int64_t> off;   // K+3 entries
  std::vector<int64_t> goff;  // K+2 entries
  std::vector<double> g, gdual;
  std::vector<double> h0, h0dual;
  int64_t C;  // sum M_k
  // device side
  bool has_device = false;
  int device = -1;
  slicq::DeviceTables d;
  slicq::KernelConfig kc;
  std::vector<slicq::PacketDev> packets;
  std::vector<int32_t> pchans;
  std::vector<uint2> fent, ient;
  std::vector<uint32_t> dpos;
  std::vector<uint2> ovbins;   // bins with overflow terms: (first term, count) in ovterm
  std::vector<uint32_t> dord;  // 1 + index into ovbins per bin (0: none)
  std::vector<uint32_t> ovterm;  // their terms in summation order (staging-row offsets)
  std::vector<float> lgw, lgdw;          // long mode filter weights
  std::vector<uint32_t> lrow, lent;      // long mode per-bin term lists
  std::vector<int32_t> lm1;              // long mode: four-step factor of M_k > 26000 (else 0)
  std::vector<uint2> cxf, cxs;           // complex-input column maps (kernels_complex.cu)
  std::vector<slicq::FChan> fchf, fchi;  // fused kernels: channel descriptors in task order
  std::vector<slicq::FTask> ftf, fti;    // fused kernels: warp tasks
  std::vector<int2> ovb;                 // fused inverse: overflow bins
  std::vector<int32_t> ovl;              // fused inverse: overflow slot lists
  std::vector<slicq::RBand> rband;       // ring kernels: bands
  std::vector<slicq::RTask> rtask;       // ring kernels: band warp tasks
  std::vector<slicq::FChan> rfch;        // ring kernels: channels in band task order
  std::vector<float> rbtw;               // ring kernels: per-band twiddles (re, im)
  std::vector<int32_t> rround;           // ring kernels: per-band round lists
  std::vector<int32_t> pbig;             // sliCQ channels with M_k > 1024 (by size class)
  std::vector<uint2> bent;               // their term destinations
  std::vector<int> bentoff, bentn;       // per channel: first entry, count
  std::vector<float> gtw;                // generic kernels: e^{-2 pi i t / N} (re, im), t < N
  std::vector<int32_t> gperm;            // generic kernels: mixed-radix digit reversal
  std::vector<slicq::P2Dev> f2pk;        // forward channel kernel v2: packets
  std::vector<slicq::FChan> f2ch;        // forward channel kernel v2: channels
  std::vector<int64_t> lsoff;            // long mode: staging scratch offset of those channels
};

namespace slicq {
int set_error(int code, const std::string &msg);
// kernels.cu
int device_supports(int logN);
int configure_kernels(slicq_plan *p);  // fills p->kc, packets (host)
int upload(slicq_plan *p);             // allocates + copies device tables
void free_device(slicq_plan *p);
int launch_forward(const slicq_plan *p, const float *x, int64_t x_len, int64_t x_stride,
                   int64_t base_off, int64_t L, int wrap, int64_t slice0, int64_t nslices,
                   int64_t batch, slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream,
                   int mode = 0);  // mode 1: full-length CQ-NSGT (one frame per row)
int launch_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t slice0, int64_t nslices,
                   int64_t total_slices, int64_t batch, int circular, int64_t n_valid,
                   int64_t L, float *y, int64_t y_stride, int64_t y_base, float *left_spill,
                   int64_t halo, void *ws, size_t ws_bytes, void *stream,
                   const float *mask = nullptr, int mask_db = 0, int mode = 0);
int launch_overlap_add(float *y, int64_t y_stride, const float *spill, int64_t count,
                       int64_t batch, void *stream);
// complex input (kernels_complex.cu)
int64_t coeffs_full(const slicq_plan *p);
size_t workspace_bytes_complex(const slicq_plan *p, int64_t nslices, int64_t batch, int64_t n);
int launch_forward_complex(const slicq_plan *p, const slicq_c32 *x, int64_t n, int64_t batch,
                           slicq_c32 *coeffs, void *ws, size_t ws_bytes, void *stream,
                           int nsgt = 0);
int launch_inverse_complex(const slicq_plan *p, const slicq_c32 *coeffs, int64_t n,
                           int64_t batch, slicq_c32 *y, void *ws, size_t ws_bytes, void *stream,
                           int nsgt = 0);
// coefficient processing (kernels_coeff.cu)
int launch_mask(const slicq_plan *p, slicq_c32 *c, const float *mask, int64_t rows, int full,
                int db, void *stream);
int launch_spectrogram(const slicq_plan *p, const slicq_c32 *c, int64_t nslices, int64_t batch,
                       float *out, void *stream);
int launch_transpose(const slicq_plan *p, const slicq_c32 *c, slicq_c32 *out, int64_t rows,
                     int shift, void *stream);
int launch_approx(const slicq_plan *ps, const slicq_plan *pl, const slicq_c32 *s,
                  const slicq_c32 *c, int64_t batch, double *out, void *stream, int full = 0);
size_t workspace_bytes(const slicq_plan *p, int64_t nslices, int64_t batch);
int kernel_launches(const slicq_plan *p, int direction, int64_t nslices, int64_t batch);
// fused kernels (fused_host.cu)
int configure_fused(slicq_plan *p);  // after configure_kernels: task tables, smem budgets
int fused_set_attrs(const slicq_plan *p);
int configure_ring(slicq_plan *p);   // after configure_fused: bands, tasks, ring sizing
int configure_fwd2(slicq_plan *p);   // after configure_fused: forward channel kernel v2
}  // namespace slicq
