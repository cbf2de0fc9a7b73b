// Internal structures shared by the host plan (plan.cpp) and the kernels (kernels.cu).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/slicq.h"

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
};

// A packet = channels of one length M = M1*M2 processed together by one warp, with at most
// 32 tasks per DFT step (nch*M2 <= 32 and nch*M1 <= 32): one task per lane.
struct PacketDev {
  int32_t m1m2;     // M1 | (M2 << 8)
  int32_t nch;      // channels in the packet
  int32_t chan_off; // offset into the packet channel list
  int32_t region;   // inverse: float2 offset of the packet's region in the chunk scratch
};

// Inverse: channels are processed in chunks whose F_k fit in shared memory; after each
// chunk, every target bin b in [blo, bhi] is gathered by exactly one thread (no atomics).
struct ChunkDev {
  int32_t pk0, pk1;   // packets [pk0, pk1) of the inverse packet list
  int32_t blo, bhi;   // target half-spectrum bins touched by the chunk
  int32_t bin_base;   // this chunk's (bhi - blo + 2) entries in bin_off
  int32_t pad0, pad1, pad2;
};

// One term of the per-bin gather: F value at chunk-scratch position (fidx & 0x7fffffff),
// conjugated if bit 31 is set (Hermitian rule, C15), times gval = dual (x 1/2 on the
// self-mirrored plateaus) / sqrt(M_k).
struct GatherEnt {
  uint32_t fidx;
  float gval;
};

struct DeviceTables {
  ChanDev *chan = nullptr;
  PacketDev *fwd_packets = nullptr;
  int32_t *fwd_pchans = nullptr;
  PacketDev *inv_packets = nullptr;
  int32_t *inv_pchans = nullptr;
  ChunkDev *chunks = nullptr;
  int32_t *bin_off = nullptr;
  GatherEnt *gents = nullptr;
  float *g = nullptr;       // fp32 g_k / sqrt(M_k) on J_k (forward)
  float *h0 = nullptr;      // fp32 h_0[t+N], t in [-N, N)
  float *h0dual = nullptr;  // fp32 h~_0[t+N]
  float *tw2n = nullptr;    // float2: [64] e^{-i pi t/N} for t < 64, then [2N/64] for t = 64 h
  float *twM = nullptr;     // float2 tables e^{+2 pi i t / M}
  void *block = nullptr;    // single allocation holding all of the above
  size_t bytes = 0;
};

struct KernelConfig {
  int logN = 0;          // N = 2^logN complex points in the r2c FFT of a 2N slice
  int threads = 0;       // CTA size
  int fwd_scr = 0;       // forward: per-warp scratch (float2 entries)
  int inv_scr = 0;       // inverse: chunk scratch (float2 entries)
  size_t fwd_smem = 0;   // dynamic shared memory bytes
  size_t inv_smem = 0;
  int fwd_npackets = 0;
  int nchunks = 0;
};

}  // namespace slicq

struct slicq_plan {
  // parameters
  double fs, fmin, fmax;
  int B;
  int64_t sl_len, N, tr;
  int raster;
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
  std::vector<slicq::PacketDev> fwd_packets, inv_packets;
  std::vector<int32_t> fwd_pchans, inv_pchans;
  std::vector<slicq::ChunkDev> chunks;
  std::vector<int32_t> bin_off;
  std::vector<slicq::GatherEnt> gents;
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
                   int64_t batch, slicq_c32 *coeffs, void *stream);
int launch_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t slice0, int64_t nslices,
                   int64_t total_slices, int64_t batch, int circular, int64_t n_valid,
                   int64_t L, float *y, int64_t y_stride, int64_t y_base, float *left_spill,
                   int64_t halo, void *ws, size_t ws_bytes, void *stream);
int launch_overlap_add(float *y, int64_t y_stride, const float *spill, int64_t count,
                       int64_t batch, void *stream);
size_t workspace_bytes(const slicq_plan *p, int64_t nslices, int64_t batch);
}  // namespace slicq
