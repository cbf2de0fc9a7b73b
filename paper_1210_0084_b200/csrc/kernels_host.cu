// Host side of the kernels: kernel configuration (channel packets, shared-memory
// budget), device-table upload and launch dispatch.  Device code: kernels_dev.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <vector>

#include "kernels_dev.cuh"

namespace slicq {
namespace {
using namespace slicq::kern;

// y += spill (the left neighbour's overlap-add spill, multi-GPU slice ranges)
__global__ void overlap_add_kernel(float *y, int64_t y_stride, const float *spill, int64_t count) {
  const int64_t row = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    y[row * y_stride + i] += spill[row * count + i];
}


const int kSizes[] = {1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 18, 20, 24, 25, 27, 30, 32};

bool in_sizes(int v) {
  for (int s : kSizes)
    if (s == v) return true;
  return false;
}

// M = M1 * M2 with both register-DFT sizes, minimising max(M1, M2) then padding.
bool factor_m(int M, int &M1, int &M2) {
  int best = 1 << 30, bp = 1 << 30;
  bool ok = false;
  for (int s : kSizes) {
    if (M % s) continue;
    const int o = M / s;
    if (!in_sizes(o)) continue;
    const int mx = std::max(s, o);
    const int pad = s * (o | 1);
    if (mx < best || (mx == best && pad < bp)) {
      best = mx;
      bp = pad;
      M1 = s;
      M2 = o;
      ok = true;
    }
  }
  return ok;
}

int threads_for(int logN) {
  switch (logN) {
    case 11: return Big<11>::T;
    case 12: return Big<12>::T;
    case 13: return Big<13>::T;
    case 14: return Big<14>::T;
  }
  return 0;
}

size_t smem_for(int logN, int scr) {
  switch (logN) {
    case 11: return smem_bytes_t<11>(scr);
    case 12: return smem_bytes_t<12>(scr);
    case 13: return smem_bytes_t<13>(scr);
    case 14: return smem_bytes_t<14>(scr);
  }
  return 0;
}

}  // namespace

int device_supports(int logN) { return logN >= 11 && logN <= 14; }

int configure_kernels(slicq_plan *p) {
  int logN = 0;
  while ((int64_t(1) << logN) < p->N) ++logN;
  if ((int64_t(1) << logN) != p->N || !device_supports(logN))
    return set_error(SLICQ_EUNSUPPORTED,
                     "CUDA path implements sl_len in {4096, 8192, 16384, 32768}");
  KernelConfig &kc = p->kc;
  kc.logN = logN;
  kc.threads = threads_for(logN);
  const int K2 = p->K + 2;
  // factor every channel length, group channels by M
  std::map<int, std::vector<int>> groups;
  std::map<int, std::pair<int, int>> fac;
  int need = 0;
  for (int k = 0; k < K2; ++k) {
    const int M = p->M[k];
    if (!fac.count(M)) {
      int m1 = 0, m2 = 0;
      if (!factor_m(M, m1, m2))
        return set_error(SLICQ_EUNSUPPORTED, "channel length M_k = " + std::to_string(M) +
                                                 " is not a product of two sizes <= 32");
      fac[M] = {m1, m2};
      need = std::max(need, m1 * (m2 | 1));
    }
    groups[M].push_back(k);
  }
  // scratch per warp: keep two CTAs per SM for N <= 8192 when the channels allow it
  const size_t smem_cap = 227 * 1024;
  int scr = std::max(need, 640);
  scr = (scr + 7) & ~7;
  if (smem_for(logN, scr) > smem_cap) scr = (need + 7) & ~7;
  if (smem_for(logN, scr) > smem_cap)
    return set_error(SLICQ_EUNSUPPORTED, "channel scratch does not fit in shared memory");
  kc.scr = scr;
  kc.smem = smem_for(logN, scr);
  // packets
  p->packets.clear();
  p->packet_chans.clear();
  for (auto &kv : groups) {
    const int M = kv.first;
    const int m1 = fac[M].first, m2 = fac[M].second;
    const int per = m1 * (m2 | 1);
    int nch = (32 + std::min(m1, m2) - 1) / std::min(m1, m2);
    nch = std::max(1, std::min({nch, scr / per, 32}));
    const std::vector<int> &ks = kv.second;
    for (size_t i = 0; i < ks.size(); i += nch) {
      PacketDev pk;
      const int n = (int)std::min<size_t>(nch, ks.size() - i);
      pk.m1m2 = m1 | (m2 << 8);
      pk.nch = n;
      pk.chan_off = (int)p->packet_chans.size();
      int lg = 0;
      while ((1 << lg) < M) ++lg;
      pk.cost = n * M * (lg + 2);
      for (int c = 0; c < n; ++c) p->packet_chans.push_back(ks[i + c]);
      p->packets.push_back(pk);
    }
  }
  std::stable_sort(p->packets.begin(), p->packets.end(),
                   [](const PacketDev &x, const PacketDev &y) { return x.cost > y.cost; });
  kc.npackets = (int)p->packets.size();
  return SLICQ_OK;
}

namespace {
template <class T>
size_t align_up(size_t x) {
  return (x + 255) & ~size_t(255);
}
}  // namespace

int upload(slicq_plan *p) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_error(SLICQ_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  p->device = dev;
  const int K2 = p->K + 2;
  const int64_t N = p->N, N2 = 2 * N;
  // channel twiddle tables e^{+2 pi i t / M}, one per distinct M
  std::map<int, int> twoff;
  std::vector<float> twM;
  for (int k = 0; k < K2; ++k) {
    const int M = p->M[k];
    if (twoff.count(M)) continue;
    twoff[M] = (int)(twM.size() / 2);
    for (int t = 0; t < M; ++t) {
      const double ang = 2.0 * 3.14159265358979323846 * (double)t / (double)M;
      twM.push_back((float)std::cos(ang));
      twM.push_back((float)std::sin(ang));
    }
  }
  std::vector<ChanDev> ch(K2);
  for (int k = 0; k < K2; ++k) {
    ChanDev &c = ch[k];
    c.lo = p->lo[k];
    c.len = p->len[k];
    c.M = p->M[k];
    c.goff = (int32_t)p->goff[k];
    c.off = (int32_t)p->off[k];
    c.twoff = twoff[c.M];
    c.scale = (float)(1.0 / std::sqrt((double)c.M));
    c.lo_mod = ((c.lo % c.M) + c.M) % c.M;
  }
  const size_t nG = p->g.size();
  std::vector<float> g(nG), gd(nG);
  for (int k = 0; k < K2; ++k) {
    const double half = (k == 0 || k == K2 - 1) ? 0.5 : 1.0;  // self-mirrored plateaus (C15)
    for (int i = 0; i < p->len[k]; ++i) {
      g[p->goff[k] + i] = (float)p->g[p->goff[k] + i];
      gd[p->goff[k] + i] = (float)(half * p->gdual[p->goff[k] + i]);
    }
  }
  std::vector<float> h0(N2), h0d(N2);
  for (int64_t i = 0; i < N2; ++i) {
    h0[i] = (float)p->h0[i];
    h0d[i] = (float)p->h0dual[i];
  }
  // e^{-i pi t/N}: t < 64, then t = 64 h
  std::vector<float> tw;
  for (int t = 0; t < 64; ++t) {
    const double a = -3.14159265358979323846 * t / (double)N;
    tw.push_back((float)std::cos(a));
    tw.push_back((float)std::sin(a));
  }
  for (int64_t h = 0; h < N2 / 64; ++h) {
    const double a = -3.14159265358979323846 * (double)(64 * h) / (double)N;
    tw.push_back((float)std::cos(a));
    tw.push_back((float)std::sin(a));
  }
  // layout of the single device block
  size_t o = 0;
  const size_t o_chan = o; o = align_up<int>(o + sizeof(ChanDev) * K2);
  const size_t o_pk = o; o = align_up<int>(o + sizeof(PacketDev) * p->packets.size());
  const size_t o_pc = o; o = align_up<int>(o + sizeof(int32_t) * p->packet_chans.size());
  const size_t o_g = o; o = align_up<int>(o + sizeof(float) * nG);
  const size_t o_gd = o; o = align_up<int>(o + sizeof(float) * nG);
  const size_t o_h0 = o; o = align_up<int>(o + sizeof(float) * N2);
  const size_t o_h0d = o; o = align_up<int>(o + sizeof(float) * N2);
  const size_t o_tw = o; o = align_up<int>(o + sizeof(float) * tw.size());
  const size_t o_twM = o; o = align_up<int>(o + sizeof(float) * twM.size());
  void *blk = nullptr;
  e = cudaMalloc(&blk, o);
  if (e != cudaSuccess) return set_error(SLICQ_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  p->d.block = blk;
  p->d.bytes = o;
  char *b = static_cast<char *>(blk);
  p->d.chan = reinterpret_cast<ChanDev *>(b + o_chan);
  p->d.packets = reinterpret_cast<PacketDev *>(b + o_pk);
  p->d.packet_chans = reinterpret_cast<int32_t *>(b + o_pc);
  p->d.g = reinterpret_cast<float *>(b + o_g);
  p->d.gdual = reinterpret_cast<float *>(b + o_gd);
  p->d.h0 = reinterpret_cast<float *>(b + o_h0);
  p->d.h0dual = reinterpret_cast<float *>(b + o_h0d);
  p->d.tw2n = reinterpret_cast<float *>(b + o_tw);
  p->d.twM = reinterpret_cast<float *>(b + o_twM);
  std::vector<char> host(o, 0);
  std::memcpy(host.data() + o_chan, ch.data(), sizeof(ChanDev) * K2);
  std::memcpy(host.data() + o_pk, p->packets.data(), sizeof(PacketDev) * p->packets.size());
  std::memcpy(host.data() + o_pc, p->packet_chans.data(), sizeof(int32_t) * p->packet_chans.size());
  std::memcpy(host.data() + o_g, g.data(), sizeof(float) * nG);
  std::memcpy(host.data() + o_gd, gd.data(), sizeof(float) * nG);
  std::memcpy(host.data() + o_h0, h0.data(), sizeof(float) * N2);
  std::memcpy(host.data() + o_h0d, h0d.data(), sizeof(float) * N2);
  std::memcpy(host.data() + o_tw, tw.data(), sizeof(float) * tw.size());
  std::memcpy(host.data() + o_twM, twM.data(), sizeof(float) * twM.size());
  e = cudaMemcpy(blk, host.data(), o, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_error(SLICQ_ECUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  int rc = 0;
  switch (p->kc.logN) {
    case 11: rc = set_attrs<11>(p->kc.smem); break;
    case 12: rc = set_attrs<12>(p->kc.smem); break;
    case 13: rc = set_attrs<13>(p->kc.smem); break;
    case 14: rc = set_attrs<14>(p->kc.smem); break;
  }
  if (rc != 0)
    return set_error(SLICQ_ECUDA, std::string("cudaFuncSetAttribute: ") +
                                      cudaGetErrorString((cudaError_t)rc));
  p->has_device = true;
  return SLICQ_OK;
}

void free_device(slicq_plan *p) {
  if (p && p->d.block) {
    cudaFree(p->d.block);
    p->d.block = nullptr;
  }
  if (p) p->has_device = false;
}

size_t workspace_bytes(const slicq_plan *p, int64_t nslices, int64_t batch) {
  const size_t cnt = align_up<int>(sizeof(unsigned) * (size_t)(batch * nslices));
  return cnt + sizeof(float) * (size_t)(batch * nslices * 2 * p->tr);
}

static KArgs base_args(const slicq_plan *p) {
  KArgs a{};
  a.tr = (int)p->tr;
  a.scr = p->kc.scr;
  a.npackets = p->kc.npackets;
  a.C = p->C;
  a.chan = p->d.chan;
  a.packets = p->d.packets;
  a.pchans = p->d.packet_chans;
  a.g = p->d.g;
  a.gdual = p->d.gdual;
  a.h0 = p->d.h0;
  a.h0dual = p->d.h0dual;
  a.tw2n = reinterpret_cast<const float2 *>(p->d.tw2n);
  a.twM = reinterpret_cast<const float2 *>(p->d.twM);
  return a;
}

static int check_device(const slicq_plan *p) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != p->device)
    return set_error(SLICQ_EINVAL, "current CUDA device differs from the plan's device");
  return SLICQ_OK;
}

int launch_forward(const slicq_plan *p, const float *x, int64_t x_len, int64_t x_stride,
                   int64_t base_off, int64_t L, int wrap, int64_t slice0, int64_t nslices,
                   int64_t batch, slicq_c32 *coeffs, void *stream) {
  int rc = check_device(p);
  if (rc) return rc;
  if (nslices > 0x7fffffff || batch > 65535) return set_error(SLICQ_ESHAPE, "grid too large");
  KArgs a = base_args(p);
  a.x = x;
  a.x_len = x_len;
  a.x_stride = x_stride;
  a.base_off = base_off;
  a.L = L;
  a.wrap = wrap;
  a.slice0 = slice0;
  a.nslices = (int)nslices;
  a.coef_out = reinterpret_cast<float2 *>(coeffs);
  dim3 grid((unsigned)nslices, (unsigned)batch);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->kc.logN) {
    case 11: e = launch_fwd<11>(a, grid, p->kc.smem, s); break;
    case 12: e = launch_fwd<12>(a, grid, p->kc.smem, s); break;
    case 13: e = launch_fwd<13>(a, grid, p->kc.smem, s); break;
    case 14: e = launch_fwd<14>(a, grid, p->kc.smem, s); break;
    default: return set_error(SLICQ_EINTERNAL, "bad logN");
  }
  if (e != cudaSuccess) return set_error(SLICQ_ECUDA, std::string("forward launch: ") + cudaGetErrorString(e));
  return SLICQ_OK;
}

int launch_inverse(const slicq_plan *p, const slicq_c32 *coeffs, int64_t slice0, int64_t nslices,
                   int64_t total_slices, int64_t batch, int circular, int64_t n_valid, int64_t L,
                   float *y, int64_t y_stride, int64_t y_base, float *left_spill, int64_t halo,
                   void *ws, size_t ws_bytes, void *stream) {
  (void)total_slices;
  int rc = check_device(p);
  if (rc) return rc;
  if (nslices > 0x7fffffff || batch > 65535) return set_error(SLICQ_ESHAPE, "grid too large");
  const size_t need = workspace_bytes(p, nslices, batch);
  if (!ws || ws_bytes < need) return set_error(SLICQ_ESHAPE, "workspace too small");
  if ((uintptr_t)ws % 16) return set_error(SLICQ_ESHAPE, "workspace must be 16-byte aligned");
  KArgs a = base_args(p);
  a.coef_in = reinterpret_cast<const float2 *>(coeffs);
  a.y = y;
  a.y_len = n_valid;
  a.y_stride = y_stride;
  a.y_base = y_base;
  a.spill = left_spill;
  a.halo = halo;
  a.L = L;
  a.circular = circular;
  a.slice0 = slice0;
  a.nslices = (int)nslices;
  a.cnt = static_cast<unsigned *>(ws);
  a.bnd = reinterpret_cast<float *>(static_cast<char *>(ws) +
                                    align_up<int>(sizeof(unsigned) * (size_t)(batch * nslices)));
  dim3 grid((unsigned)nslices, (unsigned)batch);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->kc.logN) {
    case 11: e = launch_inv<11>(a, grid, p->kc.smem, s); break;
    case 12: e = launch_inv<12>(a, grid, p->kc.smem, s); break;
    case 13: e = launch_inv<13>(a, grid, p->kc.smem, s); break;
    case 14: e = launch_inv<14>(a, grid, p->kc.smem, s); break;
    default: return set_error(SLICQ_EINTERNAL, "bad logN");
  }
  if (e != cudaSuccess) return set_error(SLICQ_ECUDA, std::string("inverse launch: ") + cudaGetErrorString(e));
  return SLICQ_OK;
}

int launch_overlap_add(float *y, int64_t y_stride, const float *spill, int64_t count,
                       int64_t batch, void *stream) {
  if (batch > 65535) return set_error(SLICQ_ESHAPE, "batch too large");
  const int T = 256;
  const unsigned blocks = (unsigned)std::min<int64_t>((count + T - 1) / T, 1024);
  overlap_add_kernel<<<dim3(blocks, (unsigned)batch), T, 0, static_cast<cudaStream_t>(stream)>>>(
      y, y_stride, spill, count);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SLICQ_ECUDA, std::string("overlap_add launch: ") + cudaGetErrorString(e));
  return SLICQ_OK;
}

}  // namespace slicq
