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

size_t fwd_smem_for(int logN, int scr) {
  switch (logN) {
    case 11: return fwd_smem_bytes<11>(scr);
    case 12: return fwd_smem_bytes<12>(scr);
    case 13: return fwd_smem_bytes<13>(scr);
    case 14: return fwd_smem_bytes<14>(scr);
  }
  return 0;
}

size_t inv_smem_for(int logN, int scr) {
  switch (logN) {
    case 11: return inv_smem_bytes<11>(scr);
    case 12: return inv_smem_bytes<12>(scr);
    case 13: return inv_smem_bytes<13>(scr);
    case 14: return inv_smem_bytes<14>(scr);
  }
  return 0;
}

constexpr size_t kSmemCap = 227 * 1024;  // per CTA
constexpr int kSmallScratch = 640;        // float2 entries a small inverse packet may use
constexpr size_t kSmemSM = 228 * 1024;   // per SM, 1 KB of it reserved per resident CTA

int minb_for(int logN) {
  switch (logN) {
    case 11: return Big<11>::MINB;
    case 12: return Big<12>::MINB;
    case 13: return Big<13>::MINB;
    case 14: return Big<14>::MINB;
  }
  return 1;
}

// shared-memory bytes a CTA may use if `ctas` CTAs are to be resident per SM
size_t smem_budget(int ctas) { return std::min(kSmemCap, kSmemSM / ctas - 1024); }

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

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
  const int N = (int)p->N, N2 = 2 * N;
  std::map<int, std::pair<int, int>> fac;
  for (int k = 0; k < K2; ++k) {
    const int M = p->M[k];
    if (fac.count(M)) continue;
    int m1 = 0, m2 = 0;
    if (M > 1024 || !factor_m(M, m1, m2))
      return set_error(SLICQ_EUNSUPPORTED, "channel length M_k = " + std::to_string(M) +
                                               " is not a product of two DFT sizes <= 32");
    fac[M] = {m1, m2};
  }
  auto nch_for = [](int m1, int m2) { return std::max(1, 32 / std::max(m1, m2)); };

  // ---------------- packets: runs of consecutive channels with the same length M and the
  // same SIMPLE flag (J_k inside [0, N]), at most 32 / max(M1, M2) channels each
  struct Pk {
    PacketDev d;
    std::vector<int> ks;
    int size;
    std::vector<std::pair<int, int>> bins;  // touched half-spectrum bins (closed intervals)
  };
  std::vector<Pk> pks;
  auto is_simple = [&](int k) { return p->lo[k] >= 0 && p->lo[k] + p->len[k] - 1 <= N; };
  for (int k = 0; k < K2;) {
    const int M = p->M[k];
    const bool simple = is_simple(k);
    const bool small = M <= 32;  // one lane per channel, DFT_M in registers
    const int m1 = small ? M : fac[M].first, m2 = small ? 1 : fac[M].second;
    const int nch = small ? std::min(32, kSmallScratch / M) : nch_for(m1, m2);
    Pk pk;
    pk.d = PacketDev{};
    pk.d.m1m2 = m1 | (m2 << 8) | ((simple ? 1 : 0) << 16) | ((small ? 1 : 0) << 17);
    pk.d.magM = (uint32_t)(((uint64_t(1) << 32) + M - 1) / M);
    pk.d.mag1 = (uint32_t)((65536 + m1 - 1) / m1);
    pk.d.mag2 = (uint32_t)((65536 + m2 - 1) / m2);
    while (k < K2 && p->M[k] == M && is_simple(k) == simple && (int)pk.ks.size() < nch)
      pk.ks.push_back(k++);
    pk.d.nch = (int)pk.ks.size();
    pk.size = small ? pk.d.nch * M : pk.d.nch * m1 * (m2 | 1);
    for (int kk : pk.ks) {  // bins the Hermitian rule of C15 touches
      const int lo = p->lo[kk], hi = p->lo[kk] + p->len[kk] - 1;
      auto clip = [&](int a0, int b0) {
        a0 = std::max(a0, 0);
        b0 = std::min(b0, N);
        if (a0 <= b0) pk.bins.push_back({a0, b0});
      };
      clip(lo, hi);                  // direct bins j in [0, N]
      clip(-hi, -lo);                // mirror of j <= 0 (DC side)
      clip(N2 - hi, N2 - lo);        // mirror of j >= N (Nyquist side)
      if (lo < 0) clip(lo + N2, hi + N2);  // j mod 2N for negative j (never <= N here)
    }
    pks.push_back(std::move(pk));
  }
  int need = 8;
  for (const Pk &pk : pks) need = std::max(need, pk.size);
  const int NW = kc.threads / 32;
  const size_t budget2 = smem_budget(minb_for(logN));
  const int cap2 = (int)((budget2 - fwd_smem_for(logN, 0)) / sizeof(float2) / NW) & ~7;
  const int cap1 = (int)((kSmemCap - fwd_smem_for(logN, 0)) / sizeof(float2) / NW) & ~7;
  if (need > cap1)
    return set_error(SLICQ_EUNSUPPORTED, "channel scratch does not fit in shared memory");
  (void)cap2;  // need <= cap2 keeps Big<LOGN>::MINB CTAs per SM
  const int scr = need;
  kc.fwd_scr = kc.inv_scr = (scr + 7) & ~7;
  kc.fwd_smem = fwd_smem_for(logN, kc.fwd_scr);
  kc.inv_smem = inv_smem_for(logN, kc.inv_scr);

  // ---------------- forward order: shape-sorted (warps of a CTA walk the list together:
  // I-cache locality), larger lengths first
  {
    std::vector<int> ord(pks.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
      const int Mx = (pks[x].d.m1m2 & 255) * ((pks[x].d.m1m2 >> 8) & 255);
      const int My = (pks[y].d.m1m2 & 255) * ((pks[y].d.m1m2 >> 8) & 255);
      if (Mx != My) return Mx > My;
      return (pks[x].d.m1m2 >> 16) < (pks[y].d.m1m2 >> 16);
    });
    p->fwd_packets.clear();
    p->fwd_pchans.clear();
    for (int i : ord) {
      PacketDev d = pks[i].d;
      d.chan_off = (int)p->fwd_pchans.size();
      for (int k : pks[i].ks) p->fwd_pchans.push_back(k);
      p->fwd_packets.push_back(d);
    }
    kc.fwd_npackets = (int)p->fwd_packets.size();
  }

  // ---------------- inverse: greedy colouring of the packet conflict graph (packets that
  // share a touched bin get different phases), shape-sorted inside a phase
  {
    auto overlap = [](const Pk &x, const Pk &y) {
      for (auto &a0 : x.bins)
        for (auto &b0 : y.bins)
          if (a0.first <= b0.second && b0.first <= a0.second) return true;
      return false;
    };
    std::vector<int> phase(pks.size(), -1);
    int nph = 0;
    for (size_t i = 0; i < pks.size(); ++i) {
      std::vector<char> used(nph + 1, 0);
      for (size_t j = 0; j < i; ++j)
        if (phase[j] >= 0 && overlap(pks[i], pks[j])) used[phase[j]] = 1;
      int ph = 0;
      while (ph < nph && used[ph]) ++ph;
      phase[i] = ph;
      nph = std::max(nph, ph + 1);
    }
    p->inv_packets.clear();
    p->inv_pchans.clear();
    p->chunks.clear();
    for (int ph = 0; ph < nph; ++ph) {
      std::vector<int> ids;
      for (size_t i = 0; i < pks.size(); ++i)
        if (phase[i] == ph) ids.push_back((int)i);
      std::stable_sort(ids.begin(), ids.end(),
                       [&](int x, int y) { return (pks[x].d.m1m2 & 0xffff) < (pks[y].d.m1m2 & 0xffff); });
      ChunkDev pr{};
      pr.pk0 = (int)p->inv_packets.size();
      for (int i : ids) {
        PacketDev d = pks[i].d;
        d.chan_off = (int)p->inv_pchans.size();
        for (int k : pks[i].ks) p->inv_pchans.push_back(k);
        p->inv_packets.push_back(d);
      }
      pr.pk1 = (int)p->inv_packets.size();
      p->chunks.push_back(pr);
    }
    kc.nchunks = nph;
  }
  return SLICQ_OK;
}

int upload(slicq_plan *p) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
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
    const double sc = 1.0 / std::sqrt((double)p->M[k]);  // Alg. 1: sqrt(M) * IFFT (1/M)
    const double half = (k == 0 || k == K2 - 1) ? 0.5 : 1.0;  // self-mirrored plateaus (C15)
    for (int i = 0; i < p->len[k]; ++i) {
      g[p->goff[k] + i] = (float)(p->g[p->goff[k] + i] * sc);
      gd[p->goff[k] + i] = (float)(p->gdual[p->goff[k] + i] * sc * half);
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
  struct Part { const void *src; size_t bytes; size_t off; };
  std::vector<Part> parts = {
      {ch.data(), sizeof(ChanDev) * ch.size(), 0},
      {p->fwd_packets.data(), sizeof(PacketDev) * p->fwd_packets.size(), 0},
      {p->fwd_pchans.data(), sizeof(int32_t) * p->fwd_pchans.size(), 0},
      {p->inv_packets.data(), sizeof(PacketDev) * p->inv_packets.size(), 0},
      {p->inv_pchans.data(), sizeof(int32_t) * p->inv_pchans.size(), 0},
      {p->chunks.data(), sizeof(ChunkDev) * p->chunks.size(), 0},
      {gd.data(), sizeof(float) * gd.size(), 0},
      {g.data(), sizeof(float) * g.size(), 0},
      {h0.data(), sizeof(float) * h0.size(), 0},
      {h0d.data(), sizeof(float) * h0d.size(), 0},
      {tw.data(), sizeof(float) * tw.size(), 0},
      {twM.data(), sizeof(float) * twM.size(), 0},
  };
  size_t o = 0;
  for (Part &pt : parts) {
    pt.off = o;
    o = align_up(o + pt.bytes + 16);
  }
  void *blk = nullptr;
  e = cudaMalloc(&blk, o);
  if (e != cudaSuccess)
    return set_error(SLICQ_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  p->d.block = blk;
  p->d.bytes = o;
  std::vector<char> host(o, 0);
  for (const Part &pt : parts)
    if (pt.bytes) std::memcpy(host.data() + pt.off, pt.src, pt.bytes);
  char *b = static_cast<char *>(blk);
  p->d.chan = reinterpret_cast<ChanDev *>(b + parts[0].off);
  p->d.fwd_packets = reinterpret_cast<PacketDev *>(b + parts[1].off);
  p->d.fwd_pchans = reinterpret_cast<int32_t *>(b + parts[2].off);
  p->d.inv_packets = reinterpret_cast<PacketDev *>(b + parts[3].off);
  p->d.inv_pchans = reinterpret_cast<int32_t *>(b + parts[4].off);
  p->d.chunks = reinterpret_cast<ChunkDev *>(b + parts[5].off);
  p->d.gdual = reinterpret_cast<float *>(b + parts[6].off);
  p->d.g = reinterpret_cast<float *>(b + parts[7].off);
  p->d.h0 = reinterpret_cast<float *>(b + parts[8].off);
  p->d.h0dual = reinterpret_cast<float *>(b + parts[9].off);
  p->d.tw2n = reinterpret_cast<float *>(b + parts[10].off);
  p->d.twM = reinterpret_cast<float *>(b + parts[11].off);
  e = cudaMemcpy(blk, host.data(), o, cudaMemcpyHostToDevice);
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  int rc = 0;
  switch (p->kc.logN) {
    case 11: rc = set_attrs<11>(p->kc.fwd_smem, p->kc.inv_smem); break;
    case 12: rc = set_attrs<12>(p->kc.fwd_smem, p->kc.inv_smem); break;
    case 13: rc = set_attrs<13>(p->kc.fwd_smem, p->kc.inv_smem); break;
    case 14: rc = set_attrs<14>(p->kc.fwd_smem, p->kc.inv_smem); break;
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
  const size_t cnt = align_up(sizeof(unsigned) * (size_t)(batch * nslices));
  return cnt + sizeof(float) * (size_t)(batch * nslices * 2 * p->tr);
}

static KArgs base_args(const slicq_plan *p) {
  KArgs a{};
  a.tr = (int)p->tr;
  a.C = p->C;
  a.chan = p->d.chan;
  a.chunks = p->d.chunks;
  a.nchunks = p->kc.nchunks;
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
  a.packets = p->d.fwd_packets;
  a.pchans = p->d.fwd_pchans;
  a.npackets = p->kc.fwd_npackets;
  a.scr = p->kc.fwd_scr;
  dim3 grid((unsigned)nslices, (unsigned)batch);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->kc.logN) {
    case 11: e = launch_fwd<11>(a, grid, p->kc.fwd_smem, s); break;
    case 12: e = launch_fwd<12>(a, grid, p->kc.fwd_smem, s); break;
    case 13: e = launch_fwd<13>(a, grid, p->kc.fwd_smem, s); break;
    case 14: e = launch_fwd<14>(a, grid, p->kc.fwd_smem, s); break;
    default: return set_error(SLICQ_EINTERNAL, "bad logN");
  }
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("forward launch: ") + cudaGetErrorString(e));
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
  a.packets = p->d.inv_packets;
  a.pchans = p->d.inv_pchans;
  a.scr = p->kc.inv_scr;
  a.cnt = static_cast<unsigned *>(ws);
  a.bnd = reinterpret_cast<float *>(static_cast<char *>(ws) +
                                    align_up(sizeof(unsigned) * (size_t)(batch * nslices)));
  dim3 grid((unsigned)nslices, (unsigned)batch);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->kc.logN) {
    case 11: e = launch_inv<11>(a, grid, p->kc.inv_smem, s); break;
    case 12: e = launch_inv<12>(a, grid, p->kc.inv_smem, s); break;
    case 13: e = launch_inv<13>(a, grid, p->kc.inv_smem, s); break;
    case 14: e = launch_inv<14>(a, grid, p->kc.inv_smem, s); break;
    default: return set_error(SLICQ_EINTERNAL, "bad logN");
  }
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("inverse launch: ") + cudaGetErrorString(e));
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
  if (e != cudaSuccess)
    return set_error(SLICQ_ECUDA, std::string("overlap_add launch: ") + cudaGetErrorString(e));
  return SLICQ_OK;
}

}  // namespace slicq

// Debug only (not part of include/slicq.h): accumulated per-phase clock64 cycles of the
// forward [0..15] and inverse [16..31] kernels, in a library built with
// -DSLICQ_PHASE_TIMING (tools/phase_timing.py).  Returns -1 in the product build.
extern "C" __attribute__((visibility("default"))) int slicq_debug_phase_times(
    int logN, unsigned long long *out32, int reset) {
  switch (logN) {
    case 11: return slicq::kern::phase_times<11>(out32, reset);
    case 12: return slicq::kern::phase_times<12>(out32, reset);
    case 13: return slicq::kern::phase_times<13>(out32, reset);
    case 14: return slicq::kern::phase_times<14>(out32, reset);
  }
  return -1;
}
