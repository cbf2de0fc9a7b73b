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

constexpr size_t kSmemCap = 227 * 1024;

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct ChanSlot {  // where a channel's F_k lives in its chunk's scratch (inverse)
  int chunk = -1, region = 0, ci = 0, m1 = 1, s2 = 1;
};

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

  // ---------------- forward: packets grouped by length, shape-sorted (I-cache locality),
  // larger packets first (dynamic scheduling tail)
  {
    std::map<int, std::vector<int>> groups;
    for (int k = 0; k < K2; ++k) groups[p->M[k]].push_back(k);
    struct G { int M, cost; };
    std::vector<G> order;
    for (auto &kv : groups) {
      const int m1 = fac[kv.first].first, m2 = fac[kv.first].second;
      order.push_back({kv.first, nch_for(m1, m2) * kv.first * (m1 + m2)});
    }
    std::stable_sort(order.begin(), order.end(), [](const G &x, const G &y) { return x.cost > y.cost; });
    p->fwd_packets.clear();
    p->fwd_pchans.clear();
    int need = 8;
    for (const G &g : order) {
      const int m1 = fac[g.M].first, m2 = fac[g.M].second, nch = nch_for(m1, m2);
      const std::vector<int> &ks = groups[g.M];
      for (size_t i = 0; i < ks.size(); i += nch) {
        PacketDev pk{};
        pk.nch = (int)std::min<size_t>(nch, ks.size() - i);
        pk.m1m2 = m1 | (m2 << 8);
        pk.chan_off = (int)p->fwd_pchans.size();
        for (int c = 0; c < pk.nch; ++c) p->fwd_pchans.push_back(ks[i + c]);
        p->fwd_packets.push_back(pk);
        need = std::max(need, pk.nch * m1 * (m2 | 1));
      }
    }
    kc.fwd_scr = (need + 7) & ~7;
    kc.fwd_smem = fwd_smem_for(logN, kc.fwd_scr);
    kc.fwd_npackets = (int)p->fwd_packets.size();
    if (kc.fwd_smem > kSmemCap)
      return set_error(SLICQ_EUNSUPPORTED, "forward scratch does not fit in shared memory");
  }

  // ---------------- inverse: packets of consecutive equal-length channels, cut into chunks
  // whose F_k fit in shared memory; per chunk a per-bin gather list (CSR).
  {
    const int cap = (int)((kSmemCap - inv_smem_for(logN, 0)) / sizeof(float2)) & ~7;
    struct Pk { PacketDev d; std::vector<int> ks; int size; };
    std::vector<Pk> pks;
    for (int k = 0; k < K2;) {
      const int M = p->M[k];
      const int m1 = fac[M].first, m2 = fac[M].second, nch = nch_for(m1, m2);
      Pk pk;
      pk.d.m1m2 = m1 | (m2 << 8);
      while (k < K2 && p->M[k] == M && (int)pk.ks.size() < nch) pk.ks.push_back(k++);
      pk.d.nch = (int)pk.ks.size();
      pk.size = pk.d.nch * m1 * (m2 | 1);
      pks.push_back(pk);
    }
    // chunks of consecutive packets
    std::vector<std::vector<int>> chunk_pk(1);
    int used = 0;
    for (int i = 0; i < (int)pks.size(); ++i) {
      if (pks[i].size > cap)
        return set_error(SLICQ_EUNSUPPORTED, "inverse channel scratch does not fit in shared memory");
      if (used + pks[i].size > cap) {
        chunk_pk.emplace_back();
        used = 0;
      }
      chunk_pk.back().push_back(i);
      used += pks[i].size;
    }
    std::vector<ChanSlot> slot(K2);
    p->inv_packets.clear();
    p->inv_pchans.clear();
    p->chunks.clear();
    p->bin_off.clear();
    p->gents.clear();
    int maxscr = 8;
    for (int c = 0; c < (int)chunk_pk.size(); ++c) {
      std::vector<int> &ids = chunk_pk[c];
      // shape-sort inside the chunk (warps walk packets pk0 + warp, pk0 + warp + NW, ...)
      std::stable_sort(ids.begin(), ids.end(),
                       [&](int x, int y) { return pks[x].d.m1m2 < pks[y].d.m1m2; });
      ChunkDev ck{};
      ck.pk0 = (int)p->inv_packets.size();
      int region = 0;
      for (int i : ids) {
        Pk &pk = pks[i];
        pk.d.region = region;
        pk.d.chan_off = (int)p->inv_pchans.size();
        const int m1 = pk.d.m1m2 & 255, m2 = pk.d.m1m2 >> 8;
        for (int ci = 0; ci < pk.d.nch; ++ci) {
          const int k = pk.ks[ci];
          p->inv_pchans.push_back(k);
          slot[k] = {c, region, ci, m1, m2 | 1};
        }
        p->inv_packets.push_back(pk.d);
        region += pk.size;
      }
      ck.pk1 = (int)p->inv_packets.size();
      maxscr = std::max(maxscr, region);
      // gather terms of the chunk's channels
      struct Term { int bin; int k; GatherEnt e; };
      std::vector<Term> terms;
      for (int i : ids)
        for (int k : pks[i].ks) {
          const ChanSlot &sl = slot[k];
          const int M = p->M[k];
          const int lo_mod = ((p->lo[k] % M) + M) % M;
          const double half = (k == 0 || k == K2 - 1) ? 0.5 : 1.0;  // self-mirrored plateaus
          const double sc = half / std::sqrt((double)M);
          for (int d = 0; d < p->len[k]; ++d) {
            const int j = p->lo[k] + d;
            int q = lo_mod + d;
            if (q >= M) q -= M;
            const uint32_t fidx = (uint32_t)(sl.region + sl.ci * sl.m1 * sl.s2 + q);
            const float gv = (float)(p->gdual[p->goff[k] + d] * sc);
            int p1 = j % N2;
            if (p1 < 0) p1 += N2;
            if (p1 <= N) terms.push_back({p1, k, {fidx, gv}});
            const int p2 = p1 == 0 ? 0 : N2 - p1;
            if (p2 <= N) terms.push_back({p2, k, {fidx | 0x80000000u, gv}});
          }
        }
      std::stable_sort(terms.begin(), terms.end(), [](const Term &x, const Term &y) {
        return x.bin != y.bin ? x.bin < y.bin : x.k < y.k;
      });
      ck.blo = terms.empty() ? 0 : terms.front().bin;
      ck.bhi = terms.empty() ? -1 : terms.back().bin;
      ck.bin_base = (int)p->bin_off.size();
      size_t t = 0;
      for (int b = ck.blo; b <= ck.bhi + 1; ++b) {
        while (t < terms.size() && terms[t].bin < b) ++t;
        p->bin_off.push_back((int32_t)(p->gents.size() + t));
      }
      for (const Term &tm : terms) p->gents.push_back(tm.e);
      p->chunks.push_back(ck);
    }
    kc.inv_scr = (maxscr + 7) & ~7;
    kc.inv_smem = inv_smem_for(logN, kc.inv_scr);
    kc.nchunks = (int)p->chunks.size();
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
  std::vector<float> g(nG);
  for (int k = 0; k < K2; ++k) {
    const double sc = 1.0 / std::sqrt((double)p->M[k]);  // Alg. 1: sqrt(M) * IFFT (1/M)
    for (int i = 0; i < p->len[k]; ++i) g[p->goff[k] + i] = (float)(p->g[p->goff[k] + i] * sc);
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
      {p->bin_off.data(), sizeof(int32_t) * p->bin_off.size(), 0},
      {p->gents.data(), sizeof(GatherEnt) * p->gents.size(), 0},
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
  p->d.bin_off = reinterpret_cast<int32_t *>(b + parts[6].off);
  p->d.gents = reinterpret_cast<GatherEnt *>(b + parts[7].off);
  p->d.g = reinterpret_cast<float *>(b + parts[8].off);
  p->d.h0 = reinterpret_cast<float *>(b + parts[9].off);
  p->d.h0dual = reinterpret_cast<float *>(b + parts[10].off);
  p->d.tw2n = reinterpret_cast<float *>(b + parts[11].off);
  p->d.twM = reinterpret_cast<float *>(b + parts[12].off);
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
  a.bin_off = p->d.bin_off;
  a.gents = p->d.gents;
  a.nchunks = p->kc.nchunks;
  a.g = p->d.g;
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
