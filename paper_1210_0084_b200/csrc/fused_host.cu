// Host side of the fused kernels (kernels_fused.cuh): warp-task tables, synthesis cores and
// overflow lists, shared-memory budgets.  Built at plan creation (fp64 plan -> int tables and
// fp32 weights); no per-call host work beyond the launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "kernels_fused.cuh"
#include "kernels_ring.cuh"
#include "slicq_internal.h"

namespace slicq {
namespace {
using namespace slicq::kern;

const int kFSizes[] = {2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 18, 20, 24, 25, 27, 30, 32};
const int kFSmall[] = {4, 6, 8, 10, 12, 16, 18, 20, 24, 30, 32};
constexpr int kScrCap = 640;  // float2 scratch entries a two-step task may use (5 KB per warp)

bool in_arr(const int *l, int n, int v) {
  for (int i = 0; i < n; ++i)
    if (l[i] == v) return true;
  return false;
}
bool fsize(int v) { return in_arr(kFSizes, sizeof(kFSizes) / sizeof(int), v); }
bool fsmall(int v) { return in_arr(kFSmall, sizeof(kFSmall) / sizeof(int), v); }

int64_t env_i(const char *name, int64_t dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoll(v);
}

// issue-slot cost model of one warp round (instructions per lane item), used only to pick
// task shapes: fold / load per point, DFT, twiddles, stores
double dft_cost(int R) { return R <= 1 ? 0.0 : R * (2.5 * std::log2((double)R) + 1.0); }
double cost_small(int M) { return M * 9.0 + dft_cost(M) + M * 0.5 + 15.0; }
double cost_s1(int M1) { return M1 * 9.0 + dft_cost(M1) + (M1 - 1) * 5.0 + M1 + 25.0; }
double cost_s2(int M2) { return M2 * 2.0 + dft_cost(M2) + 12.0; }

uint32_t mag16(int m) { return (uint32_t)((65536 + m - 1) / m); }
bool mag_exact(int m, int qmax) {  // (q * ceil(2^16/m)) >> 16 == q / m for q < qmax
  const uint32_t g = mag16(m);
  for (int q = 0; q < qmax; ++q)
    if ((int)((q * g) >> 16) != q / m) return false;
  return true;
}

struct Shape {
  bool small = false;
  int m1 = 0, m2 = 0, nch = 1;
  double cost = 1e300;
};

// best task shape for a group of G channels of length M: returns the shape and the task
// sizes (as equal as possible)
Shape best_shape(int M, int G) {
  Shape best;
  if (fsmall(M)) {
    const int nt = (G + 31) / 32;
    best.small = true;
    best.m1 = M;
    best.m2 = 1;
    best.nch = (G + nt - 1) / nt;
    best.cost = nt * (cost_small(M) + 20.0);
  }
  for (int m1 : kFSizes) {
    if (M % m1) continue;
    const int m2 = M / m1;
    if (!fsize(m2)) continue;
    for (int n = 1; n <= G; ++n) {
      if (n * m1 * (m2 | 1) > kScrCap) break;
      if (!mag_exact(m2, n * m2) || !mag_exact(m1, n * m1)) continue;
      const int nt = (G + n - 1) / n;
      const int nn = (G + nt - 1) / nt;  // channels per task after balancing
      const double c = nt * (((nn * m2 + 31) / 32) * cost_s1(m1) + ((nn * m1 + 31) / 32) * cost_s2(m2) + 30.0);
      if (c < best.cost) {
        best.small = false;
        best.m1 = m1;
        best.m2 = m2;
        best.nch = nn;
        best.cost = c;
      }
    }
  }
  return best;
}

// ring kernels: the cost of G channels of length M per unit, as tasks of nch channels with sf
// units side by side in the lanes (each lane item runs rounds of 32)
struct RShape {
  bool small = false;
  int m1 = 0, m2 = 0, nch = 1, sf = 1;
  double cost = 1e300;
};
RShape ring_shape(int M, int G, int bt, int scr_cap) {
  RShape best;
  const int sf = bt;  // a channel item runs every task for all bt units
  if (fsmall(M)) {
    for (int n = 1; n <= G && n <= 32; ++n) {
      const int nt = (G + n - 1) / n, nn = (G + nt - 1) / nt;
      if (!mag_exact(nn, sf * nn)) continue;
      const double c = nt * (((sf * nn + 31) / 32) * cost_small(M) + 10.0) / sf;
      if (c < best.cost) best = RShape{true, M, 1, nn, sf, c};
    }
  }
  for (int m1 : kFSizes) {
    if (M % m1) continue;
    const int m2 = M / m1;
    if (!fsize(m2)) continue;
    for (int n = 1; n <= G; ++n) {
      if (sf * n * m1 * (m2 | 1) > scr_cap) break;
      const int nt = (G + n - 1) / n, nn = (G + nt - 1) / nt;
      const int pa = nn * m2, pb = nn * m1;
      if (!mag_exact(pa, sf * pa) || !mag_exact(m2, pa) || !mag_exact(pb, sf * pb) ||
          !mag_exact(m1, pb))
        continue;
      const double c = nt * (((sf * pa + 31) / 32) * cost_s1(m1) + ((sf * pb + 31) / 32) * cost_s2(m2) + 10.0) / sf;
      if (c < best.cost) best = RShape{false, m1, m2, nn, sf, c};
    }
  }
  return best;
}

}  // namespace

int configure_fused(slicq_plan *p) {
  KernelConfig &kc = p->kc;
  kc.fused = kc.ftables = false;
  kc.cluster = 0;
  // the fused per-slice forward (opt-in: measured slower), the ring kernel
  // (opt-in) and the band-major channel kernel share these tables
  const bool want = env_i("SLICQ_FUSED", 0) || env_i("SLICQ_CLUSTER", 0) || env_i("SLICQ_RING", 0) || env_i("SLICQ_BAND", 0) ||
                    env_i("SLICQ_FWD2", 0);
  if (!want) return SLICQ_OK;
  if (kc.longmode || kc.large || kc.logN < 11 || kc.logN > 14 || !p->painless) return SLICQ_OK;
  const int K2 = p->K + 2;
  const int N = (int)p->N, N2 = 2 * N;
  for (int k = 0; k < K2; ++k)
    if (p->M[k] > 1024) return SLICQ_OK;  // (two sizes <= 32)

  // fp32 weights g_k / sqrt(M_k) and g~_k / sqrt(M_k) (x 1/2 on the self-mirrored plateaus,
  // C15), at the filter offsets goff_k (Alg. 1 sqrt(M) IFFT incl. 1/M; Alg. 2 FFT / sqrt(M); C1)
  const int64_t nterms = (int64_t)p->g.size();
  p->lgw.assign(nterms, 0.f);
  p->lgdw.assign(nterms, 0.f);
  for (int k = 0; k < K2; ++k) {
    const double sc = 1.0 / std::sqrt((double)p->M[k]);
    const double half = (k == 0 || k == K2 - 1) ? 0.5 : 1.0;
    for (int d = 0; d < p->len[k]; ++d) {
      const int64_t e = p->goff[k] + d;
      p->lgw[e] = (float)(p->g[e] * sc);
      p->lgdw[e] = (float)(p->gdual[e] * sc * half);
    }
  }

  // ---- synthesis cores (I3): CQ channel k adds its terms d in [d0, d1) straight into bin
  // lo + d of the shared half spectrum in phase k & 1; within a phase the cores are
  // disjoint, so the adds need no atomics and the sum order is fixed.  Eligible: bins
  // 1..N-1 (single, unconjugated target, C15) covered by no other channel of the same phase.
  std::vector<int> d0(K2, 0), d1(K2, 0);
  {
    std::vector<uint8_t> cover[2] = {std::vector<uint8_t>(N + 1, 0), std::vector<uint8_t>(N + 1, 0)};
    for (int k = 1; k < K2 - 1; ++k)
      for (int d = 0; d < p->len[k]; ++d) {
        const int j = p->lo[k] + d;
        if (j >= 1 && j <= N - 1 && cover[k & 1][j] < 2) ++cover[k & 1][j];
      }
    for (int k = 1; k < K2 - 1; ++k) {
      int bs = 0, be = 0, s = -1;
      for (int d = 0; d <= p->len[k]; ++d) {
        const int j = p->lo[k] + d;
        const bool ok = d < p->len[k] && j >= 1 && j <= N - 1 && cover[k & 1][j] == 1;
        if (ok && s < 0) s = d;
        if (!ok && s >= 0) {
          if (d - s > be - bs) bs = s, be = d;
          s = -1;
        }
      }
      d0[k] = bs;
      d1[k] = be;
    }
  }
  // ---- overflow: every non-core term gets one slot per unit (its weighted value); the bins
  // it reaches (direct j mod 2N if <= N, conjugate at -j mod 2N if <= N; C15) list the slot
  std::vector<int> ovoff(K2, 0);
  std::vector<std::vector<int32_t>> lists(N + 1);
  int nov = 0;
  for (int k = 0; k < K2; ++k) {
    ovoff[k] = nov;
    for (int d = 0; d < p->len[k]; ++d) {
      if (d >= d0[k] && d < d1[k]) continue;
      const int slot = nov++;
      const int j = p->lo[k] + d;
      int p1 = j % N2;
      if (p1 < 0) p1 += N2;
      const int p2 = p1 == 0 ? 0 : N2 - p1;
      if (p1 <= N) lists[p1].push_back(slot);
      if (p2 <= N) lists[p2].push_back(slot | (int32_t)0x80000000);
    }
  }
  p->ovb.clear();
  p->ovl.clear();
  for (int b = 0; b <= N; ++b) {
    if (lists[b].empty()) continue;
    if (p->ovl.size() >= (1u << 20) || lists[b].size() >= (1u << 11)) return SLICQ_OK;
    p->ovb.push_back(make_int2(b, (int)p->ovl.size() | ((int)lists[b].size() << 20)));
    p->ovl.insert(p->ovl.end(), lists[b].begin(), lists[b].end());
  }
  kc.nov = nov;
  kc.novb = (int)p->ovb.size();

  // ---- warp tasks: forward groups = runs of equal M; inverse groups = the same split by
  // channel parity (phase A even, phase B odd; plateaus are all overflow, any phase)
  auto interior = [&](int k) { return p->lo[k] >= 0 && p->lo[k] + p->len[k] - 1 <= N; };
  int fscr = 2;
  auto build = [&](bool inv, std::vector<FChan> &fch, std::vector<FTask> &tasks, int &nphase_a) {
    struct T {
      int phase;
      FTask t;
      std::vector<int> ks;
    };
    std::vector<T> ts;
    for (int k = 0; k < K2;) {
      int e = k;
      while (e < K2 && p->M[e] == p->M[k]) ++e;
      for (int ph = 0; ph < (inv ? 2 : 1); ++ph) {
        std::vector<int> grp;
        for (int q = k; q < e; ++q)
          if (!inv || (q & 1) == ph) grp.push_back(q);
        if (grp.empty()) continue;
        const int M = p->M[k];
        const Shape sh = best_shape(M, (int)grp.size());
        if (sh.cost >= 1e299) return false;
        for (size_t i = 0; i < grp.size(); i += sh.nch) {
          T t;
          t.phase = ph;
          for (size_t q = i; q < std::min(grp.size(), i + sh.nch); ++q) t.ks.push_back(grp[q]);
          bool in = true;
          for (int q : t.ks) in = in && interior(q);
          t.t.code = sh.m1 | (sh.m2 << 8) | ((sh.small ? 1 : 0) << 16) | ((in ? 1 : 0) << 17);
          t.t.nch = (int)t.ks.size();
          t.t.mags = sh.small ? 0u : (mag16(sh.m2) | (mag16(sh.m1) << 16));
          if (!sh.small) fscr = std::max(fscr, t.t.nch * sh.m1 * (sh.m2 | 1));
          ts.push_back(std::move(t));
        }
      }
      k = e;
    }
    // phase, then code shape (warps of a CTA run the same code at the same time), longer first
    std::stable_sort(ts.begin(), ts.end(), [](const T &x, const T &y) {
      if (x.phase != y.phase) return x.phase < y.phase;
      return (x.t.code & 0x1ffff) > (y.t.code & 0x1ffff);
    });
    fch.clear();
    tasks.clear();
    nphase_a = 0;
    for (T &t : ts) {
      t.t.coff = (int)fch.size();
      for (int k : t.ks) {
        FChan c{};
        const int M = p->M[k];
        const int m2 = (t.t.code >> 16) & 1 ? 1 : (t.t.code >> 8) & 255;
        c.lo = p->lo[k];
        c.len = p->len[k];
        c.M = M;
        c.goff = (int)p->goff[k];
        c.off = (int)p->off[k];
        c.twoff = k;  // channel index: upload() replaces it with the twiddle-table offset
        c.lo_mod = ((c.lo % M) + M) % M;
        c.lom2 = ((c.lo % m2) + m2) % m2;
        c.d0 = d0[k];
        c.d1 = d1[k];
        c.ovoff = ovoff[k];
        c.flags = interior(k) ? 1 : 0;
        fch.push_back(c);
      }
      if (t.phase == 0) ++nphase_a;
      tasks.push_back(t.t);
    }
    return true;
  };
  if (!build(false, p->fchf, p->ftf, kc.nphase_a)) return SLICQ_OK;
  if (!build(true, p->fchi, p->fti, kc.nphase_a)) return SLICQ_OK;
  kc.nftf = (int)p->ftf.size();
  kc.nfti = (int)p->fti.size();
  kc.fscr = (fscr + 1) & ~1;
  size_t fs = 0;
  switch (kc.logN) {
    case 11: fs = fused_fwd_smem<11>((int)p->tr, kc.fscr); break;
    case 12: fs = fused_fwd_smem<12>((int)p->tr, kc.fscr); break;
    case 13: fs = fused_fwd_smem<13>((int)p->tr, kc.fscr); break;
    case 14: fs = fused_fwd_smem<14>((int)p->tr, kc.fscr); break;
  }
  if (fs > 227 * 1024) return SLICQ_OK;
  kc.fsmem_f = fs;
  kc.ftables = true;
  kc.fused = env_i("SLICQ_FUSED", 0) != 0;
  {
    const int64_t G = env_i("SLICQ_CLUSTER", 0);
    if (!kc.fused && G >= 2 && G <= 16) kc.cluster = (int)G;
  }
  return SLICQ_OK;
}

// ---- ring kernels (kernels_ring.cuh): bands, tasks, ring sizing
int configure_ring(slicq_plan *p) {
  KernelConfig &kc = p->kc;
  kc.ring = false;
  const bool dbg = env_i("SLICQ_DEBUG", 0) != 0;
  auto off = [&](const char *why) {
    if (dbg) std::fprintf(stderr, "ring off: %s\n", why);
    return SLICQ_OK;
  };
  kc.band = false;
  if (!kc.ftables) return off("no fused tables");
  if (kc.logN != 12 && kc.logN != 13) return off("2N");  // spectrum role: 256-thread CTAs
  const int K2 = p->K + 2;
  const int N = (int)p->N, N2 = 2 * N;
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (nsm <= 0) nsm = 148;
  const int bt = (int)std::max<int64_t>(1, env_i("SLICQ_RING_BT", 8));
  int nb = (int)std::max<int64_t>(1, env_i("SLICQ_RING_NB", 48));
  const int la = (int)std::max<int64_t>(1, env_i("SLICQ_RING_LA", 4));
  const int grp = (int)std::max<int64_t>(1, env_i("SLICQ_RING_G", 4));
  const int scr_cap = (int)env_i("SLICQ_RING_SCR", 4096);
  // contiguous channel runs of balanced cost (channel order = frequency order)
  std::vector<double> cst(K2);
  double tot = 0, mx = 0;
  for (int k = 0; k < K2; ++k) {
    const double M = p->M[k];
    cst[k] = M * (11.0 + 2.5 * std::log2(M)) + 10.0;
    tot += cst[k];
    mx = std::max(mx, cst[k]);
  }
  auto pack = [&](double W, std::vector<int> *cuts) {
    int n = 1;
    double acc = 0;
    if (cuts) cuts->assign(1, 0);
    for (int k = 0; k < K2; ++k) {
      if (acc > 0 && acc + cst[k] > W) {
        ++n;
        acc = 0;
        if (cuts) cuts->push_back(k);
      }
      acc += cst[k];
    }
    if (cuts) cuts->push_back(K2);
    return n;
  };
  double lo = std::max(mx, tot / nb), hi = tot;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (pack(mid, nullptr) <= nb) hi = mid; else lo = mid;
  }
  std::vector<int> cuts;
  nb = pack(hi, &cuts);
  auto xidx = [&](int j) {  // X index a bin j reads (C15)
    int jj = j % N2;
    if (jj < 0) jj += N2;
    return jj > N ? N2 - jj : jj;
  };
  p->rband.clear();
  p->rtask.clear();
  p->rfch.clear();
  p->rbtw.clear();
  p->rround.clear();
  int fscr = 2, xstride = 2, wmax = 0, twmax = 0, meta = 0;
  for (int bi = 0; bi < nb; ++bi) {
    const int k0 = cuts[bi], k1 = cuts[bi + 1];
    RBand B{};
    int xmin = N, xmax = 0;
    for (int k = k0; k < k1; ++k)
      for (int d = 0; d < p->len[k]; ++d) {
        const int x = xidx(p->lo[k] + d);
        xmin = std::min(xmin, x);
        xmax = std::max(xmax, x);
      }
    B.blo = xmin & ~1;
    B.bspan = ((xmax + 2) & ~1) - B.blo;
    B.g0 = (int)p->goff[k0];
    B.ng = (int)(p->goff[k1 - 1] + p->len[k1 - 1] - p->goff[k0]);
    if ((p->rbtw.size() / 2) & 1) p->rbtw.insert(p->rbtw.end(), {0.f, 0.f});  // 16-byte tables
    B.tw0 = (int)(p->rbtw.size() / 2);
    B.task0 = (int)p->rtask.size();
    // band twiddle tables, one per distinct M
    std::vector<std::pair<int, int>> twl;  // (M, local offset)
    auto twoff_of = [&](int M) {
      for (auto &e : twl)
        if (e.first == M) return e.second;
      const int o = (int)(p->rbtw.size() / 2) - B.tw0;
      for (int t = 0; t < M; ++t) {
        const double ang = 2.0 * 3.14159265358979323846 * (double)t / (double)M;
        p->rbtw.push_back((float)std::cos(ang));
        p->rbtw.push_back((float)std::sin(ang));
      }
      twl.emplace_back(M, o);
      return o;
    };
    // tasks: channels of one length (any order within the band), largest first
    std::vector<int> Ms;
    for (int k = k0; k < k1; ++k)
      if (std::find(Ms.begin(), Ms.end(), p->M[k]) == Ms.end()) Ms.push_back(p->M[k]);
    std::sort(Ms.begin(), Ms.end(), std::greater<int>());
    for (int M : Ms) {
      std::vector<int> grp;
      for (int k = k0; k < k1; ++k)
        if (p->M[k] == M) grp.push_back(k);
      const RShape sh = ring_shape(M, (int)grp.size(), bt, scr_cap);
      if (sh.cost >= 1e299) return off("no task shape");
      const int tof = twoff_of(M);
      for (size_t i = 0; i < grp.size(); i += sh.nch) {
        RTask t{};
        t.nch = (int)std::min<size_t>(sh.nch, grp.size() - i);
        t.coff = (int)p->rfch.size();
        bool in = true;
        for (int c = 0; c < t.nch; ++c) {
          const int k = grp[i + c];
          FChan f{};
          f.lo = p->lo[k];
          f.len = p->len[k];
          f.M = M;
          f.goff = (int)(p->goff[k] - B.g0);
          f.off = (int)p->off[k];
          f.twoff = tof;
          f.lo_mod = ((f.lo % M) + M) % M;
          f.lom2 = sh.small ? 0 : ((f.lo % sh.m2) + sh.m2) % sh.m2;
          f.flags = (f.lo >= 0 && f.lo + f.len - 1 <= N) ? 1 : 0;
          in = in && f.flags;
          p->rfch.push_back(f);
        }
        t.code = sh.m1 | (sh.m2 << 8) | ((sh.small ? 1 : 0) << 16) | ((in ? 1 : 0) << 17);
        if (sh.small) {
          t.magPa = mag16(t.nch);
          if (!mag_exact(t.nch, bt * t.nch)) return off("magic");
        } else {
          const int pa = t.nch * sh.m2, pb = t.nch * sh.m1;
          t.magPa = mag16(pa);
          t.magM2 = mag16(sh.m2);
          t.magPb = mag16(pb);
          t.magM1 = mag16(sh.m1);
          if (!mag_exact(pa, bt * pa) || !mag_exact(sh.m2, pa) || !mag_exact(pb, bt * pb) ||
              !mag_exact(sh.m1, pb))
            return off("magic");
        }
        p->rtask.push_back(t);
      }
    }
    B.ntask = (int)p->rtask.size() - B.task0;
    B.ntw = (int)(p->rbtw.size() / 2) - B.tw0;
    // item scratch offsets of the two-step tasks; the band's 32-lane rounds per phase
    {
      int so = 0;
      std::vector<int32_t> r1, r2;
      for (int ti = 0; ti < B.ntask; ++ti) {
        RTask &t = p->rtask[B.task0 + ti];
        const int m1 = t.code & 255, m2 = (t.code >> 8) & 255;
        const bool small = (t.code >> 16) & 1;
        const int n1 = small ? bt * t.nch : bt * t.nch * m2;
        for (int q = 0; q < (n1 + 31) / 32; ++q) r1.push_back((ti << 16) | q);
        if (!small) {
          t.soff = so;
          so += bt * t.nch * m1 * (m2 | 1);
          const int n2 = bt * t.nch * m1;
          for (int q = 0; q < (n2 + 31) / 32; ++q) r2.push_back((ti << 16) | q);
        }
      }
      if (B.ntask >= (1 << 15)) return off("tasks");
      fscr = std::max(fscr, so);
      auto pad4 = [&]() {
        while (p->rround.size() & 3) p->rround.push_back(0);
      };
      pad4();
      B.r1off = (int)p->rround.size();
      B.nr1 = (int)r1.size();
      p->rround.insert(p->rround.end(), r1.begin(), r1.end());
      pad4();
      B.r2off = (int)p->rround.size();
      B.nr2 = (int)r2.size();
      p->rround.insert(p->rround.end(), r2.begin(), r2.end());
      pad4();
      B.f0 = p->rtask[B.task0].coff;
      B.nf = (int)p->rfch.size() - B.f0;
      meta = std::max(meta, (int)(sizeof(RTask) * B.ntask + sizeof(FChan) * B.nf) +
                                4 * (((B.nr1 + 3) & ~3) + ((B.nr2 + 3) & ~3)));
    }
    xstride = std::max(xstride, B.bspan);
    wmax = std::max(wmax, ((B.g0 + B.ng + 3) & ~3) - (B.g0 & ~3));
    twmax = std::max(twmax, (B.ntw + 1) & ~1);
    p->rband.push_back(B);
  }
  p->rbtw.insert(p->rbtw.end(), {0.f, 0.f, 0.f, 0.f});  // the last table's 16-byte tail
  kc.rnb = nb;
  kc.rq = 0;
  kc.rbt = bt;
  kc.rla = la;
  kc.rnspec = 2 * nsm;  // CTAs of the launch (two per SM)
  kc.rnchan = 0;
  kc.rxstride = (xstride + 1) & ~1;
  kc.rwmax = wmax;
  kc.rtwmax = twmax;
  kc.rfscr = (fscr + 1) & ~1;
  kc.rslot = N + 2;
  kc.rgroup = grp;
  kc.rmeta = (meta + 15) & ~15;
  const ChanSmem L = chan_smem_layout(bt, kc.rxstride, wmax, twmax, kc.rfscr, kc.rmeta);
  kc.rsmem = kc.logN == 12 ? ring_smem<12>((int)p->tr, L.total) : ring_smem<13>((int)p->tr, L.total);
  if (dbg)
    std::fprintf(stderr, "ring smem: meta %d w+tw %zu xset %zu scr %zu chan %zu total %zu (xstride %d iscr %d)\n",
                 kc.rmeta, L.set[0] - L.w, L.set[1] - L.set[0], L.total - L.scr, L.total, kc.rsmem, kc.rxstride, kc.rfscr);
  kc.rchsmem = L.total;
  if (kc.rchsmem <= 112 * 1024) kc.band = env_i("SLICQ_BAND", 0) != 0;
  if (kc.rsmem > 112 * 1024) return off("shared memory");  // two CTAs per SM
  const int64_t ring_mb = env_i("SLICQ_RING_MB", 32);
  const int64_t need = (int64_t)(la + 2) * bt * grp + 2 * (int64_t)kc.rnspec;
  kc.rR = (int)std::max<int64_t>(need, (ring_mb << 20) / (kc.rslot * 8));
  kc.ring = env_i("SLICQ_RING", 0) != 0;
  if (env_i("SLICQ_DEBUG", 0))
    std::fprintf(stderr, "ring: nb=%d la=%d bt=%d grid=%d xstride=%d wmax=%d twmax=%d fscr=%d "
                         "smem=%zu R=%d tasks=%zu\n",
                 nb, la, bt, kc.rnspec, kc.rxstride, wmax, twmax, kc.rfscr, kc.rsmem, kc.rR,
                 p->rtask.size());
  if (env_i("SLICQ_DEBUG", 0) > 1)
    for (size_t bi = 0; bi < p->rband.size(); ++bi) {
      const RBand &B = p->rband[bi];
      std::fprintf(stderr, "band %zu: blo=%d bspan=%d ng=%d ntw=%d\n", bi, B.blo, B.bspan, B.ng, B.ntw);
      for (int t = B.task0; t < B.task0 + B.ntask; ++t) {
        const RTask &T = p->rtask[t];
        std::fprintf(stderr, "  task m1=%d m2=%d small=%d inter=%d nch=%d soff=%d k0.lo=%d\n",
                     T.code & 255, (T.code >> 8) & 255, (T.code >> 16) & 1, (T.code >> 17) & 1,
                     T.nch, T.soff, p->rfch[T.coff].lo);
      }
    }
  return SLICQ_OK;
}

// ---- forward channel kernel v2 (kernels_chan2.cuh): packets of equal-length channels with
// multi-round warp tasks (shapes chosen to fill the lanes), table-free contiguous folds
int configure_fwd2(slicq_plan *p) {
  KernelConfig &kc = p->kc;
  kc.fwd2 = false;
  if (!kc.ftables || kc.large || env_i("SLICQ_FWD2", 0) == 0) return SLICQ_OK;
  const int K2 = p->K + 2;
  const int N = (int)p->N;
  const int tile = kc.tile;
  const int SCR = (int)env_i("SLICQ_FWD2_SCR", 1024), RMAX = 4;
  auto interior = [&](int k) { return p->lo[k] >= 0 && p->lo[k] + p->len[k] - 1 <= N; };
  struct Pk {
    P2Dev d;
    std::vector<int> ks;
    int var;
  };
  std::vector<Pk> pks;
  std::vector<int> Ms;
  for (int k = 0; k < K2; ++k)
    if (std::find(Ms.begin(), Ms.end(), p->M[k]) == Ms.end()) Ms.push_back(p->M[k]);
  int scr = 2;
  for (int M : Ms) {
    std::vector<int> grp;
    for (int k = 0; k < K2; ++k)
      if (p->M[k] == M) grp.push_back(k);
    const int G = (int)grp.size();
    // best (small | m1, m2, nch, nu) by issue cost per channel-unit
    struct Best {
      double cost = 1e300;
      bool small = false;
      int m1 = 0, m2 = 0, nch = 1, nu = 1;
    } best;
    auto consider = [&](bool small, int m1, int m2, int nch, int nu) {
      const int nvc = nch * nu;
      if (nu > tile) return;
      double c;
      if (small) {
        if (nvc > 32 || !mag_exact(nch, nvc)) return;
        c = (cost_small(M) + 20.0) / nvc;
      } else {
        const int i1 = nvc * m2, i2 = nvc * m1;
        if ((i1 + 31) / 32 > RMAX || (i2 + 31) / 32 > RMAX) return;
        if (nvc * m1 * (m2 | 1) > SCR) return;
        if (!mag_exact(m2, i1) || !mag_exact(m1, i2) || !mag_exact(nch, nvc)) return;
        c = (((i1 + 31) / 32) * cost_s1(m1) + ((i2 + 31) / 32) * cost_s2(m2) + 40.0) / nvc;
      }
      // coalescing: lanes of one unit read neighbouring bins and write neighbouring columns;
      // lanes spread over units do neither (each touches another row)
      c *= 1.0 + 0.5 * (1.0 - (double)nch / nvc);
      if (c < best.cost - 1e-9) best = Best{c, small, m1, m2, nch, nu};
    };
    for (int nch = 1; nch <= std::min(G, 32); ++nch)
      for (int nu = 1; nu <= 32; ++nu) {
        if (fsmall(M)) consider(true, M, 1, nch, nu);
        for (int m1 : kFSizes) {
          if (M % m1 || !fsize(M / m1)) continue;
          consider(false, m1, M / m1, nch, nu);
        }
      }
    if (best.cost >= 1e299) return SLICQ_OK;
    for (int i = 0; i < G; i += best.nch) {
      Pk pk;
      for (int q = i; q < std::min(G, i + best.nch); ++q) pk.ks.push_back(grp[q]);
      const int r = (int)pk.ks.size();
      // units per task for this packet's channel count (the last packet may be shorter)
      int nu = std::max(1, best.nu * best.nch / r);
      while (nu > 1) {
        const int nvc = r * nu;
        const bool ok = best.small ? (nvc <= 32 && mag_exact(r, nvc))
                                   : ((nvc * best.m2 + 31) / 32 <= RMAX && (nvc * best.m1 + 31) / 32 <= RMAX &&
                                      nvc * best.m1 * (best.m2 | 1) <= SCR && mag_exact(best.m2, nvc * best.m2) &&
                                      mag_exact(best.m1, nvc * best.m1) && mag_exact(r, nvc));
        if (ok) break;
        --nu;
      }
      if (!mag_exact(r, r * nu)) return SLICQ_OK;
      bool in = true;
      for (int k : pk.ks) in = in && interior(k);
      pk.d = P2Dev{};
      pk.d.code = best.m1 | (best.m2 << 8) | ((best.small ? 1 : 0) << 16) | ((in ? 1 : 0) << 17);
      pk.d.nch = r;
      pk.d.nu = nu;
      pk.d.magA = mag16(best.m2);
      pk.d.magB = mag16(best.m1);
      pk.d.magC = mag16(r);
      pk.var = std::max(best.m1, best.m2) <= 16 ? 0 : 1;
      if (!best.small) scr = std::max(scr, r * nu * best.m1 * (best.m2 | 1));
      pks.push_back(std::move(pk));
    }
  }
  std::stable_sort(pks.begin(), pks.end(), [](const Pk &x, const Pk &y) {
    if (x.var != y.var) return x.var < y.var;
    return (x.d.code & 0x1ffff) > (y.d.code & 0x1ffff);
  });
  p->f2pk.clear();
  p->f2ch.clear();
  kc.f2voff[0] = kc.f2voff[1] = kc.f2voff[2] = 0;
  for (Pk &pk : pks) {
    pk.d.coff = (int)p->f2ch.size();
    const int m2 = (pk.d.code >> 16) & 1 ? 1 : (pk.d.code >> 8) & 255;
    for (int k : pk.ks) {
      FChan c{};
      const int M = p->M[k];
      c.lo = p->lo[k];
      c.len = p->len[k];
      c.M = M;
      c.goff = (int)p->goff[k];
      c.off = (int)p->off[k];
      c.twoff = k;  // channel index: upload() replaces it with the twiddle-table offset
      c.lo_mod = ((c.lo % M) + M) % M;
      c.lom2 = ((c.lo % m2) + m2) % m2;
      c.flags = interior(k) ? 1 : 0;
      p->f2ch.push_back(c);
    }
    ++kc.f2voff[pk.var + 1];
    p->f2pk.push_back(pk.d);
  }
  kc.f2voff[2] += kc.f2voff[1];
  kc.f2scr = (scr + 1) & ~1;
  kc.fwd2 = true;
  if (env_i("SLICQ_DEBUG", 0))
    std::fprintf(stderr, "fwd2: %zu packets (lite %d, full %d), scratch %d\n", p->f2pk.size(),
                 kc.f2voff[1], kc.f2voff[2] - kc.f2voff[1], kc.f2scr);
  if (env_i("SLICQ_DEBUG", 0) > 1)
    for (const P2Dev &d : p->f2pk)
      std::fprintf(stderr, "  pk m1=%d m2=%d small=%d inter=%d nch=%d nu=%d\n", d.code & 255,
                   (d.code >> 8) & 255, (d.code >> 16) & 1, (d.code >> 17) & 1, d.nch, d.nu);
  return SLICQ_OK;
}

int fused_set_attrs(const slicq_plan *p) {
  int rc = 0;
  switch (p->kc.logN) {
    case 11: rc = fused_attrs<11>(); break;
    case 12: rc = fused_attrs<12>(); break;
    case 13: rc = fused_attrs<13>(); break;
    case 14: rc = fused_attrs<14>(); break;
  }
  if (rc == 0 && (p->kc.ring || p->kc.band)) {
    if (p->kc.logN == 12) rc = ring_attrs<12>();
    if (p->kc.logN == 13) rc = ring_attrs<13>();
  }
  return rc;
}

}  // namespace slicq
