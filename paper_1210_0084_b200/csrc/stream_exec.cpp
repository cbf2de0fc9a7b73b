// Native streaming executor: host-to-host sliCQ round trip of a long signal, pipelined over
// slice ranges (slicq_process_host, include/slicq.h).
//
// The S slices of the signal are cut into P contiguous ranges.  Range r runs on three
// streams forked from the caller's stream:
//   in : host -> device copy of its input samples [s0 N - halo, (s0 + ns) N) (circular for
//        range 0; zeros past the signal end, C13)
//   k  : slicq_forward_range -> optional coefficient hook -> slicq_inverse_range, then the
//        overlap-add of this range's left spill into range r-1's tail (slicq_overlap_add)
//   out: device -> host copy of range r-1's samples once that spill has been added
// Device buffers are a ring of R slots (input, coefficients, output, spill) carved from
// the caller's workspace; slot reuse waits for the device -> host copy of the range that
// last used it.  The arithmetic is exactly that of slicq_forward + slicq_inverse (the same
// range kernels the multi-GPU path uses; tests check bit equality).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "slicq_internal.h"

namespace {
#ifndef SLICQ_EXEC_SLOTS
#define SLICQ_EXEC_SLOTS 4
#endif
constexpr int kSlots = SLICQ_EXEC_SLOTS;
#ifndef SLICQ_EXEC_SPLIT
#define SLICQ_EXEC_SPLIT 1
#endif
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Range boundaries over S slices: the first and last kRamp ranges are shorter (weights
// 1/kRamp, 2/kRamp, ...) so that the pipeline fills and drains quickly -- the first
// copy-in and the last copy-out are not overlapped with anything.
constexpr int kRamp = 4;
std::vector<int64_t> range_bounds(int64_t S, int P) {
  std::vector<double> w(P);
  double tot = 0.0;
  for (int r = 0; r < P; ++r) {
    const int d = std::min(r + 1, P - r);
    w[r] = d >= kRamp ? 1.0 : (double)d / kRamp;
    tot += w[r];
  }
  std::vector<int64_t> b(P + 1, 0);
  double acc = 0.0;
  for (int r = 0; r < P; ++r) {
    acc += w[r];
    b[r + 1] = (int64_t)(S * acc / tot + 0.5);
    b[r + 1] = std::max(b[r + 1], b[r] + 1);                 // every range >= 1 slice
    b[r + 1] = std::min(b[r + 1], S - (int64_t)(P - 1 - r));  // room for the rest
  }
  b[P] = S;
  return b;
}

struct ExecLayout {
  int P = 0;             // ranges
  int64_t S = 0, N = 0, halo = 0, nsmax = 0, C = 0;
  int64_t xw = 0, yw = 0;  // row widths (floats) of the input / output slot buffers
  size_t x = 0, c = 0, y = 0, sp = 0, slot = 0;  // slot-relative offsets, slot size
  size_t sp0 = 0, ws = 0, ws_bytes = 0, total = 0;
};

ExecLayout exec_layout(const slicq_plan *p, int64_t n, int64_t batch, int pieces) {
  ExecLayout e;
  e.N = p->N;
  const int64_t L2N = 2 * p->N;
  const int64_t Lpad = ((n + L2N - 1) / L2N) * L2N;
  e.S = Lpad / p->N;
  e.P = (int)std::max<int64_t>(1, std::min<int64_t>(pieces, e.S / 2));
  e.halo = ((p->N + p->tr) / 2 + 1) & ~int64_t(1);  // >= slicq_halo, even
  {
    const std::vector<int64_t> b = range_bounds(e.S, e.P);
    for (int r = 0; r < e.P; ++r) e.nsmax = std::max(e.nsmax, b[r + 1] - b[r]);
  }
  e.C = p->C;
  e.xw = e.halo + e.nsmax * p->N;
  e.yw = e.nsmax * p->N;
  e.x = 0;
  e.c = align256(e.x + sizeof(float) * (size_t)(batch * e.xw));
  e.y = align256(e.c + sizeof(slicq_c32) * (size_t)(batch * e.nsmax * e.C));
  e.sp = align256(e.y + sizeof(float) * (size_t)(batch * e.yw));
  e.slot = align256(e.sp + sizeof(float) * (size_t)(batch * e.halo));
  e.sp0 = e.slot * kSlots;
  e.ws = align256(e.sp0 + sizeof(float) * (size_t)(batch * e.halo));
  e.ws_bytes = slicq::workspace_bytes(p, e.nsmax, batch);
  e.total = e.ws + e.ws_bytes;
  return e;
}
}  // namespace

using slicq::set_error;

extern "C" {

size_t slicq_process_host_workspace_bytes(const slicq_plan *p, int64_t n, int64_t batch,
                                          int pieces) {
  if (!p || !p->has_device || n < 1 || batch < 1 || pieces < 1) return 0;
  return exec_layout(p, n, batch, pieces).total;
}

int slicq_process_host(const slicq_plan *p, const float *x_host, float *y_host, int64_t n,
                       int64_t batch, int pieces, slicq_coeff_fn fn, void *user, void *ws,
                       size_t ws_bytes, void *stream) {
  if (!p) return set_error(SLICQ_EINVAL, "plan is NULL");
  if (!p->has_device) return set_error(SLICQ_EINVAL, "host-only plan");
  if (!x_host || !y_host || n < 1 || batch < 1 || pieces < 1)
    return set_error(SLICQ_ESHAPE, "bad process_host arguments");
  const ExecLayout e = exec_layout(p, n, batch, pieces);
  if (!ws || ws_bytes < e.total) return set_error(SLICQ_ESHAPE, "workspace too small");
  if ((uintptr_t)ws % 256) return set_error(SLICQ_ESHAPE, "workspace must be 256-byte aligned");
  const int64_t N = e.N, S = e.S, L = S * N, halo = e.halo, B = batch;
  const int P = e.P;
  const std::vector<int64_t> bounds = range_bounds(S, P);
  char *base = static_cast<char *>(ws);
  auto slot_x = [&](int r) { return reinterpret_cast<float *>(base + (r % kSlots) * e.slot + e.x); };
  auto slot_c = [&](int r) {
    return reinterpret_cast<slicq_c32 *>(base + (r % kSlots) * e.slot + e.c);
  };
  auto slot_y = [&](int r) { return reinterpret_cast<float *>(base + (r % kSlots) * e.slot + e.y); };
  auto spill = [&](int r) {
    return r == 0 ? reinterpret_cast<float *>(base + e.sp0)
                  : reinterpret_cast<float *>(base + (r % kSlots) * e.slot + e.sp);
  };
  void *rws = base + e.ws;

  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};  // in, k, out
  std::vector<cudaEvent_t> evs;
  auto mkev = [&]() {
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) evs.push_back(ev);
    return ev;
  };
  int rc = SLICQ_OK;
  auto cu = [&](cudaError_t err, const char *what) {
    if (err != cudaSuccess && rc == SLICQ_OK)
      rc = set_error(SLICQ_ECUDA, std::string(what) + ": " + cudaGetErrorString(err));
    return rc == SLICQ_OK;
  };
  auto lib = [&](int r2) {
    if (r2 != SLICQ_OK && rc == SLICQ_OK) rc = r2;
    return rc == SLICQ_OK;
  };
  for (auto &s : st) cu(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  cudaEvent_t ev0 = mkev();
  if (rc == SLICQ_OK && cu(cudaEventRecord(ev0, caller), "cudaEventRecord"))
    for (auto &s : st) cu(cudaStreamWaitEvent(s, ev0, 0), "cudaStreamWaitEvent");
  std::vector<cudaEvent_t> ev_in(P), ev_ready(P), ev_free(P);
  for (int r = 0; r < P; ++r) {
    ev_in[r] = mkev();
    ev_ready[r] = mkev();
    ev_free[r] = mkev();
  }
  const float *xh = x_host;

  // host -> device: global samples [a, b) (circular mod L, zeros at >= n) -> dst[:, 0:b-a]
  auto copy_in = [&](float *dst, int64_t a, int64_t b) {
    int64_t pos = a, o = 0;
    while (pos < b && rc == SLICQ_OK) {
      int64_t g = pos % L;
      if (g < 0) g += L;
      const int64_t seg = std::min(b - pos, L - g);
      const int64_t hi = std::min(g + seg, n);
      if (hi > g)
        cu(cudaMemcpy2DAsync(dst + o, sizeof(float) * e.xw, xh + g, sizeof(float) * n,
                             sizeof(float) * (hi - g), B, cudaMemcpyHostToDevice, st[0]),
           "cudaMemcpy2DAsync (in)");
      const int64_t z0 = std::max(hi - g, (int64_t)0);
      if (seg > z0)
        cu(cudaMemset2DAsync(dst + o + z0, sizeof(float) * e.xw, 0, sizeof(float) * (seg - z0), B,
                             st[0]),
           "cudaMemset2DAsync");
      pos += seg;
      o += seg;
    }
  };
  // range r's samples -> y_host, [lo, hi) of the range's global samples (clipped to n)
  auto copy_seg = [&](int r, int64_t lo, int64_t hi) {
    const int64_t a = bounds[r] * N;
    hi = std::min(hi, n);
    if (hi > lo)
      cu(cudaMemcpy2DAsync(y_host + lo, sizeof(float) * n, slot_y(r) + (lo - a), sizeof(float) * e.yw,
                           sizeof(float) * (hi - lo), B, cudaMemcpyDeviceToHost, st[2]),
         "cudaMemcpy2DAsync (out)");
  };
  // all but the last halo samples of a range are final once its own inverse ran (only the
  // next range's spill adds to the tail): they go out right away (SLICQ_EXEC_SPLIT)
  auto copy_out_head = [&](int r) {
    copy_seg(r, bounds[r] * N, bounds[r + 1] * N - halo);
  };
  auto copy_out = [&](int r, bool head_done) {
    const int64_t a = bounds[r] * N, b = bounds[r + 1] * N;
    copy_seg(r, head_done ? std::max(a, b - halo) : a, b);
    cu(cudaEventRecord(ev_free[r], st[2]), "cudaEventRecord");
  };
  const bool split = SLICQ_EXEC_SPLIT != 0;

  // host enqueue order per range: in(r), k(r) (completes range r-1), out(r-1); a slot is
  // refilled only after the copy-out of the range that used it kSlots ranges earlier
  for (int r = 0; r < P && rc == SLICQ_OK; ++r) {
    const int64_t s0 = bounds[r], ns = bounds[r + 1] - bounds[r];
    if (r >= kSlots) cu(cudaStreamWaitEvent(st[0], ev_free[r - kSlots], 0), "cudaStreamWaitEvent");
    copy_in(slot_x(r), s0 * N - halo, (s0 + ns) * N);
    cu(cudaEventRecord(ev_in[r], st[0]), "cudaEventRecord");
    if (rc != SLICQ_OK) break;
    cu(cudaStreamWaitEvent(st[1], ev_in[r], 0), "cudaStreamWaitEvent");
    if (r >= kSlots) cu(cudaStreamWaitEvent(st[1], ev_free[r - kSlots], 0), "cudaStreamWaitEvent");
    if (rc != SLICQ_OK) break;
    if (!lib(slicq_forward_range(p, slot_x(r), halo + ns * N, e.xw, halo, s0, ns, S, B,
                                 slot_c(r), rws, e.ws_bytes, st[1])))
      break;
    if (fn && !lib(fn(user, slot_c(r), s0, ns, B, st[1]) == 0
                       ? SLICQ_OK
                       : set_error(SLICQ_EINVAL, "coefficient hook failed")))
      break;
    if (!lib(slicq_inverse_range(p, slot_c(r), s0, ns, S, B, slot_y(r), e.yw, spill(r), halo,
                                 rws, e.ws_bytes, st[1])))
      break;
    if (split) {  // the head of range r is final now
      cu(cudaEventRecord(ev_in[r], st[1]), "cudaEventRecord");  // (ev_in[r] reused: k(r) done)
      cu(cudaStreamWaitEvent(st[2], ev_in[r], 0), "cudaStreamWaitEvent");
      copy_out_head(r);
    }
    if (r > 0) {  // range r's spill completes range r-1's tail
      if (!lib(slicq_overlap_add(slot_y(r - 1) + (bounds[r] - bounds[r - 1]) * N - halo, e.yw,
                                 spill(r), halo, B, st[1])))
        break;
      cu(cudaEventRecord(ev_ready[r - 1], st[1]), "cudaEventRecord");
      cu(cudaStreamWaitEvent(st[2], ev_ready[r - 1], 0), "cudaStreamWaitEvent");
      copy_out(r - 1, split);
    }
  }
  if (rc == SLICQ_OK) {  // circular wrap: range 0's spill completes the last range's tail
    const int r = P - 1;
    if (lib(slicq_overlap_add(slot_y(r) + (bounds[r + 1] - bounds[r]) * N - halo, e.yw, spill(0),
                              halo, B, st[1]))) {
      cu(cudaEventRecord(ev_ready[r], st[1]), "cudaEventRecord");
      cu(cudaStreamWaitEvent(st[2], ev_ready[r], 0), "cudaStreamWaitEvent");
      copy_out(r, split);
    }
  }
  // join: the caller's stream waits for all three (also on error, for what was enqueued)
  for (auto &s : st)
    if (s) {
      cudaEvent_t evj = mkev();
      if (evj && cudaEventRecord(evj, s) == cudaSuccess) cudaStreamWaitEvent(caller, evj, 0);
    }
  for (auto ev : evs) cudaEventDestroy(ev);  // released once their work completes
  for (auto &s : st)
    if (s) cudaStreamDestroy(s);
  return rc;
}

}  // extern "C"
