// Host-buffer execution of one layer step (forward, backward-data, weight
// update) — the reference's execute calls take HOST tensors and return
// finished results (propagation.cpp:56-61 forward_into, :237-261 backward_with,
// :377-458 weight_update). This entry streams the batch through the GPU in
// image chunks on three CUDA streams so that, per chunk, the host->device copy
// of chunk i+1, the conv kernels of chunk i and the device->host copy of chunk
// i-1 overlap (PCIe is full duplex; the kernels are ~10x faster than the link).
//
// Included at the end of dconv_capi.cu (shares its error plumbing).
#pragma once
#include <algorithm>
#include <map>
#include <set>
#include <vector>

struct dconv_host_step {
  dconv_spec_t spec;  // whole-batch layer
  int math;
  int chunk;  // images per chunk
  cudaStream_t h2d = nullptr, d2h = nullptr;
  static constexpr int kSlots = 3;  // staging depth: H2D of chunk i waits only for chunk i-3's compute
  cudaEvent_t ev_start = nullptr, ev_w = nullptr, ev_in[kSlots] = {}, ev_comp[kSlots] = {}, ev_out[kSlots] = {};
  // plans per chunk size (the schedule ramps 1, 2, 4, ... images up and down)
  struct Plans {
    int n = 0, y_hh = -1, y_hw = -1;
    dconv_fwd_plan_t f = nullptr;
    dconv_bwd_plan_t b = nullptr;
    dconv_upd_plan_t u = nullptr;
  };
  std::map<int, Plans> plans;
  // device staging: two slots per streamed tensor, one weight / weight-gradient buffer
  void* slot[4][kSlots] = {};  // x, dy, y, dx
  size_t slot_bytes[4] = {};
  void* w_dev = nullptr;
  void* dw_dev = nullptr;
  size_t w_bytes = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int last_launches = 0;
};

namespace {

size_t act_bytes_per_image(const dconv_act_t& a) {
  const size_t es = a.dtype == DCONV_BF16 ? 2 : 4;
  return static_cast<size_t>(cdiv(a.c, a.vlen)) * (a.h + 2 * a.halo_h) * (a.w + 2 * a.halo_w) * a.vlen * es;
}

void hs_free(dconv_host_step& h) {
  for (auto& kv : h.plans) {
    auto& pl = kv.second;
    if (pl.f) dconv_fwd_plan_destroy(pl.f);
    if (pl.b) dconv_bwd_plan_destroy(pl.b);
    if (pl.u) dconv_upd_plan_destroy(pl.u);
  }
  h.plans.clear();
  for (auto& s : h.slot)
    for (auto& p : s) {
      if (p) cudaFree(p);
      p = nullptr;
    }
  for (void** p : {&h.w_dev, &h.dw_dev, &h.ws})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
}

void ck(int st) {
  if (st != DCONV_OK) {
    const std::string msg = g_err;
    fail(st, msg);
  }
}

void ensure(void*& p, size_t& have, size_t want) {
  if (want <= have && p) return;
  if (p) cuda_check(cudaFree(p), "cudaFree");
  p = nullptr;
  cuda_check(cudaMalloc(&p, want), "cudaMalloc (host-step staging)");
  have = want;
}

}  // namespace

extern "C" {

int dconv_host_step_create(const dconv_spec_t* spec, int math, int chunk_images, dconv_host_step_t* out) {
  return guarded([&] {
    if (!spec || !out) fail(DCONV_ERR_INVALID_ARGUMENT, "host_step_create: null argument");
    validate_spec(*spec);
    if (math != DCONV_MATH_F32 && math != DCONV_MATH_BF16) fail(DCONV_ERR_INVALID_ARGUMENT, "bad math mode");
    auto* h = new dconv_host_step();
    h->spec = *spec;
    h->math = math;
    h->chunk = chunk_images > 0 ? std::min(chunk_images, spec->N) : std::max(1, spec->N / 4);
    cuda_check(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t* e : {&h->ev_start, &h->ev_w})
      cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    for (int b = 0; b < dconv_host_step::kSlots; ++b)
      for (cudaEvent_t* e : {&h->ev_in[b], &h->ev_comp[b], &h->ev_out[b]})
        cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    *out = h;
  });
}

void dconv_host_step_destroy(dconv_host_step_t h) {
  if (!h) return;
  cudaDeviceSynchronize();
  hs_free(*h);
  for (cudaEvent_t e : {h->ev_start, h->ev_w})
    if (e) cudaEventDestroy(e);
  for (int b = 0; b < dconv_host_step::kSlots; ++b)
    for (cudaEvent_t e : {h->ev_in[b], h->ev_comp[b], h->ev_out[b]})
    if (e) cudaEventDestroy(e);
  if (h->h2d) cudaStreamDestroy(h->h2d);
  if (h->d2h) cudaStreamDestroy(h->d2h);
  delete h;
}

int dconv_host_step_chunk(dconv_host_step_t h) { return h ? h->chunk : 0; }
int dconv_host_step_launches(dconv_host_step_t h) { return h ? h->last_launches : 0; }

int dconv_host_step_run(dconv_host_step_t h, const dconv_act_t* x, const dconv_wt_t* w, const dconv_act_t* dy,
                        const dconv_act_t* y, const dconv_act_t* dx, const dconv_wt_t* dw, dconv_stream_t stream) {
  return guarded([&] {
    if (!h) fail(DCONV_ERR_INVALID_ARGUMENT, "null host step");
    const dconv_spec_t& s = h->spec;
    const bool do_f = y != nullptr, do_b = dx != nullptr, do_u = dw != nullptr;
    if ((do_f || do_u) && !x) fail(DCONV_ERR_INVALID_ARGUMENT, "host_step: forward / update need the input");
    if ((do_b || do_u) && !dy) fail(DCONV_ERR_INVALID_ARGUMENT, "host_step: backward / update need grad_out");
    if ((do_f || do_b) && !w) fail(DCONV_ERR_INVALID_ARGUMENT, "host_step: forward / backward need weights");
    const int P = out_P(s), Q = out_Q(s);
    // shapes as the device entries check them (propagation.cpp:56-61, :383-393)
    if (x && (x->n != s.N || x->c != s.C || x->h != s.H || x->w != s.W || x->vlen != s.vlen || !x->data))
      fail(DCONV_ERR_SHAPE_MISMATCH, "host_step: input does not match the layer spec");
    if (dy && (dy->n != s.N || dy->c != s.K || dy->h != P || dy->w != Q || dy->vlen != s.vlen || !dy->data))
      fail(DCONV_ERR_SHAPE_MISMATCH, "host_step: grad_out does not match the layer spec");
    if (y && (y->n != s.N || y->c != s.K || y->h != P || y->w != Q || y->vlen != s.vlen || !y->data))
      fail(DCONV_ERR_SHAPE_MISMATCH, "host_step: output does not match the layer spec");
    if (dx && (dx->n != s.N || dx->c != s.C || dx->h != s.H || dx->w != s.W || dx->vlen != s.vlen || !dx->data))
      fail(DCONV_ERR_SHAPE_MISMATCH, "host_step: grad_in does not match the layer spec");
    const dconv_wt_t* wref = w ? w : dw;
    if (!wref || wref->k != s.K || wref->c != s.C || wref->r != s.R || wref->s != s.S || wref->vlen != s.vlen ||
        !wref->data)
      fail(DCONV_ERR_SHAPE_MISMATCH, "host_step: weights do not match the layer spec");
    if (w && dw && w->dtype != dw->dtype) fail(DCONV_ERR_INVALID_ARGUMENT, "host_step: w / dw dtypes differ");

    // chunk schedule: ramp 1, 2, 4, ... images up to the chunk size and back down,
    // so the link's fill (first H2D) and drain (last D2H) move small chunks while
    // the middle of the step runs both directions at once
    std::vector<int> sched;
    if (const char* env = getenv("DCONV_HOST_SCHED")) {  // debug: explicit comma-separated chunk sizes
      int tot = 0;
      for (const char* q = env; *q;) {
        const int v = std::atoi(q);
        if (v > 0) sched.push_back(v), tot += v;
        while (*q && *q != ',') ++q;
        if (*q) ++q;
      }
      if (tot != s.N) sched.clear();
    }
    if (sched.empty()) {
      std::vector<int> up;
      for (int r = 1; r < h->chunk; r *= 2) up.push_back(r);
      int ramp = 0;
      for (int r : up) ramp += 2 * r;
      if (ramp < s.N) {
        sched = up;
        for (int mid = s.N - ramp; mid > 0;) {
          const int c = std::min(h->chunk, mid);
          sched.push_back(c);
          mid -= c;
        }
        sched.insert(sched.end(), up.rbegin(), up.rend());
      } else {
        for (int n0 = 0; n0 < s.N; n0 += h->chunk) sched.push_back(std::min(h->chunk, s.N - n0));
      }
    }
    const int max_chunk = *std::max_element(sched.begin(), sched.end());
    // staging buffers (two slots per streamed tensor)
    const dconv_act_t* acts[4] = {x, dy, y, dx};
    for (int t = 0; t < 4; ++t)
      if (acts[t]) {
        const size_t want = act_bytes_per_image(*acts[t]) * max_chunk;
        if (want > h->slot_bytes[t] || !h->slot[t][0]) {
          for (int b = 0; b < dconv_host_step::kSlots; ++b) {
            size_t have = h->slot_bytes[t];
            ensure(h->slot[t][b], have, want);
          }
          h->slot_bytes[t] = want;
        }
      }
    const size_t wbytes = wt_elems(*wref) * (wref->dtype == DCONV_BF16 ? 2 : 4);
    {
      size_t a = h->w_bytes, b = h->w_bytes;
      if (wbytes > h->w_bytes || !h->w_dev || !h->dw_dev) {
        ensure(h->w_dev, a, wbytes);
        ensure(h->dw_dev, b, wbytes);
        h->w_bytes = wbytes;
      }
    }

    const int n_chunks = static_cast<int>(sched.size());
    const int yhh = y ? y->halo_h : 0, yhw = y ? y->halo_w : 0;
    auto plans_for = [&](int n) -> dconv_host_step::Plans& {
      dconv_host_step::Plans& pl = h->plans[n];
      if (pl.n != n || pl.y_hh != yhh || pl.y_hw != yhw) {
        if (pl.f) dconv_fwd_plan_destroy(pl.f);
        if (pl.b) dconv_bwd_plan_destroy(pl.b);
        if (pl.u) dconv_upd_plan_destroy(pl.u);
        pl = dconv_host_step::Plans{};
        dconv_spec_t sc = s;
        sc.N = n;
        ck(dconv_fwd_plan_create(&sc, nullptr, nullptr, h->math, yhh, yhw, &pl.f));
        ck(dconv_bwd_plan_create(&sc, nullptr, h->math, &pl.b));
        ck(dconv_upd_plan_create(&sc, nullptr, h->math, &pl.u));
        pl.n = n;
        pl.y_hh = yhh;
        pl.y_hw = yhw;
      }
      return pl;
    };
    auto chunk_act = [&](const dconv_act_t* a, void* data, int n) {
      dconv_act_t c = *a;
      c.data = data;
      c.n = n;
      return c;
    };
    // workspace: max over the passes and chunk sizes
    size_t ws_need = 256;
    for (int n : std::set<int>(sched.begin(), sched.end())) {
      dconv_host_step::Plans& pl = plans_for(n);
      if (do_f) ws_need = std::max(ws_need, dconv_fwd_workspace_bytes(pl.f));
      if (do_b) ws_need = std::max(ws_need, dconv_bwd_workspace_bytes(pl.b));
      if (do_u) {
        const dconv_act_t xc = chunk_act(x, h->slot[0][0], n), dc = chunk_act(dy, h->slot[1][0], n);
        ws_need = std::max(ws_need, dconv_upd_workspace_bytes(pl.u, &xc, &dc));
      }
    }
    if (ws_need > h->ws_bytes || !h->ws) {
      size_t have = h->ws_bytes;
      ensure(h->ws, have, ws_need);
      h->ws_bytes = ws_need;
    }

    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    // everything queued before this call on `stream` happens first
    cuda_check(cudaEventRecord(h->ev_start, cs), "event record");
    cuda_check(cudaStreamWaitEvent(h->h2d, h->ev_start, 0), "stream wait");
    cuda_check(cudaStreamWaitEvent(h->d2h, h->ev_start, 0), "stream wait");
    dconv_wt_t wd{}, dwd{};
    if (w) {
      wd = *w;
      wd.data = h->w_dev;
      cuda_check(cudaMemcpyAsync(h->w_dev, w->data, wbytes, cudaMemcpyHostToDevice, h->h2d), "H2D weights");
    }
    if (dw) {
      dwd = *dw;
      dwd.data = h->dw_dev;
    }
    cuda_check(cudaEventRecord(h->ev_w, h->h2d), "event record");
    cuda_check(cudaStreamWaitEvent(cs, h->ev_w, 0), "stream wait");

    int launches = 0;
    // debug timeline (DCONV_HOST_STEP_TRACE=1): timing events around every copy / compute
    static const bool trace = getenv("DCONV_HOST_STEP_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
      if (!trace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      tev.push_back(e);
    };
    mark(cs);
    for (int i = 0, n0 = 0; i < n_chunks; n0 += sched[i], ++i) {
      const int b = i % dconv_host_step::kSlots;
      const int n = sched[i];
      dconv_host_step::Plans& pl = plans_for(n);
      // the slot's previous chunk (i-2) must be done computing before its inputs are overwritten
      if (i >= dconv_host_step::kSlots) cuda_check(cudaStreamWaitEvent(h->h2d, h->ev_comp[b], 0), "stream wait");
      mark(h->h2d);
      for (int t = 0; t < 2; ++t)
        if (acts[t]) {
          const size_t per = act_bytes_per_image(*acts[t]);
          cuda_check(cudaMemcpyAsync(h->slot[t][b], static_cast<const char*>(acts[t]->data) + per * n0, per * n,
                                     cudaMemcpyHostToDevice, h->h2d),
                     "H2D chunk");
        }
      mark(h->h2d);
      cuda_check(cudaEventRecord(h->ev_in[b], h->h2d), "event record");
      cuda_check(cudaStreamWaitEvent(cs, h->ev_in[b], 0), "stream wait");
      // ... and its outputs (i-2) must have left the device before they are overwritten
      if (i >= dconv_host_step::kSlots) cuda_check(cudaStreamWaitEvent(cs, h->ev_out[b], 0), "stream wait");
      dconv_act_t xc{}, dyc{}, yc{}, dxc{};
      if (x) xc = chunk_act(x, h->slot[0][b], n);
      if (dy) dyc = chunk_act(dy, h->slot[1][b], n);
      if (y) yc = chunk_act(y, h->slot[2][b], n);
      if (dx) dxc = chunk_act(dx, h->slot[3][b], n);
      mark(cs);
      if (do_f) {
        ck(dconv_forward(pl.f, &xc, &wd, &yc, h->ws, stream));
        launches += dconv_fwd_launches(pl.f);
      }
      if (do_b) {
        ck(dconv_backward_data(pl.b, &wd, &dyc, &dxc, h->ws, stream));
        launches += dconv_bwd_launches(pl.b);
      }
      if (do_u) {
        ck(dconv_weight_update(pl.u, &xc, &dyc, &dwd, i > 0 ? 1 : 0, h->ws, stream));
        launches += dconv_upd_launches(pl.u, &xc, &dyc);
      }
      mark(cs);
      cuda_check(cudaEventRecord(h->ev_comp[b], cs), "event record");
      cuda_check(cudaStreamWaitEvent(h->d2h, h->ev_comp[b], 0), "stream wait");
      mark(h->d2h);
      for (int t = 2; t < 4; ++t)
        if (acts[t]) {
          const size_t per = act_bytes_per_image(*acts[t]);
          cuda_check(cudaMemcpyAsync(static_cast<char*>(acts[t]->data) + per * n0, h->slot[t][b], per * n,
                                     cudaMemcpyDeviceToHost, h->d2h),
                     "D2H chunk");
        }
      mark(h->d2h);
      cuda_check(cudaEventRecord(h->ev_out[b], h->d2h), "event record");
    }
    if (do_u)
      cuda_check(cudaMemcpyAsync(dw->data, h->dw_dev, wbytes, cudaMemcpyDeviceToHost, cs), "D2H weight gradient");
    // the caller's stream completes after every copy of this step
    for (int b = 0; b < std::min(n_chunks, dconv_host_step::kSlots); ++b)
      cuda_check(cudaStreamWaitEvent(cs, h->ev_out[b], 0), "stream wait");
    mark(cs);
    if (trace) {
      cudaStreamSynchronize(cs);
      auto rel = [&](size_t k) {
        float ms = 0;
        cudaEventElapsedTime(&ms, tev[0], tev[k]);
        return ms * 1e3f;
      };
      for (int i = 0; i < n_chunks; ++i) {
        const size_t k = 1 + 6 * i;
        std::fprintf(stderr, "chunk %d (%d img): h2d %.0f-%.0f  comp %.0f-%.0f  d2h %.0f-%.0f us\n", i, sched[i],
                     rel(k), rel(k + 1), rel(k + 2), rel(k + 3), rel(k + 4), rel(k + 5));
      }
      std::fprintf(stderr, "end %.0f us\n", rel(tev.size() - 1));
      for (auto e : tev) cudaEventDestroy(e);
    }
    h->last_launches = launches;
  });
}

}  // extern "C"
