// dconv_graph: the data-parallel layer-graph executor, native.
//
// The reference's run_chain (harness.cpp:311-358) runs a LINEAR chain of
// forward convs, each layer writing straight into the next layer's input
// surface (:348-353), after checking that consecutive layers chain (:331-341).
// This is its training-time, multi-GPU generalisation, written as a client of
// the C ABI (it calls the same dconv_forward_ex / dconv_backward_data_ex /
// dconv_weight_update a user would):
//  * a DAG of convs (residual adds, projection shortcuts) and 3x3/s2 max-pools;
//  * forward with ReLU / residual add fused into the producing conv's epilogue;
//  * backward-data with the ReLU mask and the two-branch gradient sum fused
//    into the consuming conv's epilogue; weight updates on a side stream,
//    forked as soon as a layer's output gradient is final;
//  * the fp32 weight gradients live in ONE flat buffer laid out in backward
//    order; buckets of it are all-reduced with NCCL on a communication stream
//    as soon as their layers' updates finish (overlapping the backward of
//    earlier layers) -- the reference's COPY_REDUCE over minibatch shards
//    (propagation.cpp:357-375, 413-457) promoted from threads to GPUs;
//  * SGD over the flat master weights in one launch;
//  * the whole step captured once into a CUDA graph (any world size: the NCCL
//    calls are captured with it) and replayed.
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy the process
// already has, e.g. PyTorch's, else the system one), so the library has no
// link-time NCCL dependency and world = 1 runs without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dconv_b200.h"

extern "C" void dconv_internal_set_error(const char* msg);  // dconv_capi.cu
extern "C" const char* dconv_internal_dev_env(const char* name);  // dconv_capi.cu (developer mode only)
extern "C" int dconv_internal_bwd_prep_launches(dconv_bwd_plan_t plan);  // dconv_capi.cu: weight preps per execute

namespace {

struct GFail {
  int code;
  std::string msg;
};

[[noreturn]] void gfail(int code, const std::string& m) { throw GFail{code, m}; }

void ck(int st, const char* what) {
  if (st != DCONV_OK) gfail(st, std::string(what) + ": " + dconv_last_error());
}
void cuck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) gfail(DCONV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int gguard(F&& f) {
  try {
    f();
    return DCONV_OK;
  } catch (const GFail& e) {
    dconv_internal_set_error(e.msg.c_str());  // dconv_last_error() reports it
    return e.code;
  } catch (const std::exception& e) {
    dconv_internal_set_error(e.what());
    return DCONV_ERR_CUDA;
  }
}

// ------------------------------------------------------------------ NCCL (run-time loaded)
struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy (PyTorch's) if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = dlerror();
      return;
    }
    n.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
    n.err = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!n.all_reduce || !n.init_rank || !n.get_unique_id)
    gfail(DCONV_ERR_UNSUPPORTED, "NCCL unavailable (libnccl.so.2): " + why);
  return n;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) gfail(DCONV_ERR_CUDA, std::string(what) + ": " + nccl().err(r));
}

// ------------------------------------------------------------------ graph state
int cdiv(int a, int b) { return (a + b - 1) / b; }

struct Tensor {
  int c, h, w;
  void* act = nullptr;   // blocked, halo 0
  void* grad = nullptr;  // dL/dz (through this tensor's ReLU), may alias another tensor's
  bool relu = false;     // produced by a ReLU (a conv with relu, or a pool of such)
  bool owns_grad = true;
  // stride-2 lattice copy (every consumer a stride-2 1x1 conv: the ResNet v1
  // downsampling blocks' input): the consumers run as stride-1 1x1 convs over it
  // (dense planes: linear / multi-image / SWIZZLE_128B plans instead of strided
  // row gathers), their data gradients sum into sub_grad, scattered back once
  int sub_consumers = 0, sh = 0, sw = 0;
  void* sub_act = nullptr;
  void* sub_grad = nullptr;
};

struct Conv {
  int node;  // index into nodes
  dconv_spec_t spec, pspec;  // layer, and as executed (space-to-depth stem, stride-2 1x1 over the lattice)
  bool s2d = false;
  bool sub = false;  // a stride-2 1x1 conv run at stride 1 over its input's lattice copy
  dconv_fwd_plan_t fp = nullptr;
  dconv_bwd_plan_t bp = nullptr;
  dconv_upd_plan_t up = nullptr;
  size_t w_off = 0, w_len = 0;  // slice of the flat weights / gradients (backward order)
  void* s2d_x = nullptr;  // space-to-depth input, weights, weight gradient
  float* s2d_w = nullptr;
  float* s2d_dw = nullptr;
  int bucket = -1;
  cudaEvent_t ev_gready = nullptr, ev_dw = nullptr;
  // prepared weights: every step's forward prepares all forward and backward-data
  // weights in one batched launch (dconv_prep_batch_*) into these per-conv workspaces
  void* ws_f = nullptr;
  void* ws_b = nullptr;
  // the backward-data epilogue operands (fixed by the graph; computed once at build):
  // the other branch's gradient to add (or this gradient itself, accumulating), the mask
  const void* b_add = nullptr;
  const void* b_mask = nullptr;
};

struct Bucket {
  size_t off = 0, len = 0;
  int n_convs = 0;
  cudaEvent_t done = nullptr;
};

}  // namespace

struct dconv_graph {
  std::vector<dconv_graph_node_t> nodes;
  dconv_graph_config_t cfg;
  int N, math, dtype;
  std::vector<Tensor> t;
  std::vector<Conv> convs;
  std::vector<int> conv_of_node;
  std::vector<void*> argmax;  // per node (pools)
  float* wflat = nullptr;
  float* gflat = nullptr;
  size_t n_params = 0;
  std::vector<Bucket> buckets;
  void* ws_main = nullptr;
  void* ws_upd = nullptr;
  size_t ws_main_bytes = 0, ws_upd_bytes = 0;
  cudaStream_t s_upd = nullptr, s_comm = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_upd_done = nullptr, ev_comm_done = nullptr;
  bool input_s2d = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;  // kernels of the last step (ours, NCCL excluded)
  bool profiling = false;  // dconv_graph_profile: one rank alone, no collectives
  std::vector<void*> allocs;
};

namespace {

void* dalloc(dconv_graph* g, size_t bytes) {
  void* p = nullptr;
  cuck(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "graph alloc");
  cuck(cudaMemset(p, 0, std::max<size_t>(bytes, 256)), "graph memset");
  g->allocs.push_back(p);
  return p;
}

int esz(int dtype) { return dtype == DCONV_BF16 ? 2 : 4; }

dconv_act_t act_of(const dconv_graph* g, int id, bool grad) {
  const Tensor& x = g->t[id];
  dconv_act_t a;
  a.data = grad ? x.grad : x.act;
  a.n = g->N;
  a.c = x.c;
  a.h = x.h;
  a.w = x.w;
  a.vlen = 16;
  a.halo_h = a.halo_w = 0;
  a.dtype = g->dtype;
  return a;
}

size_t act_bytes(const dconv_graph* g, const Tensor& x) {
  return static_cast<size_t>(g->N) * cdiv(x.c, 16) * x.h * x.w * 16 * esz(g->dtype);
}

dconv_wt_t wt_view(float* data, int k, int c, int r, int s) {
  dconv_wt_t w;
  w.data = data;
  w.k = k;
  w.c = c;
  w.r = r;
  w.s = s;
  w.vlen = 16;
  w.dtype = DCONV_F32;
  return w;
}

size_t wt_len(int k, int c, int r, int s) { return static_cast<size_t>(cdiv(k, 16)) * cdiv(c, 16) * r * s * 256; }

dconv_wt_t conv_w(const dconv_graph* g, const Conv& cv, bool grad) {
  const dconv_spec_t& s = cv.spec;
  return wt_view((grad ? g->gflat : g->wflat) + cv.w_off, s.K, s.C, s.R, s.S);
}

// a conv's input (grad: its data gradient) as executed: the space-to-depth copy, the
// stride-2 lattice copy, or the tensor itself
dconv_act_t conv_in(const dconv_graph* g, const Conv& cv, bool grad) {
  const int src = g->nodes[cv.node].src;
  dconv_act_t a = act_of(g, src, grad);
  if (cv.s2d && !grad) {
    a.data = cv.s2d_x;
    a.c = cv.pspec.C;
    a.h = cv.pspec.H;
    a.w = cv.pspec.W;
  }
  if (cv.sub) {
    const Tensor& x = g->t[src];
    a.data = grad ? x.sub_grad : x.sub_act;
    a.h = x.sh;
    a.w = x.sw;
  }
  return a;
}

void build(dconv_graph* g, int in_c, int in_h, int in_w) {
  const int n_t = static_cast<int>(g->nodes.size()) + 1;  // tensor 0 = input, node i writes tensor i + 1
  g->t.assign(n_t, Tensor{});
  g->t[0] = Tensor{in_c, in_h, in_w};
  g->conv_of_node.assign(g->nodes.size(), -1);
  g->argmax.assign(g->nodes.size(), nullptr);
  for (size_t i = 0; i < g->nodes.size(); ++i) {
    const dconv_graph_node_t& nd = g->nodes[i];
    if (nd.src < 0 || nd.src > static_cast<int>(i) || nd.add > static_cast<int>(i))
      gfail(DCONV_ERR_CHAIN_SHAPE_MISMATCH, "graph node " + std::to_string(i) + ": inputs must precede the node");
    const Tensor& src = g->t[nd.src];
    Tensor& out = g->t[i + 1];
    if (nd.kind == DCONV_NODE_MAXPOOL) {
      out = Tensor{src.c, (src.h + 2 - 3) / 2 + 1, (src.w + 2 - 3) / 2 + 1};
      out.relu = src.relu;  // max-pool of a ReLU output: the pooled values are the mask
      continue;
    }
    if (nd.kind != DCONV_NODE_CONV) gfail(DCONV_ERR_INVALID_ARGUMENT, "graph node: unknown kind");
    // harness.cpp:331-341: a layer's input channels and spatial extent must chain
    if (nd.C != src.c)
      gfail(DCONV_ERR_CHAIN_SHAPE_MISMATCH, "graph node " + std::to_string(i) + ": C=" + std::to_string(nd.C) +
                                                " but its input has " + std::to_string(src.c) + " channels");
    dconv_spec_t s;
    ck(dconv_make_spec(g->N, nd.C, nd.K, src.h, src.w, nd.R, nd.S, nd.stride, nd.pad_h, nd.pad_w, 16, &s),
       "graph conv spec");
    int P = 0, Q = 0;
    ck(dconv_output_shape(&s, &P, &Q), "graph conv shape");
    out = Tensor{nd.K, P, Q};
    out.relu = nd.relu != 0;
    if (nd.add >= 0) {
      const Tensor& a = g->t[nd.add];
      if (a.c != nd.K || a.h != P || a.w != Q)
        gfail(DCONV_ERR_CHAIN_SHAPE_MISMATCH, "graph node " + std::to_string(i) + ": residual shape differs");
    }
    Conv cv;
    cv.node = static_cast<int>(i);
    cv.spec = cv.pspec = s;
    // narrow stride-2 input convs (the 7x7/s2 stem, C=3) run as a stride-1 conv over a
    // space-to-depth copy of their input: 4x4 taps over 12 of 16 lanes instead of 49
    // taps over 3 of 16 (the MMA K dimension is a 16-lane channel block)
    if (nd.stride == 2 && nd.C * 4 <= 16 && nd.R > 1 && nd.S > 1) {
      const int r2 = (nd.R + 1) / 2, s2 = (nd.S + 1) / 2;
      ck(dconv_make_spec(g->N, 4 * nd.C, nd.K, P + r2 - 1, Q + s2 - 1, r2, s2, 1, 0, 0, 16, &cv.pspec), "s2d spec");
      cv.s2d = true;
    }
    g->conv_of_node[i] = static_cast<int>(g->convs.size());
    g->convs.push_back(cv);
  }
  // stride-2 1x1 consumers over a lattice copy (Tensor::sub_*): every consumer of the
  // tensor such a conv, the tensor no residual operand, not the image
  for (int id = 1; id < n_t; ++id) {
    int strided = 0, other = 0;
    for (size_t i = 0; i < g->nodes.size(); ++i) {
      const dconv_graph_node_t& nd = g->nodes[i];
      if (nd.add == id) ++other;
      if (nd.src != id) continue;
      const int ci = g->conv_of_node[i];
      if (nd.kind == DCONV_NODE_CONV && ci >= 0 && !g->convs[ci].s2d && nd.stride == 2 && nd.R == 1 && nd.S == 1 &&
          nd.pad_h == 0 && nd.pad_w == 0)
        ++strided;
      else
        ++other;
    }
    if (strided == 0 || other > 0 || dconv_internal_dev_env("DCONV_GRAPH_NO_LATTICE")) continue;
    Tensor& x = g->t[id];
    x.sub_consumers = strided;
    x.sh = (x.h + 1) / 2;
    x.sw = (x.w + 1) / 2;
    for (size_t i = 0; i < g->nodes.size(); ++i)
      if (g->nodes[i].src == id) {
        Conv& cv = g->convs[g->conv_of_node[i]];
        const dconv_graph_node_t& nd = g->nodes[i];
        ck(dconv_make_spec(g->N, nd.C, nd.K, x.sh, x.sw, 1, 1, 1, 0, 0, 16, &cv.pspec), "lattice spec");
        cv.sub = true;
      }
  }
  // tensors and gradients; a projection's output only feeds a residual add, so its
  // dL/dz is the block output's (aliased buffer)
  for (int id = 0; id < n_t; ++id) {
    g->t[id].act = dalloc(g, act_bytes(g, g->t[id]));
    if (g->t[id].sub_consumers > 0) {
      const size_t sb = static_cast<size_t>(g->N) * cdiv(g->t[id].c, 16) * g->t[id].sh * g->t[id].sw * 16 * esz(g->dtype);
      g->t[id].sub_act = dalloc(g, sb);
      g->t[id].sub_grad = dalloc(g, sb);
    }
  }
  for (size_t i = 0; i < g->nodes.size(); ++i) {
    const dconv_graph_node_t& nd = g->nodes[i];
    if (nd.kind == DCONV_NODE_CONV && nd.add >= 1) {
      const dconv_graph_node_t& pn = g->nodes[nd.add - 1];
      if (pn.kind == DCONV_NODE_CONV && !pn.relu) {
        g->t[nd.add].owns_grad = false;  // filled below from the consumer
      }
    }
  }
  for (int id = 1; id < n_t; ++id)
    if (g->t[id].owns_grad) g->t[id].grad = dalloc(g, act_bytes(g, g->t[id]));
  for (size_t i = 0; i < g->nodes.size(); ++i) {
    const dconv_graph_node_t& nd = g->nodes[i];
    if (nd.kind == DCONV_NODE_CONV && nd.add >= 1 && !g->t[nd.add].owns_grad) g->t[nd.add].grad = g->t[i + 1].grad;
    if (nd.kind == DCONV_NODE_MAXPOOL) g->argmax[i] = dalloc(g, act_bytes(g, g->t[i + 1]) / esz(g->dtype));
  }
  for (int id = 1; id < n_t; ++id)
    if (!g->t[id].grad) gfail(DCONV_ERR_INVALID_ARGUMENT, "graph: a non-ReLU conv output must feed a residual add");
  // flat weights / gradients in BACKWARD order (the first bucket is ready first)
  size_t off = 0;
  for (int ci = static_cast<int>(g->convs.size()) - 1; ci >= 0; --ci) {
    Conv& cv = g->convs[ci];
    cv.w_off = off;
    cv.w_len = wt_len(cv.spec.K, cv.spec.C, cv.spec.R, cv.spec.S);
    off += cv.w_len;
  }
  g->n_params = off;
  g->wflat = static_cast<float*>(dalloc(g, off * 4));
  g->gflat = static_cast<float*>(dalloc(g, off * 4));
  // He-normal masters from the seeded host generator (util.hpp:40-71 stream), packed on the device
  for (size_t ci = 0; ci < g->convs.size(); ++ci) {
    const dconv_spec_t& s = g->convs[ci].spec;
    const int64_t n = static_cast<int64_t>(s.K) * s.C * s.R * s.S;
    std::vector<float> host(static_cast<size_t>(n));
    dconv_fill_he_normal_host(static_cast<uint64_t>(g->cfg.seed) * 1000 + ci,
                              static_cast<float>(std::sqrt(2.0 / (s.C * s.R * s.S))), host.data(), n);
    void* tmp = nullptr;
    cuck(cudaMalloc(&tmp, n * 4), "weight staging");
    cuck(cudaMemcpy(tmp, host.data(), n * 4, cudaMemcpyHostToDevice), "weight upload");
    const dconv_wt_t w = conv_w(g, g->convs[ci], false);
    ck(dconv_pack_wt(tmp, DCONV_F32, &w, nullptr), "weight pack");
    cuck(cudaDeviceSynchronize(), "weight pack");
    cudaFree(tmp);
  }
  // buckets: contiguous runs of layers (backward order) of >= bucket_bytes
  const size_t bb = g->cfg.bucket_bytes > 0 ? static_cast<size_t>(g->cfg.bucket_bytes) : (8u << 20);
  Bucket cur;
  for (int ci = static_cast<int>(g->convs.size()) - 1; ci >= 0; --ci) {
    Conv& cv = g->convs[ci];
    if (cur.n_convs == 0) cur.off = cv.w_off;
    cv.bucket = static_cast<int>(g->buckets.size());
    cur.len += cv.w_len;
    ++cur.n_convs;
    if (cur.len * 4 >= bb || ci == 0) {
      g->buckets.push_back(cur);
      cur = Bucket{};
    }
  }
  for (auto& b : g->buckets) cuck(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming), "event");
  // plans and workspaces
  for (Conv& cv : g->convs) {
    const dconv_graph_node_t& nd = g->nodes[cv.node];
    ck(dconv_fwd_plan_create(&cv.pspec, nullptr, nullptr, g->math, 0, 0, &cv.fp), "graph forward plan");
    if (nd.src != 0) ck(dconv_bwd_plan_create(cv.sub ? &cv.pspec : &cv.spec, nullptr, g->math, &cv.bp), "graph backward plan");
    ck(dconv_upd_plan_create(&cv.pspec, nullptr, g->math, &cv.up), "graph update plan");
    g->ws_main_bytes = std::max(g->ws_main_bytes, dconv_fwd_workspace_bytes(cv.fp));
    if (cv.bp) g->ws_main_bytes = std::max(g->ws_main_bytes, dconv_bwd_workspace_bytes(cv.bp));
    if (cv.s2d) {
      const dconv_spec_t& p = cv.pspec;
      cv.s2d_x = dalloc(g, static_cast<size_t>(g->N) * cdiv(p.C, 16) * p.H * p.W * 16 * esz(g->dtype));
      cv.s2d_w = static_cast<float*>(dalloc(g, wt_len(p.K, p.C, p.R, p.S) * 4));
      cv.s2d_dw = static_cast<float*>(dalloc(g, wt_len(p.K, p.C, p.R, p.S) * 4));
    }
    cuck(cudaEventCreateWithFlags(&cv.ev_gready, cudaEventDisableTiming), "event");
    cuck(cudaEventCreateWithFlags(&cv.ev_dw, cudaEventDisableTiming), "event");
  }
  for (Conv& cv : g->convs) {
    const dconv_act_t in = conv_in(g, cv, false), gout = act_of(g, cv.node + 1, true);
    g->ws_upd_bytes = std::max(g->ws_upd_bytes, dconv_upd_workspace_bytes(cv.up, &in, &gout));
  }
  g->ws_main = dalloc(g, g->ws_main_bytes);
  g->ws_upd = dalloc(g, g->ws_upd_bytes);
  for (Conv& cv : g->convs) {
    cv.ws_f = dalloc(g, dconv_fwd_workspace_bytes(cv.fp));
    if (cv.bp) cv.ws_b = dalloc(g, dconv_bwd_workspace_bytes(cv.bp));
  }
  // backward-data epilogue operands, in the backward walk's order: a tensor's first
  // data-gradient contribution adds the identity-shortcut consumer's gradient (if any),
  // later ones accumulate in place; lattice consumers sum into the lattice gradient
  {
    std::vector<char> written(g->t.size(), 0);
    std::vector<int> sub_done(g->t.size(), 0);
    for (int i = static_cast<int>(g->nodes.size()) - 1; i >= 0; --i) {
      const dconv_graph_node_t& nd = g->nodes[i];
      if (nd.kind == DCONV_NODE_MAXPOOL) {
        written[nd.src] = 1;
        continue;
      }
      Conv& cv = g->convs[g->conv_of_node[i]];
      if (nd.src == 0) continue;
      Tensor& x = g->t[nd.src];
      if (cv.sub) {
        cv.b_add = sub_done[nd.src] > 0 ? x.sub_grad : nullptr;
        cv.b_mask = x.relu ? x.sub_act : nullptr;
        if (++sub_done[nd.src] == x.sub_consumers) written[nd.src] = 1;
        continue;
      }
      cv.b_mask = x.relu ? x.act : nullptr;
      cv.b_add = nullptr;
      if (written[nd.src]) {
        cv.b_add = x.grad;  // second contribution: accumulate in place
      } else {
        for (size_t j = 0; j < g->nodes.size(); ++j)  // identity-shortcut consumer of src
          if (g->nodes[j].kind == DCONV_NODE_CONV && g->nodes[j].add == nd.src) {
            cv.b_add = g->t[j + 1].grad;
            break;
          }
      }
      written[nd.src] = 1;
    }
  }
  cuck(cudaStreamCreateWithFlags(&g->s_upd, cudaStreamNonBlocking), "stream");
  cuck(cudaStreamCreateWithFlags(&g->s_comm, cudaStreamNonBlocking), "stream");
  cuck(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming), "event");
  cuck(cudaEventCreateWithFlags(&g->ev_upd_done, cudaEventDisableTiming), "event");
  cuck(cudaEventCreateWithFlags(&g->ev_comm_done, cudaEventDisableTiming), "event");
}

dconv_epilogue_t epi(const void* add, const void* mask, int relu) {
  dconv_epilogue_t e;
  e.add = add;
  e.mask = mask;
  e.relu = relu;
  e.flags = 0;
  return e;
}

// the data-gradient tensor a conv's backward-data writes (lattice consumers: the lattice gradient)
dconv_act_t bwd_out(const dconv_graph* g, const Conv& cv) {
  return cv.sub ? conv_in(g, cv, true) : act_of(g, g->nodes[cv.node].src, true);
}

// every conv's forward and backward-data weights, prepared in one batched launch
void prepare_weights(dconv_graph* g, cudaStream_t s) {
  dconv_stream_t st = reinterpret_cast<dconv_stream_t>(s);
  for (Conv& cv : g->convs)
    if (cv.s2d) {  // the space-to-depth stem's weights are transformed first
      const dconv_wt_t w = conv_w(g, cv, false);
      const dconv_wt_t w2 = wt_view(cv.s2d_w, cv.pspec.K, cv.pspec.C, cv.pspec.R, cv.pspec.S);
      ck(dconv_s2d_wt(&w, &w2, 0, st), "graph s2d weights");
      g->launches += 1;
    }
  ck(dconv_prep_batch_begin(), "graph weight prep");
  int jobs = 0;
  const int rc = gguard([&] {
    for (Conv& cv : g->convs) {
      const dconv_graph_node_t& nd = g->nodes[cv.node];
      dconv_epilogue_t e = epi(nd.add >= 0 ? g->t[nd.add].act : nullptr, nullptr, nd.relu);
      e.flags = DCONV_EP_PREP_ONLY;
      const dconv_act_t x = conv_in(g, cv, false), out = act_of(g, cv.node + 1, false);
      const dconv_wt_t w = cv.s2d ? wt_view(cv.s2d_w, cv.pspec.K, cv.pspec.C, cv.pspec.R, cv.pspec.S)
                                  : conv_w(g, cv, false);
      ck(dconv_forward_ex(cv.fp, &x, &w, &out, &e, cv.ws_f, st), "graph forward weight prep");
      jobs += 1;
      if (!cv.bp) continue;
      dconv_epilogue_t eb = epi(cv.b_add, cv.b_mask, 0);
      eb.flags = DCONV_EP_PREP_ONLY;
      const dconv_act_t go = act_of(g, cv.node + 1, true), gi = bwd_out(g, cv);
      const dconv_wt_t wb = conv_w(g, cv, false);
      ck(dconv_backward_data_ex(cv.bp, &wb, &go, &gi, &eb, cv.ws_b, st), "graph backward weight prep");
      jobs += dconv_internal_bwd_prep_launches(cv.bp);
    }
  });
  const int rc_end = dconv_prep_batch_end(st);  // (closes the batch even after an error)
  if (rc != DCONV_OK) gfail(rc, dconv_last_error());
  ck(rc_end, "graph weight prep launch");
  g->launches += (jobs + 127) / 128;
}

void forward(dconv_graph* g, cudaStream_t s) {
  dconv_stream_t st = reinterpret_cast<dconv_stream_t>(s);
  std::vector<char> subbed(g->t.size(), 0);
  prepare_weights(g, s);
  for (size_t i = 0; i < g->nodes.size(); ++i) {
    const dconv_graph_node_t& nd = g->nodes[i];
    const dconv_act_t src = act_of(g, nd.src, false), out = act_of(g, static_cast<int>(i) + 1, false);
    if (nd.kind == DCONV_NODE_MAXPOOL) {
      ck(dconv_maxpool_fwd(&src, &out, g->argmax[i], st), "graph maxpool");
      g->launches += 1;
      continue;
    }
    Conv& cv = g->convs[g->conv_of_node[i]];
    dconv_epilogue_t e = epi(nd.add >= 0 ? g->t[nd.add].act : nullptr, nullptr, nd.relu);
    e.flags = DCONV_EP_WEIGHTS_READY;  // prepare_weights
    dconv_act_t x = src;
    dconv_wt_t w = conv_w(g, cv, false);
    if (cv.s2d) {
      dconv_act_t xs = src;
      xs.data = cv.s2d_x;
      xs.c = cv.pspec.C;
      xs.h = cv.pspec.H;
      xs.w = cv.pspec.W;
      if (!(nd.src == 0 && g->input_s2d)) {  // dconv_graph_load_input packed it already
        ck(dconv_s2d_act(&src, &xs, nd.pad_h, st), "graph s2d input");
        g->launches += 1;
      }
      x = xs;
      w = wt_view(cv.s2d_w, cv.pspec.K, cv.pspec.C, cv.pspec.R, cv.pspec.S);
    }
    if (cv.sub) {  // the first strided consumer makes the lattice copy
      x = conv_in(g, cv, false);
      if (!subbed[nd.src]) {
        ck(dconv_subsample2(&src, &x, 0, st), "graph lattice copy");
        g->launches += 1;
        subbed[nd.src] = 1;
      }
    }
    ck(dconv_forward_ex(cv.fp, &x, &w, &out, &e, cv.ws_f, st), "graph forward");
    g->launches += dconv_fwd_launches(cv.fp) - 1;  // (weights prepared)
  }
}

void update(dconv_graph* g, Conv& cv, cudaStream_t s) {
  dconv_stream_t st = reinterpret_cast<dconv_stream_t>(s);
  const dconv_act_t in = conv_in(g, cv, false);  // (s2d / lattice copies: made by this step's forward)
  const dconv_act_t gout = act_of(g, cv.node + 1, true);
  dconv_wt_t dw = conv_w(g, cv, true);
  if (cv.s2d) {
    const dconv_wt_t dw2 = wt_view(cv.s2d_dw, cv.pspec.K, cv.pspec.C, cv.pspec.R, cv.pspec.S);
    ck(dconv_weight_update(cv.up, &in, &gout, &dw2, 0, g->ws_upd, st), "graph update");
    ck(dconv_s2d_wt(&dw, &dw2, 1, st), "graph s2d gradient");
    g->launches += dconv_upd_launches(cv.up, &in, &gout) + 1;
    return;
  }
  ck(dconv_weight_update(cv.up, &in, &gout, &dw, 0, g->ws_upd, st), "graph update");
  g->launches += dconv_upd_launches(cv.up, &in, &gout);
}

void backward(dconv_graph* g, const dconv_act_t* dtop, cudaStream_t s) {
  dconv_stream_t st = reinterpret_cast<dconv_stream_t>(s);
  const int top = static_cast<int>(g->nodes.size());
  const dconv_act_t gtop = act_of(g, top, true), atop = act_of(g, top, false);
  if (dtop->n != gtop.n || dtop->c != gtop.c || dtop->h != gtop.h || dtop->w != gtop.w || dtop->dtype != gtop.dtype ||
      dtop->halo_h || dtop->halo_w || dtop->vlen != 16)
    gfail(DCONV_ERR_SHAPE_MISMATCH, "graph backward: the top gradient must match the last tensor (halo 0, vlen 16)");
  cuck(cudaMemcpyAsync(gtop.data, dtop->data, act_bytes(g, g->t[top]), cudaMemcpyDeviceToDevice, s), "dtop copy");
  if (g->t[top].relu) {
    ck(dconv_relu_mask(&gtop, &atop, st), "graph top mask");
    g->launches += 1;
  }
  std::vector<int> left(g->buckets.size());
  for (size_t b = 0; b < g->buckets.size(); ++b) left[b] = g->buckets[b].n_convs;
  const bool comm = g->cfg.nccl_comm != nullptr && !g->profiling;
  std::vector<char> written(g->t.size(), 0);
  std::vector<int> sub_done(g->t.size(), 0);
  for (int i = static_cast<int>(g->nodes.size()) - 1; i >= 0; --i) {
    const dconv_graph_node_t& nd = g->nodes[i];
    if (nd.kind == DCONV_NODE_MAXPOOL) {
      const dconv_act_t go = act_of(g, i + 1, true), gi = act_of(g, nd.src, true);
      if (g->t[nd.src].relu) {  // ReLU mask of the pooled input, read off the pooled output
        const dconv_act_t pooled = act_of(g, i + 1, false);
        ck(dconv_maxpool_bwd_pooled_mask(&go, g->argmax[i], &gi, &pooled, st), "graph maxpool backward");
      } else {
        ck(dconv_maxpool_bwd(&go, g->argmax[i], &gi, nullptr, st), "graph maxpool backward");
      }
      g->launches += 1;
      written[nd.src] = 1;
      continue;
    }
    Conv& cv = g->convs[g->conv_of_node[i]];
    // weight gradient on the side stream, forked once this conv's dL/dz is final
    cudaStream_t su = g->s_upd ? g->s_upd : s;
    if (su != s) {
      cuck(cudaEventRecord(cv.ev_gready, s), "event");
      cuck(cudaStreamWaitEvent(su, cv.ev_gready, 0), "event wait");
    }
    update(g, cv, su);
    if (comm && --left[cv.bucket] == 0) {
      // every layer of the bucket has its dW: all-reduce it on the communication stream
      const Bucket& b = g->buckets[cv.bucket];
      cuck(cudaEventRecord(cv.ev_dw, su), "event");
      cuck(cudaStreamWaitEvent(g->s_comm, cv.ev_dw, 0), "event wait");
      nck(nccl().all_reduce(g->gflat + b.off, g->gflat + b.off, b.len, ncclFloat, ncclSum,
                            static_cast<ncclComm_t>(g->cfg.nccl_comm), g->s_comm),
          "ncclAllReduce");
    }
    if (nd.src == 0) continue;  // the image gradient is not needed
    if (cv.sub) {
      // lattice consumers: stride-1 backward-data into the lattice gradient (the
      // consumers' sum and the ReLU mask -- the lattice copy -- fused), scattered back
      // to the full-size gradient (zeros off the lattice) after the last consumer
      const dconv_act_t go = act_of(g, i + 1, true), gi = bwd_out(g, cv);
      Tensor& x = g->t[nd.src];
      dconv_epilogue_t e = epi(cv.b_add, cv.b_mask, 0);
      e.flags = DCONV_EP_WEIGHTS_READY;  // prepare_weights
      const dconv_wt_t w = conv_w(g, cv, false);
      ck(dconv_backward_data_ex(cv.bp, &w, &go, &gi, &e, cv.ws_b, st), "graph backward");
      g->launches += dconv_bwd_launches(cv.bp) - dconv_internal_bwd_prep_launches(cv.bp);
      if (++sub_done[nd.src] == x.sub_consumers) {
        const dconv_act_t full = act_of(g, nd.src, true);
        ck(dconv_subsample2(&full, &gi, 1, st), "graph lattice scatter");
        g->launches += 1;
        written[nd.src] = 1;
      }
      continue;
    }
    // data gradient of the conv input, through the ReLU of that tensor, summing branches
    // (epilogue operands: Conv::b_add / b_mask, fixed at build)
    const dconv_act_t go = act_of(g, i + 1, true), gi = bwd_out(g, cv);
    dconv_epilogue_t e = epi(cv.b_add, cv.b_mask, 0);
    e.flags = DCONV_EP_WEIGHTS_READY;  // prepare_weights
    const dconv_wt_t w = conv_w(g, cv, false);
    ck(dconv_backward_data_ex(cv.bp, &w, &go, &gi, &e, cv.ws_b, st), "graph backward");
    g->launches += dconv_bwd_launches(cv.bp) - dconv_internal_bwd_prep_launches(cv.bp);
    written[nd.src] = 1;
  }
  if (g->s_upd) {  // join: every dW final
    cuck(cudaEventRecord(g->ev_upd_done, g->s_upd), "event");
    cuck(cudaStreamWaitEvent(s, g->ev_upd_done, 0), "event wait");
  }
}

void apply(dconv_graph* g, cudaStream_t s) {
  dconv_stream_t st = reinterpret_cast<dconv_stream_t>(s);
  if (g->cfg.nccl_comm) {
    cuck(cudaEventRecord(g->ev_comm_done, g->s_comm), "event");
    cuck(cudaStreamWaitEvent(s, g->ev_comm_done, 0), "event wait");
  }
  const int n256 = static_cast<int>(g->n_params / 256);
  const dconv_wt_t gw = wt_view(g->gflat, 16, 16, 1, n256), ww = wt_view(g->wflat, 16, 16, 1, n256);
  if (g->cfg.world > 1) {  // all-reduced sum -> mean over the global minibatch shards
    ck(dconv_scale_wt(&gw, 1.0f / static_cast<float>(g->cfg.world), st), "graph grad scale");
    g->launches += 1;
  }
  ck(dconv_sgd(&ww, &gw, g->cfg.lr, st), "graph sgd");
  g->launches += 1;
}

}  // namespace

extern "C" {

void dconv_graph_config_default(dconv_graph_config_t* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->lr = 1e-4f;
  c->seed = 1;
  c->bucket_bytes = 8 << 20;
  c->world = 1;
  c->rank = 0;
  c->nccl_comm = nullptr;
  c->overlap_update = 1;
  c->act_dtype = DCONV_BF16;
}

int dconv_graph_create(const dconv_graph_node_t* nodes, int n_nodes, int batch, int in_c, int in_h, int in_w, int math,
                       const dconv_graph_config_t* cfg, dconv_graph_t* out) {
  dconv_graph* g = nullptr;
  const int st = gguard([&] {
    if (!nodes || n_nodes < 1 || !out || batch < 1) gfail(DCONV_ERR_INVALID_ARGUMENT, "graph_create: bad arguments");
    g = new dconv_graph();
    g->nodes.assign(nodes, nodes + n_nodes);
    if (cfg)
      g->cfg = *cfg;
    else
      dconv_graph_config_default(&g->cfg);
    if (g->cfg.world < 1 || g->cfg.rank < 0 || g->cfg.rank >= g->cfg.world)
      gfail(DCONV_ERR_INVALID_ARGUMENT, "graph_create: bad rank / world");
    g->N = batch;
    g->math = math;
    g->dtype = g->cfg.act_dtype;
    if (math == DCONV_MATH_F32 && g->dtype != DCONV_F32)
      gfail(DCONV_ERR_UNSUPPORTED, "graph_create: fp32-accurate math needs fp32 activations");
    build(g, in_c, in_h, in_w);
    if (!g->cfg.overlap_update) {
      cudaStreamDestroy(g->s_upd);
      g->s_upd = nullptr;
    }
    *out = g;
  });
  if (st != DCONV_OK && g) dconv_graph_destroy(g);
  return st;
}

void dconv_graph_destroy(dconv_graph_t g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  for (Conv& cv : g->convs) {
    if (cv.fp) dconv_fwd_plan_destroy(cv.fp);
    if (cv.bp) dconv_bwd_plan_destroy(cv.bp);
    if (cv.up) dconv_upd_plan_destroy(cv.up);
    if (cv.ev_gready) cudaEventDestroy(cv.ev_gready);
    if (cv.ev_dw) cudaEventDestroy(cv.ev_dw);
  }
  for (auto& b : g->buckets)
    if (b.done) cudaEventDestroy(b.done);
  for (cudaEvent_t e : {g->ev_fork, g->ev_upd_done, g->ev_comm_done})
    if (e) cudaEventDestroy(e);
  if (g->s_upd) cudaStreamDestroy(g->s_upd);
  if (g->s_comm) cudaStreamDestroy(g->s_comm);
  for (void* p : g->allocs) cudaFree(p);
  delete g;
}

int dconv_graph_load_input(dconv_graph_t g, const float* nchw, dconv_stream_t stream) {
  return gguard([&] {
    if (!g || !nchw) gfail(DCONV_ERR_INVALID_ARGUMENT, "graph_load_input: null argument");
    const Tensor& x = g->t[0];
    const int stem = g->conv_of_node.empty() ? -1 : g->conv_of_node[0];
    // straight into the stem's space-to-depth layout when the stem runs that way (one
    // pass, no full-resolution 16-lane copy); the stem's own s2d is then skipped
    for (Conv& cv : g->convs)
      if (g->nodes[cv.node].src == 0 && cv.s2d) {
        dconv_act_t xs = act_of(g, 0, false);
        xs.data = cv.s2d_x;
        xs.c = cv.pspec.C;
        xs.h = cv.pspec.H;
        xs.w = cv.pspec.W;
        ck(dconv_pack_s2d(nchw, g->N, x.c, x.h, x.w, &xs, g->nodes[cv.node].pad_h, stream), "graph load input");
        g->input_s2d = true;
        return;
      }
    (void)stem;
    const dconv_act_t a = act_of(g, 0, false);
    ck(dconv_pack_act(nchw, DCONV_F32, &a, stream), "graph load input");
  });
}

int dconv_graph_forward(dconv_graph_t g, dconv_stream_t stream) {
  return gguard([&] {
    if (!g) gfail(DCONV_ERR_INVALID_ARGUMENT, "null graph");
    g->launches = 0;
    forward(g, reinterpret_cast<cudaStream_t>(stream));
  });
}

int dconv_graph_backward(dconv_graph_t g, const dconv_act_t* dtop, dconv_stream_t stream) {
  return gguard([&] {
    if (!g || !dtop) gfail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    backward(g, dtop, reinterpret_cast<cudaStream_t>(stream));
  });
}

int dconv_graph_apply(dconv_graph_t g, dconv_stream_t stream) {
  return gguard([&] {
    if (!g) gfail(DCONV_ERR_INVALID_ARGUMENT, "null graph");
    apply(g, reinterpret_cast<cudaStream_t>(stream));
  });
}

int dconv_graph_step(dconv_graph_t g, const dconv_act_t* dtop, dconv_stream_t stream) {
  return gguard([&] {
    if (!g || !dtop) gfail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    g->launches = 0;
    forward(g, s);
    backward(g, dtop, s);
    apply(g, s);
  });
}

int dconv_graph_capture(dconv_graph_t g, const dconv_act_t* dtop, dconv_stream_t stream) {
  return gguard([&] {
    if (!g || !dtop) gfail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!s) gfail(DCONV_ERR_INVALID_ARGUMENT, "graph_capture: needs a non-default stream");
    if (g->exec) cudaGraphExecDestroy(g->exec), g->exec = nullptr;
    if (g->graph) cudaGraphDestroy(g->graph), g->graph = nullptr;
    cuck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      g->launches = 0;
      forward(g, s);
      backward(g, dtop, s);
      apply(g, s);
    } catch (...) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(s, &junk);
      if (junk) cudaGraphDestroy(junk);
      throw;
    }
    cuck(cudaStreamEndCapture(s, &g->graph), "end capture");
    cuck(cudaGraphInstantiate(&g->exec, g->graph, 0), "graph instantiate");
  });
}

int dconv_graph_replay(dconv_graph_t g, dconv_stream_t stream) {
  return gguard([&] {
    if (!g || !g->exec) gfail(DCONV_ERR_INVALID_ARGUMENT, "graph_replay: no captured step");
    cuck(cudaGraphLaunch(g->exec, reinterpret_cast<cudaStream_t>(stream)), "graph launch");
  });
}

int dconv_graph_profile(dconv_graph_t g, const dconv_act_t* dtop, int reps, float* ms, dconv_stream_t stream) {
  return gguard([&] {
    if (!g || !dtop || !ms || reps < 1) gfail(DCONV_ERR_INVALID_ARGUMENT, "graph_profile: bad arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    dconv_stream_t st = stream;
    // one whole step first: every tensor holds this step's values (and every plan is resolved)
    g->profiling = true;
    struct Reset {
      dconv_graph* g;
      ~Reset() { g->profiling = false; }
    } reset{g};
    forward(g, s);
    backward(g, dtop, s);
    cuck(cudaStreamSynchronize(s), "profile sync");
    cudaEvent_t e0, e1;
    cuck(cudaEventCreate(&e0), "event");
    cuck(cudaEventCreate(&e1), "event");
    auto timed = [&](auto&& fn) -> float {
      fn();  // warm
      float best = 1e30f;
      for (int trial = 0; trial < 2; ++trial) {
        cuck(cudaEventRecord(e0, s), "event");
        for (int r = 0; r < reps; ++r) fn();
        cuck(cudaEventRecord(e1, s), "event");
        cuck(cudaEventSynchronize(e1), "event sync");
        float t = 0;
        cuck(cudaEventElapsedTime(&t, e0, e1), "elapsed");
        best = std::min(best, t / reps);
      }
      return best;
    };
    for (size_t ci = 0; ci < g->convs.size(); ++ci) {
      Conv& cv = g->convs[ci];
      const dconv_graph_node_t& nd = g->nodes[cv.node];
      const dconv_act_t out = act_of(g, cv.node + 1, false);
      const dconv_act_t x = conv_in(g, cv, false);
      dconv_wt_t w = conv_w(g, cv, false);
      if (cv.s2d) w = wt_view(cv.s2d_w, cv.pspec.K, cv.pspec.C, cv.pspec.R, cv.pspec.S);
      // as the step runs them: weights prepared (by the forward above), fused epilogues
      dconv_epilogue_t e = epi(nd.add >= 0 ? g->t[nd.add].act : nullptr, nullptr, nd.relu);
      e.flags = DCONV_EP_WEIGHTS_READY;
      ms[3 * ci + 0] = timed([&] { ck(dconv_forward_ex(cv.fp, &x, &w, &out, &e, cv.ws_f, st), "profile fwd"); });
      ms[3 * ci + 1] = 0.0f;
      if (cv.bp) {
        const dconv_act_t go = act_of(g, cv.node + 1, true), gi = bwd_out(g, cv);
        dconv_epilogue_t eb = epi(cv.b_add, cv.b_mask, 0);
        eb.flags = DCONV_EP_WEIGHTS_READY;
        const dconv_wt_t wf = conv_w(g, cv, false);
        ms[3 * ci + 1] =
            timed([&] { ck(dconv_backward_data_ex(cv.bp, &wf, &go, &gi, &eb, cv.ws_b, st), "profile bwd"); });
      }
      ms[3 * ci + 2] = timed([&] { update(g, cv, s); });
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int dconv_graph_launches(dconv_graph_t g) { return g ? g->launches : -1; }
int dconv_graph_num_tensors(dconv_graph_t g) { return g ? static_cast<int>(g->t.size()) : -1; }
int dconv_graph_num_convs(dconv_graph_t g) { return g ? static_cast<int>(g->convs.size()) : -1; }

int dconv_graph_tensor(dconv_graph_t g, int id, int grad, dconv_act_t* out) {
  return gguard([&] {
    if (!g || !out || id < 0 || id >= static_cast<int>(g->t.size()) || (grad && id == 0))
      gfail(DCONV_ERR_INVALID_ARGUMENT, "graph_tensor: bad id");
    *out = act_of(g, id, grad != 0);
  });
}

int dconv_graph_conv(dconv_graph_t g, int conv, int* node, dconv_wt_t* w, dconv_wt_t* dw) {
  return gguard([&] {
    if (!g || conv < 0 || conv >= static_cast<int>(g->convs.size())) gfail(DCONV_ERR_INVALID_ARGUMENT, "bad conv");
    const Conv& cv = g->convs[conv];
    if (node) *node = cv.node;
    if (w) *w = conv_w(g, cv, false);
    if (dw) *dw = conv_w(g, cv, true);
  });
}

int dconv_graph_grads(dconv_graph_t g, float** flat, size_t* n) {
  return gguard([&] {
    if (!g || !flat || !n) gfail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    *flat = g->gflat;
    *n = g->n_params;
  });
}

int dconv_graph_weights(dconv_graph_t g, float** flat, size_t* n) {
  return gguard([&] {
    if (!g || !flat || !n) gfail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    *flat = g->wflat;
    *n = g->n_params;
  });
}

int dconv_graph_buckets(dconv_graph_t g) { return g ? static_cast<int>(g->buckets.size()) : -1; }

int dconv_nccl_unique_id(char* id, size_t len) {
  return gguard([&] {
    if (!id || len < sizeof(ncclUniqueId)) gfail(DCONV_ERR_INVALID_ARGUMENT, "nccl id buffer too small (128 bytes)");
    ncclUniqueId u;
    nck(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int dconv_nccl_comm_create(const char* id, size_t len, int world, int rank, void** comm) {
  return gguard([&] {
    if (!id || len < sizeof(ncclUniqueId) || !comm) gfail(DCONV_ERR_INVALID_ARGUMENT, "nccl comm: bad arguments");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    nck(nccl().init_rank(&c, world, u, rank), "ncclCommInitRank");
    *comm = c;
  });
}

int dconv_nccl_comm_destroy(void* comm) {
  return gguard([&] {
    if (comm) nck(nccl().destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

}  // extern "C"
