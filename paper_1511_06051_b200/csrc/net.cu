// class Net (model.hpp:50-597) on one B200: shape inference and init on the host
// (bit-exact with the reference RNG), flat fp32 parameter / gradient / velocity
// buffers in HBM, NHWC activations, and one CUDA graph per training step
// (gather -> forward -> loss -> backward -> fused SGD update).
#include <mutex>
#include <unordered_map>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "runtime.h"

namespace psg {

namespace {

constexpr size_t kAlign = 32;  // tensor offsets in floats (128 B)

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

bool is_param_layer(int kind) { return kind == PSG_LAYER_CONV || kind == PSG_LAYER_LINEAR; }

int pool_out(int in, int k, int s, int p, int ceil_mode) {
  int o;
  if (ceil_mode) {
    o = (in + 2 * p - k + s - 1) / s + 1;
    if (p > 0 && (o - 1) * s >= in + p) --o;
  } else {
    o = (in + 2 * p - k) / s + 1;  // model.hpp:244-245
  }
  return o;
}

// Guard bands (PSG_GUARD=1; compute-sanitizer is not available on the GPU pool): every
// net allocation gets kGuardBytes of 0xA5 before and after it (plus the tail up to the next
// 256 bytes); psg_debug_guard_violations() / dfree compare them after the kernels ran, so a
// kernel writing outside any activation / gradient / parameter / workspace buffer is caught.
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;

bool guard_on() {
  static const bool v = [] {
    const char* e = std::getenv("PSG_GUARD");
    return e && std::atoi(e) != 0;
  }();
  return v;
}

struct GuardAlloc {
  size_t bytes, padded;
};
std::mutex g_guard_mu;
std::unordered_map<uintptr_t, GuardAlloc> g_guard_live;  // user pointer -> sizes
unsigned long long g_guard_bad = 0;
std::string g_guard_first;

unsigned long long guard_check(uintptr_t user, const GuardAlloc& a) {
  std::vector<unsigned char> h(kGuardBytes + (a.padded - a.bytes) + kGuardBytes);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(user) - kGuardBytes;
  PSG_CUDA(cudaMemcpy(h.data(), base, kGuardBytes, cudaMemcpyDeviceToHost));
  PSG_CUDA(cudaMemcpy(h.data() + kGuardBytes, base + kGuardBytes + a.bytes,
                      h.size() - kGuardBytes, cudaMemcpyDeviceToHost));
  unsigned long long bad = 0;
  for (unsigned char c : h) bad += c != kGuardByte;
  if (bad && g_guard_first.empty())
    g_guard_first = "allocation of " + std::to_string(a.bytes) + " bytes: " + std::to_string(bad) +
                    " guard bytes overwritten";
  return bad;
}

template <class T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (!n) return p;
  if (!guard_on()) {
    PSG_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return p;
  }
  const size_t bytes = n * sizeof(T), padded = (bytes + 255) / 256 * 256;
  unsigned char* base = nullptr;
  PSG_CUDA(cudaMalloc(&base, padded + 2 * kGuardBytes));
  PSG_CUDA(cudaMemset(base, kGuardByte, kGuardBytes));
  PSG_CUDA(cudaMemset(base + kGuardBytes + bytes, kGuardByte, padded - bytes + kGuardBytes));
  PSG_CUDA(cudaDeviceSynchronize());  // the non-blocking net streams do not wait for memsets
  std::lock_guard<std::mutex> lock(g_guard_mu);
  g_guard_live[reinterpret_cast<uintptr_t>(base + kGuardBytes)] = GuardAlloc{bytes, padded};
  return reinterpret_cast<T*>(base + kGuardBytes);
}

void dfree(void* p) {
  if (!p) return;
  if (guard_on()) {
    std::lock_guard<std::mutex> lock(g_guard_mu);
    auto it = g_guard_live.find(reinterpret_cast<uintptr_t>(p));
    if (it != g_guard_live.end()) {
      cudaDeviceSynchronize();
      g_guard_bad += guard_check(it->first, it->second);
      g_guard_live.erase(it);
      cudaFree(static_cast<unsigned char*>(p) - kGuardBytes);
      return;
    }
  }
  cudaFree(p);
}

std::string lname(const psg_layer_desc& d) { return std::string(d.name); }

// NetSpec::validate (net_spec.hpp:112-169) on the C descriptors.
void validate(const psg_layer_desc* layers, int n) {
  int n_data = 0, n_label = 0, n_loss = 0;
  for (int li = 0; li < n; ++li) {
    const psg_layer_desc& d = layers[li];
    if (d.name[0] == 0) throw std::invalid_argument("net: layer with empty name");
    for (int j = 0; j < li; ++j)
      if (std::strncmp(layers[j].name, d.name, sizeof d.name) == 0)
        throw std::invalid_argument("net: duplicate layer name '" + lname(d) + "'");
    if (d.n_inputs < 0 || d.n_inputs > 8) throw std::invalid_argument("net: bad input count");
    for (int i = 0; i < d.n_inputs; ++i)
      if (d.inputs[i] < 0 || d.inputs[i] >= li)
        throw std::invalid_argument("net: layer '" + lname(d) +
                                    "' references a layer which is not declared earlier");
    switch (d.kind) {
      case PSG_LAYER_DATA:
        ++n_data;
        if (d.batch < 1 || d.channels < 1 || d.height < 1 || d.width < 1)
          throw std::invalid_argument("net: data layer needs [b,c,h,w]");
        break;
      case PSG_LAYER_LABEL:
        ++n_label;
        break;
      case PSG_LAYER_CONV:
        if (d.n_inputs != 1) throw std::invalid_argument("net: conv takes one input");
        if (d.kernel_h < 1 || d.kernel_w < 1 || d.num_output < 1 || d.stride_h < 1 ||
            d.stride_w < 1 || d.pad_h < 0 || d.pad_w < 0 || d.group < 1)
          throw std::invalid_argument("net: conv '" + lname(d) + "' has non-positive geometry");
        break;
      case PSG_LAYER_POOL:
        if (d.n_inputs != 1) throw std::invalid_argument("net: pool takes one input");
        if (d.kernel_h < 1 || d.kernel_w < 1 || d.stride_h < 1 || d.stride_w < 1 ||
            d.kernel_h * d.kernel_w > 255)
          throw std::invalid_argument("net: pool '" + lname(d) + "' has non-positive geometry");
        break;
      case PSG_LAYER_LINEAR:
        if (d.n_inputs != 1) throw std::invalid_argument("net: linear takes one input");
        if (d.num_output < 1)
          throw std::invalid_argument("net: linear '" + lname(d) + "' needs positive outputs");
        break;
      case PSG_LAYER_RELU:
      case PSG_LAYER_LRN:
      case PSG_LAYER_DROPOUT:
        if (d.n_inputs != 1) throw std::invalid_argument("net: layer takes one input");
        if (d.kind == PSG_LAYER_LRN && (d.local_size < 1 || d.local_size % 2 == 0))
          throw std::invalid_argument("net: lrn local_size must be odd");
        if (d.kind == PSG_LAYER_DROPOUT && !(d.dropout_ratio >= 0.0 && d.dropout_ratio < 1.0))
          throw std::invalid_argument("net: dropout ratio must be in [0,1)");
        break;
      case PSG_LAYER_SOFTMAX_LOSS:
        ++n_loss;
        if (d.n_inputs != 2) throw std::invalid_argument("net: softmax loss takes [logits, label]");
        break;
      case PSG_LAYER_CONCAT:
        if (d.n_inputs < 1) throw std::invalid_argument("net: concat needs inputs");
        break;
      default:
        throw std::invalid_argument("net: unsupported layer kind");
    }
  }
  if (n_data != 1) throw std::invalid_argument("net: exactly one data layer required");
  if (n_label != 1) throw std::invalid_argument("net: exactly one label layer required");
  if (n_loss < 1) throw std::invalid_argument("net: at least one softmax loss layer required");
}

void free_batch_buffers(psg_net* net) {
  for (LayerRt& l : net->L)
    if (l.fwd_relu >= 0) l.out = nullptr;  // aliases the ReLU's buffer
  for (LayerRt& l : net->L) {
    dfree(l.out);
    dfree(l.grad);
    dfree(l.route);
    dfree(l.col);
    for (float* p : l.acc_scratch) dfree(p);
    l.acc_scratch.clear();
    l.out = l.grad = l.col = nullptr;
    l.route = nullptr;
  }
  dfree(net->row_loss);
  dfree(net->labels);
  dfree(net->ws.ptr);
  for (Workspace& w : net->ws_lane) {
    dfree(w.ptr);
    w = Workspace{};
  }
  net->row_loss = nullptr;
  net->labels = nullptr;
  net->ws = Workspace{};
  net->cap = 0;
}

ConvGeom geom_for(const LayerRt& l, size_t n) {
  ConvGeom g = l.cg;
  g.n = static_cast<int>(n);
  return g;
}

}  // namespace

unsigned long long guard_violations(std::string* first) {
  if (!guard_on()) throw std::logic_error("guard bands are off (set PSG_GUARD=1)");
  PSG_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lock(g_guard_mu);
  unsigned long long bad = g_guard_bad;
  for (const auto& kv : g_guard_live) bad += guard_check(kv.first, kv.second);
  if (first) *first = g_guard_first;
  return bad;
}

// Synchronous copy ordered on the net's stream.  A plain cudaMemcpy runs on the legacy
// default stream, which the non-blocking net stream neither waits for nor is waited on by,
// and a pageable H2D cudaMemcpy may return before its DMA lands: stream-ordered + synced.
void copy_sync(psg_net* net, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  PSG_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, net->stream));
  PSG_CUDA(cudaStreamSynchronize(net->stream));
}

void invalidate_graph(psg_net* net) {
  if (net->graph) cudaGraphExecDestroy(net->graph);
  if (net->host_graph) cudaGraphExecDestroy(net->host_graph);
  for (auto& gx : net->host_graph2) {
    if (gx) cudaGraphExecDestroy(gx);
    gx = nullptr;
  }
  if (net->grad_graph) cudaGraphExecDestroy(net->grad_graph);
  if (net->round_graph) cudaGraphExecDestroy(net->round_graph);
  net->round_graph = nullptr;
  net->round_graph_batch = 0;
  net->graph = nullptr;
  net->host_graph = nullptr;
  net->grad_graph = nullptr;
  net->graph_batch = 0;
  net->grad_graph_batch = 0;
}

void plan_fusion(psg_net* net) {
  for (LayerRt& l : net->L)
    l.fwd_relu = l.fused_from = l.bwd_by = l.bwd_relu = l.lrn_pool = l.pool_lrn = -1;
  if (!net->fuse) return;
  static const bool lrn_pool = [] {  // PSG_FUSE_LRN_POOL=0: keep LRN and pool separate (A/B)
    const char* e = std::getenv("PSG_FUSE_LRN_POOL");
    return e ? std::atoi(e) != 0 : true;
  }();
  for (size_t li = 0; lrn_pool && li < net->L.size(); ++li) {
    LayerRt& l = net->L[li];
    if (l.kind != PSG_LAYER_LRN || l.consumers.size() != 1) continue;
    LayerRt& p = net->L[l.consumers[0]];
    if (p.kind == PSG_LAYER_POOL && p.inputs.size() == 1 && lrn_maxpool_fusable(l.lg, p.pg)) {
      l.lrn_pool = l.consumers[0];
      p.pool_lrn = static_cast<int>(li);
    }
  }
  for (size_t ri = 0; ri < net->L.size(); ++ri) {
    LayerRt& r = net->L[ri];
    if (r.kind != PSG_LAYER_RELU) continue;
    LayerRt& p = net->L[r.inputs[0]];
    if ((p.kind == PSG_LAYER_CONV || p.kind == PSG_LAYER_LINEAR) && p.consumers.size() == 1) {
      p.fwd_relu = static_cast<int>(ri);
      r.fused_from = r.inputs[0];
    }
    if (p.kind != PSG_LAYER_DATA && p.consumers.size() == 1 && r.consumers.size() == 1) {
      LayerRt& c = net->L[r.consumers[0]];
      if (c.kind == PSG_LAYER_LRN) {
        r.bwd_by = r.consumers[0];
        c.bwd_relu = static_cast<int>(ri);
      }
    }
  }
}

// Branch lanes (psg_net::lane_of): a layer inherits its input's lane; the k-th consumer of a
// layer with several consumers takes lane (lane + k) % kLanes; joins (several inputs) and the
// loss layers (they accumulate one device loss in layer order) run on lane 0.  Fan-out lanes
// are off for nets without fan-out; PSG_LANES=0 turns every lane (and the wgrad lane) off.
void assign_lanes(psg_net* net) {
  const char* lanes_env = std::getenv("PSG_LANES");  // read per build (tests toggle it)
  const bool env = !lanes_env || std::atoi(lanes_env) != 0;
  const int nl = static_cast<int>(net->L.size());
  net->lane_of.assign(nl, 0);
  bool fanout = false;
  for (const LayerRt& l : net->L)
    if (l.kind != PSG_LAYER_DATA && l.kind != PSG_LAYER_LABEL && l.consumers.size() > 1)
      fanout = true;
  const char* wl = std::getenv("PSG_WGRAD_LANE");
  net->wgrad_lane = env && (!wl || std::atoi(wl) != 0);
  net->lanes_on = (env && fanout) || net->wgrad_lane;
  net->fanout = env && fanout;
  if (!net->lanes_on) return;
  for (int li = 0; li < nl && fanout; ++li) {
    const LayerRt& l = net->L[li];
    if (l.inputs.size() != 1 || l.kind == PSG_LAYER_SOFTMAX_LOSS) continue;  // lane 0
    const LayerRt& p = net->L[l.inputs[0]];
    int k = 0;
    if (p.kind != PSG_LAYER_DATA && p.consumers.size() > 1)
      for (size_t c = 0; c < p.consumers.size(); ++c)
        if (p.consumers[c] == li) k = static_cast<int>(c);
    net->lane_of[li] = (net->lane_of[l.inputs[0]] + k) % psg_net::kLanes;
  }
  for (int k = 1; k < psg_net::kStreams; ++k)
    PSG_CUDA(cudaStreamCreateWithFlags(&net->lane_stream[k], cudaStreamNonBlocking));
  PSG_CUDA(cudaEventCreateWithFlags(&net->lane_fork, cudaEventDisableTiming));
  for (int k = 0; k < psg_net::kStreams; ++k)
    PSG_CUDA(cudaEventCreateWithFlags(&net->lane_join[k], cudaEventDisableTiming));
  net->ev_fwd.resize(nl);
  net->ev_bwd.resize(nl);
  net->ev_sum.resize(nl);
  for (int li = 0; li < nl; ++li) {
    PSG_CUDA(cudaEventCreateWithFlags(&net->ev_fwd[li], cudaEventDisableTiming));
    PSG_CUDA(cudaEventCreateWithFlags(&net->ev_bwd[li], cudaEventDisableTiming));
    PSG_CUDA(cudaEventCreateWithFlags(&net->ev_sum[li], cudaEventDisableTiming));
  }
}

void release_batch_buffers(psg_net* net) {
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  invalidate_graph(net);
  free_batch_buffers(net);
}

// Activation / gradient buffers for a batch of n rows.
void ensure_capacity(psg_net* net, size_t n) {
  if (net->cap >= n) return;
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  invalidate_graph(net);
  free_batch_buffers(net);
  size_t ws = 0;
  for (LayerRt& l : net->L) {
    if (l.kind == PSG_LAYER_LABEL) continue;
    const size_t elems = n * l.vol();
    if (l.fwd_relu < 0 && l.lrn_pool < 0) l.out = dalloc<float>(elems);
    if (l.kind != PSG_LAYER_DATA && l.lrn_pool < 0) l.grad = dalloc<float>(elems);
    if (l.kind == PSG_LAYER_POOL && l.d.pool == PSG_POOL_MAX) l.route = dalloc<uint8_t>(elems);
    if (l.kind == PSG_LAYER_CONV) l.col = dalloc<float>(conv_col_elems(geom_for(l, n), net->mode));
    if (is_param_layer(l.kind)) {
      for (Mode m : {Mode::Strict, Mode::Tf32})
        ws = std::max(ws, conv_workspace_elems(geom_for(l, n), m));
    }
  }
  for (LayerRt& l : net->L)
    if (l.fwd_relu >= 0) l.out = net->L[l.fwd_relu].out;
  // branch lanes: scratch for every gradient writer after the first (consumers, and the
  // consumers of a single-consumer ReLU among them that fold its backward)
  for (LayerRt& l : net->L) {
    if (!net->fanout || !l.grad) continue;
    size_t writers = l.consumers.size();
    for (int c : l.consumers)
      if (net->L[c].kind == PSG_LAYER_RELU) writers += net->L[c].consumers.size();
    for (size_t j = 1; j < writers; ++j) l.acc_scratch.push_back(dalloc<float>(n * l.vol()));
  }
  // the data layer's grad is never produced (first-layer dgrad is skipped)
  net->row_loss = dalloc<double>(n);
  net->labels = dalloc<int32_t>(n);
  net->ws.ptr = dalloc<float>(ws);
  net->ws.elems = ws;
  for (int k = 1; net->lanes_on && k < psg_net::kStreams; ++k) {
    net->ws_lane[k].ptr = dalloc<float>(ws);
    net->ws_lane[k].elems = ws;
  }
  net->cap = n;
}

namespace {

void ensure_stage(psg_net* net, size_t floats, size_t rows) {
  if (net->h_stage_cap >= floats && net->h_lab) return;
  if (net->h_stage) cudaFreeHost(net->h_stage);
  if (net->h_lab) cudaFreeHost(net->h_lab);
  PSG_CUDA(cudaMallocHost(&net->h_stage, std::max<size_t>(floats, 1) * sizeof(float)));
  PSG_CUDA(cudaMallocHost(&net->h_lab, std::max<size_t>(rows, 1024) * sizeof(int32_t)));
  net->h_stage_cap = floats;
}

void build_chunks(psg_net* net) {
  std::vector<UpdateChunk> ch;
  constexpr uint32_t piece = 8192;
  for (LayerRt& l : net->L) l.chunk0 = l.nchunk = 0;
  for (const TensorRec& t : net->tensors) {
    LayerRt& l = net->L[t.layer];
    if (l.nchunk == 0) l.chunk0 = static_cast<int>(ch.size());
    l.nchunk += static_cast<int>((t.int_count + piece - 1) / piece);
    const float lr = static_cast<float>(net->lr * t.lr_mult);
    const float wd = static_cast<float>(net->wd * t.decay_mult);
    for (size_t b = t.int_off; b < t.int_off + t.int_count; b += piece) {
      const size_t e = std::min(t.int_off + t.int_count, b + piece);
      ch.push_back(UpdateChunk{static_cast<uint32_t>(b), static_cast<uint32_t>(e), lr, wd});
    }
  }
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  if (static_cast<int>(ch.size()) != net->nchunks) {
    dfree(net->d_chunks);
    net->d_chunks = dalloc<UpdateChunk>(ch.size());
    net->nchunks = static_cast<int>(ch.size());
    invalidate_graph(net);
  }
  if (!ch.empty())
    copy_sync(net, net->d_chunks, ch.data(), ch.size() * sizeof(UpdateChunk),
                        cudaMemcpyHostToDevice);
}

// Host NCHW fp64 batch -> device NHWC (channel stride cs) into the data layer.
void upload_batch(psg_net* net, const double* images, const int32_t* labels, size_t n) {
  const LayerRt& d = net->L[net->data_idx];
  if (n < 1) throw std::invalid_argument("forward: label count does not match batch");
  for (size_t i = 0; i < n; ++i)
    if (labels[i] < 0 || labels[i] >= net->classes)
      throw std::invalid_argument("forward: label out of range");
  ensure_capacity(net, n);
  const size_t vol = d.vol();
  ensure_stage(net, n * vol, n);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  const int C = d.C, H = d.H, W = d.W, cs = d.cs;
  for (size_t b = 0; b < n; ++b)
    for (int h = 0; h < H; ++h)
      for (int w = 0; w < W; ++w)
        for (int c = 0; c < cs; ++c)
          net->h_stage[((b * H + h) * W + w) * cs + c] =
              c < C ? static_cast<float>(images[((b * C + c) * H + h) * W + w]) : 0.f;
  std::memcpy(net->h_lab, labels, n * sizeof(int32_t));
  PSG_CUDA(cudaMemcpyAsync(d.out, net->h_stage, n * vol * sizeof(float), cudaMemcpyHostToDevice,
                           net->stream));
  PSG_CUDA(cudaMemcpyAsync(net->labels, net->h_lab, n * sizeof(int32_t), cudaMemcpyHostToDevice,
                           net->stream));
}

double read_loss(psg_net* net) {
  PSG_CUDA(cudaMemcpyAsync(net->hsc, net->dsc, sizeof(DeviceScalars), cudaMemcpyDeviceToHost,
                           net->stream));
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  if (net->hsc->flag) {
    const int zero = 0;
    copy_sync(net, &net->dsc->flag, &zero, sizeof(int), cudaMemcpyHostToDevice);
    throw std::runtime_error("softmax loss: non-finite loss");
  }
  return net->hsc->loss;
}

}  // namespace

size_t TensorRec::to_int(size_t i) const {
  switch (map) {
    case 1: {  // ref [F][Cg][kh][kw] -> int [F][kh][kw][Cgs]
      const size_t v = i % kw, u = (i / kw) % kh, c = (i / (kw * kh)) % Cg,
                   f = i / (static_cast<size_t>(kw) * kh * Cg);
      return f * Kp + (u * kw + v) * Cgs + c;
    }
    case 2: {  // ref [O][c*h*w] (CHW flatten, model.hpp:409) -> int [O][h][w][pcs]
      const size_t D = static_cast<size_t>(pc) * ph * pw;
      const size_t o = i / D, d = i % D;
      const size_t ww = d % pw, hh = (d / pw) % ph, c = d / (static_cast<size_t>(pw) * ph);
      return o * (static_cast<size_t>(ph) * pw * pcs) + (hh * pw + ww) * pcs + c;
    }
    default:
      return i;
  }
}

void net_build(psg_net* net, const psg_layer_desc* layers, int n, uint64_t seed) {
  validate(layers, n);
  net->seed = seed;
  net->L.resize(n);
  size_t ref_off = 0, int_off = 0;
  for (int li = 0; li < n; ++li) {
    LayerRt& l = net->L[li];
    l.d = layers[li];
    l.kind = layers[li].kind;
    for (int i = 0; i < l.d.n_inputs; ++i) {
      l.inputs.push_back(l.d.inputs[i]);
      net->L[l.d.inputs[i]].consumers.push_back(li);
    }
    const LayerRt* src = l.inputs.empty() ? nullptr : &net->L[l.inputs[0]];
    switch (l.kind) {
      case PSG_LAYER_DATA:
        net->data_idx = li;
        net->spec_batch = l.d.batch;
        l.C = l.d.channels;
        l.H = l.d.height;
        l.W = l.d.width;
        l.cs = l.C;
        break;
      case PSG_LAYER_LABEL:
        net->label_idx = li;
        l.C = l.H = l.W = l.cs = 1;
        break;
      case PSG_LAYER_CONV: {
        const int C = src->C, G = l.d.group;
        if (src->H + 2 * l.d.pad_h < l.d.kernel_h || src->W + 2 * l.d.pad_w < l.d.kernel_w)
          throw std::invalid_argument("net: conv '" + lname(l.d) + "' kernel exceeds input");
        if (C % G || l.d.num_output % G)
          throw std::invalid_argument("net: conv '" + lname(l.d) +
                                      "' group must divide channels and filters");
        if (G > 1 && src->cs != C)
          throw std::invalid_argument("net: grouped conv on a padded input");
        l.C = l.cs = l.d.num_output;
        l.H = (src->H + 2 * l.d.pad_h - l.d.kernel_h) / l.d.stride_h + 1;
        l.W = (src->W + 2 * l.d.pad_w - l.d.kernel_w) / l.d.stride_w + 1;
        ConvGeom& g = l.cg;
        g.H = src->H;
        g.W = src->W;
        g.cs_in = src->cs;
        g.OH = l.H;
        g.OW = l.W;
        g.F = l.C;
        g.kh = l.d.kernel_h;
        g.kw = l.d.kernel_w;
        g.sh = l.d.stride_h;
        g.sw = l.d.stride_w;
        g.ph = l.d.pad_h;
        g.pw = l.d.pad_w;
        g.G = G;
        g.kp = static_cast<int>(round_up(static_cast<size_t>(g.Kf()), 4));  // 16-byte rows
        TensorRec k;
        k.layer = li;
        k.slot = 0;
        k.rank = 4;
        k.shape[0] = l.C;
        k.shape[1] = C / G;
        k.shape[2] = g.kh;
        k.shape[3] = g.kw;
        k.ref_count = static_cast<size_t>(l.C) * (C / G) * g.kh * g.kw;
        k.int_count = static_cast<size_t>(l.C) * g.Kp();
        k.map = 1;
        k.F = l.C;
        k.Cg = C / G;
        k.Cgs = g.Cgs();
        k.kh = g.kh;
        k.kw = g.kw;
        k.Kp = g.Kp();
        k.lr_mult = static_cast<float>(l.d.lr_mult_w);
        k.decay_mult = static_cast<float>(l.d.decay_mult_w);
        net->tensors.push_back(k);
        break;
      }
      case PSG_LAYER_POOL:
        if (src->H + 2 * l.d.pad_h < l.d.kernel_h || src->W + 2 * l.d.pad_w < l.d.kernel_w)
          throw std::invalid_argument("net: pool '" + lname(l.d) + "' kernel exceeds input");
        l.C = src->C;
        l.cs = src->cs;
        l.H = pool_out(src->H, l.d.kernel_h, l.d.stride_h, l.d.pad_h, l.d.ceil_mode);
        l.W = pool_out(src->W, l.d.kernel_w, l.d.stride_w, l.d.pad_w, l.d.ceil_mode);
        l.pg = PoolGeom{0,         src->H,     src->W,     l.cs,        l.H,
                        l.W,       l.d.kernel_h, l.d.kernel_w, l.d.stride_h, l.d.stride_w,
                        l.d.pad_h, l.d.pad_w,  l.d.pool};
        break;
      case PSG_LAYER_LINEAR: {
        l.C = l.cs = l.d.num_output;
        l.H = l.W = 1;
        const size_t Dint = src->vol();
        ConvGeom& g = l.cg;
        g.H = g.W = g.OH = g.OW = 1;
        g.cs_in = static_cast<int>(Dint);
        g.F = l.C;
        TensorRec k;
        k.layer = li;
        k.slot = 0;
        k.rank = 2;
        k.shape[0] = l.C;
        k.shape[1] = static_cast<int64_t>(src->C) * src->H * src->W;
        k.ref_count = static_cast<size_t>(k.shape[0]) * k.shape[1];
        k.int_count = static_cast<size_t>(l.C) * Dint;
        k.map = (src->H == 1 && src->W == 1 && src->cs == src->C) ? 0 : 2;
        k.O = l.C;
        k.pc = src->C;
        k.ph = src->H;
        k.pw = src->W;
        k.pcs = src->cs;
        k.lr_mult = static_cast<float>(l.d.lr_mult_w);
        k.decay_mult = static_cast<float>(l.d.decay_mult_w);
        net->tensors.push_back(k);
        break;
      }
      case PSG_LAYER_RELU:
      case PSG_LAYER_LRN:
      case PSG_LAYER_DROPOUT:
        l.C = src->C;
        l.H = src->H;
        l.W = src->W;
        l.cs = src->cs;
        if (l.kind == PSG_LAYER_LRN) {
          if (l.cs != l.C) throw std::invalid_argument("net: lrn on a padded input");
          l.lg = LrnGeom{0, l.C, l.d.local_size, static_cast<float>(l.d.alpha),
                         static_cast<float>(l.d.beta), static_cast<float>(l.d.k)};
        }
        if (l.kind == PSG_LAYER_DROPOUT) {
          if (l.cs != l.C) throw std::invalid_argument("net: dropout on a padded input");
          const uint64_t p[2] = {kStreamDropout, static_cast<uint64_t>(li)};
          l.dg = DropGeom{0, l.C, l.H, l.W, static_cast<float>(l.d.dropout_ratio),
                          derive_seed(seed, p, 2)};
        }
        break;
      case PSG_LAYER_SOFTMAX_LOSS:
        if (net->L[l.inputs[1]].kind != PSG_LAYER_LABEL)
          throw std::invalid_argument("net: softmax loss second input must be the label layer");
        if (src->H != 1 || src->W != 1 || src->cs != src->C)
          throw std::invalid_argument("net: softmax logits must be [classes]");
        // several weighted losses (auxiliary heads) share the labels: same class count;
        // probabilities and test() use the last loss layer
        if (net->classes && net->classes != src->C)
          throw std::invalid_argument("net: loss layers disagree on the class count");
        net->loss_idx = li;
        l.C = l.cs = src->C;
        l.H = l.W = 1;
        net->classes = l.C;
        break;
      case PSG_LAYER_CONCAT:  // Caffe Concat along channels
        l.C = 0;
        l.H = src->H;
        l.W = src->W;
        for (int in : l.inputs) {
          const LayerRt& x = net->L[in];
          if (x.H != l.H || x.W != l.W)
            throw std::invalid_argument("net: concat inputs differ in height/width");
          if (x.cs != x.C) throw std::invalid_argument("net: concat of a padded input");
          l.coff.push_back(l.C);
          l.C += x.C;
        }
        l.cs = l.C;
        break;
    }
    if (is_param_layer(l.kind)) {
      TensorRec& k = net->tensors.back();
      k.ref_off = ref_off;
      ref_off += k.ref_count;
      k.int_off = int_off;
      int_off = round_up(int_off + k.int_count, kAlign);
      l.kern_t = static_cast<int>(net->tensors.size()) - 1;
      TensorRec b;
      b.layer = li;
      b.slot = 1;
      b.rank = 1;
      b.shape[0] = l.C;
      b.ref_count = b.int_count = static_cast<size_t>(l.C);
      b.ref_off = ref_off;
      ref_off += b.ref_count;
      b.int_off = int_off;
      int_off = round_up(int_off + b.int_count, kAlign);
      b.lr_mult = static_cast<float>(l.d.lr_mult_b);
      b.decay_mult = static_cast<float>(l.d.decay_mult_b);
      net->tensors.push_back(b);
      l.bias_t = static_cast<int>(net->tensors.size()) - 1;
    }
  }
  if (net->classes < 1) throw std::invalid_argument("net: need at least one class");
  plan_fusion(net);
  net->P_ref = ref_off;
  net->P_int = int_off;
  // divisible into 4-aligned slices for up to 8 ranks (ordered reduce-scatter)
  net->P_alloc = round_up(std::max<size_t>(int_off, 1), 4 * 840);

  // model.hpp:200-283 initialisation, bit-exact fp64 then one rounding to fp32.
  std::vector<float> host(net->P_alloc, 0.f);
  for (int li = 0; li < n; ++li) {
    LayerRt& l = net->L[li];
    if (!is_param_layer(l.kind)) continue;
    const TensorRec& k = net->tensors[l.kern_t];
    Rng r(derive_seed2(seed, kStreamWeights, static_cast<uint64_t>(li)));
    double s;
    if (l.kind == PSG_LAYER_CONV) {
      const double khw = static_cast<double>(l.d.kernel_h * l.d.kernel_w);
      s = std::sqrt(6.0 / (static_cast<double>(k.Cg) * khw +
                           static_cast<double>(l.C / l.d.group) * khw));
    } else {
      s = std::sqrt(6.0 / (static_cast<double>(k.shape[1]) + static_cast<double>(l.C)));
    }
    for (size_t i = 0; i < k.ref_count; ++i)
      host[k.int_off + k.to_int(i)] = static_cast<float>(r.uniform(-s, s));
  }
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaStreamCreateWithFlags(&net->stream, cudaStreamNonBlocking));
  net->w = dalloc<float>(net->P_alloc);
  net->g = dalloc<float>(net->P_alloc);
  net->v = dalloc<float>(net->P_alloc);
  copy_sync(net, net->w, host.data(), net->P_alloc * sizeof(float), cudaMemcpyHostToDevice);
  PSG_CUDA(cudaMemset(net->g, 0, net->P_alloc * sizeof(float)));
  PSG_CUDA(cudaMemset(net->v, 0, net->P_alloc * sizeof(float)));
  PSG_CUDA(cudaMalloc(&net->dsc, sizeof(DeviceScalars)));
  PSG_CUDA(cudaMemset(net->dsc, 0, sizeof(DeviceScalars)));
  PSG_CUDA(cudaMallocHost(&net->hsc, sizeof(DeviceScalars)));
  PSG_CUDA(cudaEventCreateWithFlags(&net->idx_ev, cudaEventDisableTiming));
  PSG_CUDA(cudaEventCreate(&net->t0));
  PSG_CUDA(cudaEventCreate(&net->t1));
  assign_lanes(net);
  build_chunks(net);
}

void net_free(psg_net* net) {
  DeviceGuard dg(net->ctx->device);
  if (net->stream) cudaStreamSynchronize(net->stream);
  invalidate_graph(net);
  free_batch_buffers(net);
  dfree(net->w);
  dfree(net->g);
  dfree(net->v);
  dfree(net->d_chunks);
  dfree(net->dsc);
  dfree(net->d_idx);
  dfree(net->d_vidx);
  if (net->hsc) cudaFreeHost(net->hsc);
  if (net->h_idx) cudaFreeHost(net->h_idx);
  if (net->h_stage) cudaFreeHost(net->h_stage);
  if (net->h_lab) cudaFreeHost(net->h_lab);
  dfree(net->d_stage);
  for (int k = 0; k < 2; ++k) {
    dfree(net->d_stage2[k]);
    dfree(net->d_lab2[k]);
    if (net->copied[k]) cudaEventDestroy(net->copied[k]);
    if (net->consumed[k]) cudaEventDestroy(net->consumed[k]);
  }
  if (net->copy_stream) cudaStreamDestroy(net->copy_stream);
  for (cudaStream_t ls : net->lane_stream)
    if (ls) cudaStreamDestroy(ls);
  if (net->lane_fork) cudaEventDestroy(net->lane_fork);
  for (cudaEvent_t e : net->lane_join)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : net->ev_fwd) cudaEventDestroy(e);
  for (cudaEvent_t e : net->ev_bwd) cudaEventDestroy(e);
  for (cudaEvent_t e : net->ev_sum) cudaEventDestroy(e);
  if (net->side_stream) cudaStreamDestroy(net->side_stream);
  if (net->side_join) cudaEventDestroy(net->side_join);
  for (cudaEvent_t e : net->bucket_ev) cudaEventDestroy(e);
  if (net->h_losses) cudaFreeHost(net->h_losses);
  if (net->h_reg) cudaHostUnregister(const_cast<void*>(net->h_reg));
  for (int k = 0; k < 2; ++k) {
    if (net->h_ring[k]) cudaFreeHost(net->h_ring[k]);
    if (net->h_ring_lab[k]) cudaFreeHost(net->h_ring_lab[k]);
    if (net->h_ring_ev[k]) cudaEventDestroy(net->h_ring_ev[k]);
  }
  for (cudaEvent_t e : net->slots)
    if (e) cudaEventDestroy(e);
  if (net->idx_ev) cudaEventDestroy(net->idx_ev);
  if (net->t0) cudaEventDestroy(net->t0);
  if (net->t1) cudaEventDestroy(net->t1);
  if (net->stream) cudaStreamDestroy(net->stream);
}

void net_check_flag(psg_net* net) {
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  int flag = 0;
  copy_sync(net, &flag, &net->dsc->flag, sizeof(int), cudaMemcpyDeviceToHost);
  if (flag) {
    const int zero = 0;
    copy_sync(net, &net->dsc->flag, &zero, sizeof(int), cudaMemcpyHostToDevice);
    throw std::runtime_error("train: produced a non-finite value");
  }
}

void net_set_sgd(psg_net* net, double lr, double mu, double wd) {
  if (!(lr > 0.0)) throw std::invalid_argument("sgd: learning rate must be > 0");
  if (mu < 0.0 || mu >= 1.0) throw std::invalid_argument("sgd: momentum must be in [0,1)");
  if (wd < 0.0) throw std::invalid_argument("sgd: weight decay must be >= 0");
  if (mu != net->mu) invalidate_graph(net);
  net->lr = lr;
  net->mu = mu;
  net->wd = wd;
  build_chunks(net);
}

void net_get_weights(psg_net* net, double* flat, size_t n, bool velocity) {
  if (n != net->P_ref) throw std::invalid_argument("get_weights: size mismatch");
  DeviceGuard dg(net->ctx->device);
  std::vector<float> host(net->P_int);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  copy_sync(net, host.data(), velocity ? net->v : net->w, net->P_int * sizeof(float),
                      cudaMemcpyDeviceToHost);
  for (const TensorRec& t : net->tensors)
    for (size_t i = 0; i < t.ref_count; ++i)
      flat[t.ref_off + i] = static_cast<double>(host[t.int_off + t.to_int(i)]);
}

void net_set_weights(psg_net* net, const double* flat, size_t n) {
  if (n != net->P_ref)
    throw std::invalid_argument("set_weights: expected " + std::to_string(net->P_ref) +
                                " values, got " + std::to_string(n));
  std::vector<float> host(net->P_int, 0.f);
  for (const TensorRec& t : net->tensors)
    for (size_t i = 0; i < t.ref_count; ++i)
      host[t.int_off + t.to_int(i)] = static_cast<float>(flat[t.ref_off + i]);
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  copy_sync(net, net->w, host.data(), net->P_int * sizeof(float), cudaMemcpyHostToDevice);
}

void net_forward_host(psg_net* net, const double* images, const int32_t* labels, size_t n,
                      double* loss, double* probs) {
  DeviceGuard dg(net->ctx->device);
  upload_batch(net, images, labels, n);
  run_forward(net, n, /*train=*/false, /*seed_grad=*/false);
  net->last_n = n;
  const double l = read_loss(net);
  if (loss) *loss = l;
  if (probs) {
    std::vector<float> p(n * net->classes);
    copy_sync(net, p.data(), net->L[net->loss_idx].out, p.size() * sizeof(float),
                        cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < p.size(); ++i) probs[i] = p[i];
  }
}

void net_backward_host(psg_net* net, const double* images, const int32_t* labels, size_t n,
                       double* loss, double* grads) {
  DeviceGuard dg(net->ctx->device);
  upload_batch(net, images, labels, n);
  run_forward(net, n, /*train=*/true, /*seed_grad=*/true);
  run_backward(net, n);
  net->last_n = n;
  const double l = read_loss(net);
  if (loss) *loss = l;
  if (grads) {
    std::vector<float> host(net->P_int);
    copy_sync(net, host.data(), net->g, net->P_int * sizeof(float), cudaMemcpyDeviceToHost);
    for (const TensorRec& t : net->tensors)
      for (size_t i = 0; i < t.ref_count; ++i)
        grads[t.ref_off + i] = static_cast<double>(host[t.int_off + t.to_int(i)]);
    for (size_t i = 0; i < net->P_ref; ++i)
      if (!std::isfinite(grads[i])) throw std::runtime_error("backward: produced a non-finite value");
  }
}

void net_apply_update_host(psg_net* net, const double* grads, size_t n) {
  if (n != net->P_ref) throw std::invalid_argument("apply_update: gradient structure mismatch");
  std::vector<float> host(net->P_int, 0.f);
  for (const TensorRec& t : net->tensors)
    for (size_t i = 0; i < t.ref_count; ++i)
      host[t.int_off + t.to_int(i)] = static_cast<float>(grads[t.ref_off + i]);
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  copy_sync(net, net->g, host.data(), net->P_int * sizeof(float), cudaMemcpyHostToDevice);
  run_update(net, /*advance=*/false);
  net_check_flag(net);
}

void net_layer_readback(psg_net* net, int layer, bool grad, double* out, size_t n) {
  if (layer < 0 || layer >= static_cast<int>(net->L.size()))
    throw std::invalid_argument("layer index out of range");
  const LayerRt& l = net->L[layer];
  const size_t rows = net->last_n;
  const size_t want = rows * static_cast<size_t>(l.C) * l.H * l.W;
  if (n != want) throw std::invalid_argument("layer readback: size mismatch");
  const float* src = grad ? l.grad : l.out;
  if (!src || rows == 0) throw std::runtime_error("layer readback: no state for this layer");
  DeviceGuard dg(net->ctx->device);
  std::vector<float> host(rows * l.vol());
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  copy_sync(net, host.data(), src, host.size() * sizeof(float), cudaMemcpyDeviceToHost);
  for (size_t b = 0; b < rows; ++b)
    for (int c = 0; c < l.C; ++c)
      for (int h = 0; h < l.H; ++h)
        for (int w = 0; w < l.W; ++w)
          out[((b * l.C + c) * l.H + h) * l.W + w] = host[((b * l.H + h) * l.W + w) * l.cs + c];
}

void net_attach_shard(psg_net* net, psg_dataset* ds, const uint64_t* idx, size_t count,
                      size_t batch, uint64_t seed, int part, int parts) {
  if (batch < 1) throw std::invalid_argument("batch iterator: batch size must be >= 1");
  if (parts < 1 || part < 0 || part >= parts)
    throw std::invalid_argument("attach: part index out of range");
  if (batch % static_cast<size_t>(parts))
    throw std::invalid_argument("run_naive: worker count must divide the batch size");
  if (batch > count) throw std::invalid_argument("batch iterator: batch size exceeds shard size");
  const LayerRt& d = net->L[net->data_idx];
  if (ds->c != d.C || ds->h != d.H || ds->w != d.W)
    throw std::invalid_argument("forward: batch extents do not match the data layer");
  if (ds->ctx->device != net->ctx->device)
    throw std::invalid_argument("attach: dataset lives on another device");
  for (size_t i = 0; i < count; ++i)
    if (idx[i] >= ds->n) throw std::invalid_argument("attach: shard index out of range");
  for (int32_t y : ds->host_labels)
    if (y < 0 || y >= net->classes) throw std::invalid_argument("forward: label out of range");
  net->train_ds = ds;
  net->shard.assign(idx, idx + count);
  net->it_batch = batch;
  net->it_seed = seed;
  net->it_epoch = 0;
  net->it_part = part;
  net->it_parts = parts;
  net->order.resize(count);
  epoch_order(net->shard.data(), count, seed, 0, net->order.data());  // ctor -> start_epoch
  net->it_cursor = 0;
}

namespace {

// ShardBatchIterator::next() x steps (data.hpp:323-331): this net's rows of each batch,
// uploaded in one copy; the device cursor restarts at row block 0.  Returns rows per step.
size_t upload_stream_indices(psg_net* net, long steps) {
  const size_t B = net->it_batch, b = B / static_cast<size_t>(net->it_parts);
  const size_t off = static_cast<size_t>(net->it_part) * b;
  const size_t need = static_cast<size_t>(steps) * b;
  if (need > net->idx_cap) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    dfree(net->d_idx);
    if (net->h_idx) cudaFreeHost(net->h_idx);
    net->idx_cap = std::max(need, static_cast<size_t>(4096));
    net->d_idx = dalloc<uint32_t>(net->idx_cap);
    PSG_CUDA(cudaMallocHost(&net->h_idx, net->idx_cap * sizeof(uint32_t)));
    invalidate_graph(net);
  }
  PSG_CUDA(cudaEventSynchronize(net->idx_ev));
  for (long s = 0; s < steps; ++s) {
    if ((net->it_cursor + 1) * B > net->order.size()) {
      ++net->it_epoch;
      epoch_order(net->shard.data(), net->shard.size(), net->it_seed, net->it_epoch,
                  net->order.data());
      net->it_cursor = 0;
    }
    for (size_t i = 0; i < b; ++i)
      net->h_idx[s * b + i] = static_cast<uint32_t>(net->order[net->it_cursor * B + off + i]);
    ++net->it_cursor;
  }
  PSG_CUDA(cudaMemcpyAsync(net->d_idx, net->h_idx, need * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           net->stream));
  PSG_CUDA(cudaEventRecord(net->idx_ev, net->stream));
  PSG_CUDA(cudaMemsetAsync(&net->dsc->cursor, 0, sizeof(int), net->stream));
  return b;
}

bool eager_mode() {
  // PSG_EAGER=1: launch the step's kernels directly instead of replaying the CUDA
  // graph (ncu cannot replay graph kernel nodes that take a __grid_constant__
  // CUtensorMap).  Same kernels, same order.
  static const bool eager = [] {
    const char* e = std::getenv("PSG_EAGER");
    return e && e[0] == '1';
  }();
  return eager;
}

}  // namespace

void net_train(psg_net* net, long steps) {
  if (steps < 0) throw std::invalid_argument("train: negative step count");
  if (steps == 0) return;
  if (!net->train_ds) throw std::runtime_error("train: no training data attached");
  DeviceGuard dg(net->ctx->device);
  const size_t b = net->it_batch / static_cast<size_t>(net->it_parts);
  ensure_capacity(net, b);
  upload_stream_indices(net, steps);
  const LayerRt& d = net->L[net->data_idx];
  psg_dataset* ds = net->train_ds;
  if (eager_mode()) {
    PSG_CUDA(cudaEventRecord(net->t0, net->stream));
    for (long s = 0; s < steps; ++s) {
      stage_gathered_batch(net, ds->images, ds->labels, net->d_idx, &net->dsc->cursor, b);
      run_forward(net, b, true, true);
      run_backward(net, b);
      run_update(net, true);
    }
    PSG_CUDA(cudaEventRecord(net->t1, net->stream));
    net->timed = true;
    net->last_n = b;
    return;
  }
  if (!net->graph || net->graph_batch != b) {
    invalidate_graph(net);
    cudaGraph_t graph;
    PSG_CUDA(cudaStreamBeginCapture(net->stream, cudaStreamCaptureModeThreadLocal));
    int launches = 0;
    try {
      stage_gathered_batch(net, ds->images, ds->labels, net->d_idx, &net->dsc->cursor, b);
      ++launches;
      launches += run_forward(net, b, true, true);
      launches += run_backward(net, b);
      launches += run_update(net, true);
    } catch (...) {
      cudaStreamEndCapture(net->stream, &graph);
      throw;
    }
    PSG_CUDA(cudaStreamEndCapture(net->stream, &graph));
    PSG_CUDA(cudaGraphInstantiate(&net->graph, graph, 0));
    cudaGraphDestroy(graph);
    net->graph_batch = b;
    net->launches_per_step = launches;
  }
  PSG_CUDA(cudaEventRecord(net->t0, net->stream));
  for (long s = 0; s < steps; ++s) PSG_CUDA(cudaGraphLaunch(net->graph, net->stream));
  PSG_CUDA(cudaEventRecord(net->t1, net->stream));
  net->timed = true;
  net->last_n = b;
}

// One SparkNet round of this worker with the fast K-way average overlapped across layers
// (SURVEY §8(e)): steps - 1 ordinary graph replays, then the round's last step as its own
// graph in which every parameter layer's SGD update is issued right after its wgrad /
// dgrad and its weights are averaged by an ncclAllReduce(avg) on a side stream while the
// backward of the layers below runs; the side stream joins before the step ends.  Same
// arithmetic as train(steps) + psg_comm_average(fast) (for K = 2 bitwise: the average of
// two values does not depend on the allreduce's chunking).
void net_train_round(psg_net* net, long steps, psg_comm* comm) {
  if (steps < 1) throw std::invalid_argument("train_round: tau must be >= 1");
  if (!net->train_ds) throw std::runtime_error("train: no training data attached");
  if (!comm || comm_device(comm) != net->ctx->device)
    throw std::invalid_argument("train_round: communicator on another device");
  DeviceGuard dg(net->ctx->device);
  if (steps > 1)
    net_train(net, steps - 1);  // records t0 at the round's start
  else
    PSG_CUDA(cudaEventRecord(net->t0, net->stream));
  const size_t b = net->it_batch / static_cast<size_t>(net->it_parts);
  ensure_capacity(net, b);
  upload_stream_indices(net, 1);
  psg_dataset* ds = net->train_ds;
  if (!net->side_stream) {
    PSG_CUDA(cudaStreamCreateWithFlags(&net->side_stream, cudaStreamNonBlocking));
    PSG_CUDA(cudaEventCreateWithFlags(&net->side_join, cudaEventDisableTiming));
  }
  int nbuckets = 0, last = -1;
  for (size_t li = 0; li < net->L.size(); ++li)
    if (net->L[li].nchunk) {
      ++nbuckets;
      if (last < 0) last = static_cast<int>(li);  // first param layer = last in backward
    }
  while (static_cast<int>(net->bucket_ev.size()) < nbuckets) {
    cudaEvent_t e;
    PSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    net->bucket_ev.push_back(e);
  }
  auto body = [&] {
    RoundOverlap ov;
    ov.comm = comm;
    ov.side = net->side_stream;
    ov.ready = net->bucket_ev;
    ov.last_param_layer = last;
    int launches = stage_gathered_batch(net, ds->images, ds->labels, net->d_idx,
                                        &net->dsc->cursor, b);
    launches += run_forward(net, b, true, true);
    // fork: the side stream joins the capture / the stream order here
    PSG_CUDA(cudaEventRecord(net->side_join, net->stream));
    PSG_CUDA(cudaStreamWaitEvent(net->side_stream, net->side_join, 0));
    launches += run_backward(net, b, nullptr, &ov);
    PSG_CUDA(cudaEventRecord(net->side_join, net->side_stream));
    PSG_CUDA(cudaStreamWaitEvent(net->stream, net->side_join, 0));
    return launches;
  };
  if (eager_mode()) {
    body();
  } else {
    if (!net->round_graph || net->round_graph_batch != b || net->round_comm != comm) {
      if (net->round_graph) cudaGraphExecDestroy(net->round_graph);
      net->round_graph = nullptr;
      cudaGraph_t graph;
      PSG_CUDA(cudaStreamBeginCapture(net->stream, cudaStreamCaptureModeThreadLocal));
      try {
        body();
      } catch (...) {
        cudaStreamEndCapture(net->stream, &graph);
        throw;
      }
      PSG_CUDA(cudaStreamEndCapture(net->stream, &graph));
      PSG_CUDA(cudaGraphInstantiate(&net->round_graph, graph, 0));
      cudaGraphDestroy(graph);
      net->round_graph_batch = b;
      net->round_comm = comm;
    }
    PSG_CUDA(cudaGraphLaunch(net->round_graph, net->stream));
  }
  PSG_CUDA(cudaEventRecord(net->t1, net->stream));
  net->timed = true;
  net->last_n = b;
}

// run_naive (schemes.hpp:233-250) on the device: one part of the next batch ->
// forward + backward, gradient left in the flat buffer g (not applied).  The SGD
// update runs separately after the K part gradients were averaged.
void net_grad_step(psg_net* net) {
  if (!net->train_ds) throw std::runtime_error("train: no training data attached");
  DeviceGuard dg(net->ctx->device);
  const size_t b = net->it_batch / static_cast<size_t>(net->it_parts);
  ensure_capacity(net, b);
  upload_stream_indices(net, 1);
  const LayerRt& d = net->L[net->data_idx];
  psg_dataset* ds = net->train_ds;
  auto body = [&] {
    stage_gathered_batch(net, ds->images, ds->labels, net->d_idx, &net->dsc->cursor, b);
    run_forward(net, b, true, true);
    run_backward(net, b);
  };
  if (eager_mode()) {
    body();
  } else {
    if (!net->grad_graph || net->grad_graph_batch != b) {
      if (net->grad_graph) cudaGraphExecDestroy(net->grad_graph);
      net->grad_graph = nullptr;
      cudaGraph_t graph;
      PSG_CUDA(cudaStreamBeginCapture(net->stream, cudaStreamCaptureModeThreadLocal));
      try {
        body();
      } catch (...) {
        cudaStreamEndCapture(net->stream, &graph);
        throw;
      }
      PSG_CUDA(cudaStreamEndCapture(net->stream, &graph));
      PSG_CUDA(cudaGraphInstantiate(&net->grad_graph, graph, 0));
      cudaGraphDestroy(graph);
      net->grad_graph_batch = b;
    }
    PSG_CUDA(cudaGraphLaunch(net->grad_graph, net->stream));
  }
  net->last_n = b;
}

// apply_update with the resident (averaged) gradient; advances the step counter.
void net_apply_grads(psg_net* net) {
  DeviceGuard dg(net->ctx->device);
  run_update(net, true);
}

void net_attach_validation(psg_net* net, psg_dataset* ds, size_t batch) {
  if (batch < 1 || batch > ds->n) throw std::invalid_argument("eval iterator: bad batch size");
  const LayerRt& d = net->L[net->data_idx];
  if (ds->c != d.C || ds->h != d.H || ds->w != d.W)
    throw std::invalid_argument("forward: batch extents do not match the data layer");
  if (ds->ctx->device != net->ctx->device)
    throw std::invalid_argument("attach: dataset lives on another device");
  for (int32_t y : ds->host_labels)
    if (y < 0 || y >= net->classes) throw std::invalid_argument("forward: label out of range");
  net->val_ds = ds;
  net->val_batch = batch;
  net->val_cursor = 0;
}

// Net::test (model.hpp:122-136) over a SequentialBatchIterator (data.hpp:355-382),
// split for sharded evaluation: this call queues batches first, first + stride, ... < steps
// of the iterator's next `steps` batches (forward-only, fused argmax/count) and advances
// the iterator by `steps`, so K nets with first = k, stride = K cover one test(steps)
// between them.  test_end collects (correct, total).
void net_test_begin(psg_net* net, long steps, long first, long stride) {
  if (steps < 1) throw std::invalid_argument("test: step count must be >= 1");
  if (first < 0 || stride < 1) throw std::invalid_argument("test: bad shard");
  if (!net->val_ds) throw std::runtime_error("test: no validation data attached");
  if (net->val_pending) throw std::logic_error("test: previous evaluation not collected");
  DeviceGuard dg(net->ctx->device);
  const size_t b = net->val_batch;
  const size_t nb = net->val_ds->n / b;  // batches before the iterator wraps
  std::vector<uint32_t> idx;
  long mine = 0;
  for (long s = first; s < steps; s += stride, ++mine) {
    const size_t cursor = (net->val_cursor + static_cast<size_t>(s)) % nb;
    for (size_t i = 0; i < b; ++i) idx.push_back(static_cast<uint32_t>(cursor * b + i));
  }
  net->val_cursor = (net->val_cursor + static_cast<size_t>(steps)) % nb;
  net->val_total = static_cast<unsigned long long>(mine) * b;
  net->val_pending = true;
  PSG_CUDA(cudaMemsetAsync(&net->dsc->correct, 0, sizeof(unsigned long long), net->stream));
  if (mine == 0) return;
  ensure_capacity(net, b);
  if (idx.size() > net->vidx_cap) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    dfree(net->d_vidx);
    net->vidx_cap = idx.size();
    net->d_vidx = dalloc<uint32_t>(net->vidx_cap);
  }
  PSG_CUDA(cudaMemcpyAsync(net->d_vidx, idx.data(), idx.size() * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, net->stream));
  const LayerRt& d = net->L[net->data_idx];
  for (long s = 0; s < mine; ++s) {
    stage_gathered_batch(net, net->val_ds->images, net->val_ds->labels, net->d_vidx + s * b,
                         nullptr, b);
    run_forward(net, b, /*train=*/false, /*seed_grad=*/false);
    argmax_count(net->L[net->loss_idx].out, net->labels, static_cast<int>(b), net->classes,
                 &net->dsc->correct, net->stream);
  }
  net->last_n = b;  // (pageable idx: the async copy stages it before returning)
}

void net_test_end(psg_net* net, unsigned long long* correct, unsigned long long* total) {
  if (!net->val_pending) throw std::logic_error("test: no evaluation in flight");
  DeviceGuard dg(net->ctx->device);
  PSG_CUDA(cudaMemcpyAsync(&net->hsc->correct, &net->dsc->correct, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, net->stream));
  PSG_CUDA(cudaStreamSynchronize(net->stream));
  net->val_pending = false;
  *correct = net->hsc->correct;
  *total = net->val_total;
}

double net_test(psg_net* net, long steps) {
  net_test_begin(net, steps, 0, 1);
  unsigned long long correct = 0, total = 0;
  net_test_end(net, &correct, &total);
  return static_cast<double>(correct) / static_cast<double>(total);
}

}  // namespace psg
