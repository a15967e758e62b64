// Launch sequences of one training step (eager, under stream capture, or with a
// per-op CUDA-event timer for bench.py's roofline numbers).
#include <cstring>

#include "runtime.h"

namespace psg {

// Under stream capture the record must become an event-record node of the graph
// (cudaEventRecordExternal); outside capture that flag is rejected.
cudaError_t OpTimer::record(cudaEvent_t e) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  PSG_CUDA(cudaStreamIsCapturing(stream, &st));
  return st == cudaStreamCaptureStatusActive
             ? cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal)
             : cudaEventRecord(e, stream);
}

void OpTimer::begin(const char* name, int layer, int phase, double flops, double bytes) {
  Rec r{};
  std::strncpy(r.info.name, name, sizeof(r.info.name) - 1);
  r.info.layer = layer;
  r.info.phase = phase;
  r.info.flops = flops;
  r.info.bytes = bytes;
  PSG_CUDA(cudaEventCreate(&r.a));
  PSG_CUDA(cudaEventCreate(&r.b));
  PSG_CUDA(record(r.a));
  recs.push_back(r);
}

void OpTimer::end(int launches) {
  recs.back().info.launches = launches;
  PSG_CUDA(record(recs.back().b));
}

OpTimer::~OpTimer() {
  for (Rec& r : recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
}

namespace {

ConvGeom geom_n(const LayerRt& l, size_t n) {
  ConvGeom g = l.cg;
  g.n = static_cast<int>(n);
  return g;
}

// Algorithmic FLOPs of one GEMM-shaped pass of a conv / linear layer (logical
// channels, not the padded internal ones).
double conv_flops(const psg_net* net, const LayerRt& l, size_t n) {
  const LayerRt& src = net->L[l.inputs[0]];
  double macs;
  if (l.kind == PSG_LAYER_CONV)
    macs = static_cast<double>(n) * l.H * l.W * l.C * l.d.kernel_h * l.d.kernel_w *
           (src.C / l.d.group);
  else
    macs = static_cast<double>(n) * l.C * src.C * src.H * src.W;
  return 2.0 * macs;
}

// PSG_CONCAT_SINGLE=0: one concat copy / split launch per input (A/B; read when recording)
bool concat_single() {
  const char* e = std::getenv("PSG_CONCAT_SINGLE");
  return !e || std::atoi(e) != 0;
}

double act_bytes(const LayerRt& l, size_t n) { return 4.0 * static_cast<double>(n) * l.vol(); }

// Branch lanes (psg_net::lane_of), off when profiling per op (the timer's events are on the
// main stream).
struct Lanes {
  psg_net* net;
  bool on;
  int lane(int li) const { return on ? net->lane_of[li] : 0; }
  cudaStream_t s(int li) const {
    const int k = lane(li);
    return k ? net->lane_stream[k] : net->stream;
  }
  const Workspace& ws(int li) const {
    const int k = lane(li);
    return k ? net->ws_lane[k] : net->ws;
  }
  void fork() const {  // every lane joins the main stream's order (and a capture)
    if (!on) return;
    PSG_CUDA(cudaEventRecord(net->lane_fork, net->stream));
    for (int k = 1; k < psg_net::kStreams; ++k)
      PSG_CUDA(cudaStreamWaitEvent(net->lane_stream[k], net->lane_fork, 0));
  }
  void join() const {
    if (!on) return;
    for (int k = 1; k < psg_net::kStreams; ++k) {
      PSG_CUDA(cudaEventRecord(net->lane_join[k], net->lane_stream[k]));
      PSG_CUDA(cudaStreamWaitEvent(net->stream, net->lane_join[k], 0));
    }
  }
  // layer li waits for the forward / backward event of layer `other` (< 0: none) when that
  // ran on another lane
  void after_fwd(int li, int other) const {
    if (on && other >= 0 && lane(other) != lane(li))
      PSG_CUDA(cudaStreamWaitEvent(s(li), net->ev_fwd[other], 0));
  }
  void after_bwd(int li, int other) const {
    if (on && other >= 0 && lane(other) != lane(li))
      PSG_CUDA(cudaStreamWaitEvent(s(li), net->ev_bwd[other], 0));
  }
  void record_fwd(int li) const {
    if (on) PSG_CUDA(cudaEventRecord(net->ev_fwd[li], s(li)));
  }
  void record_bwd(int li) const {
    if (on) PSG_CUDA(cudaEventRecord(net->ev_bwd[li], s(li)));
  }
};

struct Dst {
  float* p;
  bool acc;
};

struct Scope {
  OpTimer* t;
  Scope(OpTimer* t_, const char* name, int layer, int phase, double flops, double bytes) : t(t_) {
    if (t) t->begin(name, layer, phase, flops, bytes);
  }
  void done(int launches) {
    if (t) t->end(launches);
  }
};

}  // namespace

int stage_gathered_batch(psg_net* net, const float* images, const int32_t* labels,
                         const uint32_t* idx, const int* cursor, size_t n) {
  const LayerRt& d = net->L[net->data_idx];
  net->data_s2d = false;
  if (net->fuse && d.consumers.size() == 1) {
    const LayerRt& c = net->L[d.consumers[0]];
    if (c.kind == PSG_LAYER_CONV && c.col) {
      const ConvGeom g = geom_n(c, n);
      if (conv_s2d_input(g, net->mode)) {
        gather_s2d(g, images, labels, idx, cursor, d.C, c.col, net->labels, net->stream);
        net->data_s2d = true;
        return 1;
      }
    }
  }
  gather_batch(images, labels, idx, cursor, static_cast<int>(n), d.H * d.W, d.C, d.cs, d.out,
               net->labels, net->stream);
  return 1;
}

int stage_host_batch(psg_net* net, const float* src, size_t n) {
  const LayerRt& d = net->L[net->data_idx];
  net->data_s2d = false;
  if (net->fuse && d.consumers.size() == 1) {
    const LayerRt& c = net->L[d.consumers[0]];
    if (c.kind == PSG_LAYER_CONV && c.col) {
      const ConvGeom g = geom_n(c, n);
      if (conv_s2d_input(g, net->mode)) {
        stage_s2d_nchw(g, src, d.C, c.col, net->stream);
        net->data_s2d = true;
        return 1;
      }
    }
  }
  stage_batch_nchw(src, static_cast<int>(n), d.C, d.H, d.W, d.cs, d.out, net->stream);
  return 1;
}

int run_forward(psg_net* net, size_t n, bool train, bool seed_grad, OpTimer* timer) {
  const Lanes ln{net, net->lanes_on && !timer};
  ln.fork();
  int launches = 0;
  bool first_loss = true;  // the total loss sums every loss layer's weighted mean
  for (size_t li = 0; li < net->L.size(); ++li) {
    LayerRt& l = net->L[li];
    const int lid = static_cast<int>(li);
    const std::string nm = std::string(l.d.name) + ".fwd";
    cudaStream_t s = ln.s(lid);
    for (int p : l.inputs) ln.after_fwd(lid, p);
    switch (l.kind) {
      case PSG_LAYER_DATA:
      case PSG_LAYER_LABEL:
        break;
      case PSG_LAYER_CONV:
      case PSG_LAYER_LINEAR: {
        const LayerRt& src = net->L[l.inputs[0]];
        const TensorRec& k = net->tensors[l.kern_t];
        const TensorRec& b = net->tensors[l.bias_t];
        const ConvGeom g = geom_n(l, n);
        Scope sc(timer, nm.c_str(), lid, 1, conv_flops(net, l, n), 0.0);
        // fused ReLU: l.out aliases the ReLU's buffer and the epilogue applies max(0, .)
        const bool xs = net->data_s2d && src.kind == PSG_LAYER_DATA;  // x' already gathered
        conv_fprop(g, src.out, net->w + k.int_off, net->w + b.int_off, l.out, l.fwd_relu >= 0,
                   ln.ws(lid), l.col, net->mode, s, xs);
        const int c = conv_launches(g, 0, net->mode) - (xs ? 1 : 0);
        sc.done(c);
        launches += c;
        break;
      }
      case PSG_LAYER_POOL: {
        PoolGeom g = l.pg;
        g.n = static_cast<int>(n);
        const LayerRt& src = net->L[l.inputs[0]];
        if (l.pool_lrn >= 0) {  // LRN computed in the pool kernel from the LRN's input
          const LayerRt& x = net->L[src.inputs[0]];
          Scope sc(timer, nm.c_str(), lid, 1, 0.0, act_bytes(x, n) + act_bytes(l, n) * 1.25);
          LrnGeom lg = src.lg;
          lg.pixels = static_cast<int>(n) * src.H * src.W;
          lrn_maxpool_fwd(lg, g, x.out, l.out, l.route, s);
          sc.done(1);
          ++launches;
          break;
        }
        Scope sc(timer, nm.c_str(), lid, 1, 0.0,
                 act_bytes(src, n) + act_bytes(l, n) * (l.route ? 1.25 : 1.0));
        pool_fwd(g, src.out, l.out, l.route, s);
        sc.done(1);
        ++launches;
        break;
      }
      case PSG_LAYER_RELU: {
        if (l.fused_from >= 0) break;  // computed by the producer's epilogue
        Scope sc(timer, nm.c_str(), lid, 1, 0.0, 2 * act_bytes(l, n));
        relu_fwd(net->L[l.inputs[0]].out, l.out, n * l.vol(), s);
        sc.done(1);
        ++launches;
        break;
      }
      case PSG_LAYER_LRN: {
        if (l.lrn_pool >= 0) break;  // computed by the consuming pool's kernel
        LrnGeom g = l.lg;
        g.pixels = static_cast<int>(n) * l.H * l.W;
        Scope sc(timer, nm.c_str(), lid, 1, 0.0, 2 * act_bytes(l, n));
        lrn_fwd(g, net->L[l.inputs[0]].out, l.out, s);
        sc.done(1);
        ++launches;
        break;
      }
      case PSG_LAYER_DROPOUT: {
        DropGeom g = l.dg;
        g.n = static_cast<int>(n);
        Scope sc(timer, nm.c_str(), lid, 1, 0.0, 2 * act_bytes(l, n));
        dropout_fwd(g, net->L[l.inputs[0]].out, l.out, &net->dsc->step, train, s);
        sc.done(1);
        ++launches;
        break;
      }
      case PSG_LAYER_SOFTMAX_LOSS: {
        LayerRt& logits = net->L[l.inputs[0]];
        Scope sc(timer, nm.c_str(), lid, 2, 0.0, 3 * act_bytes(l, n));
        softmax_loss(logits.out, net->labels, static_cast<int>(n), net->classes, l.d.loss_weight,
                     l.out, seed_grad ? logits.grad : nullptr, net->row_loss, &net->dsc->loss,
                     &net->dsc->flag, !first_loss, s);
        first_loss = false;
        sc.done(2);
        launches += 2;
        break;
      }
      case PSG_LAYER_CONCAT: {
        const size_t pixels = n * static_cast<size_t>(l.H) * l.W;
        Scope sc(timer, nm.c_str(), lid, 1, 0.0, 2 * act_bytes(l, n));
        ConcatSeg seg[kConcatMax];
        const int k = static_cast<int>(l.inputs.size());
        for (int i = 0; i < k && i < kConcatMax; ++i) {
          const LayerRt& x = net->L[l.inputs[i]];
          seg[i] = {x.out, nullptr, nullptr, x.C, l.coff[i], false};
        }
        int c = 1;
        if (!concat_single() || !concat_copy_all(seg, k, l.out, l.C, pixels, s)) {
          for (int i = 0; i < k; ++i) {
            const LayerRt& x = net->L[l.inputs[i]];
            concat_copy(x.out, x.C, l.out, l.C, l.coff[i], pixels, s);
          }
          c = k;
        }
        sc.done(c);
        launches += c;
        break;
      }
    }
    if (ln.on)
      for (int c : l.consumers)
        if (ln.lane(c) != ln.lane(lid)) {
          ln.record_fwd(lid);
          break;
        }
  }
  ln.join();
  net->data_s2d = false;  // one-shot: set by stage_gathered_batch for this forward only
  return launches;
}

namespace {
// Fusion: the ReLU whose backward the layer `c` (its only consumer) can fold into its own
// input-gradient pass (a tensor-core dgrad epilogue or the max/ave pool backward), else -1.
// Input `ri` of a layer, when it is a ReLU whose backward that layer (its only consumer)
// may fold in, else -1.
int foldable_relu_input(const psg_net* net, int ri) {
  const LayerRt& r = net->L[ri];
  if (!net->fuse || r.kind != PSG_LAYER_RELU || r.bwd_by >= 0 || r.consumers.size() != 1 ||
      net->L[r.inputs[0]].kind == PSG_LAYER_DATA)
    return -1;
  return ri;
}

int foldable_relu(const psg_net* net, const LayerRt& c) {
  if (!net->fuse || c.inputs.size() != 1) return -1;
  const int ri = foldable_relu_input(net, c.inputs[0]);
  if (ri < 0) return -1;
  if (c.kind == PSG_LAYER_POOL || c.kind == PSG_LAYER_DROPOUT) return ri;
  if ((c.kind == PSG_LAYER_CONV || c.kind == PSG_LAYER_LINEAR) && net->mode == Mode::Tf32 &&
      conv_dgrad_masks(c.cg, net->mode))
    return ri;
  return -1;
}
}  // namespace

int run_backward(psg_net* net, size_t n, OpTimer* timer, RoundOverlap* ov) {
  const Lanes ln{net, net->lanes_on && !timer};
  ln.fork();
  int launches = 0;
  std::vector<char> written(net->L.size(), 0);
  std::vector<char> relu_folded(net->L.size(), 0);  // backward done by the consumer
  // lanes: the layer whose backward last wrote / accumulated into each gradient buffer; a
  // reader or the next accumulator on another lane waits for its event (same order as one
  // stream, so the sums are bitwise those of one stream)
  std::vector<int> last_writer(net->L.size(), -1);
  std::vector<std::vector<int>> pend(net->L.size());  // scratch writers per gradient, in order
  for (const LayerRt& l : net->L)  // every loss seed writes its logits grad
    if (l.kind == PSG_LAYER_SOFTMAX_LOSS) written[l.inputs[0]] = 1;
  for (int li = static_cast<int>(net->L.size()) - 1; li >= 0; --li) {
    LayerRt& l = net->L[li];
    if (l.kind == PSG_LAYER_DATA || l.kind == PSG_LAYER_LABEL || l.kind == PSG_LAYER_SOFTMAX_LOSS)
      continue;
    cudaStream_t s = ln.s(li);
    // gradient scratch of this layer (lanes): add the later writers' buffers, in writer
    // order, into the first writer's gradient before anything reads it
    bool summed = false;
    if (!pend[li].empty()) {
      ln.after_bwd(li, last_writer[li]);
      for (int w : pend[li]) ln.after_bwd(li, w);
      launches += grad_accumulate(l.grad, l.acc_scratch.data(), static_cast<int>(pend[li].size()),
                                  n * l.vol(), s);
      PSG_CUDA(cudaEventRecord(net->ev_sum[li], s));
      pend[li].clear();
      last_writer[li] = li;  // later readers wait for this layer's own event
      summed = true;
    } else {
      ln.after_bwd(li, last_writer[li]);
    }
    // destination of li's write into L[buf].grad: the gradient itself (waiting for its last
    // writer when that ran on another lane), or — a fan-out layer's 2nd, 3rd, ... writer under
    // branch lanes — a scratch buffer written without waiting (summed in order above)
    auto dest = [&](int buf) -> Dst {
      LayerRt& X = net->L[buf];
      if (ln.on && written[buf] && !X.acc_scratch.empty()) {
        const size_t j = pend[buf].size();
        if (j >= X.acc_scratch.size()) throw std::logic_error("backward: gradient scratch exhausted");
        pend[buf].push_back(li);
        return {X.acc_scratch[j], false};
      }
      ln.after_bwd(li, last_writer[buf]);
      last_writer[buf] = li;
      const bool a = written[buf] != 0;
      written[buf] = 1;
      return {X.grad, a};
    };
    if (l.kind == PSG_LAYER_CONCAT) {  // dx_i (+)= dy[:, off_i : off_i + C_i]
      const size_t pixels = n * static_cast<size_t>(l.H) * l.W;
      Scope sc(timer, (std::string(l.d.name) + ".bwd").c_str(), li, 5, 0.0, 2 * act_bytes(l, n));
      // one launch for every branch (concat_split_all), else one per branch
      const int k = static_cast<int>(l.inputs.size());
      std::vector<ConcatSeg> seg(k);
      int c = 0;
      for (int i = 0; i < k; ++i) {
        const int in = l.inputs[i];
        LayerRt& x = net->L[in];
        seg[i] = {nullptr, nullptr, nullptr, x.C, l.coff[i], false};
        if (x.kind == PSG_LAYER_DATA) continue;
        const int ri = foldable_relu_input(net, in);
        if (ri >= 0) {  // the branch's ReLU backward folded into the split (mask by its output)
          const Dst d = dest(net->L[ri].inputs[0]);
          seg[i].dst = d.p;
          seg[i].acc = d.acc;
          seg[i].mask = x.out;
          relu_folded[ri] = 1;
          written[in] = 1;
        } else {
          const Dst d = dest(in);
          seg[i].dst = d.p;
          seg[i].acc = d.acc;
        }
        ++c;
      }
      if (c > 0 && concat_single() &&
          concat_split_all(l.grad, l.C, seg.data(), k, pixels, s)) {
        c = 1;
      } else {
        for (int i = 0; i < k; ++i)
          if (seg[i].dst)
            concat_split(l.grad, l.C, seg[i].off, seg[i].dst, seg[i].ci, pixels, seg[i].acc, s,
                         seg[i].mask);
      }
      sc.done(c);
      launches += c;
      ln.record_bwd(li);
      continue;
    }
    const int pi = l.inputs[0];
    LayerRt& src = net->L[pi];
    const bool need_dx = src.kind != PSG_LAYER_DATA;

    const std::string nm = std::string(l.d.name);
    switch (l.kind) {
      case PSG_LAYER_CONV:
      case PSG_LAYER_LINEAR: {
        const TensorRec& k = net->tensors[l.kern_t];
        const TensorRec& b = net->tensors[l.bias_t];
        const ConvGeom g = geom_n(l, n);
        {
          Scope sc(timer, (nm + ".wgrad").c_str(), li, 3, conv_flops(net, l, n), 0.0);
          // wgrad lane: a lane-0 layer's weight gradient on its own stream, overlapping its
          // dgrad and the layers below; it reads l.grad (complete at its last writer's event)
          // and the forward activations, writes only its own gradients and workspace (the
          // overlapped-average path keeps it on the layer's lane: the bucket update follows)
          const bool wl = ln.on && net->wgrad_lane && !ov && ln.lane(li) == 0;
          cudaStream_t sw = s;
          if (wl) {
            sw = net->lane_stream[psg_net::kWgLane];
            if (summed)
              PSG_CUDA(cudaStreamWaitEvent(sw, net->ev_sum[li], 0));
            else if (last_writer[li] >= 0)
              PSG_CUDA(cudaStreamWaitEvent(sw, net->ev_bwd[last_writer[li]], 0));
          }
          conv_wgrad(g, src.out, l.grad, net->g + k.int_off, net->g + b.int_off,
                     wl ? net->ws_lane[psg_net::kWgLane] : ln.ws(li), l.col, net->mode, sw);
          const int c = conv_launches(g, 2, net->mode);
          sc.done(c);
          launches += c;
        }
        if (need_dx) {
          Scope sc(timer, (nm + ".dgrad").c_str(), li, 4, conv_flops(net, l, n), 0.0);
          const int ri = foldable_relu(net, l);
          if (ri >= 0) {  // write the ReLU's input gradient, masked by the ReLU's output
            const int pi2 = net->L[ri].inputs[0];
            const Dst d = dest(pi2);
            conv_dgrad(g, l.grad, net->w + k.int_off, d.p, d.acc, ln.ws(li), net->mode, s,
                       net->L[ri].out, l.col);
            relu_folded[ri] = 1;
          } else {
            const Dst d = dest(pi);
            conv_dgrad(g, l.grad, net->w + k.int_off, d.p, d.acc, ln.ws(li), net->mode, s,
                       nullptr, l.col);
          }
          const int c = conv_launches(g, 1, net->mode);
          sc.done(c);
          launches += c;
        }
        if (ov && l.nchunk) {  // bucket li: update, then its average on the side stream
          const bool last = static_cast<int>(li) == ov->last_param_layer;
          sgd_update(net->d_chunks + l.chunk0, l.nchunk, net->w, net->v, net->g,
                     static_cast<float>(net->mu), &net->dsc->flag,
                     last ? &net->dsc->cursor : nullptr, last ? &net->dsc->step : nullptr, s);
          cudaEvent_t ev = ov->ready[ov->buckets++];
          PSG_CUDA(cudaEventRecord(ev, s));
          PSG_CUDA(cudaStreamWaitEvent(ov->side, ev, 0));
          const size_t lo = k.int_off, hi = b.int_off + b.int_count;
          comm_allreduce_avg(ov->comm, net->w + lo, hi - lo, ov->side);
          launches += 1;
        }
        break;
      }
      case PSG_LAYER_POOL:
        if (l.pool_lrn >= 0) break;  // gathered inside the fused LRN backward
        if (need_dx) {
          PoolGeom g = l.pg;
          g.n = static_cast<int>(n);
          Scope sc(timer, (nm + ".bwd").c_str(), li, 5, 0.0,
                   act_bytes(src, n) + act_bytes(l, n) * (l.route ? 1.25 : 1.0));
          const int ri = foldable_relu(net, l);
          if (ri >= 0) {  // ReLU backward folded in: mask by the ReLU's output
            const int pi2 = net->L[ri].inputs[0];
            const Dst d = dest(pi2);
            pool_bwd(g, l.grad, l.route, d.p, d.acc, s, net->L[ri].out);
            relu_folded[ri] = 1;
          } else {
            const Dst d = dest(pi);
            pool_bwd(g, l.grad, l.route, d.p, d.acc, s);
          }
          sc.done(1);
          ++launches;
        }
        break;
      case PSG_LAYER_RELU:
        if (l.bwd_by >= 0 || relu_folded[li]) break;  // done by the consumer's backward
        if (need_dx) {
          Scope sc(timer, (nm + ".bwd").c_str(), li, 5, 0.0, 3 * act_bytes(l, n));
          const Dst d = dest(pi);
          relu_bwd(src.out, l.grad, d.p, n * l.vol(), d.acc, s);
          sc.done(1);
          ++launches;
        }
        break;
      case PSG_LAYER_LRN:
        if (need_dx) {
          LrnGeom g = l.lg;
          g.pixels = static_cast<int>(n) * l.H * l.W;
          Scope sc(timer, (nm + ".bwd").c_str(), li, 5, 0.0, 3 * act_bytes(l, n));
          // the ReLU below folded in: mask by x > 0, write its input grad
          const Dst d = dest(l.bwd_relu >= 0 ? net->L[l.bwd_relu].inputs[0] : pi);
          float* dx = d.p;
          const bool dacc = d.acc;
          if (l.lrn_pool >= 0) {  // the max pool's backward gathered in the same kernel
            const LayerRt& p = net->L[l.lrn_pool];
            ln.after_bwd(li, last_writer[l.lrn_pool]);
            PoolGeom pg = p.pg;
            pg.n = static_cast<int>(n);
            lrn_maxpool_bwd(g, pg, src.out, p.grad, p.route, dx, dacc, l.bwd_relu >= 0, s);
          } else {
            lrn_bwd(g, src.out, l.grad, dx, dacc, s, l.bwd_relu >= 0);
          }
          sc.done(1);
          ++launches;
        }
        break;
      case PSG_LAYER_DROPOUT:
        if (need_dx) {
          DropGeom g = l.dg;
          g.n = static_cast<int>(n);
          Scope sc(timer, (nm + ".bwd").c_str(), li, 5, 0.0, 2 * act_bytes(l, n));
          const int ri = foldable_relu(net, l);
          if (ri >= 0) {  // ReLU backward folded in: mask by the ReLU's output
            const int pi2 = net->L[ri].inputs[0];
            const Dst d = dest(pi2);
            dropout_bwd(g, l.grad, d.p, &net->dsc->step, d.acc, s, net->L[ri].out);
            relu_folded[ri] = 1;
          } else {
            const Dst d = dest(pi);
            dropout_bwd(g, l.grad, d.p, &net->dsc->step, d.acc, s);
          }
          sc.done(1);
          ++launches;
        }
        break;
      default:
        break;
    }
    ln.record_bwd(li);
  }
  ln.join();
  return launches;
}

int run_update(psg_net* net, bool advance, OpTimer* timer) {
  if (net->nchunks == 0) return 0;
  const double bytes = 4.0 * static_cast<double>(net->P_int) * (net->mu > 0.0 ? 5.0 : 3.0);
  Scope sc(timer, "sgd_update", -1, 6, 0.0, bytes);
  sgd_update(net->d_chunks, net->nchunks, net->w, net->v, net->g, static_cast<float>(net->mu),
             &net->dsc->flag, advance ? &net->dsc->cursor : nullptr,
             advance ? &net->dsc->step : nullptr, net->stream);
  sc.done(1);
  return 1;
}

}  // namespace psg
