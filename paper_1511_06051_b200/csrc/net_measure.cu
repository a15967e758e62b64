// Measurement paths of a Net: per-op CUDA-event profile of one training step,
// and the host-fed (end-to-end) training loop used for bench.py's `e2e` number.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "runtime.h"

namespace psg {

void net_profile_step(psg_net* net, int repeats, psg_op_time* out, int max_ops, int* n_ops) {
  if (repeats < 1) throw std::invalid_argument("profile: repeats must be >= 1");
  if (!net->train_ds || !net->d_idx)
    throw std::runtime_error("profile: attach training data and train at least one step first");
  DeviceGuard dg(net->ctx->device);
  const size_t b = net->it_batch;
  ensure_capacity(net, b);
  const LayerRt& d = net->L[net->data_idx];
  psg_dataset* ds = net->train_ds;
  std::vector<psg_op_time> acc;
  // The step is captured with its per-op event records into a CUDA graph and replayed, as
  // the training loop runs it (eager launches would add the host's launch cost to every
  // short op); PSG_EAGER=1 profiles eager launches.
  static const bool eager = [] {
    const char* e = std::getenv("PSG_EAGER");
    return e && std::atoi(e) != 0;
  }();
  for (int r = 0; r <= repeats; ++r) {  // r = 0 is an untimed warm-up
    OpTimer t(net->stream);
    cudaGraph_t graph = nullptr;
    if (!eager) PSG_CUDA(cudaStreamBeginCapture(net->stream, cudaStreamCaptureModeThreadLocal));
    try {
      PSG_CUDA(cudaMemsetAsync(&net->dsc->cursor, 0, sizeof(int), net->stream));
      t.begin("gather", net->data_idx, 0, 0.0, 2.0 * 4.0 * static_cast<double>(b) * d.vol());
      stage_gathered_batch(net, ds->images, ds->labels, net->d_idx, &net->dsc->cursor, b);
      t.end(1);
      run_forward(net, b, true, true, &t);
      run_backward(net, b, &t);
      run_update(net, true, &t);
    } catch (...) {
      if (!eager) cudaStreamEndCapture(net->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    if (!eager) {
      PSG_CUDA(cudaStreamEndCapture(net->stream, &graph));
      cudaGraphExec_t exec = nullptr;
      PSG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      PSG_CUDA(cudaGraphLaunch(exec, net->stream));
      PSG_CUDA(cudaStreamSynchronize(net->stream));
      cudaGraphExecDestroy(exec);
    }
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    if (r == 0) {
      acc.resize(t.recs.size());
      for (size_t i = 0; i < t.recs.size(); ++i) {
        acc[i] = t.recs[i].info;
        acc[i].ms = 0.f;
      }
      continue;
    }
    for (size_t i = 0; i < t.recs.size(); ++i) {
      float ms = 0.f;
      PSG_CUDA(cudaEventElapsedTime(&ms, t.recs[i].a, t.recs[i].b));
      acc[i].ms += ms / static_cast<float>(repeats);
    }
  }
  net_check_flag(net);
  const int n = std::min<int>(max_ops, static_cast<int>(acc.size()));
  for (int i = 0; i < n; ++i) out[i] = acc[i];
  *n_ops = static_cast<int>(acc.size());
}

void net_train_host(psg_net* net, const float* images, const int32_t* labels, long steps,
                    double* losses) {
  if (steps < 0) throw std::invalid_argument("train: negative step count");
  if (steps == 0) return;
  DeviceGuard dg(net->ctx->device);
  const LayerRt& d = net->L[net->data_idx];
  const size_t b = static_cast<size_t>(net->spec_batch);
  const size_t chw = static_cast<size_t>(d.C) * d.H * d.W;
  for (long s = 0; s < steps; ++s)
    for (size_t i = 0; i < b; ++i) {
      const int32_t y = labels[s * b + i];
      if (y < 0 || y >= net->classes) throw std::invalid_argument("forward: label out of range");
    }
  ensure_capacity(net, b);
  if (net->d_stage_cap < b * chw) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    if (net->d_stage) cudaFree(net->d_stage);
    PSG_CUDA(cudaMalloc(&net->d_stage, b * chw * sizeof(float)));
    net->d_stage_cap = b * chw;
    invalidate_graph(net);
  }
  if (net->h_losses_cap < static_cast<size_t>(steps)) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    if (net->h_losses) cudaFreeHost(net->h_losses);
    PSG_CUDA(cudaMallocHost(&net->h_losses, steps * sizeof(double)));
    net->h_losses_cap = static_cast<size_t>(steps);
  }
  static const bool eager = [] {  // PSG_EAGER=1: no graph replay (see net_train)
    const char* e = std::getenv("PSG_EAGER");
    return e && e[0] == '1';
  }();
  if (eager) {
    PSG_CUDA(cudaEventRecord(net->t0, net->stream));
    for (long s = 0; s < steps; ++s) {
      PSG_CUDA(cudaMemcpyAsync(net->d_stage, images + s * b * chw, b * chw * sizeof(float),
                               cudaMemcpyHostToDevice, net->stream));
      PSG_CUDA(cudaMemcpyAsync(net->labels, labels + s * b, b * sizeof(int32_t),
                               cudaMemcpyHostToDevice, net->stream));
      stage_host_batch(net, net->d_stage, b);
      run_forward(net, b, true, true);
      run_backward(net, b);
      run_update(net, true);
      PSG_CUDA(cudaMemcpyAsync(net->h_losses + s, &net->dsc->loss, sizeof(double),
                               cudaMemcpyDeviceToHost, net->stream));
    }
    PSG_CUDA(cudaEventRecord(net->t1, net->stream));
    net->timed = true;
    net->last_n = b;
    net_check_flag(net);
    if (losses) std::memcpy(losses, net->h_losses, steps * sizeof(double));
    return;
  }
  // Graph path: two staging buffers, the H2D copies on a copy stream.  Step s waits for
  // its buffer's copy; the copy of step s+1 (other buffer) runs during step s.
  if (net->d_stage2_cap < b * chw) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    for (int k = 0; k < 2; ++k) {
      if (net->d_stage2[k]) cudaFree(net->d_stage2[k]);
      if (net->d_lab2[k]) cudaFree(net->d_lab2[k]);
      PSG_CUDA(cudaMalloc(&net->d_stage2[k], b * chw * sizeof(float)));
      PSG_CUDA(cudaMalloc(&net->d_lab2[k], b * sizeof(int32_t)));
      if (net->host_graph2[k]) cudaGraphExecDestroy(net->host_graph2[k]);
      net->host_graph2[k] = nullptr;
    }
    net->d_stage2_cap = b * chw;
  }
  if (!net->copy_stream) {
    PSG_CUDA(cudaStreamCreateWithFlags(&net->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      PSG_CUDA(cudaEventCreateWithFlags(&net->copied[k], cudaEventDisableTiming));
      PSG_CUDA(cudaEventCreateWithFlags(&net->consumed[k], cudaEventDisableTiming));
    }
  }
  if (net->graph_batch != b) invalidate_graph(net);
  for (int k = 0; k < 2; ++k) {
    if (net->host_graph2[k]) continue;
    cudaGraph_t graph;
    PSG_CUDA(cudaStreamBeginCapture(net->stream, cudaStreamCaptureModeThreadLocal));
    try {
      PSG_CUDA(cudaMemcpyAsync(net->labels, net->d_lab2[k], b * sizeof(int32_t),
                               cudaMemcpyDeviceToDevice, net->stream));
      stage_host_batch(net, net->d_stage2[k], b);
      run_forward(net, b, true, true);
      run_backward(net, b);
      run_update(net, true);
    } catch (...) {
      cudaStreamEndCapture(net->stream, &graph);
      throw;
    }
    PSG_CUDA(cudaStreamEndCapture(net->stream, &graph));
    PSG_CUDA(cudaGraphInstantiate(&net->host_graph2[k], graph, 0));
    cudaGraphDestroy(graph);
  }
  net->graph_batch = b;
  PSG_CUDA(cudaEventRecord(net->t0, net->stream));
  PSG_CUDA(cudaStreamWaitEvent(net->copy_stream, net->t0, 0));  // copies inside the timing
  for (int k = 0; k < 2; ++k) {  // buffers are free once the stream's prior work is done
    PSG_CUDA(cudaEventRecord(net->consumed[k], net->stream));
  }
  for (long s = 0; s < steps; ++s) {
    const int k = static_cast<int>(s & 1);
    PSG_CUDA(cudaStreamWaitEvent(net->copy_stream, net->consumed[k], 0));
    PSG_CUDA(cudaMemcpyAsync(net->d_stage2[k], images + s * b * chw, b * chw * sizeof(float),
                             cudaMemcpyHostToDevice, net->copy_stream));
    PSG_CUDA(cudaMemcpyAsync(net->d_lab2[k], labels + s * b, b * sizeof(int32_t),
                             cudaMemcpyHostToDevice, net->copy_stream));
    PSG_CUDA(cudaEventRecord(net->copied[k], net->copy_stream));
    PSG_CUDA(cudaStreamWaitEvent(net->stream, net->copied[k], 0));
    PSG_CUDA(cudaGraphLaunch(net->host_graph2[k], net->stream));
    PSG_CUDA(cudaEventRecord(net->consumed[k], net->stream));
    PSG_CUDA(cudaMemcpyAsync(net->h_losses + s, &net->dsc->loss, sizeof(double),
                             cudaMemcpyDeviceToHost, net->stream));
  }
  PSG_CUDA(cudaEventRecord(net->t1, net->stream));
  net->timed = true;
  net->last_n = b;
  net_check_flag(net);
  if (losses) std::memcpy(losses, net->h_losses, steps * sizeof(double));
}

}  // namespace psg
