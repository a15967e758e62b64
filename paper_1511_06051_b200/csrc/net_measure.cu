// Measurement paths of a Net: per-op CUDA-event profile of one training step,
// and the host-fed (end-to-end) training loop used for bench.py's `e2e` number.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

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

// Two device staging buffers and their step graphs (host-fed training).
void host_graphs_prepare(psg_net* net, size_t b, size_t chw) {
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
}

// Step s of a host-fed run: H2D of its batch into buffer s % 2 (copy stream, after the
// buffer's previous step consumed it), the step graph, the D2H of its loss.
void host_step_enqueue(psg_net* net, const float* img, const int32_t* lab, long s, size_t b,
                       size_t chw) {
  const int k = static_cast<int>(s & 1);
  PSG_CUDA(cudaStreamWaitEvent(net->copy_stream, net->consumed[k], 0));
  PSG_CUDA(cudaMemcpyAsync(net->d_stage2[k], img, b * chw * sizeof(float),
                           cudaMemcpyHostToDevice, net->copy_stream));
  PSG_CUDA(cudaMemcpyAsync(net->d_lab2[k], lab, b * sizeof(int32_t), cudaMemcpyHostToDevice,
                           net->copy_stream));
  PSG_CUDA(cudaEventRecord(net->copied[k], net->copy_stream));
  PSG_CUDA(cudaStreamWaitEvent(net->stream, net->copied[k], 0));
  PSG_CUDA(cudaGraphLaunch(net->host_graph2[k], net->stream));
  PSG_CUDA(cudaEventRecord(net->consumed[k], net->stream));
  PSG_CUDA(cudaMemcpyAsync(net->h_losses + s, &net->dsc->loss, sizeof(double),
                           cudaMemcpyDeviceToHost, net->stream));
}

// Device staging + pinned loss slots for `steps` host-fed steps.
void host_steps_prepare(psg_net* net, size_t b, size_t chw, long steps) {
  ensure_capacity(net, b);
  if (net->h_losses_cap < static_cast<size_t>(steps)) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    if (net->h_losses) cudaFreeHost(net->h_losses);
    PSG_CUDA(cudaMallocHost(&net->h_losses, steps * sizeof(double)));
    net->h_losses_cap = static_cast<size_t>(steps);
  }
  (void)chw;
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
  host_graphs_prepare(net, b, chw);
  PSG_CUDA(cudaEventRecord(net->t0, net->stream));
  PSG_CUDA(cudaStreamWaitEvent(net->copy_stream, net->t0, 0));  // copies inside the timing
  for (int k = 0; k < 2; ++k) {  // buffers are free once the stream's prior work is done
    PSG_CUDA(cudaEventRecord(net->consumed[k], net->stream));
  }
  for (long s = 0; s < steps; ++s)
    host_step_enqueue(net, images + s * b * chw, labels + s * b, s, b, chw);
  PSG_CUDA(cudaEventRecord(net->t1, net->stream));
  net->timed = true;
  net->last_n = b;
  net_check_flag(net);
  if (losses) std::memcpy(losses, net->h_losses, steps * sizeof(double));
}

// train(steps) fed by a host-side loader: per step, `threads` host threads gather the step's
// rows (NCHW fp32 ds_images[rows[s * b + i]]) and labels into one of two pinned staging
// buffers — the reference's gather_batch (data.hpp:292-304) on the host — while the GPU runs
// the previous step; then the same H2D copy / step graph / D2H of the loss as
// net_train_host.  A staging buffer is refilled once its copy to the device has completed.
void net_train_host_rows(psg_net* net, const float* ds_images, const int32_t* ds_labels,
                         size_t ds_rows, const uint64_t* rows, long steps, double* losses,
                         int threads) {
  if (steps < 0) throw std::invalid_argument("train: negative step count");
  if (steps == 0) return;
  threads = std::max(1, threads);
  DeviceGuard dg(net->ctx->device);
  const LayerRt& d = net->L[net->data_idx];
  const size_t b = static_cast<size_t>(net->spec_batch);
  const size_t chw = static_cast<size_t>(d.C) * d.H * d.W;
  for (long s = 0; s < steps; ++s)
    for (size_t i = 0; i < b; ++i) {
      const uint64_t r = rows[s * b + i];
      if (r >= ds_rows) throw std::invalid_argument("gather: row index out of range");
      if (ds_labels[r] < 0 || ds_labels[r] >= net->classes)
        throw std::invalid_argument("forward: label out of range");
    }
  host_steps_prepare(net, b, chw, steps);
  host_graphs_prepare(net, b, chw);
  if (net->h_ring_cap < b * chw) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    for (int k = 0; k < 2; ++k) {
      if (net->h_ring[k]) cudaFreeHost(net->h_ring[k]);
      if (net->h_ring_lab[k]) cudaFreeHost(net->h_ring_lab[k]);
      PSG_CUDA(cudaMallocHost(&net->h_ring[k], b * chw * sizeof(float)));
      PSG_CUDA(cudaMallocHost(&net->h_ring_lab[k], b * sizeof(int32_t)));
      if (!net->h_ring_ev[k])
        PSG_CUDA(cudaEventCreateWithFlags(&net->h_ring_ev[k], cudaEventDisableTiming));
    }
    net->h_ring_cap = b * chw;
  }
  // Large rows can be gathered by the DMA engine straight from the (registered,
  // page-locked) dataset into device staging — no host copy — instead of host threads
  // copying them into pinned staging for one H2D.  Measured on AlexNet's 618 KB rows with a
  // 16-thread host: 1 GPU (16 threads) host 59.7–67K vs DMA 59.5–60K img/s e2e; 2 GPUs
  // (8 threads per rank) 93K vs 118K; 4 GPUs (4 per rank) 101K vs 172K — so the DMA engine
  // takes every row when a rank has fewer than 12 host threads (rows >= 64 KB), the host
  // otherwise.  A split (both in parallel) was slower than either: the copies serialise on
  // the copy engine.  PSG_HOST_ROW_DMA_FRAC (0..1) sets the DMA share of the rows.
  const size_t row_bytes = chw * sizeof(float);
  double frac = row_bytes >= (size_t{64} << 10) && threads < 12 ? 1.0 : 0.0;
  if (const char* e = std::getenv("PSG_HOST_ROW_DMA_FRAC")) frac = std::atof(e);
  const size_t nd = std::min(b, static_cast<size_t>(std::max(0.0, frac) * b + 0.5));
  if (nd && (net->h_reg != ds_images || net->h_reg_bytes != ds_rows * row_bytes)) {
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    PSG_CUDA(cudaStreamSynchronize(net->copy_stream));
    if (net->h_reg) PSG_CUDA(cudaHostUnregister(const_cast<void*>(net->h_reg)));
    net->h_reg = nullptr;
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, ds_images) == cudaSuccess &&
                        pa.type == cudaMemoryTypeHost;
    cudaGetLastError();  // unregistered host memory: not an error worth keeping
    if (!pinned) {
      PSG_CUDA(cudaHostRegister(const_cast<float*>(ds_images), ds_rows * row_bytes,
                                cudaHostRegisterDefault));
      net->h_reg = ds_images;
      net->h_reg_bytes = ds_rows * row_bytes;
    }
  }
  PSG_CUDA(cudaEventRecord(net->t0, net->stream));
  PSG_CUDA(cudaStreamWaitEvent(net->copy_stream, net->t0, 0));
  for (int k = 0; k < 2; ++k) {
    PSG_CUDA(cudaEventRecord(net->consumed[k], net->stream));
    PSG_CUDA(cudaEventRecord(net->h_ring_ev[k], net->copy_stream));
  }
  for (long s = 0; s < steps; ++s) {
    const int k = static_cast<int>(s & 1);
    PSG_CUDA(cudaEventSynchronize(net->h_ring_ev[k]));  // this buffer's last H2D is done
    float* dst = net->h_ring[k];
    const uint64_t* rs = rows + s * b;
    // DMA rows first (asynchronous: they stream while the host threads gather the rest)
    PSG_CUDA(cudaStreamWaitEvent(net->copy_stream, net->consumed[k], 0));
    for (size_t i = 0; i < nd; ++i)
      PSG_CUDA(cudaMemcpyAsync(net->d_stage2[k] + i * chw, ds_images + rs[i] * chw, row_bytes,
                               cudaMemcpyHostToDevice, net->copy_stream));
    const size_t nh = b - nd;
    auto work = [&](size_t i0, size_t i1) {
      for (size_t i = i0; i < i1; ++i)
        std::memcpy(dst + i * chw, ds_images + rs[nd + i] * chw, row_bytes);
    };
    const size_t per = (nh + threads - 1) / threads;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads && static_cast<size_t>(t) * per < nh; ++t)
      pool.emplace_back(work, t * per, std::min(nh, (t + 1) * per));
    work(0, std::min(nh, per));
    for (std::thread& th : pool) th.join();
    for (size_t i = 0; i < b; ++i) net->h_ring_lab[k][i] = ds_labels[rs[i]];
    if (nh)
      PSG_CUDA(cudaMemcpyAsync(net->d_stage2[k] + nd * chw, dst, nh * row_bytes,
                               cudaMemcpyHostToDevice, net->copy_stream));
    PSG_CUDA(cudaMemcpyAsync(net->d_lab2[k], net->h_ring_lab[k], b * sizeof(int32_t),
                             cudaMemcpyHostToDevice, net->copy_stream));
    PSG_CUDA(cudaEventRecord(net->h_ring_ev[k], net->copy_stream));  // after its H2D
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
