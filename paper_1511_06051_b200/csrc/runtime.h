// Runtime objects behind the opaque C handles (psg_ctx / psg_dataset / psg_net /
// psg_buffer / psg_comm).
#pragma once

#include <vector>

#include "psg_internal.h"

struct psg_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
};

struct psg_dataset {
  psg_ctx* ctx = nullptr;
  size_t n = 0;
  int c = 0, h = 0, w = 0, classes = 0;
  float* images = nullptr;   // device NHWC [n][h][w][c]
  int32_t* labels = nullptr; // device [n]
  std::vector<int32_t> host_labels;
};

struct psg_buffer {
  psg_ctx* ctx = nullptr;
  float* ptr = nullptr;
  size_t n = 0;
};

namespace psg {

// One WeightCollection tensor: reference (NCHW-order) view <-> internal slot.
struct TensorRec {
  int layer = 0, slot = 0, rank = 1;
  int64_t shape[4] = {0, 0, 0, 0};
  size_t ref_off = 0, ref_count = 0;
  size_t int_off = 0, int_count = 0;
  int map = 0;  // 0 identity, 1 conv kernel, 2 linear weight
  int F = 0, Cg = 0, Cgs = 0, kh = 0, kw = 0, Kp = 0;  // conv kernel (Kp: row stride)
  int O = 0, pc = 0, ph = 0, pw = 0, pcs = 0;    // linear: producer logical dims + channel stride
  float lr_mult = 1.f, decay_mult = 1.f;
  // reference flat index i (within tensor) -> internal flat index
  size_t to_int(size_t i) const;
};

struct LayerRt {
  psg_layer_desc d{};
  int chunk0 = 0, nchunk = 0;  // this layer's SGD-update chunks (UpdateChunk table range)
  int kind = 0;
  std::vector<int> inputs, consumers;
  int C = 0, H = 1, W = 1;  // logical per-example dims
  int cs = 0;               // internal channel stride (NHWC)
  size_t vol() const { return static_cast<size_t>(H) * W * cs; }
  float* out = nullptr;
  float* grad = nullptr;
  uint8_t* route = nullptr;
  float* col = nullptr;  // im2col matrix (TF32 im2col route only)
  std::vector<int> coff;  // concat: channel offset of each input
  // ReLU fusion (psg_net_set_fusion): a conv / linear whose only consumer is a ReLU writes
  // relu(out) into the ReLU's buffer from its epilogue (fwd_relu = that ReLU, out aliases
  // it); a ReLU whose only consumer is an LRN has its backward folded into the LRN's
  // (bwd_by = that LRN; the LRN masks with its input and writes the ReLU's input grad).
  int fwd_relu = -1, fused_from = -1, bwd_by = -1, bwd_relu = -1;
  // LRN -> max pool fusion: an LRN whose only consumer is a fusable 3x3 max pool is
  // computed inside the pool's kernel (lrn_pool = that pool, pool_lrn = the LRN), and the
  // pool's backward is gathered inside the LRN backward (lrn_maxpool_bwd), so the LRN output
  // and gradient are never materialised.
  int lrn_pool = -1, pool_lrn = -1;
  int kern_t = -1, bias_t = -1;
  // lanes: gradient scratch for the 2nd, 3rd, ... writer into this layer's gradient when
  // its consumers run on several lanes (summed into grad, in writer order, before use)
  std::vector<float*> acc_scratch;
  ConvGeom cg;  // conv / linear (per-example; n filled per call)
  PoolGeom pg;
  LrnGeom lg;
  DropGeom dg;
};

struct DeviceScalars {
  double loss;
  int flag;
  int cursor;
  uint64_t step;
  unsigned long long correct;
};

}  // namespace psg

struct psg_net {
  psg_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  uint64_t seed = 0;
  std::vector<psg::LayerRt> L;
  int data_idx = -1, label_idx = -1, loss_idx = -1, classes = 0, spec_batch = 0;
  std::vector<psg::TensorRec> tensors;
  size_t P_ref = 0, P_int = 0, P_alloc = 0;
  float* w = nullptr;
  float* g = nullptr;
  float* v = nullptr;
  psg::UpdateChunk* d_chunks = nullptr;
  int nchunks = 0;
  double lr = 0.01, mu = 0.0, wd = 0.0;
  psg::Mode mode = psg::Mode::Strict;
  bool fuse = true;
  // the current batch was gathered straight into the first conv's space-to-depth input
  // (stage_gathered_batch); consumed (cleared) by the next run_forward
  bool data_s2d = false;
  psg::DeviceScalars* dsc = nullptr;
  psg::DeviceScalars* hsc = nullptr;  // pinned mirror
  double* row_loss = nullptr;
  int32_t* labels = nullptr;
  psg::Workspace ws;
  // Branch lanes (nets whose layers fan out, e.g. GoogLeNet's inception modules): layer li
  // runs on lane lane_of[li] (0 = stream, k = lane_stream[k]); a layer waits for the events
  // of its inputs (forward) / of the last writer of the gradient it reads or accumulates into
  // (backward) when they ran on another lane; each lane has its own GEMM workspace.  The
  // launch order per buffer is unchanged, so results are bitwise those of one stream.
  static constexpr int kLanes = 4;             // branch lanes (0 = stream)
  static constexpr int kWgLane = kLanes;       // the wgrad lane's own stream
  static constexpr int kStreams = kLanes + 1;
  bool lanes_on = false;
  bool fanout = false;                // branch lanes active (some layer fans out)
  std::vector<cudaEvent_t> ev_sum;    // per layer: its scratch gradients summed
  // wgrad lane (PSG_WGRAD_LANE, default on): the weight gradients of lane-0 layers run on
  // their own stream (kWgLane) — after the last writer of the gradient they read —
  // overlapping the dgrad chain
  bool wgrad_lane = false;
  std::vector<int> lane_of;
  cudaStream_t lane_stream[kStreams] = {};
  cudaEvent_t lane_fork = nullptr, lane_join[kStreams] = {};
  std::vector<cudaEvent_t> ev_fwd, ev_bwd;
  psg::Workspace ws_lane[kStreams];
  size_t cap = 0;       // batch capacity of the activation buffers
  size_t last_n = 0;    // batch of the last forward
  // training stream (ShardBatchIterator, data.hpp:312-351)
  psg_dataset* train_ds = nullptr;
  std::vector<uint64_t> shard, order;
  size_t it_batch = 0, it_cursor = 0;
  uint64_t it_seed = 0, it_epoch = 0;
  int it_part = 0, it_parts = 1;  // this net consumes rows [part*b/parts, +b/parts) of a batch
  uint32_t* d_idx = nullptr;
  uint32_t* h_idx = nullptr;  // pinned staging
  size_t idx_cap = 0;
  cudaEvent_t idx_ev = nullptr;
  // validation stream (SequentialBatchIterator, data.hpp:355-382)
  psg_dataset* val_ds = nullptr;
  size_t val_batch = 0, val_cursor = 0;
  uint32_t* d_vidx = nullptr;  // queued evaluation batches (test_begin .. test_end)
  size_t vidx_cap = 0;
  unsigned long long val_total = 0;
  bool val_pending = false;
  // explicit-batch staging
  float* h_stage = nullptr;
  size_t h_stage_cap = 0;
  int32_t* h_lab = nullptr;
  // graph of one training step
  cudaGraphExec_t graph = nullptr;
  size_t graph_batch = 0;
  cudaGraphExec_t grad_graph = nullptr;  // gather + forward + backward (run_naive parts)
  cudaGraphExec_t round_graph = nullptr;  // last step of an overlapped round (+ NCCL)
  size_t round_graph_batch = 0;
  psg_comm* round_comm = nullptr;
  cudaStream_t side_stream = nullptr;
  std::vector<cudaEvent_t> bucket_ev;
  cudaEvent_t side_join = nullptr;
  size_t grad_graph_batch = 0;
  int launches_per_step = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  bool timed = false;
  // host-fed (e2e) training: NCHW staging buffer + its own step graph
  float* d_stage = nullptr;        // eager path (one buffer)
  size_t d_stage_cap = 0;
  cudaGraphExec_t host_graph = nullptr;
  // graph path: double-buffered staging, H2D of step s+1 on copy_stream overlaps step s
  float* d_stage2[2] = {nullptr, nullptr};
  int32_t* d_lab2[2] = {nullptr, nullptr};
  size_t d_stage2_cap = 0;
  cudaGraphExec_t host_graph2[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
  double* h_losses = nullptr;
  // host-side loader (net_train_host_rows): two pinned batches gathered on the host
  float* h_ring[2] = {nullptr, nullptr};
  int32_t* h_ring_lab[2] = {nullptr, nullptr};
  cudaEvent_t h_ring_ev[2] = {nullptr, nullptr};
  size_t h_ring_cap = 0;
  // net_train_host_rows' DMA share of large rows: the dataset registered (page-locked) once
  // and those rows copied by the DMA engine straight into device staging
  const void* h_reg = nullptr;
  size_t h_reg_bytes = 0;
  size_t h_losses_cap = 0;
  cudaEvent_t slots[16] = {};
};

namespace psg {

// Per-op CUDA-event timer (psg_net_profile_step).
struct OpTimer {
  cudaStream_t stream = nullptr;
  struct Rec {
    psg_op_time info;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  explicit OpTimer(cudaStream_t s) : stream(s) {}
  ~OpTimer();
  void begin(const char* name, int layer, int phase, double flops, double bytes);
  void end(int launches);
  cudaError_t record(cudaEvent_t e);
};

// Gather the step's batch from the HBM-resident dataset rows idx[cursor * n + i]: into the
// data layer, or (fusion on, TF32) straight into the space-to-depth input of a strided
// first conv that is the data layer's only consumer.  Returns the launches enqueued.
int stage_gathered_batch(psg_net* net, const float* images, const int32_t* labels,
                         const uint32_t* idx, const int* cursor, size_t n);
// A host-fed NCHW batch (already copied to the device) into the data layer, or straight
// into the space-to-depth input of the first conv (as stage_gathered_batch).
int stage_host_batch(psg_net* net, const float* src, size_t n);
int run_forward(psg_net* net, size_t n, bool train, bool seed_grad, OpTimer* timer = nullptr);
// The last step of a SparkNet round with the K-way average overlapped across layers: as soon
// as a parameter layer's wgrad and dgrad are enqueued, its SGD update runs and its weights
// go to an ncclAllReduce(avg) on the side stream while the backward of the layers below
// continues (the bucket of layer L is final once dgrad_L has read W_L).
struct RoundOverlap {
  psg_comm* comm = nullptr;
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ready;  // per bucket: update done on the main stream
  cudaEvent_t join = nullptr;      // side stream done
  int last_param_layer = -1;       // the last bucket in backward order advances the counters
  int buckets = 0;
};
int run_backward(psg_net* net, size_t n, OpTimer* timer = nullptr, RoundOverlap* ov = nullptr);
int run_update(psg_net* net, bool advance, OpTimer* timer = nullptr);
void ensure_capacity(psg_net* net, size_t n);
void release_batch_buffers(psg_net* net);  // drops activations + graphs; realloc on demand
void invalidate_graph(psg_net* net);
unsigned long long guard_violations(std::string* first);
void copy_sync(psg_net* net, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind);
void plan_fusion(psg_net* net);

void net_profile_step(psg_net* net, int repeats, psg_op_time* out, int max_ops, int* n_ops);
void net_train_host(psg_net* net, const float* images, const int32_t* labels, long steps,
                    double* losses);
void net_train_host_rows(psg_net* net, const float* ds_images, const int32_t* ds_labels,
                         size_t ds_rows, const uint64_t* rows, long steps, double* losses,
                         int threads);

void net_build(psg_net* net, const psg_layer_desc* layers, int n, uint64_t seed);
void net_free(psg_net* net);
void net_check_flag(psg_net* net);  // throws std::runtime_error on the sticky flag
void net_set_sgd(psg_net* net, double lr, double mu, double wd);
void net_get_weights(psg_net* net, double* flat, size_t n, bool velocity);
void net_set_weights(psg_net* net, const double* flat, size_t n);
void net_forward_host(psg_net* net, const double* images, const int32_t* labels, size_t n,
                      double* loss, double* probs);
void net_backward_host(psg_net* net, const double* images, const int32_t* labels, size_t n,
                       double* loss, double* grads);
void net_apply_update_host(psg_net* net, const double* grads, size_t n);
void net_layer_readback(psg_net* net, int layer, bool grad, double* out, size_t n);
void net_attach_shard(psg_net* net, psg_dataset* ds, const uint64_t* idx, size_t count,
                      size_t batch, uint64_t seed, int part = 0, int parts = 1);
void net_train(psg_net* net, long steps);
// train(tau) + the fast K-way average, the average's buckets overlapped with the last
// step's backward
void net_train_round(psg_net* net, long steps, psg_comm* comm);
void comm_allreduce_avg(psg_comm* c, float* ptr, size_t count, cudaStream_t s);
int comm_device(const psg_comm* c);
void net_grad_step(psg_net* net);
void net_apply_grads(psg_net* net);
void net_attach_validation(psg_net* net, psg_dataset* ds, size_t batch);
double net_test(psg_net* net, long steps);
void net_test_begin(psg_net* net, long steps, long first, long stride);
void net_test_end(psg_net* net, unsigned long long* correct, unsigned long long* total);

void comm_unique_id(unsigned char id[128]);
psg_comm* comm_create(psg_ctx* ctx, int nranks, int rank, const unsigned char id[128]);
void comm_create_all(psg_ctx* const* ctxs, int ndev, psg_comm** out);
void comm_destroy(psg_comm* c);
// which: 0 = parameters (weights_mean), 1 = gradients (run_naive's per-step mean)
void comm_average_nets(psg_comm* const* comms, psg_net* const* nets, int count, int mode,
                       int which = 0);
void comm_broadcast_nets(psg_comm* const* comms, psg_net* const* nets, int count, int root);
void comm_average_buffers(psg_comm* const* comms, psg_buffer* const* bufs, int count, int mode,
                          float* device_ms);
}  // namespace psg
