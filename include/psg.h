/*
 * psg.h — C ABI of the B200-native SparkNet data-parallel hot path (libpsg.so).
 *
 * The reference (`/root/reference/proj`, "parasgd") is header-only C++ with no FFI
 * layer; its drop-in surface is the declarations in model.hpp / weights.hpp /
 * data.hpp / schemes.hpp.  This header is the thin C boundary that a C++ (or
 * ctypes / cgo / JNI) host binds to; every entry point below names the
 * reference interface it replaces.  Plain pointers and sizes only, no torch
 * types.  All host-visible tensors use the reference's layouts:
 *   images  : [n, c, h, w] row-major (NCHW), as Batch::images (batch.hpp:11-16)
 *   weights : WeightCollection order (weights.hpp:19-86): layer declaration
 *             order x {kernel, bias} x row-major; conv kernels [F, C/G, kh, kw],
 *             linear weights [O, D] with D flattened in CHW order
 *             (model.hpp:409).
 * Internally the device keeps activations NHWC and conv kernels [F, kh, kw, C/G];
 * the boundary converts.
 *
 * Error model: every call returns a status code; the message of
 * the last failure on the calling thread is psg_last_error().
 *   PSG_EINVAL   <-> std::invalid_argument  (structure / shape / argument errors)
 *   PSG_ERUNTIME <-> std::runtime_error     (non-finite values, missing data)
 *   PSG_ECUDA    <-> CUDA / NCCL failures
 *   PSG_ELOGIC   <-> std::logic_error
 */
#ifndef PSG_H_
#define PSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSG_ABI_VERSION 1

enum psg_status {
  PSG_OK = 0,
  PSG_EINVAL = 1,
  PSG_ERUNTIME = 2,
  PSG_ECUDA = 3,
  PSG_ELOGIC = 4
};

/* LayerKind (net_spec.hpp:11) plus the Caffe kinds the BASELINE configs need. */
enum psg_layer_kind {
  PSG_LAYER_DATA = 0,
  PSG_LAYER_LABEL = 1,
  PSG_LAYER_CONV = 2,
  PSG_LAYER_POOL = 3,
  PSG_LAYER_LINEAR = 4,
  PSG_LAYER_RELU = 5,
  PSG_LAYER_SOFTMAX_LOSS = 6,
  PSG_LAYER_LRN = 7,      /* extension: Caffe LRN ACROSS_CHANNELS */
  PSG_LAYER_DROPOUT = 8,  /* extension: Caffe dropout (counter-hash mask) */
  PSG_LAYER_CONCAT = 9    /* extension: Caffe Concat along channels (GoogLeNet inception) */
};

enum psg_pool_method { PSG_POOL_MAX = 0, PSG_POOL_AVE = 1 };

enum psg_precision {
  PSG_PRECISION_FP32 = 0, /* strict mode: fp32 SIMT FFMA, 1e-5 parity bar */
  PSG_PRECISION_TF32 = 1  /* fast mode: tcgen05 kind::tf32, fp32 accumulate, 1e-2 bar */
};

enum psg_average_mode {
  PSG_AVERAGE_FAST = 0,    /* NCCL allreduce-sum x 1/K */
  PSG_AVERAGE_ORDERED = 1  /* ascending-k fp64 accumulation, /K, one rounding (weights.hpp:90-107) */
};

/*
 * One declarative layer: LayerSpec (net_spec.hpp:28-38) widened with Caffe
 * geometry.  Zero/defaults (psg_layer_desc_init) reproduce the reference:
 * stride 1, no pad, group 1, floor-mode pooling, lr/decay multipliers 1.
 */
typedef struct psg_layer_desc {
  int kind;                /* psg_layer_kind */
  char name[48];
  int n_inputs;
  int inputs[8];           /* indices of earlier layers (topological order) */
  int batch, channels, height, width; /* data: [b,c,h,w]; label: batch */
  int num_output;          /* conv filters / linear outputs */
  int kernel_h, kernel_w;
  int stride_h, stride_w;
  int pad_h, pad_w;
  int group;
  int pool;                /* psg_pool_method */
  int ceil_mode;           /* 0: reference floor mode (model.hpp:244); 1: Caffe ceil */
  int local_size;          /* LRN */
  double alpha, beta, k;   /* LRN */
  double dropout_ratio;    /* dropout */
  double loss_weight;      /* softmax loss (1.0 = reference) */
  double lr_mult_w, lr_mult_b, decay_mult_w, decay_mult_b;
} psg_layer_desc;

/* Fills defaults; name is truncated to 47 bytes. */
void psg_layer_desc_init(psg_layer_desc* d, int kind, const char* name);

typedef struct psg_ctx psg_ctx;
typedef struct psg_dataset psg_dataset;
typedef struct psg_net psg_net;
typedef struct psg_comm psg_comm;
typedef struct psg_buffer psg_buffer;

const char* psg_last_error(void);
int psg_abi_version(void);
int psg_device_count(int* n);

/* ---- host-side reference semantics (bit-exact integer work) ---------------- */
/* splitmix64 / derive_seed (rng.hpp:11-25). */
uint64_t psg_splitmix64(uint64_t x);
uint64_t psg_derive_seed(uint64_t base, const uint64_t* parts, int nparts);
/* shard() permutation + split (data.hpp:261-288): perm[n], offsets[workers+1]. */
int psg_shard(size_t n, int workers, uint64_t seed, uint64_t* perm, uint64_t* offsets);
/* worker_stream_seed (data.hpp:386-388). */
uint64_t psg_worker_stream_seed(uint64_t global_seed, int worker_id);
/* ShardBatchIterator::start_epoch order (data.hpp:338-343). */
int psg_epoch_order(const uint64_t* shard_indices, size_t n, uint64_t stream_seed,
                    uint64_t epoch, uint64_t* order);
/* generate_synthetic (data.hpp:111-155), NCHW fp64 on the host. */
int psg_generate_synthetic(int classes, size_t c, size_t h, size_t w, size_t per_class,
                           double separation, uint64_t seed, uint64_t variant, double* images,
                           int32_t* labels);

/* ---- device context --------------------------------------------------------- */
int psg_ctx_create(int device, psg_ctx** out);
int psg_ctx_destroy(psg_ctx* ctx);
int psg_ctx_sync(psg_ctx* ctx);

/* ---- datasets: Dataset (data.hpp:21-41) resident in HBM --------------------- */
int psg_dataset_upload_f64(psg_ctx* ctx, const double* images, const int32_t* labels, size_t n,
                           int c, int h, int w, int num_classes, psg_dataset** out);
int psg_dataset_upload_f32(psg_ctx* ctx, const float* images, const int32_t* labels, size_t n,
                           int c, int h, int w, int num_classes, psg_dataset** out);
/* Host generator (bit-exact with the reference) followed by upload. */
int psg_dataset_synthetic(psg_ctx* ctx, int classes, int c, int h, int w, size_t per_class,
                          double separation, uint64_t seed, uint64_t variant, psg_dataset** out);
/* generate_synthetic's distribution generated on the device: class
 * means bit-exact with data.hpp:121-131, within-class noise from a counter-based RNG
 * (same law, not the reference's serial stream).  For AX/GN-sized datasets. */
int psg_dataset_synthetic_device(psg_ctx* ctx, int classes, int c, int h, int w,
                                 size_t per_class, double separation, uint64_t seed,
                                 uint64_t variant, psg_dataset** out);
/* load_idx / load_csv (data.hpp:163-255): same format checks and messages (runtime
 * errors).  psg_read_* parse on the host only (images may be NULL to query n / extents;
 * pixels p/255 in fp64 rounded to fp32); psg_dataset_load_* put the data in HBM, IDX
 * bytes converted on the device. */
int psg_read_idx(const char* images_path, const char* labels_path, size_t* n, int* h, int* w,
                 int* num_classes, float* images, int32_t* labels);
int psg_read_csv(const char* path, int c, int h, int w, int num_classes, size_t* n, float* images,
                 int32_t* labels);
int psg_dataset_load_idx(psg_ctx* ctx, const char* images_path, const char* labels_path,
                         psg_dataset** out);
int psg_dataset_load_csv(psg_ctx* ctx, const char* path, int c, int h, int w, int num_classes,
                         psg_dataset** out);
/* Read rows [first, first+count) back as NCHW fp32 + labels (tests, inspection). */
int psg_dataset_read_f32(const psg_dataset* ds, size_t first, size_t count, float* images_nchw,
                         int32_t* labels);
int psg_dataset_size(const psg_dataset* ds, size_t* n);
int psg_dataset_destroy(psg_dataset* ds);

/* ---- nets: class Net (model.hpp:50-597) ------------------------------------- */
/* Net(NetSpec, seed) (model.hpp:52-55, init at :200-283). */
int psg_net_create(psg_ctx* ctx, const psg_layer_desc* layers, int n_layers, uint64_t seed,
                   psg_net** out);
int psg_net_destroy(psg_net* net);
int psg_net_num_classes(const psg_net* net, int* classes);
/* Flat parameter count P (sum of WeightCollection tensor volumes). */
int psg_net_param_count(const psg_net* net, size_t* n);
/* WeightCollection structure: tensors in order; layer index, tensor slot
 * (0 kernel / 1 bias), rank and reference-order shape, flat offset. */
int psg_net_num_tensors(const psg_net* net, int* n);
int psg_net_tensor_info(const psg_net* net, int t, int* layer, int* slot, int* rank,
                        int64_t shape[4], size_t* offset);
int psg_net_set_precision(psg_net* net, int precision);
/* set_sgd (model.hpp:60-66) + weight decay extension (0 = reference). */
int psg_net_set_sgd(psg_net* net, double learning_rate, double momentum, double weight_decay);
/* get_weights / set_weights (model.hpp:140-171); fp32 <-> fp64 exact widening,
 * round-to-nearest narrowing.  Momentum untouched by set. */
int psg_net_get_weights_f64(psg_net* net, double* flat, size_t n);
int psg_net_set_weights_f64(psg_net* net, const double* flat, size_t n);
int psg_net_get_velocity_f64(psg_net* net, double* flat, size_t n);
int psg_net_reset_velocity(psg_net* net);
/* forward(Batch) (model.hpp:74-78): loss + probabilities [n, classes]. */
int psg_net_forward(psg_net* net, const double* images, const int32_t* labels, size_t n,
                    double* loss, double* probs);
/* backward(Batch) (model.hpp:83-86): gradient in WeightCollection order. */
int psg_net_backward(psg_net* net, const double* images, const int32_t* labels, size_t n,
                     double* loss, double* grads);
/* apply_update(grads) (model.hpp:90-107). */
int psg_net_apply_update(psg_net* net, const double* grads, size_t n);
/* Per-layer state of the last forward/backward, reference NCHW order (parity harness). */
int psg_net_layer_shape(const psg_net* net, int layer, int64_t shape[4]);
int psg_net_layer_output(psg_net* net, int layer, double* out, size_t n);
int psg_net_layer_grad(psg_net* net, int layer, double* out, size_t n);
/* set_training_data(make_worker_iterator(...)) with the shard kept on device:
 * ShardBatchIterator semantics (data.hpp:312-351). */
int psg_net_attach_shard(psg_net* net, psg_dataset* ds, const uint64_t* shard_indices,
                         size_t count, size_t batch, uint64_t stream_seed);
/* run_naive (schemes.hpp:201-262): the net consumes rows [part*batch/parts, +batch/parts)
 * of every batch of the stream (batch = the full minibatch; parts must divide it). */
int psg_net_attach_shard_part(psg_net* net, psg_dataset* ds, const uint64_t* shard_indices,
                              size_t count, size_t batch, uint64_t stream_seed, int part,
                              int parts);
/* One step of run_naive's per-part work (schemes.hpp:233-247): next batch part ->
 * forward + backward; the gradient stays in the net's flat gradient buffer. */
int psg_net_grad_step(psg_net* net);
/* apply_update (model.hpp:90-107) with the resident (e.g. averaged) gradient. */
int psg_net_apply_grads(psg_net* net);
/* Iterator position (epoch, cursor) of the attached shard stream.  Lets a host
 * share one ShardBatchIterator between nets (the warm-start master consumes
 * worker 0's stream, schemes.hpp:314). */
int psg_net_get_stream_position(const psg_net* net, uint64_t* epoch, uint64_t* cursor);
int psg_net_set_stream_position(psg_net* net, uint64_t epoch, uint64_t cursor);
/* train(steps) (model.hpp:111-118); enqueued on the net's stream.  A non-finite
 * value raises PSG_ERUNTIME at the next psg_net_sync (sticky device flag). */
int psg_net_train(psg_net* net, long steps);
int psg_net_sync(psg_net* net);
/* One SparkNet round of this worker (schemes.hpp:323-336 for one worker): train(steps)
 * followed by the fast K-way weight average over `comm` (as psg_comm_average(FAST)), the
 * average overlapped with the last step's backward: each parameter layer's update and
 * ncclAllReduce(avg) are issued as soon as its gradients are done, on a side stream,
 * in reverse layer order (extension). */
int psg_net_train_round(psg_net* net, long steps, psg_comm* comm);
/* Device time of the last psg_net_train call's kernels (CUDA events on the
 * net's stream), ms; valid after psg_net_sync. */
int psg_net_last_train_ms(psg_net* net, float* ms);
int psg_net_last_loss(psg_net* net, double* loss);
/* set_validation_data(SequentialBatchIterator) + test(steps) (model.hpp:122-136). */
int psg_net_attach_validation(psg_net* net, psg_dataset* ds, size_t batch);
int psg_net_test(psg_net* net, long steps, double* accuracy);
/* Sharded evaluation: queue batches first, first+stride, ... < steps of the iterator's
 * next `steps` batches (the iterator advances by `steps`); test_end returns the counts.
 * K nets with first = k, stride = K split one test(steps) exactly. */
int psg_net_test_begin(psg_net* net, long steps, long first, long stride);
int psg_net_test_end(psg_net* net, unsigned long long* correct, unsigned long long* total);
/* ReLU fusion (default on): a conv / linear whose only consumer is a ReLU applies the ReLU
 * in its GEMM epilogue (its stored output is then the post-ReLU value), and a ReLU feeding
 * only an LRN has its backward folded into the LRN's (its own gradient buffer is not
 * written).  Results are bitwise identical; turn it off to inspect every layer's state
 * (per-layer parity tests). */
int psg_net_set_fusion(psg_net* net, int on);
/* tcgen05 CTA-pair policy of the net's TF32 GEMMs (extension, no reference counterpart):
 * AUTO = the throughput heuristic (pairs for K-major-A GEMMs with >= 2 waves of clusters),
 * NEVER = single-CTA kernels only, ALWAYS = a CTA pair (cta_group::2) wherever legal.
 * Results are correct either way; the parity tests use ALWAYS / NEVER to run the pair and
 * single-CTA kernel variants at small batch sizes where AUTO would not pick pairs. */
enum psg_tc_pair { PSG_TC_PAIR_AUTO = 0, PSG_TC_PAIR_NEVER = 1, PSG_TC_PAIR_ALWAYS = 2 };
int psg_net_set_tc_options(psg_net* net, int pair_policy);
/* Kernel launches of one training step (device-side work count). */
int psg_net_kernels_per_step(const psg_net* net, int* launches);

/* Debug (tests; no reference counterpart): with PSG_GUARD=1 in the environment every net
 * buffer is allocated between two 4 KB guard bands of 0xA5; the count of overwritten guard
 * bytes over all live (and already freed) net buffers, and the first offender. */
int psg_debug_guard_violations(unsigned long long* bad_bytes, char* first, size_t first_len);
/* Debug (profiling tools; no reference counterpart): with PSG_TC_PROF=1 in the environment
 * every tcgen05 GEMM launch records clock64 counters of its pipeline waits; one line per
 * launch: "index|plan label|loop wait_full wait_acc stages prod_wait prod_loop epi_wait
 * epi_loop" (cycles summed over the leader CTAs).  reset != 0 zeroes the counters. */
int psg_debug_tc_prof(char* buf, size_t len, int reset);

/* ---- measurement ------------------------------------------------------------ */
/* One op of a training step: algorithmic work and its CUDA-event device time. */
typedef struct psg_op_time {
  char name[64];
  int layer;
  int phase;     /* 0 gather, 1 forward, 2 loss, 3 wgrad, 4 dgrad, 5 backward (other), 6 update */
  double flops;  /* algorithmic FLOPs (GEMM-shaped ops), else 0 */
  double bytes;  /* algorithmic HBM bytes (bandwidth ops), else 0 */
  float ms;      /* mean device time over `repeats` eager replays */
  int launches;
} psg_op_time;
/* Replays one training step eagerly `repeats` times on the attached stream's
 * current batch with an event pair around every op (a real step: it updates). */
int psg_net_profile_step(psg_net* net, int repeats, psg_op_time* out, int max_ops, int* n_ops);
/* train(steps) fed from HOST memory: per step, an H2D copy of that step's batch
 * (NCHW fp32, labels int32) then the step, then a D2H read of its loss.  The
 * end-to-end path of the C ABI (pinned memory from psg_host_alloc is fastest). */
int psg_net_train_host(psg_net* net, const float* images, const int32_t* labels, long steps,
                       double* losses);
/* train(steps) with a host-side loader: per step `threads` host threads gather the step's
 * rows ds_images[rows[s*b + i]] (NCHW fp32, row = c*h*w floats) and their labels into a
 * pinned staging buffer (gather_batch, data.hpp:292-304) while the GPU runs the previous
 * step, then H2D copy, the step, and a D2H read of its loss.  Rows of >= 64 KB with fewer
 * than 12 threads (PSG_HOST_ROW_DMA_FRAC overrides the share) are instead copied row by row
 * by the DMA engine straight into device staging: ds_images is then page-locked with
 * cudaHostRegister (unless already pinned) until the net is freed or another dataset
 * pointer is passed — it must stay allocated that long. */
int psg_net_train_host_rows(psg_net* net, const float* ds_images, const int32_t* ds_labels,
                            size_t ds_rows, const uint64_t* rows, long steps, double* losses,
                            int threads);
int psg_host_alloc(size_t bytes, void** ptr);
int psg_host_free(void* ptr);
/* Event slots (0..15) on the net's stream for device-side timing of regions. */
int psg_net_event_record(psg_net* net, int slot);
int psg_net_event_elapsed(psg_net* net, int start_slot, int end_slot, float* ms);

/* ---- averaging: weights_mean (weights.hpp:90-107) ---------------------------- */
/* K nets on one device: ordered mean written back into every net. */
int psg_average_local(psg_net* const* nets, int count);
/* Same, over the nets' flat gradient buffers (run_naive's weights_mean of part gradients). */
int psg_average_grads_local(psg_net* const* nets, int count);
/* NCCL communicators (one per rank/device). */
int psg_comm_unique_id(unsigned char id[128]);
int psg_comm_create(psg_ctx* ctx, int nranks, int rank, const unsigned char id[128],
                    psg_comm** out);
int psg_comm_create_all(psg_ctx* const* ctxs, int ndev, psg_comm** out);
int psg_comm_destroy(psg_comm* comm);
/* In-place average of every net's flat parameters across the communicator.
 * count = nets driven by this caller (1 per process, or ndev in one process). */
int psg_comm_average(psg_comm* const* comms, psg_net* const* nets, int count, int mode);
/* In-place average of every net's flat gradient buffer (run_naive, schemes.hpp:248). */
int psg_comm_average_grads(psg_comm* const* comms, psg_net* const* nets, int count, int mode);
int psg_comm_broadcast(psg_comm* const* comms, psg_net* const* nets, int count, int root);

/* ---- raw flat buffers (averaging-only sweep) -------------------------------- */
int psg_buffer_create(psg_ctx* ctx, size_t n, psg_buffer** out);
int psg_buffer_fill_uniform(psg_buffer* buf, uint64_t seed, double lo, double hi);
int psg_buffer_read(psg_buffer* buf, float* host, size_t n);
int psg_buffer_write(psg_buffer* buf, const float* host, size_t n);
int psg_buffer_destroy(psg_buffer* buf);
int psg_buffer_average_local(psg_buffer* const* bufs, int count);
int psg_comm_average_buffer(psg_comm* const* comms, psg_buffer* const* bufs, int count,
                            int mode, float* device_ms);

#ifdef __cplusplus
}
#endif

#endif /* PSG_H_ */
