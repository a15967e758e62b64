/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.  CPU fp64 restatement of the reference's
 * SparkNet data-parallel path (/root/reference/proj/include/parasgd/*.hpp) plus the
 * Caffe layer semantics the BASELINE configs need and the reference lacks
 * (pad/stride/group conv, AVE and ceil-mode pooling, LRN, dropout, weight decay).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker or the timed CPU
 * baseline.  The product (libpsg.so) never links or calls it.
 *
 * Parity pinning: the reference-layer subset is checked bit-for-bit against the
 * unmodified reference compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile) through golden fixtures in tests/golden/.  The Caffe
 * extensions are pinned by finite differences (the reference's own method,
 * tests/unit/test_helpers.hpp:51-73) and by the pad/stride identities of
 * SURVEY §8(c).
 *
 * Layout: NCHW, row-major, exactly as the reference.
 */
#ifndef PSG_ORACLE_H_
#define PSG_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/psg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:11-81 */
typedef struct orc_rng {
  uint64_t state;
  double spare;
  int has_spare;
} orc_rng;

uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_derive_seed(uint64_t base, const uint64_t* parts, int nparts);
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_normal(orc_rng* r);
void orc_rng_shuffle_u64(orc_rng* r, uint64_t* v, size_t n);

/* data.hpp */
void orc_generate_synthetic(int classes, size_t c, size_t h, size_t w, size_t per_class,
                            double separation, uint64_t seed, uint64_t variant, double* images,
                            int32_t* labels);
int orc_shard(size_t n, int workers, uint64_t seed, uint64_t* perm, uint64_t* offsets);
uint64_t orc_worker_stream_seed(uint64_t global_seed, int worker);
void orc_epoch_order(const uint64_t* shard, size_t n, uint64_t stream_seed, uint64_t epoch,
                     uint64_t* order);

/* model.hpp */
typedef struct orc_net orc_net;
orc_net* orc_net_create(const psg_layer_desc* layers, int n_layers, uint64_t seed);
const char* orc_last_error(void);
void orc_net_destroy(orc_net* net);
size_t orc_net_param_count(const orc_net* net);
int orc_net_num_classes(const orc_net* net);
void orc_net_get_weights(const orc_net* net, double* flat);
void orc_net_set_weights(orc_net* net, const double* flat);
void orc_net_get_velocity(const orc_net* net, double* flat);
void orc_net_reset_velocity(orc_net* net);
void orc_net_set_sgd(orc_net* net, double lr, double momentum, double weight_decay);
void orc_net_set_dropout_step(orc_net* net, uint64_t step);
/* train != 0 selects the training phase (dropout active). */
int orc_net_forward(orc_net* net, const double* images, const int32_t* labels, size_t n,
                    int train, double* loss, double* probs);
int orc_net_backward(orc_net* net, const double* images, const int32_t* labels, size_t n,
                     double* loss, double* grads);
int orc_net_apply_update(orc_net* net, const double* grads);
/* Per-layer access (shape = per-example dims [c,h,w] or [d,1,1]). */
int orc_net_layer_dims(const orc_net* net, int layer, int64_t dims[3]);
const double* orc_net_layer_out(const orc_net* net, int layer);
const double* orc_net_layer_grad(const orc_net* net, int layer);
/* Per-layer isolation: run one layer on explicit inputs (batch n), keeping the
 * forward state so orc_layer_backward can use it. */
int orc_layer_forward(orc_net* net, int layer, size_t n, const double* const* inputs,
                      double* out);
int orc_layer_backward(orc_net* net, int layer, size_t n, const double* dy, double* dx,
                       double* dparams);
/* Offset of layer's first parameter in the flat vector, and its count. */
void orc_net_layer_params(const orc_net* net, int layer, size_t* offset, size_t* count);

/* weights.hpp:90-107 + tensor.hpp:166-179 */
void orc_weights_mean(const double* const* items, int k, size_t n, double* out);

/* schemes.hpp:274-351, worker jobs on `threads` pthreads. */
typedef struct orc_record {
  long serial_iters, parallel_iters, rounds;
  double sim_time, accuracy;
} orc_record;
typedef struct orc_sparknet_args {
  const psg_layer_desc* layers;
  int n_layers;
  const double* train_images;
  const int32_t* train_labels;
  size_t train_n;
  const double* eval_images;
  const int32_t* eval_labels;
  size_t eval_n;
  int c, h, w;
  size_t batch;
  double lr, momentum, weight_decay;
  uint64_t seed;
  double compute_seconds, sync_seconds;
  double target_accuracy;
  long eval_steps;
  int workers, tau;
  long rounds, warm;
  int threads;
  int skip_eval; /* timing runs: skip the per-round evaluation */
  double sublinearity; /* CostModel::sublinearity (run_naive clock); 0 reads as 1 */
} orc_sparknet_args;
/* Returns number of records written (<= max_records) or -1 on error.
 * round_weights (optional) receives rounds x P averaged weights. */
long orc_run_sparknet(const orc_sparknet_args* args, orc_record* records, long max_records,
                      uint64_t* warm_digest, double* round_weights);
uint64_t orc_weights_digest(const orc_net* net, const double* flat);
/* schemes.hpp:201-262 run_naive: each batch of worker 0's single-shard stream is split
 * into `workers` parts, the part gradients are averaged (weights_mean) and applied once.
 * Uses args->workers / batch / lr / ...; evaluation every eval_every steps.  step_weights
 * (optional) receives iter_budget x P weights after every step.  Returns records or -1. */
long orc_run_naive(const orc_sparknet_args* args, long iter_budget, long eval_every,
                   orc_record* records, long max_records, double* step_weights);

#ifdef __cplusplus
}
#endif

#endif
