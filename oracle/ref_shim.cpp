// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  A C-ABI wrapper around the
// UNMODIFIED reference headers at /root/reference/proj/include (header-only
// C++20, compiled in place by oracle/Makefile into oracle/_ref/).  Used to
// (1) generate the golden fixtures under tests/golden/ that pin the C oracle,
// and (2) time the reference CPU path as bench.py's reference arm.
//
// The per-layer activations/gradients of Net are private (model.hpp:174-185,
// :588).  As SURVEY §8(c) describes, only model.hpp (and data.hpp, for the
// iterator's private order_) is wrapped in `#define private public`, after every
// standard header has been included, so the reference sources stay untouched.
#include <algorithm>
#include <array>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <optional>
#include <set>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "parasgd/batch.hpp"
#include "parasgd/net_spec.hpp"
#include "parasgd/rng.hpp"
#include "parasgd/tensor.hpp"
#include "parasgd/threadpool.hpp"
#include "parasgd/weights.hpp"
#define private public
#include "parasgd/data.hpp"
#include "parasgd/model.hpp"
#undef private
#include "parasgd/schemes.hpp"
#include "parasgd/analysis.hpp"
#include "parasgd/csv.hpp"

#include "oracle.h"

using namespace parasgd;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PSG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PSG_EINVAL;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return PSG_ELOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PSG_ERUNTIME;
  }
}

NetSpec to_spec(const psg_layer_desc* layers, int n) {
  NetSpec spec;
  auto in = [&](int li, int i) { return std::string(layers[layers[li].inputs[i]].name); };
  for (int li = 0; li < n; ++li) {
    const psg_layer_desc& d = layers[li];
    switch (d.kind) {
      case PSG_LAYER_DATA:
        spec.layers.push_back(data_layer(d.name, static_cast<std::size_t>(d.batch),
                                         static_cast<std::size_t>(d.channels),
                                         static_cast<std::size_t>(d.height),
                                         static_cast<std::size_t>(d.width)));
        break;
      case PSG_LAYER_LABEL:
        spec.layers.push_back(label_layer(d.name, static_cast<std::size_t>(d.batch)));
        break;
      case PSG_LAYER_CONV:
        if (d.pad_h || d.pad_w || d.stride_h != 1 || d.stride_w != 1 || d.group != 1)
          throw std::invalid_argument("reference: conv supports valid, stride 1, group 1 only");
        spec.layers.push_back(conv_layer(d.name, in(li, 0), d.kernel_h, d.kernel_w, d.num_output));
        break;
      case PSG_LAYER_POOL:
        if (d.pool != PSG_POOL_MAX || d.ceil_mode || d.pad_h || d.pad_w)
          throw std::invalid_argument("reference: pool supports max, floor mode, no pad only");
        spec.layers.push_back(
            pool_layer(d.name, in(li, 0), d.kernel_h, d.kernel_w, d.stride_h, d.stride_w));
        break;
      case PSG_LAYER_LINEAR:
        spec.layers.push_back(linear_layer(d.name, in(li, 0), d.num_output));
        break;
      case PSG_LAYER_RELU:
        spec.layers.push_back(relu_layer(d.name, in(li, 0)));
        break;
      case PSG_LAYER_SOFTMAX_LOSS:
        spec.layers.push_back(softmax_loss_layer(d.name, in(li, 0), in(li, 1)));
        break;
      default:
        throw std::invalid_argument("reference: layer kind not expressible");
    }
  }
  spec.validate();
  return spec;
}

std::vector<double> flatten(const WeightCollection& w) {
  std::vector<double> out;
  for (const auto& e : w)
    for (const NDArray& t : e.second) out.insert(out.end(), t.values().begin(), t.values().end());
  return out;
}

WeightCollection unflatten(const WeightCollection& like, const double* flat) {
  WeightCollection out;
  std::size_t pos = 0;
  for (const auto& e : like) {
    std::vector<NDArray> ts;
    for (const NDArray& t : e.second) {
      std::vector<double> v(flat + pos, flat + pos + t.size());
      pos += t.size();
      ts.emplace_back(t.shape(), std::move(v));
    }
    out.add(e.first, std::move(ts));
  }
  return out;
}

Batch make_batch(const Net& net, const double* images, const int32_t* labels, std::size_t n) {
  const LayerSpec& d = net.spec().data_spec();
  const std::size_t vol = d.shape[1] * d.shape[2] * d.shape[3];
  std::vector<double> v(images, images + n * vol);
  return Batch{NDArray({n, d.shape[1], d.shape[2], d.shape[3]}, std::move(v)),
               std::vector<int>(labels, labels + n)};
}

Dataset make_dataset(const double* images, const int32_t* labels, std::size_t n, int c, int h,
                     int w, int classes) {
  const std::size_t vol = static_cast<std::size_t>(c) * h * w;
  Dataset ds{NDArray({n, static_cast<std::size_t>(c), static_cast<std::size_t>(h),
                      static_cast<std::size_t>(w)},
                     std::vector<double>(images, images + n * vol)),
             std::vector<int>(labels, labels + n), classes};
  ds.validate();
  return ds;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_net_create(const psg_layer_desc* layers, int n, uint64_t seed) {
  Net* out = nullptr;
  if (guarded([&] { out = new Net(to_spec(layers, n), seed); })) return nullptr;
  return out;
}

void ref_net_destroy(void* net) { delete static_cast<Net*>(net); }

size_t ref_net_param_count(void* net) {
  return flatten(static_cast<Net*>(net)->get_weights()).size();
}

int ref_net_set_sgd(void* net, double lr, double momentum) {
  return guarded([&] { static_cast<Net*>(net)->set_sgd({lr, momentum}); });
}

void ref_net_get_weights(void* net, double* flat) {
  const std::vector<double> v = flatten(static_cast<Net*>(net)->get_weights());
  std::copy(v.begin(), v.end(), flat);
}

int ref_net_set_weights(void* net, const double* flat) {
  Net* n = static_cast<Net*>(net);
  return guarded([&] { n->set_weights(unflatten(n->get_weights(), flat)); });
}

int ref_net_forward(void* net, const double* images, const int32_t* labels, size_t n,
                    double* loss, double* probs) {
  Net* nn = static_cast<Net*>(net);
  return guarded([&] {
    const ForwardResult r = nn->forward(make_batch(*nn, images, labels, n));
    if (loss) *loss = r.loss;
    if (probs) std::copy(r.probabilities.values().begin(), r.probabilities.values().end(), probs);
  });
}

int ref_net_backward(void* net, const double* images, const int32_t* labels, size_t n,
                     double* loss, double* grads) {
  Net* nn = static_cast<Net*>(net);
  return guarded([&] {
    const WeightCollection g = nn->backward(make_batch(*nn, images, labels, n));
    const std::vector<double> v = flatten(g);
    std::copy(v.begin(), v.end(), grads);
    if (loss) *loss = nn->last_loss_;
  });
}

int ref_net_apply_update(void* net, const double* grads) {
  Net* nn = static_cast<Net*>(net);
  return guarded([&] { nn->apply_update(unflatten(nn->get_weights(), grads)); });
}

// Per-layer out / grad of the last forward/backward (private state).
size_t ref_net_layer_size(void* net, int layer) {
  return static_cast<Net*>(net)->layers_.at(static_cast<std::size_t>(layer)).out.size();
}
int ref_net_layer_out(void* net, int layer, double* out) {
  return guarded([&] {
    const NDArray& t = static_cast<Net*>(net)->layers_.at(static_cast<std::size_t>(layer)).out;
    std::copy(t.values().begin(), t.values().end(), out);
  });
}
int ref_net_layer_grad(void* net, int layer, double* out) {
  return guarded([&] {
    const NDArray& t = static_cast<Net*>(net)->layers_.at(static_cast<std::size_t>(layer)).grad;
    std::copy(t.values().begin(), t.values().end(), out);
  });
}

int ref_shard(size_t n, int workers, uint64_t seed, uint64_t* perm, uint64_t* offsets) {
  return guarded([&] {
    std::vector<double> img(n, 0.0);
    std::vector<int32_t> lab(n, 0);
    const Dataset ds = make_dataset(img.data(), lab.data(), n, 1, 1, 1, 1);
    const std::vector<Shard> s = shard(ds, workers, seed);
    std::size_t pos = 0;
    offsets[0] = 0;
    for (std::size_t k = 0; k < s.size(); ++k) {
      for (std::size_t i : s[k].indices) perm[pos++] = i;
      offsets[k + 1] = pos;
    }
  });
}

// Indices emitted by worker k's ShardBatchIterator over `steps` next() calls:
// a dataset whose row i holds the value i makes next() reveal its indices.
int ref_worker_indices(size_t n, int workers, int k, size_t batch, uint64_t seed, long steps,
                       uint64_t* out) {
  return guarded([&] {
    std::vector<double> img(n);
    std::vector<int32_t> lab(n, 0);
    for (std::size_t i = 0; i < n; ++i) img[i] = static_cast<double>(i);
    const Dataset ds = make_dataset(img.data(), lab.data(), n, 1, 1, 1, 1);
    const std::vector<Shard> s = shard(ds, workers, seed);
    auto it = make_worker_iterator(s, k, batch, seed);
    for (long t = 0; t < steps; ++t) {
      const Batch b = it->next();
      for (std::size_t i = 0; i < batch; ++i)
        out[static_cast<std::size_t>(t) * batch + i] = static_cast<uint64_t>(b.images[i]);
    }
  });
}

void ref_generate_synthetic(int classes, size_t c, size_t h, size_t w, size_t per_class,
                            double separation, uint64_t seed, uint64_t variant, double* images,
                            int32_t* labels) {
  const Dataset ds = generate_synthetic(classes, c, h, w, per_class, separation, seed, variant);
  std::copy(ds.images.values().begin(), ds.images.values().end(), images);
  std::copy(ds.labels.begin(), ds.labels.end(), labels);
}

void ref_weights_mean(const double* const* items, int k, size_t n, double* out) {
  std::vector<WeightCollection> cols;
  for (int j = 0; j < k; ++j) {
    WeightCollection w;
    w.add("t", {NDArray({n}, std::vector<double>(items[j], items[j] + n))});
    cols.push_back(std::move(w));
  }
  const WeightCollection m = weights_mean(cols);
  const NDArray& t = m.entry(0).second[0];
  std::copy(t.values().begin(), t.values().end(), out);
}

uint64_t ref_net_digest(void* net) { return static_cast<Net*>(net)->get_weights().digest(); }

// run_sparknet (schemes.hpp:274-351) on the reference's own ThreadPool.
long ref_run_sparknet(const orc_sparknet_args* a, orc_record* records, long max_records,
                      uint64_t* warm_digest, double* round_weights) {
  long nrec = -1;
  guarded([&] {
    const NetSpec spec = to_spec(a->layers, a->n_layers);
    Net probe(spec, a->seed);
    const int classes = probe.num_classes();
    const Dataset train = make_dataset(a->train_images, a->train_labels, a->train_n, a->c, a->h,
                                       a->w, classes);
    const Dataset eval =
        make_dataset(a->eval_images, a->eval_labels, a->eval_n, a->c, a->h, a->w, classes);
    SchemeContext ctx;
    ctx.net = spec;
    ctx.train_data = &train;
    ctx.eval_data = &eval;
    ctx.batch = a->batch;
    ctx.sgd = {a->lr, a->momentum};
    ctx.seed = a->seed;
    ctx.cost = {a->compute_seconds, a->sync_seconds, 1.0};
    ctx.target_accuracy = a->target_accuracy;
    ctx.eval_steps = a->eval_steps;
    SchemeObserver obs;
    long round_idx = 0;
    std::size_t P = 0;
    obs.on_round = [&](long, const WeightCollection& w) {
      if (round_weights) {
        const std::vector<double> v = flatten(w);
        P = v.size();
        std::copy(v.begin(), v.end(), round_weights + static_cast<std::size_t>(round_idx) * P);
      }
      ++round_idx;
    };
    const RunTrace t =
        run_sparknet(ctx, a->workers, a->tau, a->rounds, a->warm, a->threads, &obs);
    if (warm_digest) *warm_digest = t.warm_digest;
    for (std::size_t i = 0; i < t.records.size() && static_cast<long>(i) < max_records; ++i) {
      records[i].serial_iters = t.records[i].serial_iters;
      records[i].parallel_iters = t.records[i].parallel_iters;
      records[i].rounds = t.records[i].rounds;
      records[i].sim_time = t.records[i].sim_time;
      records[i].accuracy = t.records[i].accuracy;
    }
    nrec = static_cast<long>(t.records.size());
  });
  return nrec;
}

long ref_run_naive(const orc_sparknet_args* a, long iter_budget, long eval_every,
                   orc_record* records, long max_records, double* step_weights) {
  long nrec = -1;
  guarded([&] {
    const NetSpec spec = to_spec(a->layers, a->n_layers);
    Net probe(spec, a->seed);
    const int classes = probe.num_classes();
    const Dataset train = make_dataset(a->train_images, a->train_labels, a->train_n, a->c, a->h,
                                       a->w, classes);
    const Dataset eval =
        make_dataset(a->eval_images, a->eval_labels, a->eval_n, a->c, a->h, a->w, classes);
    SchemeContext ctx;
    ctx.net = spec;
    ctx.train_data = &train;
    ctx.eval_data = &eval;
    ctx.batch = a->batch;
    ctx.sgd = {a->lr, a->momentum};
    ctx.seed = a->seed;
    ctx.cost = {a->compute_seconds, a->sync_seconds,
                a->sublinearity > 0.0 ? a->sublinearity : 1.0};
    ctx.target_accuracy = a->target_accuracy;
    ctx.eval_steps = a->eval_steps;
    SchemeObserver obs;
    obs.on_step = [&](long it, const Net& net) {
      if (step_weights) {
        const std::vector<double> v = flatten(net.get_weights());
        std::copy(v.begin(), v.end(), step_weights + static_cast<std::size_t>(it - 1) * v.size());
      }
    };
    const RunTrace t = run_naive(ctx, a->workers, iter_budget, eval_every, &obs);
    for (std::size_t i = 0; i < t.records.size() && static_cast<long>(i) < max_records; ++i) {
      records[i].serial_iters = t.records[i].serial_iters;
      records[i].parallel_iters = t.records[i].parallel_iters;
      records[i].rounds = t.records[i].rounds;
      records[i].sim_time = t.records[i].sim_time;
      records[i].accuracy = t.records[i].accuracy;
    }
    nrec = static_cast<long>(t.records.size());
  });
  return nrec;
}

// csv::format_double (csv.hpp:22-33) for the CSV-schema pins.
int ref_format_double(double v, char* out, int cap) {
  const std::string s = csv::format_double(v);
  if (static_cast<int>(s.size()) + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

// The analysis.hpp closed forms.
double ref_naive_speedup(double c, int k, double s) { return naive_speedup(c, k, s); }
double ref_sparknet_speedup(double n, double c, double tau, double s, double m) {
  return sparknet_speedup(n, c, tau, s, m);
}

}  // extern "C"
