// parasgd_b200/model.hpp — drop-in replacement for parasgd/model.hpp (the reference's
// class Net, /root/reference/proj/include/parasgd/model.hpp:50-597) running on a B200
// through the C ABI in psg.h.
//
// Same declarations: Net(NetSpec, seed), set_sgd, set_training_data / set_validation_data,
// forward, backward, apply_update, train, test, get_weights / set_weights, num_classes,
// spec, sgd; same exception types.  The reference's value types (NDArray, NetSpec, Batch,
// BatchIterator, WeightCollection) are used as-is: include this header INSTEAD of
// parasgd/model.hpp.  Additive extensions: Net(spec, seed, device), set_precision,
// set_training_shard (HBM-resident shard stream), SparkNet-style camelCase aliases and the
// scalar_divide / average helpers.
#pragma once

#include <psg.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "parasgd/batch.hpp"
#include "parasgd/data.hpp"
#include "parasgd/net_spec.hpp"
#include "parasgd/tensor.hpp"
#include "parasgd/weights.hpp"

namespace parasgd {

struct ForwardResult {  // model.hpp:18-21
  double loss = 0.0;
  NDArray probabilities;
};

struct SgdOptions {  // model.hpp:23-26
  double learning_rate = 0.01;
  double momentum = 0.0;
};

namespace b200 {

// Status code -> the reference's exception types.
inline void check(int rc) {
  if (rc == PSG_OK) return;
  const std::string msg = psg_last_error();
  switch (rc) {
    case PSG_EINVAL:
      throw std::invalid_argument(msg);
    case PSG_ELOGIC:
      throw std::logic_error(msg);
    default:
      throw std::runtime_error(msg);
  }
}

// One context (device + stream) per device, process-wide.
inline psg_ctx* context(int device) {
  static std::vector<psg_ctx*> ctxs(64, nullptr);
  if (device < 0 || device >= 64) throw std::invalid_argument("device index out of range");
  if (!ctxs[device]) check(psg_ctx_create(device, &ctxs[device]));
  return ctxs[device];
}

inline int default_device() {
  const char* e = std::getenv("PARASGD_DEVICE");
  return e ? std::atoi(e) : 0;
}

// NetSpec (net_spec.hpp:28-38) -> psg_layer_desc[] (reference defaults: stride 1, no pad).
inline std::vector<psg_layer_desc> to_desc(const NetSpec& spec) {
  std::vector<psg_layer_desc> out(spec.layers.size());
  auto index_of = [&](const std::string& n) {
    for (std::size_t i = 0; i < spec.layers.size(); ++i)
      if (spec.layers[i].name == n) return static_cast<int>(i);
    throw std::invalid_argument("net: unknown layer '" + n + "'");
  };
  for (std::size_t i = 0; i < spec.layers.size(); ++i) {
    const LayerSpec& l = spec.layers[i];
    psg_layer_desc& d = out[i];
    int kind = PSG_LAYER_DATA;
    switch (l.kind) {
      case LayerKind::Data: kind = PSG_LAYER_DATA; break;
      case LayerKind::Label: kind = PSG_LAYER_LABEL; break;
      case LayerKind::Conv: kind = PSG_LAYER_CONV; break;
      case LayerKind::Pool: kind = PSG_LAYER_POOL; break;
      case LayerKind::Linear: kind = PSG_LAYER_LINEAR; break;
      case LayerKind::Activation: kind = PSG_LAYER_RELU; break;
      case LayerKind::SoftmaxWithLoss: kind = PSG_LAYER_SOFTMAX_LOSS; break;
    }
    psg_layer_desc_init(&d, kind, l.name.c_str());
    if (l.name.size() >= sizeof(d.name)) throw std::invalid_argument("net: layer name too long");
    d.n_inputs = static_cast<int>(l.inputs.size());
    for (std::size_t j = 0; j < l.inputs.size(); ++j) d.inputs[j] = index_of(l.inputs[j]);
    if (l.kind == LayerKind::Data) {
      d.batch = static_cast<int>(l.shape[0]);
      d.channels = static_cast<int>(l.shape[1]);
      d.height = static_cast<int>(l.shape[2]);
      d.width = static_cast<int>(l.shape[3]);
    } else if (l.kind == LayerKind::Label) {
      d.batch = static_cast<int>(l.shape[0]);
    }
    d.num_output = l.kind == LayerKind::Conv ? l.num_filters : l.num_outputs;
    d.kernel_h = l.kernel_h;
    d.kernel_w = l.kernel_w;
    if (l.kind == LayerKind::Pool) {
      d.stride_h = l.stride_h;
      d.stride_w = l.stride_w;
    }
  }
  return out;
}

// Page-locked fp32 staging for host-fed steps.
struct Pinned {
  float* p = nullptr;
  std::size_t n = 0;
  Pinned() = default;
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  // moves transfer ownership of the pinned block (Net is movable, model.hpp /
  // schemes.hpp:141-147 return it by value)
  Pinned(Pinned&& o) noexcept : p(std::exchange(o.p, nullptr)), n(std::exchange(o.n, 0)) {}
  Pinned& operator=(Pinned&& o) noexcept {
    if (this != &o) {
      if (p) psg_host_free(p);
      p = std::exchange(o.p, nullptr);
      n = std::exchange(o.n, 0);
    }
    return *this;
  }
  void ensure(std::size_t want) {
    if (want <= n) return;
    if (p) psg_host_free(p);
    void* q = nullptr;
    check(psg_host_alloc(want * sizeof(float), &q));
    p = static_cast<float*>(q);
    n = want;
  }
  ~Pinned() {
    if (p) psg_host_free(p);
  }
};

}  // namespace b200

/// class Net (model.hpp:50) on a B200.  One Net = one device context; confined to one
/// host thread at a time (model.hpp:48-49).
class Net {
 public:
  Net(NetSpec spec, std::uint64_t seed) : Net(std::move(spec), seed, b200::default_device()) {}

  Net(NetSpec spec, std::uint64_t seed, int device) : spec_(std::move(spec)), device_(device) {
    spec_.validate();
    create(b200::to_desc(spec_), seed);
  }

  /// Extension: a graph of psg_layer_desc (Caffe layers the reference's NetSpec cannot
  /// express — parasgd_b200/presets.hpp: cifar10_quick, AlexNet, GoogLeNet).  spec() is
  /// then the empty NetSpec; layer names come from the descriptors.
  Net(std::vector<psg_layer_desc> layers, std::uint64_t seed, int device) : device_(device) {
    create(std::move(layers), seed);
  }

  Net(Net&&) noexcept = default;
  Net& operator=(Net&&) noexcept = default;

  const NetSpec& spec() const noexcept { return spec_; }
  int num_classes() const noexcept { return num_classes_; }
  const SgdOptions& sgd() const noexcept { return sgd_; }
  int device() const noexcept { return device_; }

  void set_sgd(SgdOptions opts) {  // model.hpp:60-66
    if (!(opts.learning_rate > 0.0)) throw std::invalid_argument("sgd: learning rate must be > 0");
    if (opts.momentum < 0.0 || opts.momentum >= 1.0)
      throw std::invalid_argument("sgd: momentum must be in [0,1)");
    b200::check(psg_net_set_sgd(net_.get(), opts.learning_rate, opts.momentum, weight_decay_));
    sgd_ = opts;
  }

  /// Extension: L2 weight decay (v = mu v + g + wd w; 0 = the reference's update), scaled
  /// per tensor by the layers' decay_mult.
  void set_weight_decay(double wd) {
    if (!(wd >= 0.0)) throw std::invalid_argument("sgd: weight decay must be >= 0");
    b200::check(psg_net_set_sgd(net_.get(), sgd_.learning_rate, sgd_.momentum, wd));
    weight_decay_ = wd;
  }
  double weight_decay() const noexcept { return weight_decay_; }

  /// Extension: fp32 SIMT (strict, default) or TF32 tensor cores.
  void set_precision(bool tf32) {
    b200::check(psg_net_set_precision(net_.get(), tf32 ? PSG_PRECISION_TF32 : PSG_PRECISION_FP32));
  }

  void set_training_data(std::shared_ptr<BatchIterator> it) {  // model.hpp:68
    train_data_ = std::move(it);
    shard_stream_ = false;
  }
  void set_validation_data(std::shared_ptr<BatchIterator> it) { val_data_ = std::move(it); }

  /// Extension: the training stream of make_worker_iterator(shards, k, batch, seed) with the
  /// shard resident in HBM (pixels never return to the host).  `dataset` must outlive it.
  void set_training_shard(const Shard& shard, std::size_t batch_size, std::uint64_t stream_seed) {
    psg_dataset* ds = upload(*shard.dataset);
    std::vector<std::uint64_t> idx(shard.indices.begin(), shard.indices.end());
    b200::check(psg_net_attach_shard(net_.get(), ds, idx.data(), idx.size(), batch_size,
                                     stream_seed));
    shard_stream_ = true;
    train_data_.reset();
  }

  ForwardResult forward(const Batch& batch) {  // model.hpp:74-78
    check_batch(batch);
    const std::size_t n = batch.size();
    ForwardResult r;
    r.probabilities = NDArray({n, static_cast<std::size_t>(num_classes_)}, 0.0);
    b200::check(psg_net_forward(net_.get(), batch.images.data(), batch.labels.data(), n, &r.loss,
                                r.probabilities.data()));
    return r;
  }

  WeightCollection backward(const Batch& batch) {  // model.hpp:83-86
    check_batch(batch);
    std::vector<double> g(P_);
    double loss = 0.0;
    b200::check(psg_net_backward(net_.get(), batch.images.data(), batch.labels.data(),
                                 batch.size(), &loss, g.data()));
    return unflatten(g.data());
  }

  void apply_update(const WeightCollection& grads) {  // model.hpp:90-107
    const std::vector<double> g = flatten(grads, "apply_update: gradient structure mismatch at ");
    b200::check(psg_net_apply_update(net_.get(), g.data(), g.size()));
  }

  /// model.hpp:111-118.  HBM-resident shard stream: one CUDA-graph replay per step; any
  /// other BatchIterator: its host batches are fed through page-locked staging.
  void train(long num_steps) {
    if (num_steps < 0) throw std::invalid_argument("train: negative step count");
    if (num_steps == 0) return;
    if (shard_stream_) {
      b200::check(psg_net_train(net_.get(), num_steps));
      b200::check(psg_net_sync(net_.get()));
      return;
    }
    if (!train_data_) throw std::runtime_error("train: no training data attached");
    for (long s = 0; s < num_steps; ++s) {
      const Batch b = train_data_->next();
      check_batch(b);
      if (b.size() != data_shape_[0]) {
        apply_update(backward(b));  // off-spec batch size: explicit path
        continue;
      }
      staging_.ensure(b.images.size());
      for (std::size_t i = 0; i < b.images.size(); ++i)
        staging_.p[i] = static_cast<float>(b.images[i]);
      std::vector<int32_t> labels(b.labels.begin(), b.labels.end());
      b200::check(psg_net_train_host(net_.get(), staging_.p, labels.data(), 1, nullptr));
    }
  }

  double test(long num_steps) {  // model.hpp:122-136
    if (num_steps < 1) throw std::invalid_argument("test: step count must be >= 1");
    if (!val_data_) throw std::runtime_error("test: no validation data attached");
    long correct = 0, total = 0;
    for (long s = 0; s < num_steps; ++s) {
      const Batch batch = val_data_->next();
      const ForwardResult r = forward(batch);
      const std::vector<int> pred = argmax_rows(r.probabilities);
      for (std::size_t i = 0; i < batch.labels.size(); ++i)
        correct += pred[i] == batch.labels[i] ? 1 : 0;
      total += static_cast<long>(batch.labels.size());
    }
    return static_cast<double>(correct) / static_cast<double>(total);
  }

  WeightCollection get_weights() const {  // model.hpp:140-144
    std::vector<double> w(P_);
    b200::check(psg_net_get_weights_f64(net_.get(), w.data(), w.size()));
    return unflatten(w.data());
  }

  void set_weights(const WeightCollection& w) {  // model.hpp:148-171 (momentum untouched)
    if (w.size() != template_.size())
      throw std::invalid_argument("set_weights: expected " + std::to_string(template_.size()) +
                                  " entries, got " + std::to_string(w.size()));
    std::vector<double> flat(P_);
    std::size_t pos = 0;
    for (const auto& e : template_) {
      const std::vector<NDArray>* t = w.find(e.first);
      if (!t) throw std::invalid_argument("set_weights: missing layer key '" + e.first + "'");
      if (t->size() != e.second.size())
        throw std::invalid_argument("set_weights: tensor count mismatch at '" + e.first + "'");
      for (std::size_t i = 0; i < t->size(); ++i) {
        if (!(*t)[i].same_shape(e.second[i]))
          throw std::invalid_argument("set_weights: shape mismatch at '" + e.first + "'");
        std::memcpy(flat.data() + pos, (*t)[i].data(), (*t)[i].size() * sizeof(double));
        pos += (*t)[i].size();
      }
    }
    b200::check(psg_net_set_weights_f64(net_.get(), flat.data(), flat.size()));
  }

  // SparkNet (Scala) spellings
  void setTrainingData(std::shared_ptr<BatchIterator> it) { set_training_data(std::move(it)); }
  void setValidationData(std::shared_ptr<BatchIterator> it) { set_validation_data(std::move(it)); }
  WeightCollection getWeights() const { return get_weights(); }
  void setWeights(const WeightCollection& w) { set_weights(w); }

  psg_net* handle() const noexcept { return net_.get(); }

  /// Extension: (epoch, cursor) of the HBM-resident shard stream, so two nets can share
  /// one ShardBatchIterator (the warm-start master consumes worker 0's, schemes.hpp:314).
  std::pair<std::uint64_t, std::uint64_t> stream_position() const {
    std::uint64_t e = 0, c = 0;
    b200::check(psg_net_get_stream_position(net_.get(), &e, &c));
    return {e, c};
  }
  void set_stream_position(std::pair<std::uint64_t, std::uint64_t> pos) {
    b200::check(psg_net_set_stream_position(net_.get(), pos.first, pos.second));
  }

  /// Extension: accuracy over `num_steps` batches of a fresh SequentialBatchIterator on an
  /// HBM-resident copy of `ds` (schemes.hpp:134-139 evaluate, gather on device).
  /// Extension (run_naive, schemes.hpp:233-247): this net consumes rows
  /// [part*b/parts, (part+1)*b/parts) of every batch of the shard stream.
  void set_training_part(const Shard& shard, std::size_t batch_size, std::uint64_t stream_seed,
                         int part, int parts) {
    psg_dataset* ds = upload(*shard.dataset);
    std::vector<std::uint64_t> idx(shard.indices.begin(), shard.indices.end());
    b200::check(psg_net_attach_shard_part(net_.get(), ds, idx.data(), idx.size(), batch_size,
                                          stream_seed, part, parts));
  }

  /// Extension: queue sharded evaluation batches first, first+stride, ... < num_steps of a
  /// fresh SequentialBatchIterator; test_shard_end returns (correct, total).
  void test_shard_begin(const Dataset& ds, std::size_t batch, long num_steps, long first,
                        long stride) {
    b200::check(psg_net_attach_validation(net_.get(), upload(ds), batch));
    b200::check(psg_net_test_begin(net_.get(), num_steps, first, stride));
  }
  std::pair<unsigned long long, unsigned long long> test_shard_end() {
    unsigned long long c = 0, t = 0;
    b200::check(psg_net_test_end(net_.get(), &c, &t));
    return {c, t};
  }

  double test_resident(const Dataset& ds, std::size_t batch, long num_steps) {
    b200::check(psg_net_attach_validation(net_.get(), upload(ds), batch));
    double acc = 0.0;
    b200::check(psg_net_test(net_.get(), num_steps, &acc));
    return acc;
  }

 private:
  struct NetDel {
    void operator()(psg_net* n) const { psg_net_destroy(n); }
  };
  struct DsDel {
    void operator()(psg_dataset* d) const { psg_dataset_destroy(d); }
  };

  void create(std::vector<psg_layer_desc> layers, std::uint64_t seed) {
    desc_ = std::move(layers);
    psg_net* h = nullptr;
    b200::check(psg_net_create(b200::context(device_), desc_.data(),
                               static_cast<int>(desc_.size()), seed, &h));
    net_.reset(h);
    for (const psg_layer_desc& d : desc_)
      if (d.kind == PSG_LAYER_DATA)
        data_shape_ = {static_cast<std::size_t>(d.batch), static_cast<std::size_t>(d.channels),
                       static_cast<std::size_t>(d.height), static_cast<std::size_t>(d.width)};
    b200::check(psg_net_num_classes(net_.get(), &num_classes_));
    b200::check(psg_net_param_count(net_.get(), &P_));
    template_ = structure();
  }

  WeightCollection structure() const {
    int nt = 0;
    b200::check(psg_net_num_tensors(net_.get(), &nt));
    std::vector<std::vector<NDArray>> per(desc_.size());
    for (int t = 0; t < nt; ++t) {
      int layer = 0, slot = 0, rank = 0;
      int64_t shape[4];
      std::size_t off = 0;
      b200::check(psg_net_tensor_info(net_.get(), t, &layer, &slot, &rank, shape, &off));
      std::vector<std::size_t> shp(shape, shape + rank);
      per[static_cast<std::size_t>(layer)].emplace_back(shp, 0.0);
    }
    WeightCollection w;
    for (std::size_t i = 0; i < desc_.size(); ++i) w.add(desc_[i].name, per[i]);
    return w;
  }

  WeightCollection unflatten(const double* flat) const {
    WeightCollection out;
    std::size_t pos = 0;
    for (const auto& e : template_) {
      std::vector<NDArray> ts;
      for (const NDArray& t : e.second) {
        ts.emplace_back(t.shape(), std::vector<double>(flat + pos, flat + pos + t.size()));
        pos += t.size();
      }
      out.add(e.first, std::move(ts));
    }
    return out;
  }

  std::vector<double> flatten(const WeightCollection& w, const char* what) const {
    if (w.size() != template_.size()) throw std::invalid_argument(std::string(what) + "size");
    std::vector<double> flat;
    flat.reserve(P_);
    for (std::size_t e = 0; e < template_.size(); ++e) {
      const auto& want = template_.entry(e);
      const auto& got = w.entry(e);
      if (got.first != want.first || got.second.size() != want.second.size())
        throw std::invalid_argument(std::string(what) + "'" + want.first + "'");
      for (std::size_t t = 0; t < got.second.size(); ++t) {
        if (!got.second[t].same_shape(want.second[t]))
          throw std::invalid_argument(std::string(what) + "'" + want.first + "'");
        flat.insert(flat.end(), got.second[t].values().begin(), got.second[t].values().end());
      }
    }
    return flat;
  }

  void check_batch(const Batch& batch) const {  // model.hpp:287-299
    if (batch.images.rank() != 4) throw std::invalid_argument("forward: images must be [n,c,h,w]");
    const std::size_t n = batch.images.extent(0);
    if (n < 1 || batch.labels.size() != n)
      throw std::invalid_argument("forward: label count does not match batch");
    const auto& d = data_shape_;
    for (int a = 0; a < 3; ++a)
      if (batch.images.extent(a + 1) != d[a + 1])
        throw std::invalid_argument("forward: batch extents do not match the data layer");
    for (int y : batch.labels)
      if (y < 0 || y >= num_classes_) throw std::invalid_argument("forward: label out of range");
  }

  psg_dataset* upload(const Dataset& ds) {
    for (auto& u : uploads_)
      if (u.first == &ds) return u.second.get();
    psg_dataset* h = nullptr;
    std::vector<int32_t> lab(ds.labels.begin(), ds.labels.end());
    b200::check(psg_dataset_upload_f64(b200::context(device_), ds.images.data(), lab.data(),
                                       ds.size(), static_cast<int>(ds.channels()),
                                       static_cast<int>(ds.height()),
                                       static_cast<int>(ds.width()), ds.num_classes, &h));
    uploads_.emplace_back(&ds, std::unique_ptr<psg_dataset, DsDel>(h));
    return h;
  }

  NetSpec spec_;
  std::vector<psg_layer_desc> desc_;
  std::vector<std::size_t> data_shape_ = {0, 0, 0, 0};
  double weight_decay_ = 0.0;
  int device_ = 0;
  std::unique_ptr<psg_net, NetDel> net_;
  int num_classes_ = 0;
  std::size_t P_ = 0;
  WeightCollection template_;
  SgdOptions sgd_;
  std::shared_ptr<BatchIterator> train_data_, val_data_;
  bool shard_stream_ = false;
  std::vector<std::pair<const Dataset*, std::unique_ptr<psg_dataset, DsDel>>> uploads_;
  b200::Pinned staging_;
};

/// SparkNet's WeightCollection.scalarDivide: every tensor / k (true division, as the
/// reference's mean_collection, tensor.hpp:175-176).
inline WeightCollection scalar_divide(const WeightCollection& w, double k) {
  WeightCollection out;
  for (const auto& e : w) {
    std::vector<NDArray> ts;
    for (const NDArray& t : e.second) {
      NDArray q = t;
      for (double& v : q.values()) v /= k;
      q.ensure_finite("scalar_divide");
      ts.push_back(std::move(q));
    }
    out.add(e.first, std::move(ts));
  }
  return out;
}

/// SparkNet's WeightCollection.average == weights_mean (weights.hpp:90-107).
inline WeightCollection average(const std::vector<WeightCollection>& items) {
  return weights_mean(items);
}

}  // namespace parasgd
