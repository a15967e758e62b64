// extern "C" boundary (include/psg.h): exceptions -> status codes, thread-local
// last error.  std::invalid_argument -> PSG_EINVAL, CudaError -> PSG_ECUDA,
// std::logic_error -> PSG_ELOGIC, everything else -> PSG_ERUNTIME
// (SURVEY §8(b) error conventions).
#include <cstring>
#include <string>

#include "runtime.h"

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PSG_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return PSG_EINVAL;
  } catch (const psg::CudaError& e) {
    g_last_error = e.what();
    return PSG_ECUDA;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return PSG_ELOGIC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PSG_ERUNTIME;
  } catch (...) {
    g_last_error = "unknown error";
    return PSG_ERUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null handle");
}

std::vector<float> nchw_to_nhwc(const double* src, const float* srcf, size_t n, int c, int h,
                                int w) {
  std::vector<float> out(n * static_cast<size_t>(c) * h * w);
  for (size_t b = 0; b < n; ++b)
    for (int ci = 0; ci < c; ++ci)
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
          const size_t s = ((b * c + ci) * h + y) * w + x;
          out[((b * h + y) * w + x) * c + ci] = src ? static_cast<float>(src[s]) : srcf[s];
        }
  return out;
}

psg_dataset* upload(psg_ctx* ctx, const double* imgd, const float* imgf, const int32_t* labels,
                    size_t n, int c, int h, int w, int classes) {
  need(ctx, "dataset");
  if (n < 1) throw std::invalid_argument("dataset: empty");
  if (c < 1 || h < 1 || w < 1) throw std::invalid_argument("dataset: images/labels mismatch");
  if (classes < 1) throw std::invalid_argument("dataset: no classes");
  for (size_t i = 0; i < n; ++i)
    if (labels[i] < 0 || labels[i] >= classes)
      throw std::invalid_argument("dataset: label out of range");
  const std::vector<float> nhwc = nchw_to_nhwc(imgd, imgf, n, c, h, w);
  psg::DeviceGuard dg(ctx->device);
  auto* ds = new psg_dataset;
  ds->ctx = ctx;
  ds->n = n;
  ds->c = c;
  ds->h = h;
  ds->w = w;
  ds->classes = classes;
  ds->host_labels.assign(labels, labels + n);
  try {
    PSG_CUDA(cudaMalloc(&ds->images, nhwc.size() * sizeof(float)));
    PSG_CUDA(cudaMalloc(&ds->labels, n * sizeof(int32_t)));
    // stream-ordered (pageable H2D cudaMemcpy may return before its DMA lands, and the
    // non-blocking net / ctx streams are not ordered after the legacy stream)
    PSG_CUDA(cudaMemcpyAsync(ds->images, nhwc.data(), nhwc.size() * sizeof(float),
                             cudaMemcpyHostToDevice, ctx->stream));
    PSG_CUDA(cudaMemcpyAsync(ds->labels, labels, n * sizeof(int32_t), cudaMemcpyHostToDevice,
                             ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaFree(ds->images);
    cudaFree(ds->labels);
    delete ds;
    throw;
  }
  return ds;
}

}  // namespace

extern "C" {

void psg_layer_desc_init(psg_layer_desc* d, int kind, const char* name) {
  std::memset(d, 0, sizeof(*d));
  d->kind = kind;
  if (name) std::strncpy(d->name, name, sizeof(d->name) - 1);
  d->stride_h = d->stride_w = 1;
  d->group = 1;
  d->pool = PSG_POOL_MAX;
  d->local_size = 5;
  d->alpha = 1e-4;
  d->beta = 0.75;
  d->k = 1.0;
  d->dropout_ratio = 0.5;
  d->loss_weight = 1.0;
  d->lr_mult_w = d->lr_mult_b = d->decay_mult_w = d->decay_mult_b = 1.0;
}

const char* psg_last_error(void) { return g_last_error.c_str(); }
int psg_abi_version(void) { return PSG_ABI_VERSION; }

int psg_device_count(int* n) {
  return guarded([&] {
    need(n, "device_count");
    PSG_CUDA(cudaGetDeviceCount(n));
  });
}

uint64_t psg_splitmix64(uint64_t x) { return psg::splitmix64(x); }
uint64_t psg_derive_seed(uint64_t base, const uint64_t* parts, int nparts) {
  return psg::derive_seed(base, parts, nparts);
}
int psg_shard(size_t n, int workers, uint64_t seed, uint64_t* perm, uint64_t* offsets) {
  return guarded([&] { psg::shard_perm(n, workers, seed, perm, offsets); });
}
uint64_t psg_worker_stream_seed(uint64_t global_seed, int worker_id) {
  return psg::worker_stream_seed(global_seed, worker_id);
}
int psg_epoch_order(const uint64_t* shard, size_t n, uint64_t stream_seed, uint64_t epoch,
                    uint64_t* order) {
  return guarded([&] { psg::epoch_order(shard, n, stream_seed, epoch, order); });
}
int psg_generate_synthetic(int classes, size_t c, size_t h, size_t w, size_t per_class,
                           double separation, uint64_t seed, uint64_t variant, double* images,
                           int32_t* labels) {
  return guarded([&] {
    psg::generate_synthetic(classes, c, h, w, per_class, separation, seed, variant, images,
                            labels);
  });
}

int psg_ctx_create(int device, psg_ctx** out) {
  return guarded([&] {
    need(out, "ctx_create");
    int count = 0;
    PSG_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw std::invalid_argument("ctx: bad device index");
    psg::DeviceGuard dg(device);
    auto* c = new psg_ctx;
    c->device = device;
    PSG_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    PSG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *out = c;
  });
}

int psg_ctx_destroy(psg_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    psg::DeviceGuard dg(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int psg_ctx_sync(psg_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx_sync");
    psg::DeviceGuard dg(ctx->device);
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int psg_dataset_upload_f64(psg_ctx* ctx, const double* images, const int32_t* labels, size_t n,
                           int c, int h, int w, int num_classes, psg_dataset** out) {
  return guarded([&] { *out = upload(ctx, images, nullptr, labels, n, c, h, w, num_classes); });
}

int psg_dataset_upload_f32(psg_ctx* ctx, const float* images, const int32_t* labels, size_t n,
                           int c, int h, int w, int num_classes, psg_dataset** out) {
  return guarded([&] { *out = upload(ctx, nullptr, images, labels, n, c, h, w, num_classes); });
}

int psg_dataset_synthetic(psg_ctx* ctx, int classes, int c, int h, int w, size_t per_class,
                          double separation, uint64_t seed, uint64_t variant, psg_dataset** out) {
  return guarded([&] {
    const size_t n = static_cast<size_t>(classes) * per_class;
    std::vector<double> img(n * static_cast<size_t>(c) * h * w);
    std::vector<int32_t> lab(n);
    psg::generate_synthetic(classes, c, h, w, per_class, separation, seed, variant, img.data(),
                            lab.data());
    *out = upload(ctx, img.data(), nullptr, lab.data(), n, c, h, w, classes);
  });
}

int psg_dataset_synthetic_device(psg_ctx* ctx, int classes, int c, int h, int w,
                                 size_t per_class, double separation, uint64_t seed,
                                 uint64_t variant, psg_dataset** out) {
  return guarded([&] {
    need(ctx, "dataset_synthetic_device");
    if (per_class < 1) throw std::invalid_argument("synthetic: need at least one example per class");
    if (c < 1 || h < 1 || w < 1) throw std::invalid_argument("dataset: images/labels mismatch");
    const size_t dim = static_cast<size_t>(c) * h * w, n = static_cast<size_t>(classes) * per_class;
    std::vector<double> means(dim * static_cast<size_t>(std::max(classes, 1)));
    psg::synthetic_means(classes, c, h, w, separation, seed, means.data());
    std::vector<float> meansf(means.begin(), means.end());
    psg::DeviceGuard dg(ctx->device);
    auto* ds = new psg_dataset;
    ds->ctx = ctx;
    ds->n = n;
    ds->c = c;
    ds->h = h;
    ds->w = w;
    ds->classes = classes;
    ds->host_labels.resize(n);
    for (size_t r = 0; r < n; ++r) ds->host_labels[r] = static_cast<int32_t>(r / per_class);
    float* d_means = nullptr;
    try {
      PSG_CUDA(cudaMalloc(&ds->images, n * dim * sizeof(float)));
      PSG_CUDA(cudaMalloc(&ds->labels, n * sizeof(int32_t)));
      PSG_CUDA(cudaMalloc(&d_means, meansf.size() * sizeof(float)));
      PSG_CUDA(cudaMemcpyAsync(d_means, meansf.data(), meansf.size() * sizeof(float),
                               cudaMemcpyHostToDevice, ctx->stream));
      psg::synthetic_rows_device(d_means, classes, c, h, w, per_class,
                                 psg::synthetic_noise_seed(seed, variant), ds->images, ds->labels,
                                 ctx->stream);
      PSG_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(d_means);
    } catch (...) {
      cudaFree(d_means);
      cudaFree(ds->images);
      cudaFree(ds->labels);
      delete ds;
      throw;
    }
    *out = ds;
  });
}

int psg_dataset_read_f32(const psg_dataset* ds, size_t first, size_t count, float* images_nchw,
                         int32_t* labels) {
  return guarded([&] {
    need(ds, "dataset_read");
    if (first + count > ds->n) throw std::invalid_argument("dataset_read: rows out of range");
    const size_t dim = static_cast<size_t>(ds->c) * ds->h * ds->w;
    std::vector<float> nhwc(count * dim);
    psg::DeviceGuard dg(ds->ctx->device);
    PSG_CUDA(cudaMemcpy(nhwc.data(), ds->images + first * dim, nhwc.size() * sizeof(float),
                        cudaMemcpyDeviceToHost));
    for (size_t r = 0; r < count; ++r)
      for (int ch = 0; ch < ds->c; ++ch)
        for (int p = 0; p < ds->h * ds->w; ++p)
          images_nchw[(r * ds->c + ch) * ds->h * ds->w + p] = nhwc[(r * ds->h * ds->w + p) * ds->c + ch];
    for (size_t r = 0; r < count; ++r) labels[r] = ds->host_labels[first + r];
  });
}

int psg_read_idx(const char* images_path, const char* labels_path, size_t* n, int* h, int* w,
                 int* num_classes, float* images, int32_t* labels) {
  return guarded([&] {
    if (!images_path || !labels_path) throw std::invalid_argument("idx: null path");
    const psg::IdxData d = psg::read_idx(images_path, labels_path);
    *n = d.n;
    *h = static_cast<int>(d.h);
    *w = static_cast<int>(d.w);
    *num_classes = d.classes;
    if (images)
      for (size_t i = 0; i < d.pixels.size(); ++i)
        images[i] = static_cast<float>(static_cast<double>(d.pixels[i]) / 255.0);
    if (labels) std::memcpy(labels, d.labels.data(), d.labels.size() * sizeof(int32_t));
  });
}

int psg_read_csv(const char* path, int c, int h, int w, int num_classes, size_t* n, float* images,
                 int32_t* labels) {
  return guarded([&] {
    if (!path) throw std::invalid_argument("csv: null path");
    if (c < 1 || h < 1 || w < 1) throw std::invalid_argument("csv: bad extents");
    const psg::CsvData d = psg::read_csv(path, c, h, w, num_classes);
    *n = d.labels.size();
    if (images) std::memcpy(images, d.images.data(), d.images.size() * sizeof(float));
    if (labels) std::memcpy(labels, d.labels.data(), d.labels.size() * sizeof(int32_t));
  });
}

int psg_dataset_load_idx(psg_ctx* ctx, const char* images_path, const char* labels_path,
                         psg_dataset** out) {
  return guarded([&] {
    need(ctx, "dataset_load_idx");
    if (!images_path || !labels_path) throw std::invalid_argument("idx: null path");
    const psg::IdxData d = psg::read_idx(images_path, labels_path);
    psg::DeviceGuard dg(ctx->device);
    auto* ds = new psg_dataset;
    ds->ctx = ctx;
    ds->n = d.n;
    ds->c = 1;
    ds->h = static_cast<int>(d.h);
    ds->w = static_cast<int>(d.w);
    ds->classes = d.classes;
    ds->host_labels = d.labels;
    unsigned char* d_px = nullptr;
    try {
      PSG_CUDA(cudaMalloc(&ds->images, d.pixels.size() * sizeof(float)));
      PSG_CUDA(cudaMalloc(&ds->labels, d.n * sizeof(int32_t)));
      PSG_CUDA(cudaMalloc(&d_px, d.pixels.size()));
      PSG_CUDA(cudaMemcpyAsync(d_px, d.pixels.data(), d.pixels.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
      PSG_CUDA(cudaMemcpyAsync(ds->labels, d.labels.data(), d.n * sizeof(int32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      psg::ingest_u8_to_f32(d_px, d.pixels.size(), ds->images, ctx->stream);
      PSG_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(d_px);
    } catch (...) {
      cudaFree(d_px);
      cudaFree(ds->images);
      cudaFree(ds->labels);
      delete ds;
      throw;
    }
    *out = ds;
  });
}

int psg_dataset_load_csv(psg_ctx* ctx, const char* path, int c, int h, int w, int num_classes,
                         psg_dataset** out) {
  return guarded([&] {
    need(ctx, "dataset_load_csv");
    if (!path) throw std::invalid_argument("csv: null path");
    const psg::CsvData d = psg::read_csv(path, c, h, w, num_classes);
    *out = upload(ctx, nullptr, d.images.data(), d.labels.data(), d.labels.size(), c, h, w,
                  num_classes);
  });
}

int psg_dataset_size(const psg_dataset* ds, size_t* n) {
  return guarded([&] {
    need(ds, "dataset_size");
    *n = ds->n;
  });
}

int psg_dataset_destroy(psg_dataset* ds) {
  return guarded([&] {
    if (!ds) return;
    psg::DeviceGuard dg(ds->ctx->device);
    cudaFree(ds->images);
    cudaFree(ds->labels);
    delete ds;
  });
}

int psg_net_create(psg_ctx* ctx, const psg_layer_desc* layers, int n_layers, uint64_t seed,
                   psg_net** out) {
  return guarded([&] {
    need(ctx, "net_create");
    need(layers, "net_create layers");
    auto* net = new psg_net;
    net->ctx = ctx;
    try {
      psg::net_build(net, layers, n_layers, seed);
    } catch (...) {
      psg::net_free(net);
      delete net;
      throw;
    }
    *out = net;
  });
}

int psg_net_destroy(psg_net* net) {
  return guarded([&] {
    if (!net) return;
    psg::net_free(net);
    delete net;
  });
}

int psg_net_num_classes(const psg_net* net, int* classes) {
  return guarded([&] {
    need(net, "num_classes");
    *classes = net->classes;
  });
}

int psg_net_param_count(const psg_net* net, size_t* n) {
  return guarded([&] {
    need(net, "param_count");
    *n = net->P_ref;
  });
}

int psg_net_num_tensors(const psg_net* net, int* n) {
  return guarded([&] {
    need(net, "num_tensors");
    *n = static_cast<int>(net->tensors.size());
  });
}

int psg_net_tensor_info(const psg_net* net, int t, int* layer, int* slot, int* rank,
                        int64_t shape[4], size_t* offset) {
  return guarded([&] {
    need(net, "tensor_info");
    if (t < 0 || t >= static_cast<int>(net->tensors.size()))
      throw std::invalid_argument("tensor index out of range");
    const psg::TensorRec& r = net->tensors[t];
    if (layer) *layer = r.layer;
    if (slot) *slot = r.slot;
    if (rank) *rank = r.rank;
    if (shape)
      for (int i = 0; i < 4; ++i) shape[i] = r.shape[i];
    if (offset) *offset = r.ref_off;
  });
}

int psg_net_set_precision(psg_net* net, int precision) {
  return guarded([&] {
    need(net, "set_precision");
    if (precision != PSG_PRECISION_FP32 && precision != PSG_PRECISION_TF32)
      throw std::invalid_argument("precision: unknown mode");
    const psg::Mode m = precision == PSG_PRECISION_TF32 ? psg::Mode::Tf32 : psg::Mode::Strict;
    if (m != net->mode) {
      psg::DeviceGuard dg(net->ctx->device);
      PSG_CUDA(cudaStreamSynchronize(net->stream));
      net->mode = m;
      psg::release_batch_buffers(net);  // TF32 may need im2col buffers; realloc on next use
    }
  });
}

int psg_net_set_sgd(psg_net* net, double lr, double momentum, double weight_decay) {
  return guarded([&] {
    need(net, "set_sgd");
    psg::net_set_sgd(net, lr, momentum, weight_decay);
  });
}

int psg_net_get_weights_f64(psg_net* net, double* flat, size_t n) {
  return guarded([&] {
    need(net, "get_weights");
    psg::net_get_weights(net, flat, n, false);
  });
}

int psg_net_set_weights_f64(psg_net* net, const double* flat, size_t n) {
  return guarded([&] {
    need(net, "set_weights");
    psg::net_set_weights(net, flat, n);
  });
}

int psg_net_get_velocity_f64(psg_net* net, double* flat, size_t n) {
  return guarded([&] {
    need(net, "get_velocity");
    psg::net_get_weights(net, flat, n, true);
  });
}

int psg_net_reset_velocity(psg_net* net) {
  return guarded([&] {
    need(net, "reset_velocity");
    psg::DeviceGuard dg(net->ctx->device);
    PSG_CUDA(cudaMemsetAsync(net->v, 0, net->P_alloc * sizeof(float), net->stream));
  });
}

int psg_net_forward(psg_net* net, const double* images, const int32_t* labels, size_t n,
                    double* loss, double* probs) {
  return guarded([&] {
    need(net, "forward");
    psg::net_forward_host(net, images, labels, n, loss, probs);
  });
}

int psg_net_backward(psg_net* net, const double* images, const int32_t* labels, size_t n,
                     double* loss, double* grads) {
  return guarded([&] {
    need(net, "backward");
    psg::net_backward_host(net, images, labels, n, loss, grads);
  });
}

int psg_net_apply_update(psg_net* net, const double* grads, size_t n) {
  return guarded([&] {
    need(net, "apply_update");
    psg::net_apply_update_host(net, grads, n);
  });
}

int psg_net_layer_shape(const psg_net* net, int layer, int64_t shape[4]) {
  return guarded([&] {
    need(net, "layer_shape");
    if (layer < 0 || layer >= static_cast<int>(net->L.size()))
      throw std::invalid_argument("layer index out of range");
    const psg::LayerRt& l = net->L[layer];
    shape[0] = static_cast<int64_t>(net->last_n);
    shape[1] = l.C;
    shape[2] = l.H;
    shape[3] = l.W;
  });
}

int psg_net_layer_output(psg_net* net, int layer, double* out, size_t n) {
  return guarded([&] {
    need(net, "layer_output");
    psg::net_layer_readback(net, layer, false, out, n);
  });
}

int psg_net_layer_grad(psg_net* net, int layer, double* out, size_t n) {
  return guarded([&] {
    need(net, "layer_grad");
    psg::net_layer_readback(net, layer, true, out, n);
  });
}

int psg_net_attach_shard(psg_net* net, psg_dataset* ds, const uint64_t* shard_indices,
                         size_t count, size_t batch, uint64_t stream_seed) {
  return guarded([&] {
    need(net, "attach_shard");
    need(ds, "attach_shard dataset");
    psg::net_attach_shard(net, ds, shard_indices, count, batch, stream_seed);
  });
}

int psg_net_attach_shard_part(psg_net* net, psg_dataset* ds, const uint64_t* shard_indices,
                              size_t count, size_t batch, uint64_t stream_seed, int part,
                              int parts) {
  return guarded([&] {
    need(net, "attach_shard_part");
    need(ds, "attach_shard_part dataset");
    psg::net_attach_shard(net, ds, shard_indices, count, batch, stream_seed, part, parts);
  });
}

int psg_net_grad_step(psg_net* net) {
  return guarded([&] {
    need(net, "grad_step");
    psg::net_grad_step(net);
  });
}

int psg_net_apply_grads(psg_net* net) {
  return guarded([&] {
    need(net, "apply_grads");
    psg::net_apply_grads(net);
  });
}

int psg_net_get_stream_position(const psg_net* net, uint64_t* epoch, uint64_t* cursor) {
  return guarded([&] {
    need(net, "get_stream_position");
    if (!net->train_ds) throw std::runtime_error("train: no training data attached");
    *epoch = net->it_epoch;
    *cursor = net->it_cursor;
  });
}

int psg_net_set_stream_position(psg_net* net, uint64_t epoch, uint64_t cursor) {
  return guarded([&] {
    need(net, "set_stream_position");
    if (!net->train_ds) throw std::runtime_error("train: no training data attached");
    if (cursor * net->it_batch > net->order.size())
      throw std::invalid_argument("stream position: cursor past the epoch");
    if (epoch != net->it_epoch) {
      net->it_epoch = epoch;
      psg::epoch_order(net->shard.data(), net->shard.size(), net->it_seed, epoch,
                       net->order.data());
    }
    net->it_cursor = cursor;
  });
}

int psg_net_train(psg_net* net, long steps) {
  return guarded([&] {
    need(net, "train");
    psg::net_train(net, steps);
  });
}

int psg_net_train_round(psg_net* net, long steps, psg_comm* comm) {
  return guarded([&] {
    need(net, "train_round");
    psg::net_train_round(net, steps, comm);
  });
}

int psg_net_sync(psg_net* net) {
  return guarded([&] {
    need(net, "sync");
    psg::net_check_flag(net);
  });
}

int psg_net_last_train_ms(psg_net* net, float* ms) {
  return guarded([&] {
    need(net, "last_train_ms");
    if (!net->timed) throw std::runtime_error("no timed train call");
    psg::DeviceGuard dg(net->ctx->device);
    PSG_CUDA(cudaEventSynchronize(net->t1));
    PSG_CUDA(cudaEventElapsedTime(ms, net->t0, net->t1));
  });
}

int psg_net_last_loss(psg_net* net, double* loss) {
  return guarded([&] {
    need(net, "last_loss");
    psg::DeviceGuard dg(net->ctx->device);
    PSG_CUDA(cudaStreamSynchronize(net->stream));
    PSG_CUDA(cudaMemcpy(loss, &net->dsc->loss, sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int psg_net_attach_validation(psg_net* net, psg_dataset* ds, size_t batch) {
  return guarded([&] {
    need(net, "attach_validation");
    need(ds, "attach_validation dataset");
    psg::net_attach_validation(net, ds, batch);
  });
}

int psg_net_test(psg_net* net, long steps, double* accuracy) {
  return guarded([&] {
    need(net, "test");
    *accuracy = psg::net_test(net, steps);
  });
}

int psg_net_test_begin(psg_net* net, long steps, long first, long stride) {
  return guarded([&] {
    need(net, "test_begin");
    psg::net_test_begin(net, steps, first, stride);
  });
}

int psg_net_test_end(psg_net* net, unsigned long long* correct, unsigned long long* total) {
  return guarded([&] {
    need(net, "test_end");
    psg::net_test_end(net, correct, total);
  });
}

int psg_net_set_fusion(psg_net* net, int on) {
  return guarded([&] {
    need(net, "set_fusion");
    if (net->fuse == (on != 0)) return;
    psg::release_batch_buffers(net);
    net->fuse = on != 0;
    psg::plan_fusion(net);
  });
}

int psg_net_set_tc_options(psg_net* net, int pair_policy) {
  return guarded([&] {
    need(net, "set_tc_options");
    if (pair_policy != PSG_TC_PAIR_AUTO && pair_policy != PSG_TC_PAIR_NEVER &&
        pair_policy != PSG_TC_PAIR_ALWAYS)
      throw std::invalid_argument("set_tc_options: unknown pair policy");
    // workspace sizes and the captured step graph depend on the policy: rebuild on next use
    psg::release_batch_buffers(net);
    for (psg::LayerRt& l : net->L) l.cg.tc_pair = pair_policy;
  });
}

int psg_debug_tc_prof(char* buf, size_t len, int reset) {
  return guarded([&] {
    const std::string r = psg::tc_prof_report(reset != 0);
    if (buf && len) {
      std::strncpy(buf, r.c_str(), len - 1);
      buf[len - 1] = 0;
    }
  });
}

int psg_debug_guard_violations(unsigned long long* bad_bytes, char* first, size_t first_len) {
  return guarded([&] {
    std::string f;
    *bad_bytes = psg::guard_violations(&f);
    if (first && first_len) {
      std::strncpy(first, f.c_str(), first_len - 1);
      first[first_len - 1] = 0;
    }
  });
}

int psg_net_kernels_per_step(const psg_net* net, int* launches) {
  return guarded([&] {
    need(net, "kernels_per_step");
    *launches = net->launches_per_step;
  });
}

int psg_net_profile_step(psg_net* net, int repeats, psg_op_time* out, int max_ops, int* n_ops) {
  return guarded([&] {
    need(net, "profile_step");
    psg::net_profile_step(net, repeats, out, max_ops, n_ops);
  });
}

int psg_net_train_host(psg_net* net, const float* images, const int32_t* labels, long steps,
                       double* losses) {
  return guarded([&] {
    need(net, "train_host");
    psg::net_train_host(net, images, labels, steps, losses);
  });
}

int psg_net_train_host_rows(psg_net* net, const float* ds_images, const int32_t* ds_labels,
                            size_t ds_rows, const uint64_t* rows, long steps, double* losses,
                            int threads) {
  return guarded([&] {
    need(net, "train_host_rows");
    psg::net_train_host_rows(net, ds_images, ds_labels, ds_rows, rows, steps, losses, threads);
  });
}

int psg_host_alloc(size_t bytes, void** ptr) {
  return guarded([&] { PSG_CUDA(cudaMallocHost(ptr, std::max<size_t>(bytes, 1))); });
}

int psg_host_free(void* ptr) {
  return guarded([&] {
    if (ptr) PSG_CUDA(cudaFreeHost(ptr));
  });
}

int psg_net_event_record(psg_net* net, int slot) {
  return guarded([&] {
    need(net, "event_record");
    if (slot < 0 || slot >= 16) throw std::invalid_argument("event slot out of range");
    psg::DeviceGuard dg(net->ctx->device);
    if (!net->slots[slot]) PSG_CUDA(cudaEventCreate(&net->slots[slot]));
    PSG_CUDA(cudaEventRecord(net->slots[slot], net->stream));
  });
}

int psg_net_event_elapsed(psg_net* net, int start_slot, int end_slot, float* ms) {
  return guarded([&] {
    need(net, "event_elapsed");
    if (start_slot < 0 || start_slot >= 16 || end_slot < 0 || end_slot >= 16 ||
        !net->slots[start_slot] || !net->slots[end_slot])
      throw std::invalid_argument("event slot not recorded");
    psg::DeviceGuard dg(net->ctx->device);
    PSG_CUDA(cudaEventSynchronize(net->slots[end_slot]));
    PSG_CUDA(cudaEventElapsedTime(ms, net->slots[start_slot], net->slots[end_slot]));
  });
}

namespace {
void average_local_nets(psg_net* const* nets, int count, int which) {
  {
    if (count < 1) throw std::invalid_argument("weights_mean: empty input");
    std::vector<float*> bufs(count);
    for (int i = 0; i < count; ++i) {
      need(nets[i], "average_local");
      if (nets[i]->ctx->device != nets[0]->ctx->device)
        throw std::invalid_argument("average_local: nets on different devices");
      if (nets[i]->P_int != nets[0]->P_int)
        throw std::invalid_argument("weights_mean: structure mismatch");
      bufs[i] = which ? nets[i]->g : nets[i]->w;
    }
    psg::DeviceGuard dg(nets[0]->ctx->device);
    // order the average after every net's queued work, and every net after it
    std::vector<cudaEvent_t> evs(count);
    for (int i = 0; i < count; ++i) {
      PSG_CUDA(cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming));
      PSG_CUDA(cudaEventRecord(evs[i], nets[i]->stream));
      PSG_CUDA(cudaStreamWaitEvent(nets[0]->stream, evs[i], 0));
    }
    psg::average_ordered(bufs.data(), count, nets[0]->P_int, &nets[0]->dsc->flag,
                         nets[0]->stream);
    PSG_CUDA(cudaEventRecord(evs[0], nets[0]->stream));
    for (int i = 1; i < count; ++i) PSG_CUDA(cudaStreamWaitEvent(nets[i]->stream, evs[0], 0));
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    psg::net_check_flag(nets[0]);
  }
}
}  // namespace

int psg_average_local(psg_net* const* nets, int count) {
  return guarded([&] { average_local_nets(nets, count, 0); });
}

int psg_average_grads_local(psg_net* const* nets, int count) {
  return guarded([&] { average_local_nets(nets, count, 1); });
}

int psg_comm_unique_id(unsigned char id[128]) {
  return guarded([&] { psg::comm_unique_id(id); });
}

int psg_comm_create(psg_ctx* ctx, int nranks, int rank, const unsigned char id[128],
                    psg_comm** out) {
  return guarded([&] {
    need(ctx, "comm_create");
    *out = psg::comm_create(ctx, nranks, rank, id);
  });
}

int psg_comm_create_all(psg_ctx* const* ctxs, int ndev, psg_comm** out) {
  return guarded([&] {
    if (ndev < 1) throw std::invalid_argument("comm_create_all: need >= 1 device");
    psg::comm_create_all(ctxs, ndev, out);
  });
}

int psg_comm_destroy(psg_comm* comm) {
  return guarded([&] { psg::comm_destroy(comm); });
}

int psg_comm_average(psg_comm* const* comms, psg_net* const* nets, int count, int mode) {
  return guarded([&] {
    if (count < 1) throw std::invalid_argument("weights_mean: empty input");
    psg::comm_average_nets(comms, nets, count, mode);
  });
}

int psg_comm_average_grads(psg_comm* const* comms, psg_net* const* nets, int count, int mode) {
  return guarded([&] {
    if (count < 1) throw std::invalid_argument("weights_mean: empty input");
    psg::comm_average_nets(comms, nets, count, mode, 1);
  });
}

int psg_comm_broadcast(psg_comm* const* comms, psg_net* const* nets, int count, int root) {
  return guarded([&] { psg::comm_broadcast_nets(comms, nets, count, root); });
}

int psg_buffer_create(psg_ctx* ctx, size_t n, psg_buffer** out) {
  return guarded([&] {
    need(ctx, "buffer_create");
    psg::DeviceGuard dg(ctx->device);
    auto* b = new psg_buffer;
    b->ctx = ctx;
    b->n = n;
    if (cudaMalloc(&b->ptr, std::max<size_t>(n, 1) * sizeof(float)) != cudaSuccess) {
      delete b;
      throw psg::CudaError("buffer: cudaMalloc failed");
    }
    *out = b;
  });
}

int psg_buffer_fill_uniform(psg_buffer* buf, uint64_t seed, double lo, double hi) {
  return guarded([&] {
    need(buf, "buffer_fill");
    psg::DeviceGuard dg(buf->ctx->device);
    psg::fill_uniform(buf->ptr, buf->n, seed, lo, hi, buf->ctx->stream);
  });
}

int psg_buffer_read(psg_buffer* buf, float* host, size_t n) {
  return guarded([&] {
    need(buf, "buffer_read");
    if (n != buf->n) throw std::invalid_argument("buffer_read: size mismatch");
    psg::DeviceGuard dg(buf->ctx->device);
    PSG_CUDA(cudaStreamSynchronize(buf->ctx->stream));
    PSG_CUDA(cudaMemcpyAsync(host, buf->ptr, n * sizeof(float), cudaMemcpyDeviceToHost,
                             buf->ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(buf->ctx->stream));
  });
}

int psg_buffer_write(psg_buffer* buf, const float* host, size_t n) {
  return guarded([&] {
    need(buf, "buffer_write");
    if (n != buf->n) throw std::invalid_argument("buffer_write: size mismatch");
    psg::DeviceGuard dg(buf->ctx->device);
    PSG_CUDA(cudaStreamSynchronize(buf->ctx->stream));
    PSG_CUDA(cudaMemcpyAsync(buf->ptr, host, n * sizeof(float), cudaMemcpyHostToDevice,
                             buf->ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(buf->ctx->stream));
  });
}

int psg_buffer_destroy(psg_buffer* buf) {
  return guarded([&] {
    if (!buf) return;
    psg::DeviceGuard dg(buf->ctx->device);
    cudaStreamSynchronize(buf->ctx->stream);
    cudaFree(buf->ptr);
    delete buf;
  });
}

int psg_buffer_average_local(psg_buffer* const* bufs, int count) {
  return guarded([&] {
    if (count < 1) throw std::invalid_argument("weights_mean: empty input");
    std::vector<float*> ptrs(count);
    for (int i = 0; i < count; ++i) {
      need(bufs[i], "buffer_average_local");
      if (bufs[i]->n != bufs[0]->n) throw std::invalid_argument("weights_mean: structure mismatch");
      if (bufs[i]->ctx != bufs[0]->ctx)
        throw std::invalid_argument("buffer_average_local: buffers must share a context");
      ptrs[i] = bufs[i]->ptr;
    }
    psg::DeviceGuard dg(bufs[0]->ctx->device);
    int* flag = nullptr;
    PSG_CUDA(cudaMalloc(&flag, sizeof(int)));
    PSG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), bufs[0]->ctx->stream));
    psg::average_ordered(ptrs.data(), count, bufs[0]->n, flag, bufs[0]->ctx->stream);
    int h = 0;
    PSG_CUDA(cudaStreamSynchronize(bufs[0]->ctx->stream));
    PSG_CUDA(cudaMemcpy(&h, flag, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(flag);
    if (h) throw std::runtime_error("mean_collection: produced a non-finite value");
  });
}

int psg_comm_average_buffer(psg_comm* const* comms, psg_buffer* const* bufs, int count, int mode,
                            float* device_ms) {
  return guarded([&] {
    if (count < 1) throw std::invalid_argument("weights_mean: empty input");
    psg::comm_average_buffers(comms, bufs, count, mode, device_ms);
  });
}

}  // extern "C"
