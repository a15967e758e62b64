/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C99, fp64, NCHW.
 *
 * Restates, function by function, the reference path under
 * /root/reference/proj/include/parasgd/.  Accumulation orders follow the
 * reference loops exactly so that, compiled without FP contraction
 * (-ffp-contract=off, oracle/Makefile), the reference-layer subset reproduces
 * the reference bit for bit (pinned by tests/golden/).
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
static void set_err(const char* msg) { snprintf(g_err, sizeof g_err, "%s", msg); }
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng ---- */
/* rng.hpp:11-16 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:20-25: s = mix(base); s = mix(s ^ part) for each part. */
uint64_t orc_derive_seed(uint64_t base, const uint64_t* parts, int nparts) {
  uint64_t s = orc_splitmix64(base);
  for (int i = 0; i < nparts; ++i) s = orc_splitmix64(s ^ parts[i]);
  return s;
}

static const uint64_t kStreamWeights = 0x57454947ULL; /* rng.hpp:28 */
static const uint64_t kStreamShard = 0x53484152ULL;   /* rng.hpp:29 */
static const uint64_t kStreamWorker = 0x574f524bULL;  /* rng.hpp:30 */
static const uint64_t kStreamData = 0x44415441ULL;    /* rng.hpp:31 */
/* Extension: dropout masks (no reference counterpart). */
static const uint64_t kStreamDropout = 0x44524f50ULL;

void orc_rng_init(orc_rng* r, uint64_t seed) {
  r->state = seed;
  r->spare = 0.0;
  r->has_spare = 0;
}

/* rng.hpp:38-43 (counter form of splitmix64) */
uint64_t orc_rng_next(orc_rng* r) {
  r->state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = r->state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:46: 53 random bits scaled by 2^-53 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_uniform_range(orc_rng* r, double lo, double hi) {
  return lo + (hi - lo) * orc_rng_uniform(r); /* rng.hpp:48 */
}

/* rng.hpp:54-66, Box-Muller with a cached spare */
double orc_rng_normal(orc_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = 1.0 - orc_rng_uniform(r);
  const double u2 = orc_rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(theta);
  r->has_spare = 1;
  return rad * cos(theta);
}

/* rng.hpp:69-75: descending Fisher-Yates, j = next % i */
void orc_rng_shuffle_u64(orc_rng* r, uint64_t* v, size_t n) {
  for (size_t i = n; i > 1; --i) {
    const size_t j = (size_t)(orc_rng_next(r) % (uint64_t)i);
    const uint64_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

/* ----------------------------------------------------------------- data ---- */
/* data.hpp:60-92 smooth_pattern: coarse node grid, bilinear upsampling. */
static void grid_cell(size_t i, size_t extent, size_t grid, size_t* lo, double* t) {
  const double f = extent > 1 ? (double)i * (double)grid / (double)(extent - 1) : 0.0;
  size_t l = (size_t)f;
  if (l > grid - 1) l = grid - 1;
  *lo = l;
  *t = f - (double)l;
}

static void smooth_pattern(orc_rng* rng, size_t channels, size_t height, size_t width,
                           int unit_var, double* pattern, double* nodes) {
  const size_t gh = height / 4 > 1 ? height / 4 : 1;
  const size_t gw = width / 4 > 1 ? width / 4 : 1;
  const size_t stride = gw + 1;
  for (size_t c = 0; c < channels; ++c) {
    for (size_t q = 0; q < (gh + 1) * (gw + 1); ++q) nodes[q] = orc_rng_normal(rng);
    for (size_t y = 0; y < height; ++y) {
      size_t y0;
      double ty;
      grid_cell(y, height, gh, &y0, &ty);
      for (size_t x = 0; x < width; ++x) {
        size_t x0;
        double tx;
        grid_cell(x, width, gw, &x0, &tx);
        const double w00 = (1.0 - ty) * (1.0 - tx), w01 = (1.0 - ty) * tx;
        const double w10 = ty * (1.0 - tx), w11 = ty * tx;
        double v = w00 * nodes[y0 * stride + x0] + w01 * nodes[y0 * stride + x0 + 1] +
                   w10 * nodes[(y0 + 1) * stride + x0] + w11 * nodes[(y0 + 1) * stride + x0 + 1];
        if (unit_var) v /= sqrt(w00 * w00 + w01 * w01 + w10 * w10 + w11 * w11);
        pattern[(c * height + y) * width + x] = v;
      }
    }
  }
}

/* data.hpp:111-155 generate_synthetic */
void orc_generate_synthetic(int classes, size_t c, size_t h, size_t w, size_t per_class,
                            double separation, uint64_t seed, uint64_t variant, double* images,
                            int32_t* labels) {
  const size_t dim = c * h * w;
  const size_t gh = h / 4 > 1 ? h / 4 : 1, gw = w / 4 > 1 ? w / 4 : 1;
  double* nodes = (double*)malloc(sizeof(double) * (gh + 1) * (gw + 1));
  double* means = (double*)malloc(sizeof(double) * dim * (size_t)classes);
  double* structure = (double*)malloc(sizeof(double) * dim);
  orc_rng mean_stream, noise_stream;
  const uint64_t mp[2] = {kStreamData, 0x4d45414eULL};
  const uint64_t np[3] = {kStreamData, 0x4e4f495345ULL, variant};
  orc_rng_init(&mean_stream, orc_derive_seed(seed, mp, 2));
  orc_rng_init(&noise_stream, orc_derive_seed(seed, np, 3));
  const double radius = separation / sqrt(2.0);
  for (int cls = 0; cls < classes; ++cls) {
    double* mu = means + (size_t)cls * dim;
    smooth_pattern(&mean_stream, c, h, w, 0, mu, nodes);
    double norm2 = 0.0;
    for (size_t d = 0; d < dim; ++d) norm2 += mu[d] * mu[d];
    const double inv = norm2 > 0.0 ? radius / sqrt(norm2) : 0.0;
    for (size_t d = 0; d < dim; ++d) mu[d] *= inv;
  }
  const double smooth_scale = 0.7; /* data.hpp:98 kStructuredNoise */
  const double white_scale = sqrt(1.0 - smooth_scale * smooth_scale);
  size_t row = 0;
  for (int cls = 0; cls < classes; ++cls) {
    const double* mu = means + (size_t)cls * dim;
    for (size_t e = 0; e < per_class; ++e, ++row) {
      labels[row] = cls;
      double* dst = images + row * dim;
      smooth_pattern(&noise_stream, c, h, w, 1, structure, nodes);
      for (size_t d = 0; d < dim; ++d) {
        dst[d] = mu[d] + smooth_scale * structure[d] + white_scale * orc_rng_normal(&noise_stream);
      }
    }
  }
  free(nodes);
  free(means);
  free(structure);
}

/* data.hpp:261-288: iota, shuffle with derive_seed(seed, kStreamShard),
 * contiguous split, first n%K shards one longer. */
int orc_shard(size_t n, int workers, uint64_t seed, uint64_t* perm, uint64_t* offsets) {
  if (workers < 1) {
    set_err("shard: need at least one worker");
    return PSG_EINVAL;
  }
  if ((size_t)workers > n) {
    set_err("shard: more workers than examples");
    return PSG_EINVAL;
  }
  for (size_t i = 0; i < n; ++i) perm[i] = i;
  orc_rng r;
  orc_rng_init(&r, orc_derive_seed(seed, &kStreamShard, 1));
  orc_rng_shuffle_u64(&r, perm, n);
  const size_t base = n / (size_t)workers, extra = n % (size_t)workers;
  size_t pos = 0;
  offsets[0] = 0;
  for (int k = 0; k < workers; ++k) {
    pos += base + ((size_t)k < extra ? 1 : 0);
    offsets[k + 1] = pos;
  }
  return PSG_OK;
}

/* data.hpp:386-388 */
uint64_t orc_worker_stream_seed(uint64_t global_seed, int worker) {
  const uint64_t parts[2] = {kStreamWorker, (uint64_t)worker};
  return orc_derive_seed(global_seed, parts, 2);
}

/* data.hpp:338-343 */
void orc_epoch_order(const uint64_t* shard, size_t n, uint64_t stream_seed, uint64_t epoch,
                     uint64_t* order) {
  memcpy(order, shard, n * sizeof(uint64_t));
  orc_rng r;
  orc_rng_init(&r, orc_derive_seed(stream_seed, &epoch, 1));
  orc_rng_shuffle_u64(&r, order, n);
}

/* ---------------------------------------------------------------- model ---- */
typedef struct orc_layer {
  psg_layer_desc d;
  int kind;
  int64_t c, h, w;          /* per-example output dims */
  int64_t ic, ih, iw;       /* per-example dims of input 0 */
  size_t poff, kcount, bcount;
  double* out;              /* [n, c, h, w] */
  double* grad;
  int64_t* route;           /* max pool */
  double* aux;              /* LRN scale / dropout mask */
  size_t cap;               /* elements allocated for out/grad/aux */
  const double* fin[8];     /* inputs of the last forward */
} orc_layer;

struct orc_net {
  orc_layer* L;
  int n;
  size_t P;
  double* params;
  double* vel;
  int data_idx, label_idx, loss_idx, classes;
  double lr, mu, wd;
  uint64_t seed, dropout_step;
  size_t batch;
  int32_t* labels;
  size_t labels_cap;
  int train_phase;
  double last_loss;
};

static int64_t vol3(const orc_layer* l) { return l->c * l->h * l->w; }

static int pool_out_dim(int64_t in, int k, int s, int p, int ceil_mode) {
  int64_t o;
  if (ceil_mode) {
    o = (in + 2 * p - k + s - 1) / s + 1; /* ceil((in+2p-k)/s)+1 */
    if (p > 0 && (o - 1) * s >= in + p) --o;
  } else {
    o = (in + 2 * p - k) / s + 1; /* model.hpp:244-245 (p = 0) */
  }
  return (int)o;
}

orc_net* orc_net_create(const psg_layer_desc* layers, int n_layers, uint64_t seed) {
  orc_net* net = (orc_net*)calloc(1, sizeof(orc_net));
  net->L = (orc_layer*)calloc((size_t)n_layers, sizeof(orc_layer));
  net->n = n_layers;
  net->seed = seed;
  net->data_idx = net->label_idx = net->loss_idx = -1;
  net->lr = 0.01;
  size_t P = 0;
  for (int li = 0; li < n_layers; ++li) {
    orc_layer* l = &net->L[li];
    l->d = layers[li];
    l->kind = layers[li].kind;
    for (int i = 0; i < l->d.n_inputs; ++i) {
      if (l->d.inputs[i] < 0 || l->d.inputs[i] >= li) {
        set_err("net: layer input not declared earlier");
        orc_net_destroy(net);
        return NULL;
      }
    }
    if (l->d.n_inputs > 0) {
      const orc_layer* src = &net->L[l->d.inputs[0]];
      l->ic = src->c;
      l->ih = src->h;
      l->iw = src->w;
    }
    switch (l->kind) {
      case PSG_LAYER_DATA:
        net->data_idx = li;
        l->c = l->d.channels;
        l->h = l->d.height;
        l->w = l->d.width;
        break;
      case PSG_LAYER_LABEL:
        net->label_idx = li;
        l->c = l->h = l->w = 1;
        break;
      case PSG_LAYER_CONV: {
        const int kh = l->d.kernel_h, kw = l->d.kernel_w, g = l->d.group;
        if (l->ih + 2 * l->d.pad_h < kh || l->iw + 2 * l->d.pad_w < kw) {
          set_err("net: conv kernel exceeds input");
          orc_net_destroy(net);
          return NULL;
        }
        if (l->ic % g || l->d.num_output % g) {
          set_err("net: conv group must divide channels and filters");
          orc_net_destroy(net);
          return NULL;
        }
        l->c = l->d.num_output;
        l->h = (l->ih + 2 * l->d.pad_h - kh) / l->d.stride_h + 1;
        l->w = (l->iw + 2 * l->d.pad_w - kw) / l->d.stride_w + 1;
        l->kcount = (size_t)(l->c * (l->ic / g) * kh * kw);
        l->bcount = (size_t)l->c;
        break;
      }
      case PSG_LAYER_POOL:
        if (l->ih + 2 * l->d.pad_h < l->d.kernel_h || l->iw + 2 * l->d.pad_w < l->d.kernel_w) {
          set_err("net: pool kernel exceeds input");
          orc_net_destroy(net);
          return NULL;
        }
        l->c = l->ic;
        l->h = pool_out_dim(l->ih, l->d.kernel_h, l->d.stride_h, l->d.pad_h, l->d.ceil_mode);
        l->w = pool_out_dim(l->iw, l->d.kernel_w, l->d.stride_w, l->d.pad_w, l->d.ceil_mode);
        break;
      case PSG_LAYER_LINEAR:
        l->c = l->d.num_output;
        l->h = l->w = 1;
        l->kcount = (size_t)(l->c * l->ic * l->ih * l->iw);
        l->bcount = (size_t)l->c;
        break;
      case PSG_LAYER_RELU:
      case PSG_LAYER_LRN:
      case PSG_LAYER_DROPOUT:
        l->c = l->ic;
        l->h = l->ih;
        l->w = l->iw;
        break;
      case PSG_LAYER_SOFTMAX_LOSS:
        /* several weighted losses (GoogLeNet's auxiliary heads): they share the labels, so
         * they must agree on the class count; probabilities / test use the last one */
        if (net->classes && net->classes != (int)(l->ic * l->ih * l->iw)) {
          set_err("net: loss layers disagree on the class count");
          orc_net_destroy(net);
          return NULL;
        }
        net->loss_idx = li;
        l->c = l->ic * l->ih * l->iw;
        l->h = l->w = 1;
        net->classes = (int)l->c;
        break;
      case PSG_LAYER_CONCAT: /* Caffe Concat along channels: inputs share h, w */
        l->c = 0;
        for (int i = 0; i < l->d.n_inputs; ++i) {
          const orc_layer* in = &net->L[l->d.inputs[i]];
          if (in->h != l->ih || in->w != l->iw) {
            set_err("net: concat inputs differ in height/width");
            orc_net_destroy(net);
            return NULL;
          }
          l->c += in->c;
        }
        l->h = l->ih;
        l->w = l->iw;
        break;
      default:
        set_err("net: unsupported layer kind in oracle");
        orc_net_destroy(net);
        return NULL;
    }
    l->poff = P;
    P += l->kcount + l->bcount;
  }
  net->P = P;
  net->params = (double*)calloc(P ? P : 1, sizeof(double));
  net->vel = (double*)calloc(P ? P : 1, sizeof(double));
  /* model.hpp:205-258: per-layer stream derive_seed(seed, kStreamWeights, li);
   * kernels U(-s, s), s = sqrt(6/(fan_in + fan_out)); biases zero. */
  for (int li = 0; li < n_layers; ++li) {
    orc_layer* l = &net->L[li];
    if (!l->kcount) continue;
    const uint64_t parts[2] = {kStreamWeights, (uint64_t)li};
    orc_rng r;
    orc_rng_init(&r, orc_derive_seed(seed, parts, 2));
    double s;
    if (l->kind == PSG_LAYER_CONV) {
      const double khw = (double)(l->d.kernel_h * l->d.kernel_w);
      const double fan_in = (double)(l->ic / l->d.group) * khw;
      const double fan_out = (double)(l->c / l->d.group) * khw;
      s = sqrt(6.0 / (fan_in + fan_out));
    } else {
      s = sqrt(6.0 / ((double)(l->ic * l->ih * l->iw) + (double)l->c));
    }
    double* k = net->params + l->poff;
    for (size_t i = 0; i < l->kcount; ++i) k[i] = rng_uniform_range(&r, -s, s);
  }
  return net;
}

void orc_net_destroy(orc_net* net) {
  if (!net) return;
  for (int i = 0; i < net->n; ++i) {
    free(net->L[i].out);
    free(net->L[i].grad);
    free(net->L[i].route);
    free(net->L[i].aux);
  }
  free(net->L);
  free(net->params);
  free(net->vel);
  free(net->labels);
  free(net);
}

size_t orc_net_param_count(const orc_net* net) { return net->P; }
int orc_net_num_classes(const orc_net* net) { return net->classes; }
void orc_net_get_weights(const orc_net* net, double* flat) {
  memcpy(flat, net->params, net->P * sizeof(double));
}
void orc_net_set_weights(orc_net* net, const double* flat) {
  memcpy(net->params, flat, net->P * sizeof(double));
}
void orc_net_get_velocity(const orc_net* net, double* flat) {
  memcpy(flat, net->vel, net->P * sizeof(double));
}
void orc_net_reset_velocity(orc_net* net) { memset(net->vel, 0, net->P * sizeof(double)); }
void orc_net_set_sgd(orc_net* net, double lr, double momentum, double weight_decay) {
  net->lr = lr;
  net->mu = momentum;
  net->wd = weight_decay;
}
void orc_net_set_dropout_step(orc_net* net, uint64_t step) { net->dropout_step = step; }
void orc_net_layer_params(const orc_net* net, int layer, size_t* offset, size_t* count) {
  *offset = net->L[layer].poff;
  *count = net->L[layer].kcount + net->L[layer].bcount;
}
int orc_net_layer_dims(const orc_net* net, int layer, int64_t dims[3]) {
  if (layer < 0 || layer >= net->n) return PSG_EINVAL;
  dims[0] = net->L[layer].c;
  dims[1] = net->L[layer].h;
  dims[2] = net->L[layer].w;
  return PSG_OK;
}
const double* orc_net_layer_out(const orc_net* net, int layer) { return net->L[layer].out; }
const double* orc_net_layer_grad(const orc_net* net, int layer) { return net->L[layer].grad; }

static void ensure_buffers(orc_layer* l, size_t n) {
  const size_t need = n * (size_t)vol3(l);
  if (l->cap >= need) return;
  free(l->out);
  free(l->grad);
  free(l->route);
  free(l->aux);
  l->out = (double*)calloc(need, sizeof(double));
  l->grad = (double*)calloc(need, sizeof(double));
  l->route = (int64_t*)calloc(need, sizeof(int64_t));
  l->aux = (double*)calloc(need, sizeof(double));
  l->cap = need;
}

static int all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* model.hpp:334-367 generalised to Caffe geometry (pad, stride, group).  Every
 * output starts at its bias and accumulates taps in (c, u, v) order. */
static void conv_fwd(const orc_net* net, const orc_layer* l, size_t n, const double* x,
                     double* y) {
  const int64_t C = l->ic, H = l->ih, W = l->iw, F = l->c, OH = l->h, OW = l->w;
  const int kh = l->d.kernel_h, kw = l->d.kernel_w, sh = l->d.stride_h, sw = l->d.stride_w;
  const int ph = l->d.pad_h, pw = l->d.pad_w, G = l->d.group;
  const int64_t Cg = C / G, Fg = F / G;
  const double* ker = net->params + l->poff;
  const double* bias = ker + l->kcount;
  for (size_t b = 0; b < n; ++b) {
    for (int64_t f = 0; f < F; ++f) {
      double* om = y + ((int64_t)b * F + f) * OH * OW;
      for (int64_t i = 0; i < OH * OW; ++i) om[i] = bias[f];
      const int64_t c0 = (f / Fg) * Cg;
      for (int64_t cl = 0; cl < Cg; ++cl) {
        const double* im = x + ((int64_t)b * C + c0 + cl) * H * W;
        const double* km = ker + (f * Cg + cl) * kh * kw;
        for (int u = 0; u < kh; ++u) {
          for (int v = 0; v < kw; ++v) {
            const double kv = km[u * kw + v];
            for (int64_t i = 0; i < OH; ++i) {
              const int64_t r = i * sh - ph + u;
              if (r < 0 || r >= H) continue;
              double* orow = om + i * OW;
              for (int64_t j = 0; j < OW; ++j) {
                const int64_t s = j * sw - pw + v;
                if (s < 0 || s >= W) continue;
                orow[j] += kv * im[r * W + s];
              }
            }
          }
        }
      }
    }
  }
}

/* model.hpp:544-585: dbias (b, i) order; dK = sum over b of per-image partial
 * sums; dx accumulated in (f, u, v) order. */
static void conv_bwd(const orc_net* net, const orc_layer* l, size_t n, const double* x,
                     const double* dy, double* dx, double* dk, double* db) {
  const int64_t C = l->ic, H = l->ih, W = l->iw, F = l->c, OH = l->h, OW = l->w;
  const int kh = l->d.kernel_h, kw = l->d.kernel_w, sh = l->d.stride_h, sw = l->d.stride_w;
  const int ph = l->d.pad_h, pw = l->d.pad_w, G = l->d.group;
  const int64_t Cg = C / G, Fg = F / G;
  const double* ker = net->params + l->poff;
  for (size_t b = 0; b < n; ++b) {
    for (int64_t f = 0; f < F; ++f) {
      const double* gm = dy + ((int64_t)b * F + f) * OH * OW;
      for (int64_t i = 0; i < OH * OW; ++i) db[f] += gm[i];
      const int64_t c0 = (f / Fg) * Cg;
      for (int64_t cl = 0; cl < Cg; ++cl) {
        const double* im = x + ((int64_t)b * C + c0 + cl) * H * W;
        double* dm = dx ? dx + ((int64_t)b * C + c0 + cl) * H * W : NULL;
        const double* km = ker + (f * Cg + cl) * kh * kw;
        double* dkm = dk + (f * Cg + cl) * kh * kw;
        for (int u = 0; u < kh; ++u) {
          for (int v = 0; v < kw; ++v) {
            const double kv = km[u * kw + v];
            double acc = 0.0;
            for (int64_t i = 0; i < OH; ++i) {
              const int64_t r = i * sh - ph + u;
              if (r < 0 || r >= H) continue;
              const double* grow = gm + i * OW;
              for (int64_t j = 0; j < OW; ++j) {
                const int64_t s = j * sw - pw + v;
                if (s < 0 || s >= W) continue;
                acc += grow[j] * im[r * W + s];
                if (dm) dm[r * W + s] += grow[j] * kv;
              }
            }
            dkm[u * kw + v] += acc;
          }
        }
      }
    }
  }
}

/* model.hpp:369-406 (max, floor mode, first max wins on ties) extended with
 * Caffe padding / ceil mode / AVE (window clipped to the image, AVE divisor
 * counts the padded window clipped to H+pad). */
static void pool_fwd(const orc_layer* l, size_t n, const double* x, double* y, int64_t* route) {
  const int64_t C = l->ic, H = l->ih, W = l->iw, OH = l->h, OW = l->w;
  const int kh = l->d.kernel_h, kw = l->d.kernel_w, sh = l->d.stride_h, sw = l->d.stride_w;
  const int ph = l->d.pad_h, pw = l->d.pad_w;
  int64_t m = 0;
  for (size_t b = 0; b < n; ++b) {
    for (int64_t c = 0; c < C; ++c) {
      const int64_t base = ((int64_t)b * C + c) * H * W;
      for (int64_t i = 0; i < OH; ++i) {
        for (int64_t j = 0; j < OW; ++j, ++m) {
          int64_t hs = i * sh - ph, ws = j * sw - pw;
          int64_t he = hs + kh, we = ws + kw;
          if (l->d.pool == PSG_POOL_AVE) {
            const int64_t hp = he < H + ph ? he : H + ph, wp = we < W + pw ? we : W + pw;
            const double size = (double)((hp - hs) * (wp - ws));
            if (hs < 0) hs = 0;
            if (ws < 0) ws = 0;
            if (he > H) he = H;
            if (we > W) we = W;
            double acc = 0.0;
            for (int64_t r = hs; r < he; ++r)
              for (int64_t s = ws; s < we; ++s) acc += x[base + r * W + s];
            y[m] = acc / size;
            route[m] = -1;
          } else {
            if (hs < 0) hs = 0;
            if (ws < 0) ws = 0;
            if (he > H) he = H;
            if (we > W) we = W;
            int64_t best = base + hs * W + ws;
            double bv = x[best];
            for (int64_t r = hs; r < he; ++r) {
              for (int64_t s = ws; s < we; ++s) {
                const int64_t idx = base + r * W + s;
                if (x[idx] > bv) {
                  bv = x[idx];
                  best = idx;
                }
              }
            }
            y[m] = bv;
            route[m] = best;
          }
        }
      }
    }
  }
}

/* model.hpp:492-498 (max: dx[route[m]] += dy[m], ascending m); AVE spreads
 * dy/size over the clipped window in ascending output order (Caffe). */
static void pool_bwd(const orc_layer* l, size_t n, const double* dy, const int64_t* route,
                     double* dx) {
  const int64_t total = (int64_t)n * vol3(l);
  if (l->d.pool == PSG_POOL_MAX) {
    for (int64_t m = 0; m < total; ++m) dx[route[m]] += dy[m];
    return;
  }
  const int64_t C = l->ic, H = l->ih, W = l->iw, OH = l->h, OW = l->w;
  const int kh = l->d.kernel_h, kw = l->d.kernel_w, sh = l->d.stride_h, sw = l->d.stride_w;
  const int ph = l->d.pad_h, pw = l->d.pad_w;
  int64_t m = 0;
  for (size_t b = 0; b < n; ++b) {
    for (int64_t c = 0; c < C; ++c) {
      const int64_t base = ((int64_t)b * C + c) * H * W;
      for (int64_t i = 0; i < OH; ++i) {
        for (int64_t j = 0; j < OW; ++j, ++m) {
          int64_t hs = i * sh - ph, ws = j * sw - pw;
          int64_t he = hs + kh, we = ws + kw;
          const int64_t hp = he < H + ph ? he : H + ph, wp = we < W + pw ? we : W + pw;
          const double size = (double)((hp - hs) * (wp - ws));
          if (hs < 0) hs = 0;
          if (ws < 0) ws = 0;
          if (he > H) he = H;
          if (we > W) we = W;
          const double g = dy[m] / size;
          for (int64_t r = hs; r < he; ++r)
            for (int64_t s = ws; s < we; ++s) dx[base + r * W + s] += g;
        }
      }
    }
  }
}

/* model.hpp:408-427: bias first, then d ascending. */
static void linear_fwd(const orc_net* net, const orc_layer* l, size_t n, const double* x,
                       double* y) {
  const int64_t D = l->ic * l->ih * l->iw, O = l->c;
  const double* wt = net->params + l->poff;
  const double* bias = wt + l->kcount;
  for (size_t b = 0; b < n; ++b) {
    const double* xr = x + (int64_t)b * D;
    for (int64_t o = 0; o < O; ++o) {
      const double* wr = wt + o * D;
      double acc = bias[o];
      for (int64_t d = 0; d < D; ++d) acc += wr[d] * xr[d];
      y[(int64_t)b * O + o] = acc;
    }
  }
}

/* model.hpp:516-542: b-outer, skip g == 0. */
static void linear_bwd(const orc_net* net, const orc_layer* l, size_t n, const double* x,
                       const double* dy, double* dx, double* dw, double* db) {
  const int64_t D = l->ic * l->ih * l->iw, O = l->c;
  const double* wt = net->params + l->poff;
  for (size_t b = 0; b < n; ++b) {
    const double* xr = x + (int64_t)b * D;
    const double* gr = dy + (int64_t)b * O;
    double* dxr = dx ? dx + (int64_t)b * D : NULL;
    for (int64_t o = 0; o < O; ++o) {
      const double g = gr[o];
      if (g == 0.0) continue;
      db[o] += g;
      double* dwr = dw + o * D;
      const double* wr = wt + o * D;
      for (int64_t d = 0; d < D; ++d) {
        dwr[d] += g * xr[d];
        if (dxr) dxr[d] += g * wr[d];
      }
    }
  }
}

/* Caffe LRN ACROSS_CHANNELS: scale = k + alpha/size * sum_{window} x^2,
 * y = x * scale^-beta (direct window sums in ascending channel order). */
static void lrn_fwd(const orc_layer* l, size_t n, const double* x, double* y, double* scale) {
  const int64_t C = l->c, HW = l->h * l->w;
  const int size = l->d.local_size, pre = (size - 1) / 2;
  const double a = l->d.alpha / size, beta = l->d.beta, k = l->d.k;
  for (size_t b = 0; b < n; ++b) {
    for (int64_t c = 0; c < C; ++c) {
      int64_t lo = c - pre, hi = c + (size - pre - 1);
      if (lo < 0) lo = 0;
      if (hi > C - 1) hi = C - 1;
      for (int64_t p = 0; p < HW; ++p) {
        double acc = 0.0;
        for (int64_t q = lo; q <= hi; ++q) {
          const double v = x[((int64_t)b * C + q) * HW + p];
          acc += v * v;
        }
        const int64_t idx = ((int64_t)b * C + c) * HW + p;
        scale[idx] = k + a * acc;
        y[idx] = x[idx] * pow(scale[idx], -beta);
      }
    }
  }
}

static void lrn_bwd(const orc_layer* l, size_t n, const double* x, const double* y,
                    const double* scale, const double* dy, double* dx) {
  const int64_t C = l->c, HW = l->h * l->w;
  const int size = l->d.local_size, pre = (size - 1) / 2, post = size - pre - 1;
  const double beta = l->d.beta, ratio = 2.0 * l->d.alpha * beta / size;
  for (size_t b = 0; b < n; ++b) {
    for (int64_t c = 0; c < C; ++c) {
      /* channels q whose window contains c: q in [c - post, c + pre] */
      int64_t lo = c - post, hi = c + pre;
      if (lo < 0) lo = 0;
      if (hi > C - 1) hi = C - 1;
      for (int64_t p = 0; p < HW; ++p) {
        double acc = 0.0;
        for (int64_t q = lo; q <= hi; ++q) {
          const int64_t j = ((int64_t)b * C + q) * HW + p;
          acc += dy[j] * y[j] / scale[j];
        }
        const int64_t idx = ((int64_t)b * C + c) * HW + p;
        dx[idx] += dy[idx] * pow(scale[idx], -beta) - ratio * x[idx] * acc;
      }
    }
  }
}

/* Extension: dropout keep-mask from a counter hash of (seed, layer, step, element). */
static uint64_t dropout_base(uint64_t net_seed, int layer, uint64_t step) {
  const uint64_t parts[3] = {kStreamDropout, (uint64_t)layer, step};
  return orc_derive_seed(net_seed, parts, 3);
}

static void dropout_fwd(const orc_net* net, int li, const orc_layer* l, size_t n, const double* x,
                        double* y, double* mask, int train) {
  const size_t total = n * (size_t)vol3(l);
  if (!train) {
    for (size_t i = 0; i < total; ++i) {
      y[i] = x[i];
      mask[i] = 1.0;
    }
    return;
  }
  const uint64_t base = dropout_base(net->seed, li, net->dropout_step);
  const double ratio = l->d.dropout_ratio, keep_scale = 1.0 / (1.0 - ratio);
  const uint32_t thresh = (uint32_t)(ratio * 16777216.0);
  for (size_t i = 0; i < total; ++i) {
    const uint32_t u = (uint32_t)(orc_splitmix64(base + (uint64_t)i) >> 40);
    mask[i] = u >= thresh ? keep_scale : 0.0;
    y[i] = x[i] * mask[i];
  }
}

/* model.hpp:429-451 softmax + mean cross-entropy (x loss_weight). */
static int softmax_fwd(orc_net* net, const orc_layer* l, size_t n, const double* logits,
                       double* probs) {
  const int64_t C = l->c;
  double loss = 0.0;
  for (size_t b = 0; b < n; ++b) {
    const double* row = logits + (int64_t)b * C;
    double mx = row[0];
    for (int64_t j = 1; j < C; ++j) mx = row[j] > mx ? row[j] : mx;
    double sum = 0.0;
    double* pr = probs + (int64_t)b * C;
    for (int64_t j = 0; j < C; ++j) {
      pr[j] = exp(row[j] - mx);
      sum += pr[j];
    }
    for (int64_t j = 0; j < C; ++j) pr[j] /= sum;
    const int y = net->labels[b];
    loss -= (row[y] - mx) - log(sum);
  }
  net->last_loss += loss / (double)n * l->d.loss_weight; /* sum of weighted losses */
  if (!isfinite(net->last_loss)) {
    set_err("softmax loss: non-finite loss");
    return PSG_ERUNTIME;
  }
  return PSG_OK;
}

/* model.hpp:463-475: d(mean loss)/d(logits) = (p - onehot)/n (x loss_weight). */
static void softmax_seed(const orc_net* net, const orc_layer* l, size_t n, const double* probs,
                         double* dlogits) {
  const int64_t C = l->c;
  const double inv_n = l->d.loss_weight * (1.0 / (double)n);
  for (size_t b = 0; b < n; ++b) {
    for (int64_t j = 0; j < C; ++j) dlogits[(int64_t)b * C + j] += probs[(int64_t)b * C + j] * inv_n;
    dlogits[(int64_t)b * C + net->labels[b]] -= inv_n;
  }
}

static int layer_forward_impl(orc_net* net, int li, size_t n) {
  orc_layer* l = &net->L[li];
  ensure_buffers(l, n);
  const double* x = l->fin[0];
  const size_t total = n * (size_t)vol3(l);
  switch (l->kind) {
    case PSG_LAYER_DATA:
    case PSG_LAYER_LABEL:
      return PSG_OK;
    case PSG_LAYER_CONV:
      conv_fwd(net, l, n, x, l->out);
      if (!all_finite(l->out, total)) {
        set_err("conv forward: produced a non-finite value");
        return PSG_ERUNTIME;
      }
      return PSG_OK;
    case PSG_LAYER_POOL:
      pool_fwd(l, n, x, l->out, l->route);
      return PSG_OK;
    case PSG_LAYER_LINEAR:
      linear_fwd(net, l, n, x, l->out);
      if (!all_finite(l->out, total)) {
        set_err("linear forward: produced a non-finite value");
        return PSG_ERUNTIME;
      }
      return PSG_OK;
    case PSG_LAYER_RELU:
      for (size_t i = 0; i < total; ++i) l->out[i] = x[i] > 0.0 ? x[i] : 0.0; /* model.hpp:324 */
      return PSG_OK;
    case PSG_LAYER_LRN:
      lrn_fwd(l, n, x, l->out, l->aux);
      return PSG_OK;
    case PSG_LAYER_DROPOUT:
      dropout_fwd(net, li, l, n, x, l->out, l->aux, net->train_phase);
      return PSG_OK;
    case PSG_LAYER_SOFTMAX_LOSS:
      return softmax_fwd(net, l, n, x, l->out);
    case PSG_LAYER_CONCAT: { /* NCHW: input i fills channels [off_i, off_i + c_i) */
      const int64_t hw = l->h * l->w;
      int64_t off = 0;
      for (int i = 0; i < l->d.n_inputs; ++i) {
        const int64_t ci = net->L[l->d.inputs[i]].c;
        for (size_t b = 0; b < n; ++b)
          memcpy(l->out + ((int64_t)b * l->c + off) * hw, l->fin[i] + (int64_t)b * ci * hw,
                 (size_t)(ci * hw) * sizeof(double));
        off += ci;
      }
      return PSG_OK;
    }
  }
  set_err("forward: unsupported layer");
  return PSG_EINVAL;
}

static int run_forward(orc_net* net, const double* images, const int32_t* labels, size_t n) {
  if (n < 1) {
    set_err("forward: label count does not match batch");
    return PSG_EINVAL;
  }
  for (size_t i = 0; i < n; ++i) {
    if (labels[i] < 0 || labels[i] >= net->classes) {
      set_err("forward: label out of range");
      return PSG_EINVAL;
    }
  }
  if (net->labels_cap < n) {
    free(net->labels);
    net->labels = (int32_t*)malloc(n * sizeof(int32_t));
    net->labels_cap = n;
  }
  memcpy(net->labels, labels, n * sizeof(int32_t));
  net->batch = n;
  net->last_loss = 0.0;
  for (int li = 0; li < net->n; ++li) {
    orc_layer* l = &net->L[li];
    if (l->kind == PSG_LAYER_DATA) {
      ensure_buffers(l, n);
      memcpy(l->out, images, n * (size_t)vol3(l) * sizeof(double));
      continue;
    }
    for (int i = 0; i < l->d.n_inputs; ++i) l->fin[i] = net->L[l->d.inputs[i]].out;
    const int rc = layer_forward_impl(net, li, n);
    if (rc) return rc;
  }
  return PSG_OK;
}

int orc_net_forward(orc_net* net, const double* images, const int32_t* labels, size_t n,
                    int train, double* loss, double* probs) {
  net->train_phase = train;
  const int rc = run_forward(net, images, labels, n);
  net->train_phase = 0;
  if (rc) return rc;
  if (loss) *loss = net->last_loss;
  if (probs) memcpy(probs, net->L[net->loss_idx].out, n * (size_t)net->classes * sizeof(double));
  return PSG_OK;
}

/* Backward of one layer into explicit buffers (dx may be NULL). */
static void layer_backward_impl(orc_net* net, int li, size_t n, const double* dy, double* dx,
                                double* dparams) {
  orc_layer* l = &net->L[li];
  const double* x = l->fin[0];
  const size_t total = n * (size_t)vol3(l);
  switch (l->kind) {
    case PSG_LAYER_RELU:
      for (size_t i = 0; i < total; ++i) dx[i] += x[i] > 0.0 ? dy[i] : 0.0; /* model.hpp:489 */
      break;
    case PSG_LAYER_POOL:
      pool_bwd(l, n, dy, l->route, dx);
      break;
    case PSG_LAYER_LINEAR:
      linear_bwd(net, l, n, x, dy, dx, dparams, dparams + l->kcount);
      break;
    case PSG_LAYER_CONV:
      conv_bwd(net, l, n, x, dy, dx, dparams, dparams + l->kcount);
      break;
    case PSG_LAYER_LRN:
      lrn_bwd(l, n, x, l->out, l->aux, dy, dx);
      break;
    case PSG_LAYER_DROPOUT:
      for (size_t i = 0; i < total; ++i) dx[i] += dy[i] * l->aux[i];
      break;
    default:
      break;
  }
}

int orc_net_backward(orc_net* net, const double* images, const int32_t* labels, size_t n,
                     double* loss, double* grads) {
  net->train_phase = 1;
  int rc = run_forward(net, images, labels, n);
  net->train_phase = 0;
  if (rc) return rc;
  /* model.hpp:455-461: zero every gradient buffer */
  for (int li = 0; li < net->n; ++li) {
    orc_layer* l = &net->L[li];
    if (l->kind == PSG_LAYER_LABEL) continue;
    memset(l->grad, 0, n * (size_t)vol3(l) * sizeof(double));
  }
  memset(grads, 0, net->P * sizeof(double));
  for (int li = 0; li < net->n; ++li) { /* every loss seeds its logits (+=) */
    const orc_layer* ls = &net->L[li];
    if (ls->kind == PSG_LAYER_SOFTMAX_LOSS)
      softmax_seed(net, ls, n, ls->out, net->L[ls->d.inputs[0]].grad);
  }
  for (int li = net->n - 1; li >= 0; --li) {
    orc_layer* l = &net->L[li];
    if (l->kind == PSG_LAYER_DATA || l->kind == PSG_LAYER_LABEL ||
        l->kind == PSG_LAYER_SOFTMAX_LOSS)
      continue;
    if (l->kind == PSG_LAYER_CONCAT) { /* dx_i += dy[:, off_i : off_i + c_i] */
      const int64_t hw = l->h * l->w;
      int64_t off = 0;
      for (int i = 0; i < l->d.n_inputs; ++i) {
        orc_layer* in = &net->L[l->d.inputs[i]];
        const int64_t ci = in->c;
        for (size_t b = 0; b < n; ++b) {
          const double* src = l->grad + ((int64_t)b * l->c + off) * hw;
          double* dst = in->grad + (int64_t)b * ci * hw;
          for (int64_t e = 0; e < ci * hw; ++e) dst[e] += src[e];
        }
        off += ci;
      }
      continue;
    }
    double* dx = net->L[l->d.inputs[0]].grad;
    if (net->L[l->d.inputs[0]].kind == PSG_LAYER_DATA && l->kind == PSG_LAYER_CONV) {
      /* the reference also computes the (unused) data-layer gradient; the
       * value is never observable, so it is skipped here */
      dx = NULL;
    }
    layer_backward_impl(net, li, n, l->grad, dx, grads + l->poff);
  }
  if (!all_finite(grads, net->P)) {
    set_err("backward: produced a non-finite value");
    return PSG_ERUNTIME;
  }
  if (loss) *loss = net->last_loss;
  return PSG_OK;
}

/* model.hpp:90-107 + tensor.hpp:60-71 (+ weight decay / multipliers extension). */
int orc_net_apply_update(orc_net* net, const double* grads) {
  for (int li = 0; li < net->n; ++li) {
    const orc_layer* l = &net->L[li];
    for (int t = 0; t < 2; ++t) {
      const size_t off = l->poff + (t ? l->kcount : 0);
      const size_t cnt = t ? l->bcount : l->kcount;
      if (!cnt) continue;
      const double lr = net->lr * (t ? l->d.lr_mult_b : l->d.lr_mult_w);
      const double wd = net->wd * (t ? l->d.decay_mult_b : l->d.decay_mult_w);
      double* w = net->params + off;
      double* v = net->vel + off;
      const double* g = grads + off;
      for (size_t i = 0; i < cnt; ++i) {
        double gi = g[i];
        if (wd != 0.0) gi = gi + wd * w[i];
        if (net->mu > 0.0) {
          v[i] = net->mu * v[i] + gi;
          w[i] += -lr * v[i];
        } else {
          w[i] += -lr * gi;
        }
      }
      if ((net->mu > 0.0 && !all_finite(v, cnt)) || !all_finite(w, cnt)) {
        set_err("add_scaled_in_place: produced a non-finite value");
        return PSG_ERUNTIME;
      }
    }
  }
  return PSG_OK;
}

int orc_layer_forward(orc_net* net, int layer, size_t n, const double* const* inputs,
                      double* out) {
  if (layer < 0 || layer >= net->n) return PSG_EINVAL;
  orc_layer* l = &net->L[layer];
  if (l->kind == PSG_LAYER_SOFTMAX_LOSS) {
    set_err("isolated forward: use orc_net_forward for the loss layer");
    return PSG_EINVAL;
  }
  for (int i = 0; i < l->d.n_inputs; ++i) l->fin[i] = inputs[i];
  net->train_phase = 1;
  const int rc = layer_forward_impl(net, layer, n);
  net->train_phase = 0;
  if (rc) return rc;
  memcpy(out, l->out, n * (size_t)vol3(l) * sizeof(double));
  return PSG_OK;
}

int orc_layer_backward(orc_net* net, int layer, size_t n, const double* dy, double* dx,
                       double* dparams) {
  if (layer < 0 || layer >= net->n) return PSG_EINVAL;
  orc_layer* l = &net->L[layer];
  const orc_layer* src = &net->L[l->d.inputs[0]];
  if (dx) memset(dx, 0, n * (size_t)vol3(src) * sizeof(double));
  if (dparams) memset(dparams, 0, (l->kcount + l->bcount) * sizeof(double));
  layer_backward_impl(net, layer, n, dy, dx, dparams);
  return PSG_OK;
}

/* weights.hpp:90-107 / tensor.hpp:166-179: acc = 0; acc += w_k ascending; acc /= K */
void orc_weights_mean(const double* const* items, int k, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = 0.0;
  for (int j = 0; j < k; ++j)
    for (size_t i = 0; i < n; ++i) out[i] += items[j][i];
  const double kk = (double)k;
  for (size_t i = 0; i < n; ++i) out[i] /= kk;
}

/* weights.hpp:66-82: FNV-1a over layer names and raw fp64 bytes. */
uint64_t orc_weights_digest(const orc_net* net, const double* flat) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int li = 0; li < net->n; ++li) {
    const orc_layer* l = &net->L[li];
    const unsigned char* nb = (const unsigned char*)l->d.name;
    for (size_t i = 0; i < strlen(l->d.name); ++i) {
      h ^= nb[i];
      h *= 0x100000001b3ULL;
    }
    const unsigned char* b = (const unsigned char*)(flat + l->poff);
    for (size_t i = 0; i < (l->kcount + l->bcount) * sizeof(double); ++i) {
      h ^= b[i];
      h *= 0x100000001b3ULL;
    }
  }
  return h;
}

/* -------------------------------------------------------- run_sparknet ---- */
typedef struct stream_state {
  const uint64_t* shard;
  size_t n, batch;
  uint64_t seed, epoch;
  uint64_t* order;
  size_t cursor;
} stream_state;

static void stream_next(stream_state* s, const double* images, const int32_t* labels, size_t dim,
                        double* bimg, int32_t* blab) {
  if ((s->cursor + 1) * s->batch > s->n) { /* data.hpp:324-327 */
    ++s->epoch;
    orc_epoch_order(s->shard, s->n, s->seed, s->epoch, s->order);
    s->cursor = 0;
  }
  const uint64_t* idx = s->order + s->cursor * s->batch;
  for (size_t i = 0; i < s->batch; ++i) { /* data.hpp:292-304 gather_batch */
    memcpy(bimg + i * dim, images + idx[i] * dim, dim * sizeof(double));
    blab[i] = labels[idx[i]];
  }
  ++s->cursor;
}

typedef struct worker_job {
  orc_net* net;
  stream_state* stream;
  const orc_sparknet_args* a;
  const double* bcast;
  double* slot;
  double *bimg, *grads;
  int32_t* blab;
  long steps;
  int rc;
} worker_job;

static int train_steps(orc_net* net, stream_state* s, const orc_sparknet_args* a, long steps,
                       double* bimg, int32_t* blab, double* grads) {
  const size_t dim = (size_t)a->c * a->h * a->w;
  for (long t = 0; t < steps; ++t) { /* model.hpp:111-118 */
    stream_next(s, a->train_images, a->train_labels, dim, bimg, blab);
    int rc = orc_net_backward(net, bimg, blab, a->batch, NULL, grads);
    if (!rc) rc = orc_net_apply_update(net, grads);
    if (rc) return rc;
    net->dropout_step++;
  }
  return PSG_OK;
}

static void* worker_main(void* p) {
  worker_job* j = (worker_job*)p;
  orc_net_set_weights(j->net, j->bcast);
  j->rc = train_steps(j->net, j->stream, j->a, j->steps, j->bimg, j->blab, j->grads);
  orc_net_get_weights(j->net, j->slot);
  return NULL;
}

typedef struct pool_arg {
  worker_job* jobs;
  int k, t, threads;
} pool_arg;

static void* pool_main(void* p) {
  pool_arg* pa = (pool_arg*)p;
  for (int k = pa->t; k < pa->k; k += pa->threads) worker_main(&pa->jobs[k]);
  return NULL;
}

/* schemes.hpp:134-139 + model.hpp:122-136 + tensor.hpp:187-201 */
static double evaluate(orc_net* net, const orc_sparknet_args* a, double* bimg, int32_t* blab,
                       double* probs) {
  const size_t dim = (size_t)a->c * a->h * a->w;
  const int C = net->classes;
  long correct = 0, total = 0;
  size_t cursor = 0;
  for (long s = 0; s < a->eval_steps; ++s) {
    if ((cursor + 1) * a->batch > a->eval_n) cursor = 0;
    for (size_t i = 0; i < a->batch; ++i) {
      const size_t r = cursor * a->batch + i;
      memcpy(bimg + i * dim, a->eval_images + r * dim, dim * sizeof(double));
      blab[i] = a->eval_labels[r];
    }
    ++cursor;
    if (orc_net_forward(net, bimg, blab, a->batch, 0, NULL, probs)) return -1.0;
    for (size_t i = 0; i < a->batch; ++i) {
      int best = 0;
      for (int j = 1; j < C; ++j)
        if (probs[i * C + j] > probs[i * C + best]) best = j;
      correct += best == blab[i] ? 1 : 0;
    }
    total += (long)a->batch;
  }
  return (double)correct / (double)total;
}

long orc_run_sparknet(const orc_sparknet_args* a, orc_record* records, long max_records,
                      uint64_t* warm_digest, double* round_weights) {
  if (a->workers < 1 || a->tau < 1 || a->rounds < 0 || a->warm < 0) {
    set_err("run_sparknet: bad arguments");
    return -1;
  }
  const int K = a->workers;
  uint64_t* perm = (uint64_t*)malloc(a->train_n * sizeof(uint64_t));
  uint64_t* offs = (uint64_t*)malloc((size_t)(K + 1) * sizeof(uint64_t));
  if (orc_shard(a->train_n, K, a->seed, perm, offs)) {
    free(perm);
    free(offs);
    return -1;
  }
  for (int k = 0; k < K; ++k) {
    if (offs[k + 1] - offs[k] < a->batch) {
      set_err("run_sparknet: shard smaller than the batch size");
      free(perm);
      free(offs);
      return -1;
    }
  }
  const size_t dim = (size_t)a->c * a->h * a->w;
  orc_net* master = orc_net_create(a->layers, a->n_layers, a->seed);
  orc_net_set_sgd(master, a->lr, a->momentum, a->weight_decay);
  const size_t P = master->P;
  worker_job* jobs = (worker_job*)calloc((size_t)K, sizeof(worker_job));
  stream_state* streams = (stream_state*)calloc((size_t)K, sizeof(stream_state));
  double* current = (double*)malloc(P * sizeof(double));
  double* slots = (double*)malloc((size_t)K * P * sizeof(double));
  const double** items = (const double**)malloc((size_t)K * sizeof(double*));
  for (int k = 0; k < K; ++k) {
    stream_state* s = &streams[k];
    s->shard = perm + offs[k];
    s->n = offs[k + 1] - offs[k];
    s->batch = a->batch;
    s->seed = orc_worker_stream_seed(a->seed, k);
    s->order = (uint64_t*)malloc(s->n * sizeof(uint64_t));
    orc_epoch_order(s->shard, s->n, s->seed, 0, s->order);
    jobs[k].net = orc_net_create(a->layers, a->n_layers, a->seed);
    orc_net_set_sgd(jobs[k].net, a->lr, a->momentum, a->weight_decay);
    jobs[k].stream = s;
    jobs[k].a = a;
    jobs[k].bcast = current;
    jobs[k].slot = slots + (size_t)k * P;
    jobs[k].bimg = (double*)malloc(a->batch * dim * sizeof(double));
    jobs[k].blab = (int32_t*)malloc(a->batch * sizeof(int32_t));
    jobs[k].grads = (double*)malloc((P ? P : 1) * sizeof(double));
    jobs[k].steps = a->tau;
    items[k] = jobs[k].slot;
  }
  long nrec = 0;
  double* probs = (double*)malloc(a->batch * (size_t)master->classes * sizeof(double));
  /* schemes.hpp:312-317: warm start on worker 0's (shared) stream */
  int rc = train_steps(master, &streams[0], a, a->warm, jobs[0].bimg, jobs[0].blab, jobs[0].grads);
  orc_net_get_weights(master, current);
  if (warm_digest) *warm_digest = orc_weights_digest(master, current);
  const int threads = a->threads < 1 ? 1 : (a->threads > K ? K : a->threads);
  for (long round = 1; !rc && round <= a->rounds; ++round) {
    if (threads == 1) {
      for (int k = 0; k < K; ++k) worker_main(&jobs[k]);
    } else {
      pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
      pool_arg* pa = (pool_arg*)malloc((size_t)threads * sizeof(pool_arg));
      for (int t = 0; t < threads; ++t) {
        pa[t].jobs = jobs;
        pa[t].k = K;
        pa[t].t = t;
        pa[t].threads = threads;
        pthread_create(&th[t], NULL, pool_main, &pa[t]);
      }
      for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
      free(th);
      free(pa);
    }
    for (int k = 0; k < K && !rc; ++k) rc = jobs[k].rc;
    if (rc) break;
    orc_weights_mean(items, K, P, current); /* schemes.hpp:336 */
    if (!all_finite(current, P)) {
      set_err("mean_collection: produced a non-finite value");
      rc = PSG_ERUNTIME;
      break;
    }
    orc_net_set_weights(master, current);
    if (round_weights) memcpy(round_weights + (size_t)(round - 1) * P, current, P * sizeof(double));
    const double sim = (double)a->warm * a->compute_seconds +
                       (double)round * ((double)a->tau * a->compute_seconds + a->sync_seconds);
    const double acc = a->skip_eval ? 0.0 : evaluate(master, a, jobs[0].bimg, jobs[0].blab, probs);
    if (nrec < max_records) {
      records[nrec].serial_iters = a->warm;
      records[nrec].parallel_iters = (long)a->tau * round;
      records[nrec].rounds = round;
      records[nrec].sim_time = sim;
      records[nrec].accuracy = acc;
    }
    ++nrec;
    if (!a->skip_eval && acc >= a->target_accuracy) break;
  }
  for (int k = 0; k < K; ++k) {
    orc_net_destroy(jobs[k].net);
    free(streams[k].order);
    free(jobs[k].bimg);
    free(jobs[k].blab);
    free(jobs[k].grads);
  }
  orc_net_destroy(master);
  free(jobs);
  free(streams);
  free(current);
  free(slots);
  free(items);
  free(probs);
  free(perm);
  free(offs);
  return rc ? -1 : nrec;
}

/* schemes.hpp:201-262 (run_naive), restated over the same stream / update helpers. */
long orc_run_naive(const orc_sparknet_args* a, long iter_budget, long eval_every,
                   orc_record* records, long max_records, double* step_weights) {
  const int K = a->workers;
  if (K < 1) {
    set_err("run_naive: need at least one worker");
    return -1;
  }
  if (a->batch % (size_t)K != 0) {
    set_err("run_naive: worker count must divide the batch size");
    return -1;
  }
  if (eval_every < 1) {
    set_err("run_naive: eval_every must be >= 1");
    return -1;
  }
  if (iter_budget < 0) {
    set_err("run_naive: negative budget");
    return -1;
  }
  uint64_t* perm = (uint64_t*)malloc((a->train_n ? a->train_n : 1) * sizeof(uint64_t));
  uint64_t offs[2];
  if (orc_shard(a->train_n, 1, a->seed, perm, offs)) { /* shard(*train, 1, seed) */
    free(perm);
    return -1;
  }
  if (offs[1] - offs[0] < a->batch) {
    set_err("batch iterator: batch size exceeds shard size");
    free(perm);
    return -1;
  }
  const size_t dim = (size_t)a->c * a->h * a->w, part = a->batch / (size_t)K;
  orc_net* net = orc_net_create(a->layers, a->n_layers, a->seed);
  if (!net) {
    free(perm);
    return -1;
  }
  orc_net_set_sgd(net, a->lr, a->momentum, a->weight_decay);
  const size_t P = net->P;
  stream_state st;
  memset(&st, 0, sizeof st);
  st.shard = perm;
  st.n = offs[1] - offs[0];
  st.batch = a->batch;
  st.seed = orc_worker_stream_seed(a->seed, 0); /* make_worker_iterator(shards, 0, ...) */
  st.order = (uint64_t*)malloc(st.n * sizeof(uint64_t));
  orc_epoch_order(st.shard, st.n, st.seed, 0, st.order);
  double* bimg = (double*)malloc(a->batch * dim * sizeof(double));
  int32_t* blab = (int32_t*)malloc(a->batch * sizeof(int32_t));
  double* grads = (double*)malloc((size_t)K * (P ? P : 1) * sizeof(double));
  const double** items = (const double**)malloc((size_t)K * sizeof(double*));
  double* mean = (double*)malloc((P ? P : 1) * sizeof(double));
  double* probs = (double*)malloc(a->batch * (size_t)net->classes * sizeof(double));
  const double sub = a->sublinearity > 0.0 ? a->sublinearity : 1.0;
  const double step_s = (sub == 1.0 ? a->compute_seconds / (double)K
                                    : a->compute_seconds * pow(1.0 / (double)K, sub)) +
                        a->sync_seconds; /* naive_step_seconds, schemes.hpp:56-61 */
  long iters = 0, nrec = 0;
  int rc = PSG_OK;
  while (!rc && iters < iter_budget) {
    const long chunk = eval_every < iter_budget - iters ? eval_every : iter_budget - iters;
    for (long s = 0; !rc && s < chunk; ++s) {
      stream_next(&st, a->train_images, a->train_labels, dim, bimg, blab);
      for (int k = 0; !rc && k < K; ++k) { /* per-part gradients, schemes.hpp:235-246 */
        items[k] = grads + (size_t)k * P;
        rc = orc_net_backward(net, bimg + (size_t)k * part * dim, blab + (size_t)k * part, part,
                              NULL, grads + (size_t)k * P);
      }
      if (rc) break;
      orc_weights_mean(items, K, P, mean); /* schemes.hpp:248 */
      rc = orc_net_apply_update(net, mean);
      net->dropout_step++;
      ++iters;
      if (step_weights) orc_net_get_weights(net, step_weights + (size_t)(iters - 1) * P);
    }
    if (rc) break;
    const double acc = evaluate(net, a, bimg, blab, probs);
    if (nrec < max_records) {
      records[nrec].serial_iters = iters;
      records[nrec].parallel_iters = 0;
      records[nrec].rounds = iters;
      records[nrec].sim_time = (double)iters * step_s;
      records[nrec].accuracy = acc;
    }
    ++nrec;
    if (acc >= a->target_accuracy) break;
  }
  orc_net_destroy(net);
  free(perm);
  free(st.order);
  free(bimg);
  free(blab);
  free(grads);
  free(items);
  free(mean);
  free(probs);
  return rc ? -1 : nrec;
}
