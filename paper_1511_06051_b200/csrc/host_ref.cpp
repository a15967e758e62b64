// Host-side reference semantics kept bit-exact: SplitMix64 streams, shard(),
// ShardBatchIterator epoch order and the synthetic generator.  These are the
// integer / fp64 host pieces of the path; pixels never
// come back through here once uploaded.
#include <cmath>
#include <cstring>

#include "psg_internal.h"

namespace psg {

// rng.hpp:11-16
uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// rng.hpp:20-25
uint64_t derive_seed(uint64_t base, const uint64_t* parts, int nparts) {
  uint64_t s = splitmix64(base);
  for (int i = 0; i < nparts; ++i) s = splitmix64(s ^ parts[i]);
  return s;
}

// rng.hpp:38-43: the counter advances by the golden gamma, then the mixer.
uint64_t Rng::next_u64() {
  state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

double Rng::normal() {  // rng.hpp:54-66
  if (has_spare) {
    has_spare = false;
    return spare;
  }
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  spare = r * std::sin(theta);
  has_spare = true;
  return r * std::cos(theta);
}

void Rng::shuffle(uint64_t* v, size_t n) {  // rng.hpp:69-75
  for (size_t i = n; i > 1; --i) {
    const size_t j = static_cast<size_t>(next_u64() % static_cast<uint64_t>(i));
    std::swap(v[i - 1], v[j]);
  }
}

// data.hpp:261-288
void shard_perm(size_t n, int workers, uint64_t seed, uint64_t* perm, uint64_t* offsets) {
  if (workers < 1) throw std::invalid_argument("shard: need at least one worker");
  if (static_cast<size_t>(workers) > n)
    throw std::invalid_argument("shard: more workers than examples");
  for (size_t i = 0; i < n; ++i) perm[i] = i;
  Rng r(derive_seed1(seed, kStreamShard));
  r.shuffle(perm, n);
  const size_t base = n / static_cast<size_t>(workers), extra = n % static_cast<size_t>(workers);
  size_t pos = 0;
  offsets[0] = 0;
  for (int k = 0; k < workers; ++k) {
    pos += base + (static_cast<size_t>(k) < extra ? 1 : 0);
    offsets[k + 1] = pos;
  }
}

// data.hpp:386-388
uint64_t worker_stream_seed(uint64_t global_seed, int worker) {
  return derive_seed2(global_seed, kStreamWorker, static_cast<uint64_t>(worker));
}

// data.hpp:338-343
void epoch_order(const uint64_t* shard, size_t n, uint64_t stream_seed, uint64_t epoch,
                 uint64_t* order) {
  std::memcpy(order, shard, n * sizeof(uint64_t));
  Rng r(derive_seed1(stream_seed, epoch));
  r.shuffle(order, n);
}

namespace {

// data.hpp:60-92: per-channel coarse grid of normals, bilinear upsampling.
void smooth_pattern(Rng& rng, size_t channels, size_t height, size_t width, bool unit_var,
                    double* pattern, std::vector<double>& nodes) {
  const size_t gh = std::max<size_t>(1, height / 4), gw = std::max<size_t>(1, width / 4);
  nodes.resize((gh + 1) * (gw + 1));
  auto cell = [](size_t i, size_t extent, size_t grid, size_t& lo, double& t) {
    const double f = extent > 1 ? static_cast<double>(i) * static_cast<double>(grid) /
                                      static_cast<double>(extent - 1)
                                : 0.0;
    lo = std::min<size_t>(static_cast<size_t>(f), grid - 1);
    t = f - static_cast<double>(lo);
  };
  const size_t st = gw + 1;
  for (size_t c = 0; c < channels; ++c) {
    for (double& v : nodes) v = rng.normal();
    for (size_t y = 0; y < height; ++y) {
      size_t y0;
      double ty;
      cell(y, height, gh, y0, ty);
      for (size_t x = 0; x < width; ++x) {
        size_t x0;
        double tx;
        cell(x, width, gw, x0, tx);
        const double w00 = (1.0 - ty) * (1.0 - tx), w01 = (1.0 - ty) * tx;
        const double w10 = ty * (1.0 - tx), w11 = ty * tx;
        double v = w00 * nodes[y0 * st + x0] + w01 * nodes[y0 * st + x0 + 1] +
                   w10 * nodes[(y0 + 1) * st + x0] + w11 * nodes[(y0 + 1) * st + x0 + 1];
        if (unit_var) v /= std::sqrt(w00 * w00 + w01 * w01 + w10 * w10 + w11 * w11);
        pattern[(c * height + y) * width + x] = v;
      }
    }
  }
}

}  // namespace

// data.hpp:111-155
// The class means of generate_synthetic (data.hpp:121-131), bit-exact: means [classes][c*h*w].
void synthetic_means(int classes, size_t c, size_t h, size_t w, double separation, uint64_t seed,
                     double* means) {
  if (classes < 1) throw std::invalid_argument("synthetic: need at least one class");
  if (separation < 0.0) throw std::invalid_argument("synthetic: negative separation");
  const size_t dim = c * h * w;
  Rng mean_stream(derive_seed2(seed, kStreamData, 0x4d45414eULL));
  std::vector<double> nodes;
  const double radius = separation / std::sqrt(2.0);
  for (int cls = 0; cls < classes; ++cls) {
    double* mu = means + static_cast<size_t>(cls) * dim;
    smooth_pattern(mean_stream, c, h, w, false, mu, nodes);
    double norm2 = 0.0;
    for (size_t d = 0; d < dim; ++d) norm2 += mu[d] * mu[d];
    const double inv = norm2 > 0.0 ? radius / std::sqrt(norm2) : 0.0;
    for (size_t d = 0; d < dim; ++d) mu[d] *= inv;
  }
}

// Seed of the within-class noise of (seed, variant) (data.hpp:120).
uint64_t synthetic_noise_seed(uint64_t seed, uint64_t variant) {
  const uint64_t np[3] = {kStreamData, 0x4e4f495345ULL, variant};
  return derive_seed(seed, np, 3);
}

void generate_synthetic(int classes, size_t c, size_t h, size_t w, size_t per_class,
                        double separation, uint64_t seed, uint64_t variant, double* images,
                        int32_t* labels) {
  if (classes < 1) throw std::invalid_argument("synthetic: need at least one class");
  if (per_class < 1) throw std::invalid_argument("synthetic: need at least one example per class");
  if (separation < 0.0) throw std::invalid_argument("synthetic: negative separation");
  const size_t dim = c * h * w;
  Rng mean_stream(derive_seed2(seed, kStreamData, 0x4d45414eULL));
  const uint64_t np[3] = {kStreamData, 0x4e4f495345ULL, variant};
  Rng noise_stream(derive_seed(seed, np, 3));
  std::vector<double> nodes, means(dim * static_cast<size_t>(classes)), structure(dim);
  const double radius = separation / std::sqrt(2.0);
  for (int cls = 0; cls < classes; ++cls) {
    double* mu = means.data() + static_cast<size_t>(cls) * dim;
    smooth_pattern(mean_stream, c, h, w, false, mu, nodes);
    double norm2 = 0.0;
    for (size_t d = 0; d < dim; ++d) norm2 += mu[d] * mu[d];
    const double inv = norm2 > 0.0 ? radius / std::sqrt(norm2) : 0.0;
    for (size_t d = 0; d < dim; ++d) mu[d] *= inv;
  }
  const double smooth_scale = 0.7;
  const double white_scale = std::sqrt(1.0 - smooth_scale * smooth_scale);
  size_t row = 0;
  for (int cls = 0; cls < classes; ++cls) {
    const double* mu = means.data() + static_cast<size_t>(cls) * dim;
    for (size_t e = 0; e < per_class; ++e, ++row) {
      labels[row] = cls;
      double* dst = images + row * dim;
      smooth_pattern(noise_stream, c, h, w, true, structure.data(), nodes);
      for (size_t d = 0; d < dim; ++d)
        dst[d] = mu[d] + smooth_scale * structure[d] + white_scale * noise_stream.normal();
    }
  }
}

}  // namespace psg
