// Elementwise / reduction kernels of the training step: ReLU, softmax-loss, argmax,
// the fused SGD update, the ordered weight average.  Every reduction is fixed-order
// (no float atomics), so a step is bitwise reproducible.
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "psg_internal.h"

namespace psg {

// Raise a kernel's dynamic shared memory limit to the device maximum once (per device and
// kernel), instead of setting it to each launch's size right before the launch: two host
// threads launching the same kernel with different sizes (nets driven from several threads)
// could otherwise lower the limit between the other thread's set and launch
// (cudaLaunchKernelEx: invalid argument).
void allow_max_dynamic_smem(const void* kern) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int d = 0;
  PSG_CUDA(cudaGetDevice(&d));
  std::lock_guard<std::mutex> lock(mu);
  if (!done.insert({d, kern}).second) return;
  int optin = 0;
  PSG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d));
  cudaFuncAttributes fa{};
  PSG_CUDA(cudaFuncGetAttributes(&fa, kern));
  PSG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - static_cast<int>(fa.sharedSizeBytes)));
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PSG_PDL");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}
namespace {

inline int grid_for(size_t n, int block = 256, int max_blocks = 148 * 16) {
  const size_t b = (n + block - 1) / block;
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(b, max_blocks)));
}

#define GRID_STRIDE(i, n)                                                          \
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < (n); \
       i += static_cast<size_t>(gridDim.x) * blockDim.x)

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:11-16
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// ------------------------------------------------------------------ relu ---
// model.hpp:319-326 (y = x > 0 ? x : 0) and :484-491 (dx += x > 0 ? dy : 0).
__global__ void relu_fwd_k(const float* __restrict__ x, float* __restrict__ y, size_t n) {
  pdl_enter();
  const size_t n4 = n / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* y4 = reinterpret_cast<float4*>(y);
  GRID_STRIDE(i, n4) {
    float4 v = x4[i];
    v.x = v.x > 0.f ? v.x : 0.f;
    v.y = v.y > 0.f ? v.y : 0.f;
    v.z = v.z > 0.f ? v.z : 0.f;
    v.w = v.w > 0.f ? v.w : 0.f;
    y4[i] = v;
  }
  GRID_STRIDE(j, n - n4 * 4) {
    const size_t i = n4 * 4 + j;
    y[i] = x[i] > 0.f ? x[i] : 0.f;
  }
}

__global__ void relu_bwd_k(const float* __restrict__ x, const float* __restrict__ dy,
                           float* __restrict__ dx, size_t n, int accumulate) {
  pdl_enter();
  const size_t n4 = n / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* g4 = reinterpret_cast<const float4*>(dy);
  float4* d4 = reinterpret_cast<float4*>(dx);
  GRID_STRIDE(i, n4) {
    const float4 xv = x4[i], gv = g4[i];
    float4 r = make_float4(xv.x > 0.f ? gv.x : 0.f, xv.y > 0.f ? gv.y : 0.f,
                           xv.z > 0.f ? gv.z : 0.f, xv.w > 0.f ? gv.w : 0.f);
    if (accumulate) {
      const float4 o = d4[i];
      r.x += o.x;
      r.y += o.y;
      r.z += o.z;
      r.w += o.w;
    }
    d4[i] = r;
  }
  GRID_STRIDE(j, n - n4 * 4) {
    const size_t i = n4 * 4 + j;
    const float g = x[i] > 0.f ? dy[i] : 0.f;
    dx[i] = accumulate ? dx[i] + g : g;
  }
}

// ---------------------------------------------------------- softmax-loss ---
// model.hpp:429-451 + :463-475.  One warp per row; the row math runs in fp64
// (tiny), probabilities and the loss seed are rounded once to fp32.
__global__ void softmax_loss_k(const float* __restrict__ logits, const int32_t* __restrict__ labels,
                               int n, int C, double scale, float* __restrict__ probs,
                               float* __restrict__ dlogits, double* __restrict__ row_loss) {
  pdl_enter();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= n) return;
  const float* row = logits + static_cast<size_t>(warp) * C;
  float mx = -FLT_MAX;
  for (int j = lane; j < C; j += 32) mx = fmaxf(mx, row[j]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (int j = lane; j < C; j += 32) sum += exp(static_cast<double>(row[j]) - mx);
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const int y = labels[warp];
  for (int j = lane; j < C; j += 32) {
    const double p = exp(static_cast<double>(row[j]) - mx) / sum;
    probs[static_cast<size_t>(warp) * C + j] = static_cast<float>(p);
    if (dlogits)
      dlogits[static_cast<size_t>(warp) * C + j] =
          static_cast<float>(p * scale - (j == y ? scale : 0.0));
  }
  if (lane == 0) row_loss[warp] = -((static_cast<double>(row[y]) - mx) - log(sum));
}

// Fixed-order reduction of the per-row losses: loss = sum / n * loss_weight.
__global__ void loss_reduce_k(const double* __restrict__ row_loss, int n, double lw,
                              double* __restrict__ loss, int* __restrict__ flag, int accumulate) {
  pdl_enter();
  __shared__ double part[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += row_loss[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double l = part[0] / n * lw + (accumulate ? *loss : 0.0);
    *loss = l;
    if (!isfinite(l)) *flag = 1;
  }
}

// tensor.hpp:187-201 argmax (lowest index wins) + model.hpp:129-133 count.
__global__ void argmax_count_k(const float* __restrict__ probs, const int32_t* __restrict__ labels,
                               int n, int C, unsigned long long* correct) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* p = probs + static_cast<size_t>(i) * C;
  int best = 0;
  for (int j = 1; j < C; ++j)
    if (p[j] > p[best]) best = j;
  if (best == labels[i]) atomicAdd(correct, 1ULL);  // integer count: order-independent
}

// ---------------------------------------------------------------- update ---
// model.hpp:90-107 + tensor.hpp:60-71 fused into one pass over the flat
// buffer: g' = g + wd*w; v = mu*v + g'; w += -lr*v  (mu = 0: w += -lr*g').
// A sticky flag replaces ensure_finite; block 0 also advances the per-step
// device counters (batch cursor, dropout step) for the next graph replay.
__global__ void sgd_update_k(const UpdateChunk* __restrict__ chunks, float* __restrict__ w,
                             float* __restrict__ v, const float* __restrict__ g, float mu,
                             int* __restrict__ flag, int* __restrict__ cursor,
                             uint64_t* __restrict__ step) {
  pdl_enter();
  const UpdateChunk ch = chunks[blockIdx.x];
  bool bad = false;
  const uint32_t vec_end = ch.begin + ((ch.end - ch.begin) / 4) * 4;
  for (uint32_t i = ch.begin + threadIdx.x * 4; i < vec_end; i += blockDim.x * 4) {
    float4 wv = *reinterpret_cast<float4*>(w + i);
    const float4 gv = *reinterpret_cast<const float4*>(g + i);
    float gg[4] = {gv.x, gv.y, gv.z, gv.w};
    float ww[4] = {wv.x, wv.y, wv.z, wv.w};
    if (ch.wd != 0.f)
      for (int q = 0; q < 4; ++q) gg[q] = fmaf(ch.wd, ww[q], gg[q]);
    if (mu > 0.f) {
      float4 vv = *reinterpret_cast<float4*>(v + i);
      float vq[4] = {vv.x, vv.y, vv.z, vv.w};
      for (int q = 0; q < 4; ++q) {
        vq[q] = fmaf(mu, vq[q], gg[q]);
        ww[q] = fmaf(-ch.lr, vq[q], ww[q]);
        bad |= !isfinite(vq[q]) || !isfinite(ww[q]);
      }
      *reinterpret_cast<float4*>(v + i) = make_float4(vq[0], vq[1], vq[2], vq[3]);
    } else {
      for (int q = 0; q < 4; ++q) {
        ww[q] = fmaf(-ch.lr, gg[q], ww[q]);
        bad |= !isfinite(ww[q]);
      }
    }
    *reinterpret_cast<float4*>(w + i) = make_float4(ww[0], ww[1], ww[2], ww[3]);
  }
  for (uint32_t i = vec_end + threadIdx.x; i < ch.end; i += blockDim.x) {
    float gi = g[i];
    if (ch.wd != 0.f) gi = fmaf(ch.wd, w[i], gi);
    if (mu > 0.f) {
      v[i] = fmaf(mu, v[i], gi);
      w[i] = fmaf(-ch.lr, v[i], w[i]);
      bad |= !isfinite(v[i]);
    } else {
      w[i] = fmaf(-ch.lr, gi, w[i]);
    }
    bad |= !isfinite(w[i]);
  }
  if (bad) *flag = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (cursor) *cursor += 1;
    if (step) *step += 1;
  }
}

// weights.hpp:90-107: acc = 0; acc += w_k for k ascending; acc /= K (fp64, one rounding).
struct PtrPack {
  float* p[64];
};

// out == nullptr: write the mean back into every input; else into out only.
__global__ void average_ordered_k(PtrPack bufs, int K, size_t n, float* out, int* flag) {
  pdl_enter();
  const size_t n4 = n / 4;
  GRID_STRIDE(i, n4) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int k = 0; k < K; ++k) {
      const float4 t = reinterpret_cast<const float4*>(bufs.p[k])[i];
      a0 += t.x;
      a1 += t.y;
      a2 += t.z;
      a3 += t.w;
    }
    const double kk = K;
    const float4 r = make_float4(static_cast<float>(a0 / kk), static_cast<float>(a1 / kk),
                                 static_cast<float>(a2 / kk), static_cast<float>(a3 / kk));
    if (!isfinite(r.x) || !isfinite(r.y) || !isfinite(r.z) || !isfinite(r.w)) *flag = 1;
    if (out)
      reinterpret_cast<float4*>(out)[i] = r;
    else
      for (int k = 0; k < K; ++k) reinterpret_cast<float4*>(bufs.p[k])[i] = r;
  }
  GRID_STRIDE(j, n - n4 * 4) {
    const size_t i = n4 * 4 + j;
    double a = 0.0;
    for (int k = 0; k < K; ++k) a += bufs.p[k][i];
    const float r = static_cast<float>(a / K);
    if (!isfinite(r)) *flag = 1;
    if (out)
      out[i] = r;
    else
      for (int k = 0; k < K; ++k) bufs.p[k][i] = r;
  }
}

__global__ void scale_k(float* x, size_t n, float a, int* flag) {
  pdl_enter();
  GRID_STRIDE(i, n) {
    const float r = x[i] * a;
    if (!isfinite(r)) *flag = 1;
    x[i] = r;
  }
}

__global__ void fill_uniform_k(float* x, size_t n, uint64_t seed, double lo, double hi) {
  pdl_enter();
  GRID_STRIDE(i, n) {
    const double u = static_cast<double>(mix64(seed + i) >> 11) * 0x1.0p-53;
    x[i] = static_cast<float>(lo + (hi - lo) * u);
  }
}

}  // namespace

// dst = ((dst + src[0]) + src[1]) + ... — the branch gradients a fan-out layer received in
// scratch buffers (lanes), added in the order the single-stream backward accumulates them
// (each accumulating pass adds its new value to the old one once), so bitwise equal to it.
struct GradSrcs {
  const float* p[8];
};
__global__ void grad_accumulate_k(float* __restrict__ dst, GradSrcs src, int k, size_t n) {
  pdl_enter();
  const size_t n4 = n / 4;
  float4* d4 = reinterpret_cast<float4*>(dst);
  GRID_STRIDE(i, n4) {
    float4 v = d4[i];
    for (int j = 0; j < k; ++j) {
      const float4 o = reinterpret_cast<const float4*>(src.p[j])[i];
      v.x += o.x;
      v.y += o.y;
      v.z += o.z;
      v.w += o.w;
    }
    d4[i] = v;
  }
  GRID_STRIDE(j, n - n4 * 4) {
    const size_t i = n4 * 4 + j;
    float v = dst[i];
    for (int q = 0; q < k; ++q) v += src.p[q][i];
    dst[i] = v;
  }
}

void relu_fwd(const float* x, float* y, size_t n, cudaStream_t s) {
  launch_k(relu_fwd_k, grid_for(n / 4 + 1), 256, 0, s, x, y, n);
  PSG_CUDA(cudaGetLastError());
}

int grad_accumulate(float* dst, float* const* src, int k, size_t n, cudaStream_t s) {
  int launches = 0;
  for (int j0 = 0; j0 < k; j0 += 8, ++launches) {
    GradSrcs g{};
    const int c = std::min(8, k - j0);
    for (int j = 0; j < c; ++j) g.p[j] = src[j0 + j];
    launch_k(grad_accumulate_k, grid_for(n / 4 + 1), 256, 0, s, dst, g, c, n);
    PSG_CUDA(cudaGetLastError());
  }
  return launches;
}

void relu_bwd(const float* x, const float* dy, float* dx, size_t n, bool accumulate,
              cudaStream_t s) {
  launch_k(relu_bwd_k, grid_for(n / 4 + 1), 256, 0, s, x, dy, dx, n, accumulate);
  PSG_CUDA(cudaGetLastError());
}

void softmax_loss(const float* logits, const int32_t* labels, int n, int C, double loss_weight,
                  float* probs, float* dlogits, double* row_loss, double* loss, int* flag,
                  bool accumulate, cudaStream_t s) {
  const double scale = loss_weight * (1.0 / static_cast<double>(n));
  launch_k(softmax_loss_k, (n * 32 + 255) / 256, 256, 0, s, logits, labels, n, C, scale, probs, dlogits,
                                                      row_loss);
  PSG_CUDA(cudaGetLastError());
  launch_k(loss_reduce_k, 1, 256, 0, s, row_loss, n, loss_weight, loss, flag, accumulate ? 1 : 0);
  PSG_CUDA(cudaGetLastError());
}

namespace {
// Concat copies over (pixel, channel-vector) with 32-bit index math; V = float4 when every
// channel count / offset is a multiple of 4 (GoogLeNet), else float.
__device__ __forceinline__ float relu_gate(float m, float v) { return m > 0.f ? v : 0.f; }
__device__ __forceinline__ float4 relu_gate(float4 m, float4 v) {
  return make_float4(relu_gate(m.x, v.x), relu_gate(m.y, v.y), relu_gate(m.z, v.z),
                     relu_gate(m.w, v.w));
}
__device__ __forceinline__ float4 operator+(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

template <typename V>
__global__ void concat_copy_k(const V* __restrict__ in, int ci, V* __restrict__ out, int ctot,
                              int off, uint32_t total) {
  pdl_enter();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t p = i / ci, c = i - p * ci;
    out[p * ctot + off + c] = in[i];
  }
}
// dx (+)= dy[:, off : off + ci]; with `mask` (a folded ReLU backward) dx (+)= mask > 0 ? . : 0
template <typename V>
__global__ void concat_split_k(const V* __restrict__ dy, int ctot, int off, V* __restrict__ dx,
                               int ci, uint32_t total, int accumulate, const V* __restrict__ mask) {
  pdl_enter();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t p = i / ci, c = i - p * ci;
    V v = dy[p * ctot + off + c];
    if (mask) v = relu_gate(__ldg(mask + i), v);
    dx[i] = accumulate ? dx[i] + v : v;
  }
}
// One launch over every (pixel, vector) of the concat: segment j owns vectors
// [off[j], off[j + 1]) of a pixel (off[k] = ctot); writes / reads coalesced over the concat row.
template <typename V>
struct ConcatAll {
  const V* src[kConcatMax];
  V* dst[kConcatMax];
  const V* mask[kConcatMax];
  int ci[kConcatMax];
  int off[kConcatMax + 1];
  int acc[kConcatMax];
  int k;
};
template <typename V>
__device__ __forceinline__ int concat_seg(const ConcatAll<V>& a, uint32_t c) {
  int j = 0;
  while (j + 1 < a.k && c >= static_cast<uint32_t>(a.off[j + 1])) ++j;
  return j;
}
template <typename V>
__global__ void concat_copy_all_k(ConcatAll<V> a, V* __restrict__ out, int ctot, uint32_t total) {
  pdl_enter();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t p = i / ctot, c = i - p * ctot;
    const int j = concat_seg(a, c);
    out[i] = a.src[j][p * a.ci[j] + (c - a.off[j])];
  }
}
template <typename V>
__global__ void concat_split_all_k(const V* __restrict__ dy, ConcatAll<V> a, int ctot,
                                   uint32_t total) {
  pdl_enter();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t p = i / ctot, c = i - p * ctot;
    const int j = concat_seg(a, c);
    V* dx = a.dst[j];
    if (!dx) continue;
    const uint32_t q = p * a.ci[j] + (c - a.off[j]);
    V v = dy[i];
    if (a.mask[j]) v = relu_gate(__ldg(a.mask[j] + q), v);
    dx[q] = a.acc[j] ? dx[q] + v : v;
  }
}
template <typename V>
bool concat_pack(const ConcatSeg* seg, int k, int ctot, int vw, ConcatAll<V>& a) {
  if (k < 1 || k > kConcatMax || ctot % vw) return false;
  a.k = k;
  int expect = 0;
  for (int j = 0; j < k; ++j) {
    if (seg[j].ci % vw || seg[j].off % vw || seg[j].off != expect) return false;
    for (int i = 0; i < j; ++i)
      if (seg[j].dst && seg[j].dst == seg[i].dst) return false;
    a.src[j] = reinterpret_cast<const V*>(seg[j].src);
    a.dst[j] = reinterpret_cast<V*>(seg[j].dst);
    a.mask[j] = reinterpret_cast<const V*>(seg[j].mask);
    a.ci[j] = seg[j].ci / vw;
    a.off[j] = seg[j].off / vw;
    a.acc[j] = seg[j].acc ? 1 : 0;
    expect += seg[j].ci;
  }
  a.off[k] = ctot / vw;
  return expect == ctot;
}
unsigned concat_blocks(size_t total) {
  return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((total + 255) / 256, 148 * 16)));
}
uint32_t concat_total(size_t pixels, int ctot) {
  if (pixels * static_cast<size_t>(ctot) >= (1ULL << 31))
    throw std::invalid_argument("concat: tensor too large");
  return static_cast<uint32_t>(pixels * static_cast<size_t>(ctot));
}
}  // namespace

void concat_copy(const float* in, int ci, float* out, int ctot, int off, size_t pixels,
                 cudaStream_t s) {
  concat_total(pixels, ctot);
  if (ci % 4 == 0 && ctot % 4 == 0 && off % 4 == 0) {
    const uint32_t total = static_cast<uint32_t>(pixels * ci / 4);
    launch_k(concat_copy_k<float4>, concat_blocks(total), 256, 0, s,
             reinterpret_cast<const float4*>(in), ci / 4, reinterpret_cast<float4*>(out), ctot / 4,
             off / 4, total);
  } else {
    const uint32_t total = static_cast<uint32_t>(pixels * ci);
    launch_k(concat_copy_k<float>, concat_blocks(total), 256, 0, s, in, ci, out, ctot, off, total);
  }
  PSG_CUDA(cudaGetLastError());
}

void concat_split(const float* dy, int ctot, int off, float* dx, int ci, size_t pixels,
                  bool accumulate, cudaStream_t s, const float* relu_mask) {
  concat_total(pixels, ctot);
  if (ci % 4 == 0 && ctot % 4 == 0 && off % 4 == 0) {
    const uint32_t total = static_cast<uint32_t>(pixels * ci / 4);
    launch_k(concat_split_k<float4>, concat_blocks(total), 256, 0, s,
             reinterpret_cast<const float4*>(dy), ctot / 4, off / 4, reinterpret_cast<float4*>(dx),
             ci / 4, total, accumulate ? 1 : 0, reinterpret_cast<const float4*>(relu_mask));
  } else {
    const uint32_t total = static_cast<uint32_t>(pixels * ci);
    launch_k(concat_split_k<float>, concat_blocks(total), 256, 0, s, dy, ctot, off, dx, ci, total,
             accumulate ? 1 : 0, relu_mask);
  }
  PSG_CUDA(cudaGetLastError());
}

bool concat_copy_all(const ConcatSeg* seg, int k, float* out, int ctot, size_t pixels,
                     cudaStream_t s) {
  concat_total(pixels, ctot);
  ConcatAll<float4> a4;
  ConcatAll<float> a1;
  if (concat_pack(seg, k, ctot, 4, a4)) {
    const uint32_t total = static_cast<uint32_t>(pixels * ctot / 4);
    launch_k(concat_copy_all_k<float4>, concat_blocks(total), 256, 0, s, a4,
             reinterpret_cast<float4*>(out), ctot / 4, total);
  } else if (concat_pack(seg, k, ctot, 1, a1)) {
    const uint32_t total = static_cast<uint32_t>(pixels * ctot);
    launch_k(concat_copy_all_k<float>, concat_blocks(total), 256, 0, s, a1, out, ctot, total);
  } else {
    return false;
  }
  PSG_CUDA(cudaGetLastError());
  return true;
}

bool concat_split_all(const float* dy, int ctot, const ConcatSeg* seg, int k, size_t pixels,
                      cudaStream_t s) {
  concat_total(pixels, ctot);
  ConcatAll<float4> a4;
  ConcatAll<float> a1;
  if (concat_pack(seg, k, ctot, 4, a4)) {
    const uint32_t total = static_cast<uint32_t>(pixels * ctot / 4);
    launch_k(concat_split_all_k<float4>, concat_blocks(total), 256, 0, s,
             reinterpret_cast<const float4*>(dy), a4, ctot / 4, total);
  } else if (concat_pack(seg, k, ctot, 1, a1)) {
    const uint32_t total = static_cast<uint32_t>(pixels * ctot);
    launch_k(concat_split_all_k<float>, concat_blocks(total), 256, 0, s, dy, a1, ctot, total);
  } else {
    return false;
  }
  PSG_CUDA(cudaGetLastError());
  return true;
}

void argmax_count(const float* probs, const int32_t* labels, int n, int C,
                  unsigned long long* correct, cudaStream_t s) {
  launch_k(argmax_count_k, (n + 255) / 256, 256, 0, s, probs, labels, n, C, correct);
  PSG_CUDA(cudaGetLastError());
}

void sgd_update(const UpdateChunk* chunks, int nchunks, float* w, float* v, const float* g,
                float momentum, int* flag, int* cursor, uint64_t* step, cudaStream_t s) {
  launch_k(sgd_update_k, nchunks, 256, 0, s, chunks, w, v, g, momentum, flag, cursor, step);
  PSG_CUDA(cudaGetLastError());
}

void average_ordered_into(float* const* bufs, int K, size_t n, float* out, int* flag,
                          cudaStream_t s) {
  if (K > 64) throw std::invalid_argument("average: at most 64 buffers");
  PtrPack pp{};
  for (int k = 0; k < K; ++k) pp.p[k] = bufs[k];
  launch_k(average_ordered_k, grid_for(n / 4 + 1), 256, 0, s, pp, K, n, out, flag);
  PSG_CUDA(cudaGetLastError());
}

void average_ordered(float* const* bufs, int K, size_t n, int* flag, cudaStream_t s) {
  average_ordered_into(bufs, K, n, nullptr, flag, s);
}

void scale_inplace(float* x, size_t n, float a, int* flag, cudaStream_t s) {
  launch_k(scale_k, grid_for(n), 256, 0, s, x, n, a, flag);
  PSG_CUDA(cudaGetLastError());
}

void fill_uniform(float* x, size_t n, uint64_t seed, double lo, double hi, cudaStream_t s) {
  launch_k(fill_uniform_k, grid_for(n), 256, 0, s, x, n, seed, lo, hi);
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
