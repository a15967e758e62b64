// Device-side generate_synthetic (and the IDX byte ingestion) (data.hpp:111-155) for AX/GN-sized datasets (SURVEY.md
// §8(f) #3): the reference's noise stream is one serial RNG over every pixel of every row,
// so the device generator keeps the DISTRIBUTION, not the bits:
//   * class means: computed on the host with the reference's mean stream (bit-exact);
//   * per row: a smooth pattern (normal nodes on a (h/4+1) x (w/4+1) grid per channel,
//     bilinear interpolation scaled to unit pixel variance, data.hpp:60-91) times 0.7 plus
//     independent N(0,1) pixel noise times sqrt(1 - 0.49);
//   * the normals come from a counter-based SplitMix64 hash of (noise seed, row, draw) with
//     Box-Muller, so every row is generated independently in parallel.
// Labels are row / per_class (classes in blocks, data.hpp:137-150).  Output is the
// device dataset layout, NHWC fp32.
#include <algorithm>

#include "psg_internal.h"

namespace psg {
namespace {

__device__ __forceinline__ uint64_t mix(uint64_t x) {  // rng.hpp:11-16 finaliser
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// N(0,1) from draw `k` of row `row`: Box-Muller on two 53-bit uniforms.
__device__ __forceinline__ double normal_at(uint64_t key, uint64_t row, uint64_t k) {
  const uint64_t a = mix(key ^ mix(row * 0x2545f4914f6cdd1dULL + 2 * k));
  const uint64_t b = mix(key ^ mix(row * 0x2545f4914f6cdd1dULL + 2 * k + 1));
  const double u1 = (static_cast<double>(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
  const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// One block per row.  Shared memory: the row's grid nodes for every channel.
__global__ void synthetic_rows_k(const float* __restrict__ means, int c, int h, int w,
                                 uint32_t per_class, uint64_t key, float* __restrict__ images,
                                 int32_t* __restrict__ labels) {
  pdl_enter();
  extern __shared__ float nodes[];
  const uint32_t row = blockIdx.x;
  const int gh = max(1, h / 4), gw = max(1, w / 4), nn = (gh + 1) * (gw + 1);
  for (int i = threadIdx.x; i < c * nn; i += blockDim.x)
    nodes[i] = static_cast<float>(normal_at(key, row, static_cast<uint64_t>(i)));
  const int cls = static_cast<int>(row / per_class);
  if (threadIdx.x == 0) labels[row] = cls;
  __syncthreads();
  const float* mu = means + static_cast<size_t>(cls) * c * h * w;  // NCHW
  float* dst = images + static_cast<size_t>(row) * h * w * c;       // NHWC
  const float ws = 0.71414284285428499f;                            // sqrt(1 - 0.7^2)
  const uint32_t dim = static_cast<uint32_t>(c) * h * w;
  for (uint32_t i = threadIdx.x; i < dim; i += blockDim.x) {  // NHWC order: coalesced
    const int ch = static_cast<int>(i % c), pix = static_cast<int>(i / c);
    const int y = pix / w, x = pix % w;
    const float fy = h > 1 ? static_cast<float>(y) * gh / (h - 1) : 0.f;
    const float fx = w > 1 ? static_cast<float>(x) * gw / (w - 1) : 0.f;
    const int y0 = min(static_cast<int>(fy), gh - 1), x0 = min(static_cast<int>(fx), gw - 1);
    const float ty = fy - y0, tx = fx - x0;
    const float w00 = (1.f - ty) * (1.f - tx), w01 = (1.f - ty) * tx, w10 = ty * (1.f - tx),
                w11 = ty * tx;
    const float* nd = nodes + ch * nn;
    const float s = (w00 * nd[y0 * (gw + 1) + x0] + w01 * nd[y0 * (gw + 1) + x0 + 1] +
                     w10 * nd[(y0 + 1) * (gw + 1) + x0] + w11 * nd[(y0 + 1) * (gw + 1) + x0 + 1]) *
                    rsqrtf(w00 * w00 + w01 * w01 + w10 * w10 + w11 * w11);
    const float white =
        static_cast<float>(normal_at(key, row, static_cast<uint64_t>(c) * nn + i));
    dst[i] = mu[(static_cast<size_t>(ch) * h + y) * w + x] + 0.7f * s + ws * white;
  }
}

__global__ void u8_to_f32_k(const unsigned char* __restrict__ px, size_t n,
                            float* __restrict__ out) {
  pdl_enter();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(static_cast<double>(px[i]) / 255.0);
}

}  // namespace

void ingest_u8_to_f32(const unsigned char* pixels, size_t n, float* images, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 16));
  launch_k(u8_to_f32_k, std::max(1u, blocks), 256, 0, s, pixels, n, images);
  PSG_CUDA(cudaGetLastError());
}

void synthetic_rows_device(const float* d_means, int classes, int c, int h, int w,
                           size_t per_class, uint64_t noise_seed, float* images, int32_t* labels,
                           cudaStream_t s) {
  const size_t n = static_cast<size_t>(classes) * per_class;
  if (n >= (1ULL << 31) || static_cast<size_t>(c) * h * w >= (1ULL << 31))
    throw std::invalid_argument("synthetic: too large");
  const int gh = std::max(1, h / 4), gw = std::max(1, w / 4);
  const size_t smem = static_cast<size_t>(c) * (gh + 1) * (gw + 1) * sizeof(float);
  if (smem > 200 * 1024) throw std::invalid_argument("synthetic: node grid too large");
  if (smem > 48 * 1024) allow_max_dynamic_smem(reinterpret_cast<const void*>(synthetic_rows_k));
  launch_k(synthetic_rows_k, static_cast<unsigned>(n), 256, smem, s, 
      d_means, c, h, w, static_cast<uint32_t>(per_class), noise_seed, images, labels);
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
