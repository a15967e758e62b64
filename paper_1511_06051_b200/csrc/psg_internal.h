// Internal declarations of libpsg (B200-native SparkNet hot path).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/psg.h"

namespace psg {

// Exceptions mapped 1:1 onto psg_status by the C ABI layer (api.cpp).
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define PSG_CUDA(x) ::psg::cuda_check((x), #x, __FILE__, __LINE__)

// Scoped device selection: every entry point sets the device of the object it
// touches (SURVEY §8(b) "Every entry point sets the device itself").
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) PSG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------- host rng --
uint64_t splitmix64(uint64_t x);
uint64_t derive_seed(uint64_t base, const uint64_t* parts, int nparts);
inline uint64_t derive_seed1(uint64_t base, uint64_t a) { return derive_seed(base, &a, 1); }
inline uint64_t derive_seed2(uint64_t base, uint64_t a, uint64_t b) {
  const uint64_t p[2] = {a, b};
  return derive_seed(base, p, 2);
}
constexpr uint64_t kStreamWeights = 0x57454947ULL;
constexpr uint64_t kStreamShard = 0x53484152ULL;
constexpr uint64_t kStreamWorker = 0x574f524bULL;
constexpr uint64_t kStreamData = 0x44415441ULL;
constexpr uint64_t kStreamDropout = 0x44524f50ULL;

struct Rng {
  uint64_t state;
  double spare = 0.0;
  bool has_spare = false;
  explicit Rng(uint64_t s) : state(s) {}
  uint64_t next_u64();
  double uniform();
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal();
  void shuffle(uint64_t* v, size_t n);
};

void shard_perm(size_t n, int workers, uint64_t seed, uint64_t* perm, uint64_t* offsets);
uint64_t worker_stream_seed(uint64_t global_seed, int worker);
void epoch_order(const uint64_t* shard, size_t n, uint64_t stream_seed, uint64_t epoch,
                 uint64_t* order);
void generate_synthetic(int classes, size_t c, size_t h, size_t w, size_t per_class,
                        double separation, uint64_t seed, uint64_t variant, double* images,
                        int32_t* labels);
void synthetic_means(int classes, size_t c, size_t h, size_t w, double separation, uint64_t seed,
                     double* means);
uint64_t synthetic_noise_seed(uint64_t seed, uint64_t variant);
// load_idx / load_csv (data.hpp:163-255): parsed on the host with the reference's checks.
struct IdxData {
  uint32_t n = 0, h = 0, w = 0;
  int classes = 0;
  std::vector<unsigned char> pixels;  // [n][h][w]
  std::vector<int32_t> labels;
};
IdxData read_idx(const std::string& images_path, const std::string& labels_path);
struct CsvData {
  std::vector<float> images;  // NCHW, p / 255 rounded to fp32
  std::vector<int32_t> labels;
};
CsvData read_csv(const std::string& path, size_t channels, size_t height, size_t width,
                 int num_classes);
// images[i] = (float)(pixels[i] / 255.0) on the device (single channel: NCHW == NHWC).
void ingest_u8_to_f32(const unsigned char* pixels, size_t n, float* images, cudaStream_t s);
// Device generator with generate_synthetic's distribution (exact class means; counter-based
// within-class noise): writes NHWC fp32 rows [n][h][w][c] and labels.
void synthetic_rows_device(const float* d_means, int classes, int c, int h, int w,
                           size_t per_class, uint64_t noise_seed, float* images, int32_t* labels,
                           cudaStream_t s);

// ------------------------------------------------------------- kernel API ---
// NHWC everywhere.  Conv kernels are stored [F][kh][kw][cs_in/G]; a linear
// layer is a 1x1 conv over a 1x1 "image" whose channels are the producer's
// flattened (h, w, c) features.
struct ConvGeom {
  int n = 0;             // batch
  int H = 0, W = 0;      // input spatial
  int cs_in = 0;         // input channel stride (>= logical channels; data layer may be padded)
  int OH = 0, OW = 0;    // output spatial
  int F = 0;             // output channels (= output channel stride)
  int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
  int G = 1;             // groups
  int kp = 0;            // row stride of the weight matrix (>= Kf, 16-byte multiple); 0 = Kf
  int tc_pair = 0;       // tcgen05 CTA pairs: PSG_TC_PAIR_AUTO / _NEVER / _ALWAYS (psg.h)
  __host__ __device__ int Cgs() const { return cs_in / G; }
  __host__ __device__ int Fg() const { return F / G; }
  // reduction length of fprop / row length of dW
  __host__ __device__ int Kf() const { return kh * kw * Cgs(); }
  // weight row stride: W[f][Kp], dW[f][Kp]
  __host__ __device__ int Kp() const { return kp ? kp : Kf(); }
};

enum class Mode { Strict = 0, Tf32 = 1 };

struct Workspace {
  float* ptr = nullptr;
  size_t elems = 0;
};

// All three passes may split K across blocks (fixed-order second-stage sums);
// the shared workspace must hold conv_workspace_elems() floats.
// `col` (conv_col_elems floats, may be null) holds an im2col matrix written by fprop (or by
// wgrad itself) and read by the same step's wgrad when a TF32 layer takes an im2col route.
// x_s2d: the space-to-depth input x' is already in `col` (written by gather_s2d).
void conv_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
                bool relu, const Workspace& ws, float* col, Mode mode, cudaStream_t s,
                bool x_s2d = false);
// A strided first conv on the space-to-depth route (TF32): its input can be gathered
// straight into x' (col) from the dataset rows idx[cursor * g.n + b] (+ the labels).
bool conv_s2d_input(const ConvGeom& g, Mode mode);
// The same from a host-fed NCHW batch already in device memory (no labels).
void stage_s2d_nchw(const ConvGeom& g, const float* src, int C, float* col, cudaStream_t s);
void gather_s2d(const ConvGeom& g, const float* ds_images, const int32_t* ds_labels,
                const uint32_t* idx, const int* cursor, int src_cs, float* col, int32_t* labels,
                cudaStream_t s);
// relu_mask (tensor-core path only, see conv_dgrad_masks): dx = (relu_mask > 0 ? dgrad : 0)
// (+ dx when accumulating) — the backward of a ReLU whose only consumer is this layer.
// col: the layer's conv_col_elems scratch (holds a K-major weight copy for some dgrads).
void conv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                const Workspace& ws, Mode mode, cudaStream_t s, const float* relu_mask = nullptr,
                float* col = nullptr);
bool conv_dgrad_masks(const ConvGeom& g, Mode mode);
// dW [F][Kp] and db [F] (written, not accumulated).
void conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                const Workspace& ws, float* col, Mode mode, cudaStream_t s);
size_t conv_workspace_elems(const ConvGeom& g, Mode mode);
size_t conv_col_elems(const ConvGeom& g, Mode mode);
int conv_launches(const ConvGeom& g, int which, Mode mode);  // 0 fprop 1 dgrad 2 wgrad

struct PoolGeom {
  int n = 0, H = 0, W = 0, C = 0, OH = 0, OW = 0;
  int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
  int method = 0;
};
void pool_fwd(const PoolGeom& g, const float* x, float* y, uint8_t* route, cudaStream_t s);
// relu_mask: dx = (relu_mask > 0 ? pool gradient : 0) (+ dx) — a folded ReLU backward.
void pool_bwd(const PoolGeom& g, const float* dy, const uint8_t* route, float* dx,
              bool accumulate, cudaStream_t s, const float* relu_mask = nullptr);

void relu_fwd(const float* x, float* y, size_t n, cudaStream_t s);
// dst += src[0], += src[1], ... in that order (k scratch gradients); returns launches
int grad_accumulate(float* dst, float* const* src, int k, size_t n, cudaStream_t s);
void relu_bwd(const float* x, const float* dy, float* dx, size_t n, bool accumulate,
              cudaStream_t s);

struct LrnGeom {
  int pixels = 0, C = 0, size = 5;
  float alpha = 1e-4f, beta = 0.75f, k = 1.f;
};
// The LRN scale is recomputed in backward from x (not stored).
void lrn_fwd(const LrnGeom& g, const float* x, float* y, cudaStream_t s);
// relu_mask: the LRN's input is a ReLU output; write dx * (x > 0), i.e. the gradient at
// the ReLU's input (the ReLU's own backward is folded in).
void lrn_bwd(const LrnGeom& g, const float* x, const float* dy, float* dx, bool accumulate,
             cudaStream_t s, bool relu_mask = false);
// LRN -> 3x3 max pool fused (the LRN output is never stored; bitwise the unfused pair).
bool lrn_maxpool_fusable(const LrnGeom& lg, const PoolGeom& pg);
void lrn_maxpool_fwd(const LrnGeom& lg, const PoolGeom& g, const float* x, float* y,
                     uint8_t* route, cudaStream_t s);
// dx (+)= LRN backward of the pool gradient gathered through `route` (relu_mask as lrn_bwd)
void lrn_maxpool_bwd(const LrnGeom& lg, const PoolGeom& g, const float* x, const float* dpool,
                     const uint8_t* route, float* dx, bool accumulate, bool relu_mask,
                     cudaStream_t s);

struct DropGeom {
  int n = 0, C = 0, H = 1, W = 1;  // logical NCHW dims for the counter index
  float ratio = 0.5f;
  uint64_t base_seed = 0;          // derive_seed(net_seed, kStreamDropout, layer)
};
void dropout_fwd(const DropGeom& g, const float* x, float* y, const uint64_t* d_step, bool train,
                 cudaStream_t s);
// relu_mask: a folded ReLU backward (dx (+)= relu_mask > 0 ? dy * mask : 0)
void dropout_bwd(const DropGeom& g, const float* dy, float* dx, const uint64_t* d_step,
                 bool accumulate, cudaStream_t s, const float* relu_mask = nullptr);

// Softmax + mean cross-entropy (x loss_weight) + the loss seed; per-row loss
// terms in fp64, reduced in fixed order into *loss.
// loss (+)= loss_weight * mean CE (accumulate: add to *loss, for several loss layers)
void softmax_loss(const float* logits, const int32_t* labels, int n, int C, double loss_weight,
                  float* probs, float* dlogits, double* row_loss, double* loss, int* flag,
                  bool accumulate, cudaStream_t s);
// Caffe Concat along channels, NHWC: out[pix][off_i + c] = in_i[pix][c]; backward
// dx_i[pix][c] (+)= dy[pix][off_i + c].
void concat_copy(const float* in, int ci, float* out, int ctot, int off, size_t pixels,
                 cudaStream_t s);
// relu_mask: a folded ReLU backward (dx (+)= relu_mask > 0 ? dy slice : 0)
void concat_split(const float* dy, int ctot, int off, float* dx, int ci, size_t pixels,
                  bool accumulate, cudaStream_t s, const float* relu_mask = nullptr);
// All inputs of a concat in one launch (same values as the per-input calls above).
// ConcatSeg i: channels [off_i, off_i + ci) of the concat; forward reads `src`; backward
// writes dx (+)= the slice into `dst` (skipped when null; `mask` = a folded ReLU backward).
// k <= kConcatMax segments, every dst distinct; false = not applicable (caller loops).
constexpr int kConcatMax = 8;
struct ConcatSeg {
  const float* src;
  float* dst;
  const float* mask;
  int ci, off;
  bool acc;
};
bool concat_copy_all(const ConcatSeg* seg, int k, float* out, int ctot, size_t pixels,
                     cudaStream_t s);
bool concat_split_all(const float* dy, int ctot, const ConcatSeg* seg, int k, size_t pixels,
                      cudaStream_t s);
void argmax_count(const float* probs, const int32_t* labels, int n, int C,
                  unsigned long long* correct, cudaStream_t s);

// Batch staging from the HBM-resident dataset: rows idx[cursor*b + i].
void gather_batch(const float* ds_images, const int32_t* ds_labels, const uint32_t* idx,
                  const int* cursor, int b, int pixels, int C, int cs, float* out,
                  int32_t* labels, cudaStream_t s);

void stage_batch_nchw(const float* src, int n, int C, int H, int W, int cs, float* dst,
                      cudaStream_t s);

struct UpdateChunk {
  uint32_t begin, end;  // element range (multiples of 4 except tails)
  float lr, wd;         // effective lr and weight decay for this tensor
};
void sgd_update(const UpdateChunk* chunks, int nchunks, float* w, float* v, const float* g,
                float momentum, int* flag, int* cursor, uint64_t* step, cudaStream_t s);

// Ordered mean of K same-device buffers: fp64 accumulation ascending k, /K, one rounding.
void average_ordered(float* const* bufs, int K, size_t n, int* flag, cudaStream_t s);
void average_ordered_into(float* const* bufs, int K, size_t n, float* out, int* flag,
                          cudaStream_t s);
void scale_inplace(float* x, size_t n, float a, int* flag, cudaStream_t s);
void fill_uniform(float* x, size_t n, uint64_t seed, double lo, double hi, cudaStream_t s);

// ------------------------------------------------- programmatic dependent launch --
// Every kernel of the library is launched with the PDL attribute (launch_k) and starts
// with pdl_enter(): it waits for its stream predecessor to complete (memory flushed)
// before touching global memory, so its launch overlaps the predecessor's tail.  The
// successor is released at exit (an early griddepcontrol.launch_dependents, built with
// -DPSG_PDL_EARLY_TRIGGER, parks waiting CTAs next to the persistent GEMMs and measured
// 2-4% slower on AlexNet / GoogLeNet).  No-ops for a kernel launched without the attribute;
// PSG_PDL=0 launches without it (A/B measurement).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef PSG_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
#endif
bool pdl_enabled();
// a kernel's dynamic shared memory limit raised to the device maximum, once per device
void allow_max_dynamic_smem(const void* kern);

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PSG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// PSG_TC_PROF=1 launch counters, one "index|label|8 counters" line per GEMM launch
std::string tc_prof_report(bool reset);

}  // namespace psg
