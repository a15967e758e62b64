// Precision-mode dispatch for the GEMM-shaped layers (conv + linear):
//   Mode::Strict -> fp32 SIMT implicit GEMM (conv_simt.cu), the 1e-5 parity mode;
//   Mode::Tf32   -> tcgen05 kind::tf32 implicit GEMM (conv_tc.cu) straight from the NHWC
//                   activations wherever the operands are TMA-rectangle-describable
//                   (stride 1, channel blocks of 16/32);
//                   otherwise (e.g. AlexNet conv1: 3 channels, stride 4) an explicit im2col
//                   buffer, written once in forward and reused by wgrad, turns fprop and
//                   wgrad into 2-D tcgen05 GEMMs; such a layer's dgrad (never needed for a
//                   first layer) stays on the SIMT kernel.
#include <algorithm>

#include "psg_internal.h"

namespace psg {

void conv_fprop_simt(const ConvGeom& g, const float* x, const float* w, const float* bias,
                     float* y, bool relu, const Workspace& ws, cudaStream_t s);
void conv_dgrad_simt(const ConvGeom& g, const float* dy, const float* w, float* dx,
                     bool accumulate, const Workspace& ws, cudaStream_t s);
void conv_wgrad_simt(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                     const Workspace& ws, cudaStream_t s);
size_t conv_workspace_elems_simt(const ConvGeom& g);
int conv_launches_simt(const ConvGeom& g, int which);

bool tc_supported(const ConvGeom& g, int which);
size_t tc_workspace_elems(const ConvGeom& g);
int tc_launches(const ConvGeom& g, int which);
void tc_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
              bool relu, const Workspace& ws, cudaStream_t s);
void tc_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
              const Workspace& ws, cudaStream_t s);
void tc_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
              const Workspace& ws, cudaStream_t s);

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" +
                    std::to_string(line) + ")");
}

namespace {

bool is_linear(const ConvGeom& g) {
  return g.H == 1 && g.W == 1 && g.OH == 1 && g.OW == 1 && g.kh == 1 && g.kw == 1;
}

// The im2col matrix [n*OH*OW][Kp] seen as a linear layer's input (D = Kp).
ConvGeom col_geom(const ConvGeom& g) {
  ConvGeom l;
  l.n = g.n * g.OH * g.OW;
  l.H = l.W = l.OH = l.OW = 1;
  l.cs_in = g.Kp();
  l.F = g.F;
  return l;
}

bool im2col_route(const ConvGeom& g) {
  return !is_linear(g) && g.G == 1 && !tc_supported(g, 0) && tc_supported(col_geom(g), 0) &&
         tc_supported(col_geom(g), 2);
}

// col[pix][k] = x at (b, oh*sh - ph + u, ow*sw - pw + v, c) for k = (u*kw + v)*C + c < Kf,
// 0 for padding taps and for Kf <= k < Kp.  A block owns kPixPerBlock consecutive output
// pixels; thread t owns columns k = t, t + blockDim, ... (tap decode once per column),
// so writes are row-contiguous and all index math is 32-bit.
constexpr int kPixPerBlock = 16;

__global__ void im2col_k(const float* __restrict__ x, ConvGeom g, float* __restrict__ col,
                         uint32_t pixels) {
  const int Kf = g.Kf(), Kp = g.Kp(), C = g.cs_in;
  const uint32_t p0 = blockIdx.x * kPixPerBlock;
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    int ku = 0, kv = 0, c = 0;
    const bool tap = k < Kf;
    if (tap) {
      c = k % C;
      const int t = k / C;
      kv = t % g.kw;
      ku = t / g.kw;
    }
    for (uint32_t p = p0; p < min(pixels, p0 + kPixPerBlock); ++p) {
      float v = 0.f;
      if (tap) {
        const int ow = static_cast<int>(p % g.OW), r = static_cast<int>(p / g.OW);
        const int oh = r % g.OH, b = r / g.OH;
        const int ih = oh * g.sh - g.ph + ku, iw = ow * g.sw - g.pw + kv;
        if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
          v = __ldg(x + ((static_cast<size_t>(b) * g.H + ih) * g.W + iw) * C + c);
      }
      col[static_cast<size_t>(p) * Kp + k] = v;
    }
  }
}

void im2col(const ConvGeom& g, const float* x, float* col, cudaStream_t s) {
  const size_t pixels = static_cast<size_t>(g.n) * g.OH * g.OW;
  if (pixels >= (1ULL << 31)) throw std::invalid_argument("im2col: too many pixels");
  const int blocks = static_cast<int>((pixels + kPixPerBlock - 1) / kPixPerBlock);
  im2col_k<<<blocks, 128, 0, s>>>(x, g, col, static_cast<uint32_t>(pixels));
  PSG_CUDA(cudaGetLastError());
}

bool use_tc(const ConvGeom& g, int which, Mode m) {
  return m == Mode::Tf32 && tc_supported(g, which);
}

}  // namespace

size_t conv_col_elems(const ConvGeom& g, Mode m) {
  if (m != Mode::Tf32 || !im2col_route(g)) return 0;
  return static_cast<size_t>(g.n) * g.OH * g.OW * g.Kp();
}

void conv_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
                bool relu, const Workspace& ws, float* col, Mode m, cudaStream_t s) {
  if (use_tc(g, 0, m)) {
    tc_fprop(g, x, w, bias, y, relu, ws, s);
  } else if (m == Mode::Tf32 && col && im2col_route(g)) {
    im2col(g, x, col, s);
    tc_fprop(col_geom(g), col, w, bias, y, relu, ws, s);
  } else {
    conv_fprop_simt(g, x, w, bias, y, relu, ws, s);
  }
}

void conv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                const Workspace& ws, Mode m, cudaStream_t s) {
  if (use_tc(g, 1, m))
    tc_dgrad(g, dy, w, dx, accumulate, ws, s);
  else
    conv_dgrad_simt(g, dy, w, dx, accumulate, ws, s);
}

void conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                const Workspace& ws, const float* col, Mode m, cudaStream_t s) {
  if (use_tc(g, 2, m))
    tc_wgrad(g, x, dy, dw, db, ws, s);
  else if (m == Mode::Tf32 && col && im2col_route(g))
    tc_wgrad(col_geom(g), col, dy, dw, db, ws, s);  // col written by this step's forward
  else
    conv_wgrad_simt(g, x, dy, dw, db, ws, s);
}

size_t conv_workspace_elems(const ConvGeom& g, Mode m) {
  size_t e = conv_workspace_elems_simt(g);
  if (m == Mode::Tf32) {
    e = std::max(e, tc_workspace_elems(g));
    if (im2col_route(g)) e = std::max(e, tc_workspace_elems(col_geom(g)));
  }
  return e;
}

int conv_launches(const ConvGeom& g, int which, Mode m) {
  if (use_tc(g, which, m)) return tc_launches(g, which);
  if (m == Mode::Tf32 && which != 1 && im2col_route(g))
    return tc_launches(col_geom(g), which) + (which == 0 ? 1 : 0);
  return conv_launches_simt(g, which);
}

}  // namespace psg
