// Precision-mode dispatch for the GEMM-shaped layers (conv + linear):
//   Mode::Strict -> fp32 SIMT implicit GEMM (conv_simt.cu), the 1e-5 parity mode;
//   Mode::Tf32   -> tcgen05 kind::tf32 GEMMs (conv_tc.cu):
//     fprop / dgrad straight from the NHWC activations wherever the operands are
//       TMA-rectangle-describable (stride 1, channel blocks of 16/32);
//     otherwise (e.g. AlexNet conv1: 3 channels, stride 4) fprop goes through an explicit
//       im2col matrix (written once per step, reused by wgrad); such a layer's dgrad
//       (never needed for a first layer) stays on the SIMT kernel;
//     wgrad runs multi-tap implicit GEMM tiles from the activations; only layers whose
//       activations TMA cannot tile (stride > 1, C/G < 16) use the im2col matrix.
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
bool tc_wgrad_col_supported(const ConvGeom& g);
size_t tc_wgrad_col_ws_elems(const ConvGeom& g);
int tc_wgrad_col_launches(const ConvGeom& g);
void tc_wgrad_col(const ConvGeom& g, const float* col, const float* dy, float* dw, float* db,
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

// The im2col matrix [n*OH*OW][Kp] seen as a linear layer's input (D = Kp), G = 1.
ConvGeom col_geom(const ConvGeom& g) {
  ConvGeom l;
  l.n = g.n * g.OH * g.OW;
  l.H = l.W = l.OH = l.OW = 1;
  l.cs_in = g.Kp();
  l.F = g.F;
  return l;
}

bool fprop_col_route(const ConvGeom& g) {
  return !is_linear(g) && g.G == 1 && !tc_supported(g, 0) && tc_supported(col_geom(g), 0) &&
         tc_wgrad_col_supported(g);
}

bool wgrad_col_route(const ConvGeom& g) {
  if (is_linear(g) || !tc_wgrad_col_supported(g)) return false;
  return fprop_col_route(g) || !tc_supported(g, 2);
}

// col[g][pix][k] = x at (b, oh*sh - ph + u, ow*sw - pw + v, g*Cgs + c) for
// k = (u*kw + v)*Cgs + c < Kf; 0 for padding taps and for Kf <= k < Kp.  A block owns
// kPixPerBlock consecutive output pixels of one group (their origins decoded once into
// shared memory); thread t owns columns k = t, t + blockDim, ...: per column the
// kPixPerBlock loads are independent (unrolled) and every store row is contiguous.
constexpr int kPixPerBlock = 16;

__global__ void __launch_bounds__(128) im2col_k(const float* __restrict__ x, ConvGeom g,
                                                float* __restrict__ col, uint32_t pixels) {
  __shared__ int s_ih[kPixPerBlock], s_iw[kPixPerBlock], s_base[kPixPerBlock];
  const int Kf = g.Kf(), Kp = g.Kp(), Cgs = g.Cgs(), grp = blockIdx.y;
  const uint32_t p0 = blockIdx.x * kPixPerBlock;
  if (threadIdx.x < kPixPerBlock) {
    const uint32_t p = min(p0 + threadIdx.x, pixels - 1);
    const int ow = static_cast<int>(p % g.OW), r = static_cast<int>(p / g.OW);
    const int oh = r % g.OH, b = r / g.OH;
    s_ih[threadIdx.x] = oh * g.sh - g.ph;
    s_iw[threadIdx.x] = ow * g.sw - g.pw;
    s_base[threadIdx.x] = b * g.H;
  }
  __syncthreads();
  const int np = static_cast<int>(min(static_cast<uint32_t>(kPixPerBlock), pixels - p0));
  float* colg = col + (static_cast<size_t>(grp) * pixels + p0) * Kp;
  const float* xg = x + grp * Cgs;
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    int ku = -(1 << 20), kv = 0, c = 0;  // padding column: every pixel out of range
    if (k < Kf) {
      c = k % Cgs;
      const int t = k / Cgs;
      kv = t % g.kw;
      ku = t / g.kw;
    }
    float v[kPixPerBlock];
#pragma unroll
    for (int i = 0; i < kPixPerBlock; ++i) {
      const int ih = s_ih[i] + ku, iw = s_iw[i] + kv;
      v[i] = (i < np && ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
                 ? __ldg(xg + (static_cast<size_t>(s_base[i] + ih) * g.W + iw) * g.cs_in + c)
                 : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kPixPerBlock; ++i)
      if (i < np) colg[static_cast<size_t>(i) * Kp + k] = v[i];
  }
}

void im2col(const ConvGeom& g, const float* x, float* col, cudaStream_t s) {
  const size_t pixels = static_cast<size_t>(g.n) * g.OH * g.OW;
  if (pixels >= (1ULL << 31)) throw std::invalid_argument("im2col: too many pixels");
  const dim3 grid(static_cast<unsigned>((pixels + kPixPerBlock - 1) / kPixPerBlock), g.G);
  im2col_k<<<grid, 128, 0, s>>>(x, g, col, static_cast<uint32_t>(pixels));
  PSG_CUDA(cudaGetLastError());
}

bool use_tc(const ConvGeom& g, int which, Mode m) {
  return m == Mode::Tf32 && tc_supported(g, which);
}

}  // namespace

size_t conv_col_elems(const ConvGeom& g, Mode m) {
  if (m != Mode::Tf32 || !(fprop_col_route(g) || wgrad_col_route(g))) return 0;
  return static_cast<size_t>(g.G) * g.n * g.OH * g.OW * g.Kp();
}

void conv_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
                bool relu, const Workspace& ws, float* col, Mode m, cudaStream_t s) {
  if (m == Mode::Tf32 && col && fprop_col_route(g)) {
    im2col(g, x, col, s);
    tc_fprop(col_geom(g), col, w, bias, y, relu, ws, s);
  } else if (use_tc(g, 0, m)) {
    tc_fprop(g, x, w, bias, y, relu, ws, s);
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
                const Workspace& ws, float* col, Mode m, cudaStream_t s) {
  if (m == Mode::Tf32 && col && wgrad_col_route(g)) {
    if (!fprop_col_route(g)) im2col(g, x, col, s);  // else written by this step's fprop
    tc_wgrad_col(g, col, dy, dw, db, ws, s);
  } else if (use_tc(g, 2, m)) {
    tc_wgrad(g, x, dy, dw, db, ws, s);
  } else {
    conv_wgrad_simt(g, x, dy, dw, db, ws, s);
  }
}

size_t conv_workspace_elems(const ConvGeom& g, Mode m) {
  size_t e = conv_workspace_elems_simt(g);
  if (m == Mode::Tf32) {
    e = std::max(e, tc_workspace_elems(g));
    if (fprop_col_route(g)) e = std::max(e, tc_workspace_elems(col_geom(g)));
    if (wgrad_col_route(g)) e = std::max(e, tc_wgrad_col_ws_elems(g));
  }
  return e;
}

int conv_launches(const ConvGeom& g, int which, Mode m) {
  if (m == Mode::Tf32 && which == 0 && fprop_col_route(g))
    return 1 + tc_launches(col_geom(g), 0);
  if (m == Mode::Tf32 && which == 2 && wgrad_col_route(g))
    return (fprop_col_route(g) ? 0 : 1) + tc_wgrad_col_launches(g);
  if (use_tc(g, which, m)) return tc_launches(g, which);
  return conv_launches_simt(g, which);
}

}  // namespace psg
