// Precision-mode dispatch for the GEMM-shaped layers (conv + linear):
//   Mode::Strict -> fp32 SIMT implicit GEMM (conv_simt.cu), the 1e-5 parity mode;
//   Mode::Tf32   -> tcgen05 kind::tf32 implicit GEMM (conv_tc.cu) wherever the operands are
//                   TMA-describable (stride 1, channel blocks of 16/32, 16-byte strides), the
//                   SIMT kernel otherwise (e.g. a 3-channel first layer).
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

static bool use_tc(const ConvGeom& g, int which, Mode m) {
  return m == Mode::Tf32 && tc_supported(g, which);
}

void conv_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
                bool relu, const Workspace& ws, Mode m, cudaStream_t s) {
  if (use_tc(g, 0, m))
    tc_fprop(g, x, w, bias, y, relu, ws, s);
  else
    conv_fprop_simt(g, x, w, bias, y, relu, ws, s);
}

void conv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                const Workspace& ws, Mode m, cudaStream_t s) {
  if (use_tc(g, 1, m))
    tc_dgrad(g, dy, w, dx, accumulate, ws, s);
  else
    conv_dgrad_simt(g, dy, w, dx, accumulate, ws, s);
}

void conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                const Workspace& ws, Mode m, cudaStream_t s) {
  if (use_tc(g, 2, m))
    tc_wgrad(g, x, dy, dw, db, ws, s);
  else
    conv_wgrad_simt(g, x, dy, dw, db, ws, s);
}

size_t conv_workspace_elems(const ConvGeom& g, Mode m) {
  return m == Mode::Tf32 ? std::max(conv_workspace_elems_simt(g), tc_workspace_elems(g))
                         : conv_workspace_elems_simt(g);
}

int conv_launches(const ConvGeom& g, int which, Mode m) {
  return use_tc(g, which, m) ? tc_launches(g, which) : conv_launches_simt(g, which);
}

}  // namespace psg
