// Precision-mode dispatch for the GEMM-shaped layers (conv + linear).
#include "psg_internal.h"

namespace psg {

void conv_fprop_simt(const ConvGeom& g, const float* x, const float* w, const float* bias,
                     float* y, bool relu, cudaStream_t s);
void conv_dgrad_simt(const ConvGeom& g, const float* dy, const float* w, float* dx,
                     bool accumulate, cudaStream_t s);
void conv_wgrad_simt(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                     const Workspace& ws, cudaStream_t s);
size_t wgrad_workspace_elems_simt(const ConvGeom& g);
int wgrad_launches_simt(const ConvGeom& g);

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" +
                    std::to_string(line) + ")");
}

void conv_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
                bool relu, Mode, cudaStream_t s) {
  conv_fprop_simt(g, x, w, bias, y, relu, s);
}

void conv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                Mode, cudaStream_t s) {
  conv_dgrad_simt(g, dy, w, dx, accumulate, s);
}

void conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                const Workspace& ws, Mode, cudaStream_t s) {
  conv_wgrad_simt(g, x, dy, dw, db, ws, s);
}

size_t wgrad_workspace_elems(const ConvGeom& g, Mode) { return wgrad_workspace_elems_simt(g); }

int conv_launches(const ConvGeom& g, int which, Mode) {
  return which == 2 ? wgrad_launches_simt(g) : 1;
}

}  // namespace psg
