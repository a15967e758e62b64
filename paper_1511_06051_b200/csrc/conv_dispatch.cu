// Precision-mode dispatch for the GEMM-shaped layers (conv + linear).
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

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" +
                    std::to_string(line) + ")");
}

void conv_fprop(const ConvGeom& g, const float* x, const float* w, const float* bias, float* y,
                bool relu, const Workspace& ws, Mode, cudaStream_t s) {
  conv_fprop_simt(g, x, w, bias, y, relu, ws, s);
}

void conv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                const Workspace& ws, Mode, cudaStream_t s) {
  conv_dgrad_simt(g, dy, w, dx, accumulate, ws, s);
}

void conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* db,
                const Workspace& ws, Mode, cudaStream_t s) {
  conv_wgrad_simt(g, x, dy, dw, db, ws, s);
}

size_t conv_workspace_elems(const ConvGeom& g, Mode) { return conv_workspace_elems_simt(g); }

int conv_launches(const ConvGeom& g, int which, Mode) { return conv_launches_simt(g, which); }

}  // namespace psg
