// The every-tau weight average (weights_mean, weights.hpp:90-107; the
// collect/average/broadcast of schemes.hpp:330-338) as NCCL collectives over
// NVLink on the flat parameter buffer.
//   fast    : one ncclAllReduce with ncclAvg (sum and 1/K fused in NCCL).
//   ordered : reduce-scatter by all-to-all (ncclSend/ncclRecv), an ascending-k fp64
//             accumulation per slice with one rounding, then an in-place allgather
//             — the reference's fixed order, same bus bytes as an allreduce.
// NCCL is bound at run time (dlopen "libnccl.so.2"): the process reuses the copy
// torch already loaded, or the system one.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "runtime.h"

struct psg_comm {
  psg_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  float* scratch = nullptr;
  size_t scratch_elems = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

namespace psg {
namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL unavailable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    if (!api.AllReduce || !api.Send || !api.GroupEnd) err = "NCCL: missing symbols";
  });
  if (!err.empty()) throw CudaError(err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}

// Slice of the padded flat buffer owned by `rank` in the ordered reduce-scatter.
size_t slice_elems(size_t P_alloc, int nranks) { return P_alloc / static_cast<size_t>(nranks); }

void ensure_scratch(psg_comm* c, size_t elems) {
  if (c->scratch_elems >= elems) return;
  if (c->scratch) cudaFree(c->scratch);
  PSG_CUDA(cudaMalloc(&c->scratch, elems * sizeof(float)));
  c->scratch_elems = elems;
}

// Average of one flat buffer per comm (count comms driven by this thread).
void average_flat(psg_comm* const* comms, float* const* bufs, const size_t* counts,
                  cudaStream_t const* streams, int* const* flags, int count, int mode) {
  const NcclApi& api = nccl();
  if (mode == PSG_AVERAGE_FAST) {
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < count; ++i) {
      DeviceGuard dg(comms[i]->ctx->device);
      nccl_check(api.AllReduce(bufs[i], bufs[i], counts[i], ncclFloat, ncclAvg, comms[i]->comm,
                               streams[i]),
                 "ncclAllReduce");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    return;
  }
  if (mode != PSG_AVERAGE_ORDERED) throw std::invalid_argument("average: unknown mode");
  // each rank's slice is reduced with float4 loads: counts[i] must split into nranks
  // 4-aligned slices (a net's P_alloc is padded to a multiple of 4 * 840 = 4 * lcm(1..8))
  for (int i = 0; i < count; ++i)
    if (counts[i] % (4 * static_cast<size_t>(comms[i]->nranks)))
      throw std::invalid_argument("average: buffer length not divisible into 4-aligned rank slices");
  nccl_check(api.GroupStart(), "ncclGroupStart");
  for (int i = 0; i < count; ++i) {
    psg_comm* c = comms[i];
    DeviceGuard dg(c->ctx->device);
    const size_t sl = slice_elems(counts[i], c->nranks);
    ensure_scratch(c, sl * c->nranks);
    for (int j = 0; j < c->nranks; ++j) {
      if (j == c->rank) continue;
      nccl_check(api.Send(bufs[i] + j * sl, sl, ncclFloat, j, c->comm, streams[i]), "ncclSend");
      nccl_check(api.Recv(c->scratch + j * sl, sl, ncclFloat, j, c->comm, streams[i]), "ncclRecv");
    }
  }
  nccl_check(api.GroupEnd(), "ncclGroupEnd");
  for (int i = 0; i < count; ++i) {
    psg_comm* c = comms[i];
    DeviceGuard dg(c->ctx->device);
    const size_t sl = slice_elems(counts[i], c->nranks);
    float* own = bufs[i] + c->rank * sl;
    PSG_CUDA(cudaMemcpyAsync(c->scratch + c->rank * sl, own, sl * sizeof(float),
                             cudaMemcpyDeviceToDevice, streams[i]));
    std::vector<float*> parts(c->nranks);
    for (int j = 0; j < c->nranks; ++j) parts[j] = c->scratch + j * sl;
    average_ordered_into(parts.data(), c->nranks, sl, own, flags[i], streams[i]);
  }
  nccl_check(api.GroupStart(), "ncclGroupStart");
  for (int i = 0; i < count; ++i) {
    psg_comm* c = comms[i];
    DeviceGuard dg(c->ctx->device);
    const size_t sl = slice_elems(counts[i], c->nranks);
    nccl_check(api.AllGather(bufs[i] + c->rank * sl, bufs[i], sl, ncclFloat, c->comm, streams[i]),
               "ncclAllGather");
  }
  nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

}  // namespace

void comm_unique_id(unsigned char id[128]) {
  ncclUniqueId u;
  nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
}

psg_comm* comm_create(psg_ctx* ctx, int nranks, int rank, const unsigned char id[128]) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("comm: bad rank");
  DeviceGuard dg(ctx->device);
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  auto* c = new psg_comm;
  c->ctx = ctx;
  c->rank = rank;
  c->nranks = nranks;
  try {
    nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    PSG_CUDA(cudaEventCreate(&c->e0));
    PSG_CUDA(cudaEventCreate(&c->e1));
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

void comm_create_all(psg_ctx* const* ctxs, int ndev, psg_comm** out) {
  std::vector<int> devs(ndev);
  for (int i = 0; i < ndev; ++i) devs[i] = ctxs[i]->device;
  std::vector<ncclComm_t> comms(ndev);
  nccl_check(nccl().CommInitAll(comms.data(), ndev, devs.data()), "ncclCommInitAll");
  for (int i = 0; i < ndev; ++i) {
    DeviceGuard dg(devs[i]);
    auto* c = new psg_comm;
    c->ctx = ctxs[i];
    c->comm = comms[i];
    c->rank = i;
    c->nranks = ndev;
    PSG_CUDA(cudaEventCreate(&c->e0));
    PSG_CUDA(cudaEventCreate(&c->e1));
    out[i] = c;
  }
}

void comm_destroy(psg_comm* c) {
  if (!c) return;
  DeviceGuard dg(c->ctx->device);
  if (c->comm) nccl().CommDestroy(c->comm);
  if (c->scratch) cudaFree(c->scratch);
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  delete c;
}

void comm_average_nets(psg_comm* const* comms, psg_net* const* nets, int count, int mode,
                       int which) {
  std::vector<float*> bufs(count);
  std::vector<size_t> counts(count);
  std::vector<cudaStream_t> streams(count);
  std::vector<int*> flags(count);
  for (int i = 0; i < count; ++i) {
    if (nets[i]->ctx->device != comms[i]->ctx->device)
      throw std::invalid_argument("average: net and communicator on different devices");
    bufs[i] = which ? nets[i]->g : nets[i]->w;
    counts[i] = mode == PSG_AVERAGE_FAST ? nets[i]->P_int : nets[i]->P_alloc;
    streams[i] = nets[i]->stream;
    flags[i] = &nets[i]->dsc->flag;
    if (i && nets[i]->P_int != nets[0]->P_int)
      throw std::invalid_argument("weights_mean: structure mismatch");
  }
  average_flat(comms, bufs.data(), counts.data(), streams.data(), flags.data(), count, mode);
}

int comm_device(const psg_comm* c) { return c->ctx->device; }

void comm_allreduce_avg(psg_comm* c, float* ptr, size_t count, cudaStream_t s) {
  nccl_check(nccl().AllReduce(ptr, ptr, count, ncclFloat, ncclAvg, c->comm, s), "ncclAllReduce");
}

void comm_broadcast_nets(psg_comm* const* comms, psg_net* const* nets, int count, int root) {
  const NcclApi& api = nccl();
  nccl_check(api.GroupStart(), "ncclGroupStart");
  for (int i = 0; i < count; ++i) {
    DeviceGuard dg(comms[i]->ctx->device);
    nccl_check(api.Broadcast(nets[i]->w, nets[i]->w, nets[i]->P_int, ncclFloat, root,
                             comms[i]->comm, nets[i]->stream),
               "ncclBroadcast");
  }
  nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

void comm_average_buffers(psg_comm* const* comms, psg_buffer* const* bufs, int count, int mode,
                          float* device_ms) {
  std::vector<float*> ptrs(count);
  std::vector<size_t> counts(count);
  std::vector<cudaStream_t> streams(count);
  std::vector<int*> flags(count);
  std::vector<int*> dflags(count);
  for (int i = 0; i < count; ++i) {
    DeviceGuard dg(comms[i]->ctx->device);
    if (mode == PSG_AVERAGE_ORDERED && bufs[i]->n % (4 * static_cast<size_t>(comms[i]->nranks)))
      throw std::invalid_argument("average: ordered mode needs n divisible by 4*nranks");
    ptrs[i] = bufs[i]->ptr;
    counts[i] = bufs[i]->n;
    streams[i] = bufs[i]->ctx->stream;
    PSG_CUDA(cudaMalloc(&dflags[i], sizeof(int)));
    PSG_CUDA(cudaMemsetAsync(dflags[i], 0, sizeof(int), streams[i]));
    flags[i] = dflags[i];
    PSG_CUDA(cudaEventRecord(comms[i]->e0, streams[i]));
  }
  average_flat(comms, ptrs.data(), counts.data(), streams.data(), flags.data(), count, mode);
  float worst = 0.f;
  for (int i = 0; i < count; ++i) {
    DeviceGuard dg(comms[i]->ctx->device);
    PSG_CUDA(cudaEventRecord(comms[i]->e1, streams[i]));
    PSG_CUDA(cudaEventSynchronize(comms[i]->e1));
    float ms = 0.f;
    PSG_CUDA(cudaEventElapsedTime(&ms, comms[i]->e0, comms[i]->e1));
    worst = std::max(worst, ms);
    int flag = 0;
    PSG_CUDA(cudaMemcpy(&flag, dflags[i], sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(dflags[i]);
    if (flag) throw std::runtime_error("mean_collection: produced a non-finite value");
  }
  if (device_ms) *device_ms = worst;
}

}  // namespace psg
