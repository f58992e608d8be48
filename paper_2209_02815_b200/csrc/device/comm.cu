// comm.cu -- exchanges of the cell-partitioned solve (see comm.cuh).
#include "comm.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>

#include "amg_device.cuh"  // DeviceError, GNW_CUDA_CHECK

namespace gnw {

std::vector<long long> partition_cells(long long N, int world) {
  if (world < 1) throw std::invalid_argument("partition: world size must be >= 1");
  std::vector<long long> lo(world + 1);
  for (int r = 0; r <= world; ++r) {
    const long long x = (N * r) / world;
    lo[r] = (r == world) ? N : std::min(N, (x + 32) / 64 * 64);
  }
  for (int r = 1; r <= world; ++r)
    if (lo[r] < lo[r - 1]) lo[r] = lo[r - 1];
  return lo;
}

// ------------------------------------------------------------------ LocalHub
void LocalHub::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  if (broken_) throw std::runtime_error("partitioned solve: another rank failed");
  const long long gen = generation_;
  if (++arrived_ == world_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
    return;
  }
  cv_.wait(lk, [&] { return generation_ != gen || broken_; });
  if (generation_ == gen) throw std::runtime_error("partitioned solve: another rank failed");
}

void LocalHub::abandon() {
  std::lock_guard<std::mutex> lk(mu_);
  broken_ = true;
  cv_.notify_all();
}

LocalComm::LocalComm(std::shared_ptr<LocalHub> hub, int r) : hub_(std::move(hub)) {
  rank = r;
  world = hub_->world();
}
LocalComm::~LocalComm() = default;

void LocalComm::allgatherv(double* buf, const std::vector<long long>& off, const std::vector<long long>& cnt,
                           cudaStream_t s) {
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));  // my slice is final
  hub_->ptrs()[rank] = buf;
  hub_->barrier();                           // every slice is final and published
  for (int r = 0; r < world; ++r) {
    if (r == rank || cnt[r] == 0) continue;
    GNW_CUDA_CHECK(cudaMemcpyAsync(buf + off[r], hub_->ptrs()[r] + off[r], cnt[r] * sizeof(double),
                                   cudaMemcpyDeviceToDevice, s));
  }
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  hub_->barrier();                           // nobody overwrites a slice another rank still reads
}

void LocalComm::allgather(const double* in, double* out, long long n, cudaStream_t s) {
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  hub_->ptrs()[rank] = in;
  hub_->barrier();
  for (int r = 0; r < world; ++r)
    GNW_CUDA_CHECK(cudaMemcpyAsync(out + static_cast<long long>(r) * n, hub_->ptrs()[r], n * sizeof(double),
                                   cudaMemcpyDeviceToDevice, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  hub_->barrier();
}

void LocalComm::alltoallv(const std::vector<const double*>& send, const std::vector<long long>&,
                          const std::vector<double*>& recv, const std::vector<long long>& rcnt, cudaStream_t s) {
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  for (int q = 0; q < world; ++q) hub_->table()[rank][q] = send[q];
  hub_->barrier();
  for (int q = 0; q < world; ++q)
    if (rcnt[q] > 0)
      GNW_CUDA_CHECK(cudaMemcpyAsync(recv[q], hub_->table()[q][rank], rcnt[q] * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
  GNW_CUDA_CHECK(cudaStreamSynchronize(s));
  hub_->barrier();
}

// ------------------------------------------------------------------- NCCL
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.Broadcast && a.Send && a.Recv && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
}

const NcclApi& nccl_or_throw() {
  const NcclApi& a = nccl();
  if (!a.ok) throw DeviceError("partitioned solve: " + a.why);
  return a;
}
}  // namespace

bool nccl_available(std::string* why) {
  const NcclApi& a = nccl();
  if (!a.ok && why) *why = a.why;
  return a.ok;
}

void nccl_unique_id(unsigned char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  nccl_check(nccl_or_throw().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
}

NcclComm::NcclComm(const unsigned char* id, int r, int w, int device) {
  rank = r;
  world = w;
  const NcclApi& a = nccl_or_throw();
  GNW_CUDA_CHECK(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclComm_t c = nullptr;
  nccl_check(a.CommInitRank(&c, w, uid, r), "ncclCommInitRank");
  comm_ = c;
}

NcclComm::~NcclComm() {
  if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::allgatherv(double* buf, const std::vector<long long>& off, const std::vector<long long>& cnt,
                          cudaStream_t s) {
  const NcclApi& a = nccl_or_throw();
  nccl_check(a.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < world; ++r)
    if (cnt[r] > 0)
      nccl_check(a.Broadcast(buf + off[r], buf + off[r], static_cast<size_t>(cnt[r]), ncclDouble, r,
                             static_cast<ncclComm_t>(comm_), s),
                 "ncclBroadcast");
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

void NcclComm::allgather(const double* in, double* out, long long n, cudaStream_t s) {
  const NcclApi& a = nccl_or_throw();
  nccl_check(a.AllGather(in, out, static_cast<size_t>(n), ncclDouble, static_cast<ncclComm_t>(comm_), s),
             "ncclAllGather");
}

void NcclComm::alltoallv(const std::vector<const double*>& send, const std::vector<long long>& scnt,
                         const std::vector<double*>& recv, const std::vector<long long>& rcnt, cudaStream_t s) {
  const NcclApi& a = nccl_or_throw();
  if (rcnt[rank] > 0)  // own chunk: a device copy
    GNW_CUDA_CHECK(cudaMemcpyAsync(recv[rank], send[rank], rcnt[rank] * sizeof(double), cudaMemcpyDeviceToDevice, s));
  nccl_check(a.GroupStart(), "ncclGroupStart");
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    if (scnt[q] > 0)
      nccl_check(a.Send(send[q], static_cast<size_t>(scnt[q]), ncclDouble, q, static_cast<ncclComm_t>(comm_), s),
                 "ncclSend");
    if (rcnt[q] > 0)
      nccl_check(a.Recv(recv[q], static_cast<size_t>(rcnt[q]), ncclDouble, q, static_cast<ncclComm_t>(comm_), s),
                 "ncclRecv");
  }
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

}  // namespace gnw
