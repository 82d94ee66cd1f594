// GPU team runtime (team.hpp). Host C++; kernels live in csrc/*.cu.
#include "team.hpp"

#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>

#include "imbalance/errors.hpp"

namespace imb::rt {

namespace {
// NVTX range for Nsight timelines (SURVEY §5 tracing): header-only NVTX v3,
// a no-op unless a tool injects itself (NVTX_INJECTION64_PATH / nsys / ncu).
struct Trace {
  explicit Trace(const char* name) { nvtxRangePushA(name); }
  ~Trace() { nvtxRangePop(); }
  Trace(const Trace&) = delete;
  Trace& operator=(const Trace&) = delete;
};
}  // namespace

#define IMB_CUDA(call)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw ::imb::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " (" +      \
                             __FILE__ + ":" + std::to_string(__LINE__) + ")");               \
  } while (0)

int step_radius(const Options& o) {
  int r = 1;
  for (int k = 2; k <= o.iord; ++k) r += o.nonos ? 2 : 1;
  return r;
}

void ring_plan(int rank, int nranks, std::int64_t ni, std::int64_t R, RingOp out[4]) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw ContractError("bad ring rank/size");
  if (ni < R || R < 1) throw ContractError("slab thinner than the halo");
  const int left = (rank + nranks - 1) % nranks, right = (rank + 1) % nranks;
  out[0] = RingOp{0, left, R, R};        // first interior planes -> left neighbour
  out[1] = RingOp{0, right, ni, R};      // last interior planes -> right neighbour
  out[2] = RingOp{1, right, R + ni, R};  // right halo <- right neighbour
  out[3] = RingOp{1, left, 0, R};        // left halo <- left neighbour
}

// ---- NCCL, loaded at run time so the library has no hard NCCL dependency --
namespace {

struct NcclApi {
  void* dl = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*async_error)(ncclComm_t, ncclResult_t*) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.dl = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.dl) break;
    }
    if (!api.dl) return;
    auto sym = [](const char* s) { return dlsym(api.dl, s); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.async_error = reinterpret_cast<decltype(api.async_error)>(sym("ncclCommGetAsyncError"));
  });
  if (!api.dl || !api.get_unique_id || !api.comm_init_rank || !api.send || !api.recv ||
      !api.group_start || !api.group_end)
    throw NcclError("NCCL (libnccl.so.2) could not be loaded");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
    throw NcclError(std::string(what) + ": " + msg);
  }
}

}  // namespace

class NcclLink {
 public:
  NcclLink(const unsigned char* id, int nranks, int rank) : nranks_(nranks), rank_(rank) {
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof uid.internal);
    nccl_check(nccl().comm_init_rank(&comm_, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclLink() {
    if (comm_ && nccl().comm_destroy) nccl().comm_destroy(comm_);
  }
  // Ring halo swap of R planes following ring_plan(), as one NCCL group.
  void swap_halos(char* buf, std::size_t plane_bytes, std::int64_t R, std::int64_t ni,
                  cudaStream_t st) {
    RingOp plan[4];
    ring_plan(rank_, nranks_, ni, R, plan);
    nccl_check(nccl().group_start(), "ncclGroupStart");
    for (const RingOp& op : plan) {
      char* p = buf + plane_bytes * static_cast<std::size_t>(op.first_plane);
      const std::size_t bytes = plane_bytes * static_cast<std::size_t>(op.planes);
      if (op.kind == 0)
        nccl_check(nccl().send(p, bytes, ncclUint8, op.peer, comm_, st), "ncclSend");
      else
        nccl_check(nccl().recv(p, bytes, ncclUint8, op.peer, comm_, st), "ncclRecv");
    }
    nccl_check(nccl().group_end(), "ncclGroupEnd");
    // A failed peer or link surfaces asynchronously (the group call itself
    // returned): poll it so the step throws instead of waiting forever.
    if (nccl().async_error) {
      ncclResult_t st = ncclSuccess;
      nccl_check(nccl().async_error(comm_, &st), "ncclCommGetAsyncError");
      if (st != ncclSuccess && st != ncclInProgress) nccl_check(st, "NCCL communicator (async)");
    }
  }
  int nranks() const { return nranks_; }

 private:
  ncclComm_t comm_ = nullptr;
  int nranks_, rank_;
};

// ---- stream memory operations (driver API, resolved through the runtime) ---
namespace {
struct MemOps {
  CUresult (*wait)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
  CUresult (*write)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
};
MemOps& memops() {
  static MemOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.wait = reinterpret_cast<decltype(ops.wait)>(fn);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.write = reinterpret_cast<decltype(ops.write)>(fn);
  });
  if (!ops.wait || !ops.write) throw CudaError("stream memory operations unavailable");
  return ops;
}
}  // namespace

bool stream_memops_available() {
  try {
    (void)memops();
    return true;
  } catch (const CudaError&) {
    return false;
  }
}

namespace {
void memop_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw CudaError(std::string(what) + " failed (CUresult " + std::to_string(r) + ")");
}
}  // namespace

void nccl_unique_id(unsigned char* out) {
  ncclUniqueId uid;
  nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
  std::memcpy(out, uid.internal, sizeof uid.internal);
}

// ---- Team -------------------------------------------------------------------
Team::Team(std::int64_t n, std::int64_t m, std::int64_t l, const Options& opt, int device,
           std::int64_t i0, std::int64_t ni)
    : n_(n), m_(m), l_(l), opt_(opt), device_(device), i0_(i0), ni_(ni) {
  if (n < 3 || m < 3 || l < 3) throw ContractError("grid extents must be >= 3");
  if (opt.iord < 1 || opt.iord > 8) throw ConfigError("iord must be in [1, 8]");
  if (i0 < 0 || i0 >= n || ni < 1 || ni > n) throw ContractError("slab outside the grid");
  R_ = step_radius(opt);
  if (ni < R_)
    throw ContractError("slab of " + std::to_string(ni) + " planes is thinner than the step radius " +
                        std::to_string(R_));
  P_ = ni_ + 2 * R_;
  int count = 0;
  IMB_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    throw ConfigError("device " + std::to_string(device) + " not present (" +
                      std::to_string(count) + " visible)");
  try {
    acquire();
  } catch (...) {
    release();  // the destructor does not run for a throwing constructor
    throw;
  }
}

void Team::acquire() {
  IMB_CUDA(cudaSetDevice(device_));
  IMB_CUDA(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device_));
  IMB_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
  IMB_CUDA(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking));
  IMB_CUDA(cudaEventCreateWithFlags(&ev_ready_, cudaEventDisableTiming));
  IMB_CUDA(cudaEventCreateWithFlags(&ev_halo_, cudaEventDisableTiming));
  const std::size_t fbytes = static_cast<std::size_t>(P_) * plane_bytes();
  // The fused kernels take any slab >= R planes (they read R halo planes);
  // every slab of a decomposition then runs the same arithmetic.
  const bool fused = dev::fused_supported(opt_.iord, opt_.nonos, m_, l_, P_);
  const int ntmp = fused ? 0 : 12;
  const int next = (fused && opt_.iord == 3) ? 6 : 0;  // psi^(2), bounds, limited velocities
  const std::size_t total = fbytes * static_cast<std::size_t>(7 + ntmp + next);
  if (cudaMalloc(&pool_, total) != cudaSuccess) {
    cudaGetLastError();
    throw ConfigError("cannot allocate " + std::to_string(total >> 20) + " MiB on device " +
                      std::to_string(device_));
  }
  IMB_CUDA(cudaMemsetAsync(pool_, 0, total, cs_));
  IMB_CUDA(cudaMalloc(&flags_, 4 * sizeof(std::uint64_t)));
  IMB_CUDA(cudaMemsetAsync(flags_, 0, 4 * sizeof(std::uint64_t), cs_));
  char* p = static_cast<char*>(pool_);
  x_ = p;
  xn_ = p + fbytes;
  x0_ = p + 2 * fbytes;
  for (int f = 0; f < 4; ++f) st_[f] = p + static_cast<std::size_t>(3 + f) * fbytes;
  for (int t = 0; t < ntmp; ++t) tmp_[t] = p + static_cast<std::size_t>(7 + t) * fbytes;
  for (int t = 0; t < next; ++t) ext_[t] = p + static_cast<std::size_t>(7 + ntmp + t) * fbytes;
  IMB_CUDA(cudaStreamSynchronize(cs_));
}

Team::~Team() { release(); }

void Team::release() noexcept {
  cudaSetDevice(device_);
  if (cs_) cudaStreamSynchronize(cs_);
  if (xs_) cudaStreamSynchronize(xs_);
  nccl_.reset();
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  if (ev_ready_) cudaEventDestroy(ev_ready_);
  if (ev_halo_) cudaEventDestroy(ev_halo_);
  if (cs_) cudaStreamDestroy(cs_);
  if (xs_) cudaStreamDestroy(xs_);
  if (ups_) cudaStreamDestroy(ups_);
  if (dns_) cudaStreamDestroy(dns_);
  for (cudaEvent_t e : ev_pipe_) cudaEventDestroy(e);
  for (cudaGraphExec_t g : graph_)
    if (g) cudaGraphExecDestroy(g);
  if (pool_) cudaFree(pool_);
  if (flags_) cudaFree(flags_);
  for (IpcPeer* p : {&ipc_left_, &ipc_right_})
    if (p->opened) {
      cudaIpcCloseMemHandle(p->pool);
      cudaIpcCloseMemHandle(p->flags);
    }
}

void* Team::fbuf(int field) const {
  switch (field) {
    case 0: return x_;
    case 1: return st_[0];
    case 2: return st_[1];
    case 3: return st_[2];
    case 4: return st_[3];
    default: throw ContractError("field id must be 0..4 (x, u, v, w, h)");
  }
}

void Team::init_recipe(int kind, std::uint64_t seed) {
  if (kind < 0 || kind > 2) throw ConfigError("unknown recipe " + std::to_string(kind));
  IMB_CUDA(cudaSetDevice(device_));
  const recipe::Params prm = recipe::make_params(kind, n_, m_, l_, seed);
  if (opt_.fp64)
    launches_ += dev::launch_init<double>(prm, i0_, R_, P_, static_cast<double*>(x_),
                                          static_cast<double*>(st_[0]), static_cast<double*>(st_[1]),
                                          static_cast<double*>(st_[2]), static_cast<double*>(st_[3]), cs_);
  else
    launches_ += dev::launch_init<float>(prm, i0_, R_, P_, static_cast<float*>(x_),
                                         static_cast<float*>(st_[0]), static_cast<float*>(st_[1]),
                                         static_cast<float*>(st_[2]), static_cast<float*>(st_[3]), cs_);
  IMB_CUDA(cudaGetLastError());
  IMB_CUDA(cudaMemcpyAsync(x0_, x_, static_cast<std::size_t>(P_) * plane_bytes(),
                           cudaMemcpyDeviceToDevice, cs_));
  IMB_CUDA(cudaStreamSynchronize(cs_));
  static_halo_ok_ = true;  // recipe halos are generated, not exchanged
  halo_fresh_ = true;
}

void Team::upload(int field, const void* host, std::size_t bytes) {
  halo_fresh_ = false;
  const std::size_t want = static_cast<std::size_t>(ni_) * plane_bytes();
  if (bytes != want)
    throw ContractError("upload of " + std::to_string(bytes) + " bytes, slab needs " +
                        std::to_string(want));
  IMB_CUDA(cudaSetDevice(device_));
  char* dst = static_cast<char*>(fbuf(field)) + static_cast<std::size_t>(R_) * plane_bytes();
  IMB_CUDA(cudaMemcpyAsync(dst, host, bytes, cudaMemcpyHostToDevice, cs_));
  if (field == 0)
    IMB_CUDA(cudaMemcpyAsync(static_cast<char*>(x0_) + static_cast<std::size_t>(R_) * plane_bytes(),
                             dst, bytes, cudaMemcpyDeviceToDevice, cs_));
  else
    static_halo_ok_ = false;
  IMB_CUDA(cudaStreamSynchronize(cs_));
}

void Team::download(int field, void* host, std::size_t bytes) {
  const std::size_t want = static_cast<std::size_t>(ni_) * plane_bytes();
  if (bytes != want)
    throw ContractError("download of " + std::to_string(bytes) + " bytes, slab holds " +
                        std::to_string(want));
  IMB_CUDA(cudaSetDevice(device_));
  const char* src = static_cast<const char*>(fbuf(field)) + static_cast<std::size_t>(R_) * plane_bytes();
  IMB_CUDA(cudaMemcpyAsync(host, src, bytes, cudaMemcpyDeviceToHost, cs_));
  IMB_CUDA(cudaStreamSynchronize(cs_));
}

void Team::reset() {
  halo_fresh_ = false;
  IMB_CUDA(cudaSetDevice(device_));
  IMB_CUDA(cudaMemcpyAsync(x_, x0_, static_cast<std::size_t>(P_) * plane_bytes(),
                           cudaMemcpyDeviceToDevice, cs_));
  IMB_CUDA(cudaStreamSynchronize(cs_));
}

// Periodic single slab: halo planes come from the opposite end of itself.
void Team::exchange_x_self(void* buf) {
  char* b = static_cast<char*>(buf);
  const std::size_t pb = plane_bytes(), bytes = pb * static_cast<std::size_t>(R_);
  IMB_CUDA(cudaMemcpyAsync(b, b + pb * static_cast<std::size_t>(ni_), bytes,
                           cudaMemcpyDeviceToDevice, cs_));
  IMB_CUDA(cudaMemcpyAsync(b + pb * static_cast<std::size_t>(R_ + ni_),
                           b + pb * static_cast<std::size_t>(R_), bytes, cudaMemcpyDeviceToDevice, cs_));
}

void Team::exchange_x_nccl(void* buf) {
  Trace tr("imb.exchange.nccl");
  IMB_CUDA(cudaEventRecord(ev_ready_, cs_));
  IMB_CUDA(cudaStreamWaitEvent(xs_, ev_ready_, 0));
  nccl_->swap_halos(static_cast<char*>(buf), plane_bytes(), R_, ni_, xs_);
  IMB_CUDA(cudaEventRecord(ev_halo_, xs_));
  IMB_CUDA(cudaStreamWaitEvent(cs_, ev_halo_, 0));
}

void Team::exchange_static() {
  Trace tr("imb.exchange.static");
  for (int f = 0; f < 4; ++f) {
    if (nccl_ && nccl_->nranks() > 1)
      exchange_x_nccl(st_[f]);
    else
      exchange_x_self(st_[f]);
  }
  static_halo_ok_ = true;
}

void Team::pull_from_ring(int field, cudaStream_t st) {
  const std::size_t pb = plane_bytes(), bytes = pb * static_cast<std::size_t>(R_);
  char* mine = static_cast<char*>(fbuf(field));
  const char* lsrc = static_cast<const char*>(left_->fbuf(field)) + pb * static_cast<std::size_t>(left_->ni_);
  const char* rsrc = static_cast<const char*>(right_->fbuf(field)) + pb * static_cast<std::size_t>(right_->R_);
  IMB_CUDA(cudaMemcpyPeerAsync(mine, device_, lsrc, left_->device_, bytes, st));
  IMB_CUDA(cudaMemcpyPeerAsync(mine + pb * static_cast<std::size_t>(R_ + ni_), device_, rsrc,
                               right_->device_, bytes, st));
}

void Team::begin_compute_window() {
  if (ev_used_ + 2 > ev_pool_.size()) {
    cudaEvent_t a, b;
    IMB_CUDA(cudaEventCreate(&a));
    IMB_CUDA(cudaEventCreate(&b));
    ev_pool_.push_back(a);
    ev_pool_.push_back(b);
  }
  IMB_CUDA(cudaEventRecord(ev_pool_[ev_used_], cs_));
}

void Team::end_compute_window() {
  IMB_CUDA(cudaEventRecord(ev_pool_[ev_used_ + 1], cs_));
  ev_used_ += 2;
}

double Team::take_compute_seconds() {
  double s = 0.0;
  if (ev_used_ > 0) IMB_CUDA(cudaEventSynchronize(ev_pool_[ev_used_ - 1]));
  for (std::size_t q = 0; q + 1 < ev_used_; q += 2) {
    float ms = 0.f;
    IMB_CUDA(cudaEventElapsedTime(&ms, ev_pool_[q], ev_pool_[q + 1]));
    s += static_cast<double>(ms) * 1e-3;
  }
  ev_used_ = 0;
  return s;
}

namespace {
// Fused launchers return the kernels launched, or < 0 when the kernel could
// not be configured for this device (shared-memory opt-in / occupancy).
int fused_launched(int n) {
  if (n < 0) {
    const cudaError_t e = cudaGetLastError();
    throw CudaError(std::string("fused step kernel could not be configured: ") +
                    cudaGetErrorString(e));
  }
  return n;
}
struct Rng {
  std::int64_t a, b;
};
Rng cap(Rng r, std::int64_t lo, std::int64_t hi) { return {std::max(r.a, lo), std::min(r.b, hi)}; }
Rng hull(Rng x, Rng y) { return {std::min(x.a, y.a), std::max(x.b, y.b)}; }
}  // namespace

// One step on a halo-complete x: xn = MPDATA(x) on the interior, then swap.
template <class T>
void Team::compute_step_t() {
  const T* x = static_cast<const T*>(x_);
  const T* u = static_cast<const T*>(st_[0]);
  const T* v = static_cast<const T*>(st_[1]);
  const T* w = static_cast<const T*>(st_[2]);
  const T* h = static_cast<const T*>(st_[3]);
  T* out = static_cast<T*>(xn_);
  if (tmp_[0] == nullptr) {
    dev::FusedShape fs{m_, l_, ni_, R_, 0, ni_};
    dev::HaloPush<T> push{static_cast<T*>(push_lo_), push_lo_ni_, static_cast<T*>(push_hi_),
                          push_sys_};
    if (opt_.iord == 3)
      launches_ += fused_launched(dev::launch_fused3<T>(
          fs, x, u, v, w, h, static_cast<T*>(ext_[0]), static_cast<T*>(ext_[1]),
          static_cast<T*>(ext_[2]), static_cast<T*>(ext_[3]), static_cast<T*>(ext_[4]),
          static_cast<T*>(ext_[5]), out, num_sms_, cs_, push));
    else
      launches_ += fused_launched(dev::launch_fused<T>(fs, opt_.iord, opt_.nonos, x, u, v, w, h,
                                                       out, num_sms_, cs_, push));
    IMB_CUDA(cudaGetLastError());
    push_lo_ = push_hi_ = nullptr;
    push_sys_ = false;
    if (swap_after_) std::swap(x_, xn_);
    return;
  }
  T* it[2] = {static_cast<T*>(tmp_[0]), static_cast<T*>(tmp_[1])};
  T* va[3] = {static_cast<T*>(tmp_[2]), static_cast<T*>(tmp_[3]), static_cast<T*>(tmp_[4])};
  T* vb[3] = {static_cast<T*>(tmp_[5]), static_cast<T*>(tmp_[6]), static_cast<T*>(tmp_[7])};
  T* mx = static_cast<T*>(tmp_[8]);
  T* mn = static_cast<T*>(tmp_[9]);
  T* bu = static_cast<T*>(tmp_[10]);
  T* bd = static_cast<T*>(tmp_[11]);
  const std::int64_t P = P_;
  auto span = [&](Rng r) { return dev::Span{m_, l_, std::max<std::int64_t>(r.a, 1), std::min(r.b, P - 1)}; };
  const Rng all{0, P};
  const Rng goal{R_, R_ + ni_};
  // Validity of every intermediate is tracked as a plane interval; each stage
  // is launched on the widest interval its inputs support.
  Rng rc{1, P - 1};
  T* cur = (opt_.iord == 1) ? out : it[0];
  launches_ += dev::launch_update<T>(span(opt_.iord == 1 ? goal : rc), x, u, v, w, h, cur, cs_);
  if (opt_.iord == 1) {
    IMB_CUDA(cudaGetLastError());
    std::swap(x_, xn_);
    return;
  }
  const T *U = u, *V = v, *W = w;
  Rng ru = all, rvw = all, rm{0, 0};
  T** vel = va;
  int nit = 1;
  for (int pass = 2; pass <= opt_.iord; ++pass) {
    const Rng nu = {std::max({rc.a + 1, rvw.a + 1, ru.a}), std::min({rc.b, rvw.b, ru.b})};
    const Rng nvw = {std::max({rc.a + 1, ru.a, rvw.a}), std::min({rc.b - 1, ru.b - 1, rvw.b})};
    launches_ += dev::launch_pseudo<T>(span(hull(nu, nvw)), cur, U, V, W, h, vel[0], vel[1], vel[2], cs_);
    Rng lu = nu, lvw = nvw;
    if (opt_.nonos) {
      const bool first = pass == 2;
      const Rng nm = first ? Rng{rc.a + 1, rc.b - 1} : cap(Rng{rc.a + 1, rc.b - 1}, rm.a, rm.b);
      launches_ += dev::launch_bounds<T>(span(nm), cur, x, first ? 1 : 0, mx, mn, cs_);
      rm = nm;
      const Rng nb = {std::max({rc.a + 1, nu.a, nvw.a, nm.a}), std::min({rc.b - 1, nu.b - 1, nvw.b, nm.b})};
      launches_ += dev::launch_beta<T>(span(nb), cur, vel[0], vel[1], vel[2], h, mx, mn, bu, bd, cs_);
      lu = {std::max(nu.a, nb.a + 1), std::min(nu.b, nb.b)};
      lvw = {std::max(nvw.a, nb.a), std::min(nvw.b, nb.b)};
      launches_ += dev::launch_limit<T>(span(hull(lu, lvw)), vel[0], vel[1], vel[2], bu, bd, cs_);
    }
    Rng nr = {std::max({rc.a + 1, lu.a, lvw.a}), std::min({rc.b - 1, lu.b - 1, lvw.b})};
    T* dst;
    if (pass == opt_.iord) {
      if (nr.a > goal.a || nr.b < goal.b)
        throw ContractError("internal: step radius does not cover the slab interior");
      nr = goal;
      dst = out;
    } else {
      dst = it[nit];
      nit ^= 1;
    }
    launches_ += dev::launch_update<T>(span(nr), cur, vel[0], vel[1], vel[2], h, dst, cs_);
    cur = dst;
    rc = nr;
    U = vel[0];
    V = vel[1];
    W = vel[2];
    ru = lu;
    rvw = lvw;
    vel = (vel == va) ? vb : va;
  }
  IMB_CUDA(cudaGetLastError());
  std::swap(x_, xn_);
}

void Team::compute_step() {
  if (opt_.fp64)
    compute_step_t<double>();
  else
    compute_step_t<float>();
}

// Fused step kernel over output planes [o0, o1) (interior coordinates), no swap.
void Team::fused_range(std::int64_t o0, std::int64_t o1) {
  if (o1 <= o0) return;
  dev::FusedShape fs{m_, l_, ni_, R_, o0, o1};
  if (opt_.fp64)
    launches_ += fused_launched(dev::launch_fused<double>(
        fs, opt_.iord, opt_.nonos, static_cast<const double*>(x_), static_cast<const double*>(st_[0]),
        static_cast<const double*>(st_[1]), static_cast<const double*>(st_[2]),
        static_cast<const double*>(st_[3]), static_cast<double*>(xn_), num_sms_, cs_));
  else
    launches_ += fused_launched(dev::launch_fused<float>(
        fs, opt_.iord, opt_.nonos, static_cast<const float*>(x_), static_cast<const float*>(st_[0]),
        static_cast<const float*>(st_[1]), static_cast<const float*>(st_[2]),
        static_cast<const float*>(st_[3]), static_cast<float*>(xn_), num_sms_, cs_));
  IMB_CUDA(cudaGetLastError());
}

// Multi-rank step with the halo exchange hidden behind the interior: the
// interior output planes [R, ni-R) read no halo plane, so they run while NCCL
// moves the halos on the exchange stream; the 2R boundary planes follow the
// exchange event. The next step's sends read planes written by the boundary
// launches, which the ev_ready record at the top of that step orders.
void Team::step_overlapped() {
  halo_fresh_ = false;
  IMB_CUDA(cudaEventRecord(ev_ready_, cs_));
  IMB_CUDA(cudaStreamWaitEvent(xs_, ev_ready_, 0));
  nccl_->swap_halos(static_cast<char*>(x_), plane_bytes(), R_, ni_, xs_);
  IMB_CUDA(cudaEventRecord(ev_halo_, xs_));
  begin_compute_window();
  fused_range(R_, ni_ - R_);
  IMB_CUDA(cudaStreamWaitEvent(cs_, ev_halo_, 0));
  fused_range(0, R_);
  fused_range(ni_ - R_, ni_);
  end_compute_window();
  std::swap(x_, xn_);
}

// Two self-pushing fused steps as one graph replay (x -> xn -> x). Captured on
// first use for each starting buffer; returns false if capture is unavailable
// (the caller then launches the step directly).
bool Team::graph_step_pair() {
  const int slot = (x_ == graph_x_[0]) ? 0 : (x_ == graph_x_[1]) ? 1 : (graph_x_[0] ? 1 : 0);
  if (graph_[slot] == nullptr || graph_x_[slot] != x_) {
    if (graph_[slot]) IMB_CUDA(cudaGraphExecDestroy(graph_[slot]));
    graph_[slot] = nullptr;
    void* x0 = x_;
    const std::int64_t l0 = launches_;
    IMB_CUDA(cudaStreamBeginCapture(cs_, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < 2; ++k) {
      push_lo_ = push_hi_ = xn_;
      push_lo_ni_ = ni_;
      compute_step();  // swaps x_ and xn_
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cs_, &g);
    graph_launches_ = launches_ - l0;
    launches_ = l0;
    if (e != cudaSuccess || g == nullptr) {  // nothing ran (x_ is back to x0)
      cudaGetLastError();
      return false;
    }
    const cudaError_t ie = cudaGraphInstantiate(&graph_[slot], g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      cudaGetLastError();
      graph_[slot] = nullptr;
      return false;
    }
    graph_x_[slot] = x0;
  }
  IMB_CUDA(cudaGraphLaunch(graph_[slot], cs_));
  launches_ += graph_launches_;
  return true;
}

void Team::run(int steps, double* compute_s, double* wall_s) {
  Trace tr("imb.team.run");
  if (steps < 0) throw ContractError("steps must be >= 0");
  if (left_ || right_) throw ContractError("ring member teams are stepped through their group");
  IMB_CUDA(cudaSetDevice(device_));
  const bool multi = nccl_ && nccl_->nranks() > 1;
  cudaEvent_t t0, t1;
  IMB_CUDA(cudaEventCreate(&t0));
  IMB_CUDA(cudaEventCreate(&t1));
  IMB_CUDA(cudaEventRecord(t0, cs_));
  // IPC ring members pull their neighbours' static halos inside ipc_step()
  // (after both neighbours posted their uploads); a self/NCCL exchange here
  // would fill them from the wrong slab and mark them valid.
  if (!static_halo_ok_ && !ipc_) exchange_static();
  ev_used_ = 0;
  // Hiding the exchange behind the interior costs two extra launches for the
  // 2R boundary planes; each streams R planes plus the warm-up on one block
  // per SM (~7 plane-times, ~75 us at C4 rows), while an NVLink exchange of
  // 2R planes takes ~20 us. So by default the exchange runs first and one
  // launch covers the slab; IMB_OVERLAP=1 selects the overlapped schedule.
  static const bool overlap_on = [] {
    const char* e = std::getenv("IMB_OVERLAP");
    return e && e[0] == '1';
  }();
  const bool overlap = overlap_on && multi && opt_.iord == 2 && tmp_[0] == nullptr && ni_ > 2 * R_;
  const bool self_push = !multi && !ipc_ && tmp_[0] == nullptr;
  static const bool graphs_on = [] {
    const char* e = std::getenv("IMB_GRAPH");
    return !(e && e[0] == '0');
  }();
  const bool use_graph = graphs_on && self_push && steps >= 4;
  for (int s = 0; s < steps; ++s) {
    if (ipc_) {
      ipc_step();
      continue;
    }
    if (overlap) {
      step_overlapped();
      continue;
    }
    if (self_push) {
      // Periodic single slab: the kernel's epilogue writes the edge planes
      // into the opposite halos of its own output, so after the first step
      // no exchange is needed at all.
      if (halo_fresh_ && use_graph && s + 2 <= steps) {
        begin_compute_window();
        if (graph_step_pair()) {
          end_compute_window();
          ++s;
          continue;
        }
        end_compute_window();
      }
      if (!halo_fresh_) exchange_x_self(x_);
      push_lo_ = push_hi_ = xn_;
      push_lo_ni_ = ni_;
      begin_compute_window();
      compute_step();
      end_compute_window();
      halo_fresh_ = true;
      continue;
    }
    if (multi)
      exchange_x_nccl(x_);
    else
      exchange_x_self(x_);
    begin_compute_window();
    compute_step();
    end_compute_window();
  }
  if (!self_push && !ipc_) halo_fresh_ = false;
  IMB_CUDA(cudaEventRecord(t1, cs_));
  IMB_CUDA(cudaEventSynchronize(t1));
  float ms = 0.f;
  IMB_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  const double comp = take_compute_seconds();
  if (compute_s) *compute_s = comp;
  if (wall_s) *wall_s = static_cast<double>(ms) * 1e-3;
}

// Host-buffer step with the PCIe copies hidden behind each other and behind
// the kernel: the slab is cut into chunks of planes; chunk c's H2D (copy
// engine 1), the fused kernel on the output planes it completes, and the
// D2H of those planes (copy engine 2) run on three streams linked by events.
// The periodic halos need the first and last R planes, so those go first.
void Team::step_host_pipelined(const void* x_in, void* x_out) {
  if (!ups_) {
    IMB_CUDA(cudaStreamCreateWithFlags(&ups_, cudaStreamNonBlocking));
    IMB_CUDA(cudaStreamCreateWithFlags(&dns_, cudaStreamNonBlocking));
  }
  // Chunk boundaries 0 = cut[0] < ... < cut[nch] = ni. Uniform chunks leave
  // the pipeline's fill (the first chunk's H2D before any kernel) and drain
  // (the last chunk's D2H after the last kernel) as large as a chunk; the
  // ramped schedule (default) starts and ends with chunks of `base` planes and
  // doubles up to `cap` in between, so both ends shrink to a few MB.
  static const int max_chunks = [] {
    const char* e = std::getenv("IMB_PIPE_CHUNKS");  // > 0: that many uniform chunks (A/B knob)
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  std::vector<std::int64_t>& cut = pipe_cuts_;
  cut.assign(1, 0);
  static const int base_env = [] {
    // first/last chunk planes (A/B knob). Measured at C4 (profiles/r02c_e2e_sweep.txt):
    // ramp from 16 planes 5.51 Gcell/s, uniform 12/16/20/24/32 chunks 5.46/5.48/5.45/5.39/5.26
    const char* e = std::getenv("IMB_PIPE_BASE");
    return e ? std::atoi(e) : 16;
  }();
  const std::int64_t base = std::max<std::int64_t>(base_env, 2 * R_), cap = std::max<std::int64_t>(base, ni_ / 16);
  std::vector<std::int64_t> ramp;
  for (std::int64_t c = base, sum = 0; c < cap && 2 * (sum + c) <= ni_ / 2; c *= 2) {
    ramp.push_back(c);
    sum += c;
  }
  std::int64_t ramp_sum = 0;
  for (std::int64_t c : ramp) ramp_sum += c;
  if (max_chunks > 0 || ramp.empty()) {
    const std::int64_t n = std::max<std::int64_t>(
        1, std::min<std::int64_t>(max_chunks > 0 ? max_chunks : 16, ni_ / (8 * R_)));
    for (std::int64_t c = 1; c <= n; ++c) cut.push_back(ni_ * c / n);
  } else {
    for (std::int64_t c : ramp) cut.push_back(cut.back() + c);
    const std::int64_t mid = ni_ - 2 * ramp_sum, nm = std::max<std::int64_t>(1, (mid + cap - 1) / cap);
    const std::int64_t m0 = cut.back();
    for (std::int64_t c = 1; c <= nm; ++c) cut.push_back(m0 + mid * c / nm);
    for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) cut.push_back(cut.back() + *it);
  }
  const int nch = static_cast<int>(cut.size()) - 1;
  while (ev_pipe_.size() < static_cast<std::size_t>(2 * nch + 2)) {
    cudaEvent_t e;
    IMB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev_pipe_.push_back(e);
  }
  const std::size_t pb = plane_bytes();
  const char* in = static_cast<const char*>(x_in);
  char* out = static_cast<char*>(x_out);
  auto xplane = [&](std::int64_t p) { return static_cast<char*>(x_) + static_cast<std::size_t>(p + R_) * pb; };
  auto nplane = [&](std::int64_t p) { return static_cast<char*>(xn_) + static_cast<std::size_t>(p + R_) * pb; };
  auto h2d = [&](std::int64_t a, std::int64_t b) {
    if (b > a)
      IMB_CUDA(cudaMemcpyAsync(xplane(a), in + static_cast<std::size_t>(a) * pb,
                               static_cast<std::size_t>(b - a) * pb, cudaMemcpyHostToDevice, ups_));
  };
  cudaEvent_t ev_start = ev_pipe_[0], ev_edges = ev_pipe_[1];
  IMB_CUDA(cudaEventRecord(ev_start, cs_));
  // IMB_PIPE_TRACE=1: per-chunk H2D / kernel / D2H completion times on stderr
  static const bool trace = [] {
    const char* e = std::getenv("IMB_PIPE_TRACE");
    return e && e[0] == '1';
  }();
  std::vector<cudaEvent_t> tr;
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    IMB_CUDA(cudaEventCreate(&e));
    IMB_CUDA(cudaEventRecord(e, st));
    tr.push_back(e);
  };
  mark(cs_);
  IMB_CUDA(cudaStreamWaitEvent(ups_, ev_start, 0));
  IMB_CUDA(cudaStreamWaitEvent(dns_, ev_start, 0));
  // edges + periodic self halos
  h2d(0, R_);
  h2d(ni_ - R_, ni_);
  const std::size_t hb = static_cast<std::size_t>(R_) * pb;
  IMB_CUDA(cudaMemcpyAsync(xplane(-R_), xplane(ni_ - R_), hb, cudaMemcpyDeviceToDevice, ups_));
  IMB_CUDA(cudaMemcpyAsync(xplane(ni_), xplane(0), hb, cudaMemcpyDeviceToDevice, ups_));
  IMB_CUDA(cudaEventRecord(ev_edges, ups_));
  std::int64_t done_out = 0;
  for (int c = 0; c < nch; ++c) {
    const std::int64_t b0 = cut[c], b1 = cut[c + 1];
    h2d(std::max(b0, R_), std::min(b1, ni_ - R_));
    cudaEvent_t up = ev_pipe_[2 + 2 * c], comp = ev_pipe_[3 + 2 * c];
    IMB_CUDA(cudaEventRecord(up, ups_));
    mark(ups_);
    IMB_CUDA(cudaStreamWaitEvent(cs_, up, 0));
    const std::int64_t o1 = (c == nch - 1) ? ni_ : std::max(done_out, b1 - R_);
    fused_range(done_out, o1);
    IMB_CUDA(cudaEventRecord(comp, cs_));
    mark(cs_);
    IMB_CUDA(cudaStreamWaitEvent(dns_, comp, 0));
    if (o1 > done_out)
      IMB_CUDA(cudaMemcpyAsync(out + static_cast<std::size_t>(done_out) * pb, nplane(done_out),
                               static_cast<std::size_t>(o1 - done_out) * pb, cudaMemcpyDeviceToHost,
                               dns_));
    mark(dns_);
    done_out = o1;
  }
  (void)ev_edges;
  IMB_CUDA(cudaStreamSynchronize(dns_));
  IMB_CUDA(cudaStreamSynchronize(cs_));
  if (trace) {
    std::string line = "imb pipe (ms from start: h2d kernel d2h per chunk):";
    for (std::size_t i = 1; i < tr.size(); ++i) {
      float ms = 0.f;
      IMB_CUDA(cudaEventElapsedTime(&ms, tr[0], tr[i]));
      line += (i % 3 == 1 ? "  | " : " ") + std::to_string(ms).substr(0, 6);
    }
    std::fprintf(stderr, "%s\n", line.c_str());
    for (cudaEvent_t e : tr) cudaEventDestroy(e);
  }
  std::swap(x_, xn_);
}

void Team::step_host(const void* x_in, void* x_out) {
  Trace tr("imb.team.step_host");
  halo_fresh_ = false;
  if (left_ || right_) throw ContractError("ring member teams are stepped through their group");
  IMB_CUDA(cudaSetDevice(device_));
  if (ipc_) {  // every rank rewrites x, then one flag-synchronised pushed step
    const std::size_t bytes = static_cast<std::size_t>(ni_) * plane_bytes();
    const std::size_t off = static_cast<std::size_t>(R_) * plane_bytes();
    IMB_CUDA(cudaMemcpyAsync(static_cast<char*>(x_) + off, x_in, bytes, cudaMemcpyHostToDevice, cs_));
    ipc_step();
    IMB_CUDA(cudaMemcpyAsync(x_out, static_cast<char*>(x_) + off, bytes, cudaMemcpyDeviceToHost, cs_));
    IMB_CUDA(cudaStreamSynchronize(cs_));
    return;
  }
  if (!static_halo_ok_) exchange_static();
  if (!(nccl_ && nccl_->nranks() > 1) && opt_.iord == 2 && tmp_[0] == nullptr && ni_ >= 4 * R_) {
    step_host_pipelined(x_in, x_out);
    return;
  }
  const std::size_t bytes = static_cast<std::size_t>(ni_) * plane_bytes();
  char* interior = static_cast<char*>(x_) + static_cast<std::size_t>(R_) * plane_bytes();
  IMB_CUDA(cudaMemcpyAsync(interior, x_in, bytes, cudaMemcpyHostToDevice, cs_));
  if (!static_halo_ok_) exchange_static();
  if (nccl_ && nccl_->nranks() > 1)
    exchange_x_nccl(x_);
  else
    exchange_x_self(x_);
  compute_step();
  interior = static_cast<char*>(x_) + static_cast<std::size_t>(R_) * plane_bytes();
  IMB_CUDA(cudaMemcpyAsync(x_out, interior, bytes, cudaMemcpyDeviceToHost, cs_));
  IMB_CUDA(cudaStreamSynchronize(cs_));
}

std::uint64_t Team::checksum() {
  std::vector<unsigned char> host(static_cast<std::size_t>(ni_) * plane_bytes());
  download(0, host.data(), host.size());
  std::uint64_t hsh = 0xcbf29ce484222325ull;
  for (unsigned char b : host) {
    hsh ^= b;
    hsh *= 0x100000001b3ull;
  }
  return hsh;
}

void Team::connect_nccl(const unsigned char* id, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw ContractError("bad NCCL rank/size");
  if (left_ || right_ || ipc_ || nccl_) throw ContractError("team is already part of a ring");
  IMB_CUDA(cudaSetDevice(device_));
  nccl_ = std::make_unique<NcclLink>(id, nranks, rank);
}

namespace {
struct IpcBlob {
  std::uint32_t magic;
  std::int32_t device;
  cudaIpcMemHandle_t pool;
  cudaIpcMemHandle_t flags;
  std::int64_t off_x, off_xn, ni, step0, plane_bytes, R;
  std::int64_t off_st[4];
};
constexpr std::uint32_t kIpcMagic = 0x1b200c0du;
static_assert(sizeof(IpcBlob) <= Team::kIpcBlobBytes, "IPC blob too large");
}  // namespace

void Team::ipc_export(unsigned char* blob) {
  IMB_CUDA(cudaSetDevice(device_));
  if (tmp_[0] != nullptr) throw ConfigError("IPC halo push needs the fused step kernel");
  IpcBlob b{};
  b.magic = kIpcMagic;
  b.device = device_;
  IMB_CUDA(cudaIpcGetMemHandle(&b.pool, pool_));
  IMB_CUDA(cudaIpcGetMemHandle(&b.flags, flags_));
  char* base = static_cast<char*>(pool_);
  b.off_x = static_cast<char*>(x_) - base;
  b.off_xn = static_cast<char*>(xn_) - base;
  b.ni = ni_;
  b.step0 = static_cast<std::int64_t>(step_count_);
  b.plane_bytes = static_cast<std::int64_t>(plane_bytes());
  b.R = R_;
  for (int f = 0; f < 4; ++f) b.off_st[f] = static_cast<char*>(st_[f]) - base;
  std::memset(blob, 0, kIpcBlobBytes);
  std::memcpy(blob, &b, sizeof b);
}

void Team::connect_ipc(const unsigned char* left_blob, const unsigned char* right_blob,
                       int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw ContractError("bad IPC rank/size");
  if (left_ || right_ || ipc_ || nccl_) throw ContractError("team is already part of a ring");
  if (tmp_[0] != nullptr) throw ConfigError("IPC halo push needs the fused step kernel");
  IMB_CUDA(cudaSetDevice(device_));
  if (nranks == 1) return;  // periodic single slab: the self push already covers it
  IpcBlob l, r;
  std::memcpy(&l, left_blob, sizeof l);
  std::memcpy(&r, right_blob, sizeof r);
  if (l.magic != kIpcMagic || r.magic != kIpcMagic) throw ContractError("not an imb IPC blob");
  if (l.plane_bytes != static_cast<std::int64_t>(plane_bytes()) || l.R != R_ ||
      r.plane_bytes != static_cast<std::int64_t>(plane_bytes()) || r.R != R_)
    throw ContractError("IPC neighbours disagree on plane size or halo radius");
  auto open = [&](const IpcBlob& b, IpcPeer& p) {
    void* pool = nullptr;
    void* fl = nullptr;
    IMB_CUDA(cudaIpcOpenMemHandle(&pool, b.pool, cudaIpcMemLazyEnablePeerAccess));
    IMB_CUDA(cudaIpcOpenMemHandle(&fl, b.flags, cudaIpcMemLazyEnablePeerAccess));
    p.pool = static_cast<char*>(pool);
    p.flags = static_cast<std::uint64_t*>(fl);
    p.off_x = b.off_x;
    p.off_xn = b.off_xn;
    p.ni = b.ni;
    p.step0 = b.step0;
    p.device = b.device;
    for (int f = 0; f < 4; ++f) p.off_st[f] = b.off_st[f];
    p.opened = true;
  };
  open(l, ipc_left_);
  if (nranks == 2) {  // one neighbour on both sides: a handle opens once per process
    ipc_right_ = ipc_left_;
    ipc_right_.opened = false;
  } else {
    open(r, ipc_right_);
  }
  if (ipc_left_.step0 != static_cast<std::int64_t>(step_count_) ||
      ipc_right_.step0 != static_cast<std::int64_t>(step_count_))
    throw ContractError("IPC ring members must connect at the same step count");
  // Probe now, while no rank steps, that this stream can write the mapped
  // flag words (peer memory over NVLink): rewrite the values they already
  // hold (only this rank writes the words that describe it), so a missing
  // capability fails here instead of leaving a neighbour waiting mid-step.
  MemOps& ops = memops();
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_left_.flags + 1), step_count_,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64 (peer)");
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_right_.flags + 0), step_count_,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64 (peer)");
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_left_.flags + 3), post_epoch_,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64 (peer)");
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_right_.flags + 2), post_epoch_,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64 (peer)");
  IMB_CUDA(cudaStreamSynchronize(cs_));
  ipc_ = true;
}

// One flag-synchronised step of a process ring (see group_flag_step): wait
// until both neighbours finished step s-1, run the fused kernel whose
// epilogue stores the edge planes into the neighbours' step-s buffers
// (mapped over NVLink), then raise the neighbours' flag words.
void Team::ipc_step() {
  Trace tr("imb.team.ipc_step");
  MemOps& ops = memops();
  const std::uint64_t s = step_count_;
  memop_check(ops.wait(cs_, reinterpret_cast<CUdeviceptr>(flags_ + 0), s, CU_STREAM_WAIT_VALUE_GEQ),
              "cuStreamWaitValue64");
  memop_check(ops.wait(cs_, reinterpret_cast<CUdeviceptr>(flags_ + 1), s, CU_STREAM_WAIT_VALUE_GEQ),
              "cuStreamWaitValue64");
  const std::size_t pb = plane_bytes(), hb = pb * static_cast<std::size_t>(R_);
  if (!halo_fresh_ || !static_halo_ok_) {
    // Fields were rewritten from the host (upload / reset / step_host) on
    // every rank: post that, wait for both neighbours' posts (flag words 2
    // and 3 count rewrite epochs), then pull their edge planes once.
    ++post_epoch_;
    memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_left_.flags + 3), post_epoch_,
                          CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
    memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_right_.flags + 2), post_epoch_,
                          CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
    memop_check(ops.wait(cs_, reinterpret_cast<CUdeviceptr>(flags_ + 2), post_epoch_,
                         CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue64");
    memop_check(ops.wait(cs_, reinterpret_cast<CUdeviceptr>(flags_ + 3), post_epoch_,
                         CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue64");
  }
  if (!static_halo_ok_) {
    for (int f = 0; f < 4; ++f) {
      char* mine = static_cast<char*>(st_[f]);
      IMB_CUDA(cudaMemcpyAsync(mine, ipc_left_.pool + ipc_left_.off_st[f] + pb * ipc_left_.ni, hb,
                               cudaMemcpyDefault, cs_));
      IMB_CUDA(cudaMemcpyAsync(mine + pb * static_cast<std::size_t>(R_ + ni_),
                               ipc_right_.pool + ipc_right_.off_st[f] + pb * R_, hb,
                               cudaMemcpyDefault, cs_));
    }
    static_halo_ok_ = true;
  }
  if (!halo_fresh_) {  // the neighbours' current x is the buffer they wrote in step s-1
    char* mine = static_cast<char*>(x_);
    const char* lsrc = static_cast<const char*>(ipc_left_.buffer(static_cast<std::int64_t>(s) - 1));
    const char* rsrc = static_cast<const char*>(ipc_right_.buffer(static_cast<std::int64_t>(s) - 1));
    IMB_CUDA(cudaMemcpyAsync(mine, lsrc + pb * ipc_left_.ni, hb, cudaMemcpyDefault, cs_));
    IMB_CUDA(cudaMemcpyAsync(mine + pb * static_cast<std::size_t>(R_ + ni_), rsrc + pb * R_, hb,
                             cudaMemcpyDefault, cs_));
  }
  begin_compute_window();
  push_lo_ = ipc_left_.buffer(static_cast<std::int64_t>(s));
  push_lo_ni_ = ipc_left_.ni;
  push_hi_ = ipc_right_.buffer(static_cast<std::int64_t>(s));
  push_sys_ = ipc_left_.device != device_ || ipc_right_.device != device_;
  swap_after_ = false;
  compute_step();
  swap_after_ = true;
  end_compute_window();
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_left_.flags + 1), s + 1,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(ipc_right_.flags + 0), s + 1,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
  std::swap(x_, xn_);
  ++step_count_;
  halo_fresh_ = true;
}

void Team::group_mark_ready() {
  IMB_CUDA(cudaSetDevice(device_));
  IMB_CUDA(cudaEventRecord(ev_ready_, cs_));
}

void Team::group_pull() {
  IMB_CUDA(cudaSetDevice(device_));
  // Both neighbours finished the previous step: their edge planes are final
  // and their kernels no longer read the buffers this step writes into.
  IMB_CUDA(cudaStreamWaitEvent(cs_, left_->ev_ready_, 0));
  IMB_CUDA(cudaStreamWaitEvent(cs_, right_->ev_ready_, 0));
  if (!static_halo_ok_) {
    for (int f = 1; f <= 4; ++f) pull_from_ring(f, cs_);
    static_halo_ok_ = true;
  }
  // Fused slabs push their edge planes into the neighbours' halos from the
  // kernel epilogue; a copy is only needed when x's halos are stale.
  if (tmp_[0] != nullptr || !halo_fresh_) pull_from_ring(0, cs_);
}

void Team::group_compute() {
  IMB_CUDA(cudaSetDevice(device_));
  begin_compute_window();
  if (tmp_[0] == nullptr) {
    // push targets: the neighbours' output buffers of this step (their
    // pointers are swapped only in group_finish, after every launch)
    push_lo_ = push_ok_ ? left_->xn_ : nullptr;
    push_lo_ni_ = left_->ni_;
    push_hi_ = push_ok_ ? right_->xn_ : nullptr;
    push_sys_ = left_->device_ != device_ || right_->device_ != device_;
    swap_after_ = false;
    compute_step();
    swap_after_ = true;
  } else {
    compute_step();
  }
  end_compute_window();
}

// Flag-synchronised group step (fused slabs only): no host phases and no
// events. Each step waits — in the stream front-end, no spinning kernel —
// until both neighbours have announced the end of the previous step through
// this team's flag words, launches the fused kernel that pushes its edge
// planes into the neighbours' step-s output buffers (device stores; NVLink
// for a peer GPU), then announces its own step in the neighbours' flags.
// Every wait depends only on work issued earlier, so the ring cannot
// deadlock. Buffers: step s writes bufs[(s+1)%2] of every team (all teams
// step together), which lets a team address a neighbour's buffer without
// reading its host-side pointers.
void Team::group_flag_step() {
  IMB_CUDA(cudaSetDevice(device_));
  MemOps& ops = memops();
  const std::uint64_t s = step_count_;
  memop_check(ops.wait(cs_, reinterpret_cast<CUdeviceptr>(flags_ + 0), s, CU_STREAM_WAIT_VALUE_GEQ),
              "cuStreamWaitValue64");
  memop_check(ops.wait(cs_, reinterpret_cast<CUdeviceptr>(flags_ + 1), s, CU_STREAM_WAIT_VALUE_GEQ),
              "cuStreamWaitValue64");
  if (!static_halo_ok_ || !halo_fresh_)
    throw ContractError("flag-synchronised step needs fresh halos (run an event step first)");
  begin_compute_window();
  push_lo_ = left_->out_buffer(s);
  push_lo_ni_ = left_->ni_;
  push_hi_ = right_->out_buffer(s);
  push_sys_ = left_->device_ != device_ || right_->device_ != device_;
  swap_after_ = false;
  compute_step();
  swap_after_ = true;
  end_compute_window();
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(left_->flags_ + 1), s + 1,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
  memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(right_->flags_ + 0), s + 1,
                        CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
  std::swap(x_, xn_);
  ++step_count_;
  halo_fresh_ = true;
}

void* Team::out_buffer(std::uint64_t s) const {
  // x_/xn_ alternate every step; step s writes the buffer that is xn_ when
  // this team has completed exactly s steps.
  return ((s - step_count_) % 2 == 0) ? xn_ : x_;
}

void Team::group_finish(bool signal) {
  if (tmp_[0] == nullptr) {
    std::swap(x_, xn_);
    halo_fresh_ = push_ok_ && left_->push_ok_ && right_->push_ok_;
  }
  if (signal) {  // keep the flag protocol's counters in step (flag mode after an event step)
    MemOps& ops = memops();
    memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(left_->flags_ + 1), step_count_ + 1,
                          CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
    memop_check(ops.write(cs_, reinterpret_cast<CUdeviceptr>(right_->flags_ + 0), step_count_ + 1,
                          CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
  }
  ++step_count_;
}

}  // namespace imb::rt
