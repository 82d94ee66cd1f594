// GPU team runtime: one Team owns one i-slab of the periodic global grid on
// one device — the B200 counterpart of imb::TeamRunner
// (/root/reference/proj/include/imbalance/workload.hpp:94-122), where a team
// of CPU threads becomes one GPU. It owns the padded-slab device buffers,
// a compute stream and a communication stream, and one of three halo
// exchangers: itself (periodic single slab), an in-process ring of teams
// (device copies; also the P-slabs-on-one-GPU test backend), or NCCL
// send/recv between processes (one process per GPU).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "mpdata_kernels.cuh"

namespace imb::rt {

struct Options {
  int iord = 2;
  int nonos = 1;
  bool fp64 = true;
};

int step_radius(const Options& o);

// One point-to-point operation of the per-step ring halo swap.
struct RingOp {
  int kind;                  // 0 = send, 1 = recv
  int peer;                  // rank in the slab ring
  std::int64_t first_plane;  // plane offset inside the padded slab
  std::int64_t planes;       // number of contiguous planes
};
// The 4-operation plan every rank issues, in this order, each step: send
// my first R interior planes left, my last R right, receive the right halo
// from the right, the left halo from the left. Operations to one peer are
// matched in issue order, so the two-rank ring (left == right) pairs
// first->right-halo and last->left-halo correctly.
void ring_plan(int rank, int nranks, std::int64_t ni, std::int64_t R, RingOp out[4]);

class NcclLink;  // defined in team.cpp

// cuStreamWaitValue64 / cuStreamWriteValue64 resolvable on this driver.
bool stream_memops_available();

class Team {
 public:
  Team(std::int64_t n, std::int64_t m, std::int64_t l, const Options& opt, int device,
       std::int64_t i0, std::int64_t ni);
  ~Team();
  Team(const Team&) = delete;
  Team& operator=(const Team&) = delete;

  void init_recipe(int kind, std::uint64_t seed);
  void upload(int field, const void* host, std::size_t bytes);
  void download(int field, void* host, std::size_t bytes);
  void reset();
  void run(int steps, double* compute_s, double* wall_s);
  void step_host(const void* x_in, void* x_out);
  std::uint64_t checksum();

  void connect_nccl(const unsigned char* id, int nranks, int rank);
  // Multi-process halo push (one process per GPU, no NCCL): export this
  // team's buffers as CUDA IPC handles, map the ring neighbours' and then
  // step with the flag protocol, the step kernel storing edge planes straight
  // into the neighbours' halos over NVLink.
  static constexpr int kIpcBlobBytes = 512;
  void ipc_export(unsigned char* blob);
  void connect_ipc(const unsigned char* left_blob, const unsigned char* right_blob, int nranks,
                   int rank);
  // In-process ring wiring (imb_group): neighbours own the adjacent slabs.
  void set_ring(Team* left, Team* right) {
    left_ = left;
    right_ = right;
  }
  // False when this team's device cannot store into a neighbour's device
  // memory (no peer access): its kernel then pushes nothing and the ring
  // falls back to pulling the edge planes with peer copies every step.
  void set_push_ok(bool ok) { push_ok_ = ok; }
  bool push_ok() const { return push_ok_; }

  // Group stepping, issued by imb_group in four host phases per step, each
  // over all teams before the next: (1) record "x of this step is complete";
  // (2) wait for both neighbours, then (staged slabs, or stale halos) pull
  // their edge planes into the halos; (3) launch the step — fused slabs push
  // their edge planes into the neighbours' next-step halos from the kernel
  // epilogue, targeting the neighbours' current output buffers; (4) swap.
  // The swap is deferred to phase 4 so phase 3 sees every team's buffers of
  // this step.
  void group_mark_ready();
  void group_pull();
  void group_compute();
  // phase 4: swap the ping-pong buffers (fused push path); with `signal`,
  // also announce the step in the neighbours' flag words. The group signals
  // on every event step whenever the flag protocol is usable, so switching
  // the sync mode at any point finds the flag words in step.
  void group_finish(bool signal = false);
  bool halos_ready() const { return static_halo_ok_ && halo_fresh_; }
  // Alternative group protocol for fused slabs: one call per team per step,
  // synchronised through device flag words (cuStreamWaitValue/WriteValue).
  void group_flag_step();
  bool fused() const { return tmp_[0] == nullptr; }

  std::int64_t launches() const { return launches_; }
  int device() const { return device_; }
  std::int64_t ni() const { return ni_; }
  std::int64_t i0() const { return i0_; }
  std::int64_t radius() const { return R_; }
  cudaStream_t stream() const { return cs_; }
  cudaEvent_t ready_event() const { return ev_ready_; }
  double take_compute_seconds();
  std::size_t elem() const { return opt_.fp64 ? 8 : 4; }

 private:
  void exchange_static();
  void exchange_x_self(void* x);
  void exchange_x_nccl(void* x);
  void pull_from_ring(int field, cudaStream_t st);
  void compute_step();  // x (halo-complete) -> xn, then swap
  void fused_range(std::int64_t o0, std::int64_t o1);
  void step_overlapped();  // NCCL exchange hidden behind the interior planes
  void step_host_pipelined(const void* x_in, void* x_out);
  cudaStream_t ups_ = nullptr, dns_ = nullptr;  // H2D / D2H copy streams (step_host)
  std::vector<cudaEvent_t> ev_pipe_;
  std::vector<std::int64_t> pipe_cuts_;  // host-step chunk boundaries (step_host_pipelined)
  template <class T>
  void compute_step_t();
  void* fbuf(int field) const;
  std::size_t plane_bytes() const { return static_cast<std::size_t>(m_ * l_) * elem(); }
  void begin_compute_window();
  void end_compute_window();

  std::int64_t n_, m_, l_;
  Options opt_;
  int device_;
  std::int64_t i0_, ni_, R_, P_;
  int num_sms_ = 148;
  cudaStream_t cs_ = nullptr, xs_ = nullptr;  // compute, exchange
  cudaEvent_t ev_ready_ = nullptr, ev_halo_ = nullptr;
  std::vector<cudaEvent_t> ev_pool_;  // begin/end pairs of compute windows
  std::size_t ev_used_ = 0;
  // device buffers (padded slabs of P_ planes)
  void* pool_ = nullptr;
  void* x_ = nullptr;
  void* xn_ = nullptr;
  void* x0_ = nullptr;
  void* st_[4] = {nullptr, nullptr, nullptr, nullptr};  // u, v, w, h
  void* tmp_[12] = {};  // iterates, 2 velocity sets, mx, mn, bu, bd
  void* ext_[6] = {};   // fused IORD=3: psi^(2), mx, mn, limited u, v, w
  bool static_halo_ok_ = false;
  // Halo push of the next fused launch (consumed by it) and whether x's halo
  // planes already hold the neighbours' edge planes (written by the previous
  // step's push), so no exchange is needed before the next step.
  void* push_lo_ = nullptr;
  void* push_hi_ = nullptr;
  std::int64_t push_lo_ni_ = 0;
  bool halo_fresh_ = false;
  bool swap_after_ = true;
  bool push_ok_ = true;
  bool push_sys_ = false;  // the current push targets include a peer GPU
  void acquire();           // device resources (streams, events, pool); throws
  void release() noexcept;  // frees whatever acquire() obtained
  std::uint64_t* flags_ = nullptr;  // [0]/[1] left/right neighbour's finished steps,
                                    // [2]/[3] their host-rewrite epochs (IPC ring)
  struct IpcPeer {
    char* pool = nullptr;            // mapped neighbour pool (or this team's own)
    std::uint64_t* flags = nullptr;  // mapped neighbour flag words
    std::int64_t off_x = 0, off_xn = 0, ni = 0, step0 = 0;
    int device = -1;
    std::int64_t off_st[4] = {0, 0, 0, 0};
    bool opened = false;             // this process opened (and must close) it
    void* buffer(std::int64_t s) const {  // the buffer that peer writes in step s
      return pool + (((s - step0) % 2 == 0) ? off_xn : off_x);
    }
  };
  IpcPeer ipc_left_, ipc_right_;
  bool ipc_ = false;
  std::uint64_t post_epoch_ = 0;  // host rewrites of x posted to the IPC neighbours
  void ipc_step();
  std::uint64_t step_count_ = 0;    // steps taken through the group protocols
  void* out_buffer(std::uint64_t s) const;
  std::int64_t launches_ = 0;
  // Periodic single slab: two fused steps (x -> xn -> x) captured as one CUDA
  // graph per starting buffer, replayed to cut per-step launch overhead.
  cudaGraphExec_t graph_[2] = {nullptr, nullptr};
  void* graph_x_[2] = {nullptr, nullptr};
  std::int64_t graph_launches_ = 0;  // kernels per replay
  bool graph_step_pair();
  Team* left_ = nullptr;
  Team* right_ = nullptr;
  std::unique_ptr<NcclLink> nccl_;
};

}  // namespace imb::rt
