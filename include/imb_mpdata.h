/*
 * imb_mpdata.h — the C-ABI drop-in boundary of the B200-native MPDATA
 * framework (libimb_b200.so). Plain pointers and sizes only; no C++ or torch
 * types cross it, and no exception escapes it.
 *
 * Every entry point names the reference interface it replaces. The
 * reference is the C++20 toolkit under /root/reference/proj (headers in
 * include/imbalance/), which has no FFI of its own; a binding a maintainer
 * would add is shown in INTEGRATION.md.
 *
 * Errors (errors.hpp:10-64): every function returns an int status. 0 is
 * success; 1..10 map one-to-one onto the reference exception types; 20+
 * are device-side failures. imb_last_error() returns the thread-local
 * message of the last failure on the calling thread.
 */
#ifndef IMB_MPDATA_H
#define IMB_MPDATA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: errors.hpp:15-64 ------------------------------------ */
enum {
  IMB_OK = 0,
  IMB_E_RANGE = 1,        /* RangeError              errors.hpp:15 */
  IMB_E_DOMAIN = 2,       /* DomainError             errors.hpp:20 */
  IMB_E_ALIGNMENT = 3,    /* AlignmentError          errors.hpp:25 */
  IMB_E_INCOMPATIBLE = 4, /* IncompatibleModelError  errors.hpp:30 */
  IMB_E_INSUFFICIENT = 5, /* InsufficientDataError   errors.hpp:35 */
  IMB_E_INFEASIBLE = 6,   /* InfeasibleError         errors.hpp:40 */
  IMB_E_TOOLARGE = 7,     /* TooLargeError           errors.hpp:45 */
  IMB_E_CONFIG = 8,       /* ConfigError             errors.hpp:50 */
  IMB_E_CONTRACT = 9,     /* ContractError           errors.hpp:55 */
  IMB_E_PARSE = 10,       /* ParseError              errors.hpp:60-64 */
  IMB_E_CUDA = 20,        /* CUDA runtime failure (no reference analogue) */
  IMB_E_NCCL = 21,        /* NCCL failure */
  IMB_E_NOMEM = 22,       /* device or host allocation failed */
  IMB_E_INTERNAL = 99
};

/* Thread-local message of the last failing call on this thread. */
const char* imb_last_error(void);
const char* imb_version(void); /* version.hpp:5 kVersion */

/* ---- grid + options: workload.hpp:14-26 (StencilDomain) ----------------- */
typedef struct imb_domain {
  int64_t n, m, l; /* interior extents; n is the slab (outermost) axis */
  int64_t halo;    /* ghost width of the host GridField layout (>= 1) */
} imb_domain;

enum { IMB_FP64 = 0, IMB_FP32 = 1 };
enum { IMB_RECIPE_UNIFORM = 0, IMB_RECIPE_GAUSS = 1, IMB_RECIPE_ROTCUBE = 2 };
enum { IMB_FIELD_X = 0, IMB_FIELD_U = 1, IMB_FIELD_V = 2, IMB_FIELD_W = 3, IMB_FIELD_H = 4 };

/* Additive to the reference (which fixes a 5-stage surrogate):
 * the real MPDATA step options. */
typedef struct imb_opts {
  int iord;      /* passes: 1 donor-cell only, 2 = +1 corrective, 3 = +2 (>= 1) */
  int nonos;     /* nonoscillatory limiter on/off */
  int precision; /* IMB_FP64 / IMB_FP32 */
} imb_opts;

/* Dependency radius of one fused step: 1 + sum_{k=2..iord} (nonos ? 2 : 1). */
int imb_step_radius(const imb_opts* opts);

/* ---- one team = one GPU owning i-slab [i0, i0+ni) of a periodic global
 * grid: workload.hpp:94-122 (TeamRunner). Host arrays are slab interiors,
 * ni*m*l values of the team precision, i outermost and k contiguous
 * (the interior order of GridField::index, workload.hpp:40-43). ---- */
typedef struct imb_team imb_team;

/* TeamRunner(domain, threads, seed, pin_base_core), workload.hpp:96-97:
 * `device` replaces `threads`; (i0, ni) is the team's slab of `global`. */
int imb_team_create(const imb_domain* global, const imb_opts* opts, int device, int64_t i0,
                    int64_t ni, imb_team** out);
int imb_team_destroy(imb_team* t); /* idempotent on NULL */

/* init_fields(domain, seed), workload.hpp:61-64: device-side seeded
 * recipe, a pure function of (seed, field, global i, j, k). */
int imb_team_init_recipe(imb_team* t, int recipe, uint64_t seed);
/* Upload/download one field's slab interior (bytes = ni*m*l*elem). */
int imb_team_upload(imb_team* t, int field, const void* host, size_t bytes);
int imb_team_download(imb_team* t, int field, void* host, size_t bytes);
/* reset(), workload.hpp:99: restore x to the state of the last init/upload. */
int imb_team_reset(imb_team* t);

/* run(steps, ...), workload.hpp:101-109: `steps` MPDATA steps including the
 * per-step halo exchange; *compute_s = summed device time of the step
 * kernels (CUDA events), *wall_s = device time of the whole run including
 * exchange. Blocks until done. Either out pointer may be NULL. */
int imb_team_run(imb_team* t, int steps, double* compute_s, double* wall_s);
/* Reference-facing host-buffer step (run_step, workload.hpp:76-80, with
 * the static fields already resident): copy x_in (host) to the device,
 * one step, copy the result to x_out (host). Pinned buffers are faster. */
int imb_team_step_host(imb_team* t, const void* x_in, void* x_out);
/* current_checksum(), workload.hpp:111: FNV-1a 64 over the interior bytes. */
int imb_team_checksum(imb_team* t, uint64_t* out);
/* Kernel launches issued by this team so far (evidence counter). */
int64_t imb_team_launch_count(const imb_team* t);

/* ---- multi-rank (one process per GPU) exchange over NCCL ---------------
 * Rank r's neighbours in the periodic slab ring are r-1 and r+1 (mod n).
 * Without a connect call a team is its own periodic neighbour. */
enum { IMB_NCCL_ID_BYTES = 128 };
int imb_nccl_unique_id(unsigned char id[IMB_NCCL_ID_BYTES]);
int imb_team_connect_nccl(imb_team* t, const unsigned char id[IMB_NCCL_ID_BYTES], int nranks,
                          int rank);
/* NVLink halo push between processes (no NCCL): every rank exports its
 * buffers as CUDA IPC handles, the blobs are exchanged by any control plane,
 * and each rank maps its ring neighbours'. From then on imb_team_run waits
 * on device flag words (cuStreamWaitValue64), the step kernel stores its edge
 * planes straight into the neighbours' halos, and the rank raises the
 * neighbours' flags (cuStreamWriteValue64). All ranks must connect at the
 * same step count and then step in lockstep; host rewrites of x (upload,
 * reset, step_host) must also happen on every rank. Connecting probes the
 * peer flag writes, so an unsupported mapping fails there (status 20)
 * before any rank steps. Synchronise all ranks (any control-plane barrier
 * after their last run) before destroying a connected team: the neighbours'
 * kernels write into its buffers. */
enum { IMB_IPC_BLOB_BYTES = 512 };
int imb_team_ipc_export(imb_team* t, unsigned char blob[IMB_IPC_BLOB_BYTES]);
int imb_team_connect_ipc(imb_team* t, const unsigned char left[IMB_IPC_BLOB_BYTES],
                         const unsigned char right[IMB_IPC_BLOB_BYTES], int nranks, int rank);
/* The 4 point-to-point operations a rank issues per step (in order):
 * kinds[q] 0 = send / 1 = recv, peers[q], and the plane range
 * [first_plane[q], first_plane[q] + planes[q]) of the padded slab
 * (ni interior planes + R halo planes on each side). Host-only; the NCCL
 * exchange executes exactly this plan. */
int imb_ring_plan(int rank, int nranks, int64_t ni, int64_t R, int kinds[4], int peers[4],
                  int64_t first_plane[4], int64_t planes[4]);
/* Slab offsets = exclusive prefix sums of the shares, in processor order
 * (the decomposition of SURVEY.md §8a-12). */
int imb_slab_offsets(const int64_t* shares, int p, int64_t* offsets);

/* ---- in-process group of teams (the fake multi-GPU backend / one host
 * thread per GPU): slabs from `shares` in ring order, exchange by device
 * copies. devices[g] may repeat (P virtual slabs on one GPU). ---------- */
typedef struct imb_group imb_group;
int imb_group_create(const imb_domain* global, const imb_opts* opts, int nteams,
                     const int* devices, const int64_t* shares, imb_group** out);
int imb_group_destroy(imb_group* g);
int imb_group_team(imb_group* g, int index, imb_team** out);
int imb_group_init_recipe(imb_group* g, int recipe, uint64_t seed);
/* Step synchronisation of a group. EVENTS (default): four stream-ordered
 * host phases per step. FLAGS (fused slabs): each team's stream waits on
 * device flag words its neighbours write after their step
 * (cuStreamWaitValue64 / cuStreamWriteValue64) — no host phases, no events;
 * the halo planes travel inside the step kernel (peer stores). */
enum { IMB_GROUP_SYNC_EVENTS = 0, IMB_GROUP_SYNC_FLAGS = 1 };
int imb_group_set_sync(imb_group* g, int mode);
/* per_team_s[g] = compute seconds of team g; *wall_s = max over teams of
 * the run span including exchange waits. */
int imb_group_run(imb_group* g, int steps, double* per_team_s, double* wall_s);

/* ---- reference stage ops on the padded GridField layout
 * ((n+2h)(m+2h)(l+2h) doubles): workload.hpp:66-74 ---------------------- */
int imb_fill_halo_clamped(const imb_domain* d, double* field);
int imb_stage_max7(const imb_domain* d, const double* in, double* out);
int imb_stage_min7(const imb_domain* d, const double* in, double* out);
/* checksum(f), workload.hpp:82-83, over the interior of a padded field. */
int imb_checksum_padded(const imb_domain* d, const double* field, uint64_t* out);

/* ---- FPM speed functions: fpm.hpp:13-127 --------------------------------
 * A speed function is passed as (unit_cells, granularity, samples, count);
 * the constructor checks of fpm.cpp:11-33 apply to every call. */
typedef struct imb_speed_sample {
  int64_t x;           /* workload units (frames of unit_cells cells) */
  double speed;        /* cells per second, > 0 */
  double ci_halfwidth; /* >= 0 */
  int64_t repetitions; /* >= 1 */
} imb_speed_sample;

int imb_speed_validate(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s, int ns);
int imb_eval_speed(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s, int ns,
                   double x, double* out); /* fpm.hpp:93-96 */
int imb_eval_time(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s, int ns,
                  double x, double* out); /* fpm.hpp:98-101 */
/* check_condition, fpm.hpp:103: up to `cap` violating pairs in viol[2i],
 * viol[2i+1]; *nviol = total; max_gain_pair = {-1,-1} when satisfied. */
int imb_check_condition(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                        int ns, int* satisfied, int64_t* viol, int cap, int* nviol,
                        int64_t max_gain_pair[2]);
/* classify_shape, fpm.hpp:107: 0 decreasing, 1 increasing-concave-then-
 * decreasing, 2 other; *peak_x = -1 when absent. */
int imb_classify_shape(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                       int ns, int* cls, int64_t* peak_x);
/* average, fpm.hpp:113: nf functions x ns samples, samples[f*ns + i]. */
int imb_average(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s, int nf,
                int ns, imb_speed_sample* out);
/* scaled, fpm.hpp:118. */
int imb_scaled(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s, int ns,
               double factor, imb_speed_sample* out);

/* Speed-function CSV (the "# unit_cells=.. granularity=..
 * label=.." header, then x,speed,ci_halfwidth,repetitions rows, doubles at
 * %.17g). The one parser/writer of the format (csrc/host/fpm.cpp); the
 * Python mirror and the CLI go through these.
 * parse: up to `cap` samples into out, *ns = the sample count (call with
 * cap = 0 to size), label copied NUL-terminated into label[label_cap];
 * IMB_E_PARSE with the 1-based line in *err_line (0 otherwise).
 * format: the text into out[cap] (NUL-terminated), *len = its length
 * without the NUL; IMB_E_RANGE when cap is too small (*len says how much). */
int imb_speed_csv_parse(const char* text, size_t len, int64_t* unit_cells, int64_t* granularity,
                        imb_speed_sample* out, int cap, int* ns, char* label, size_t label_cap,
                        int* err_line);
int imb_speed_csv_format(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                         int ns, const char* label, char* out, size_t cap, size_t* len);

/* slice_surface, fpm.hpp:123 (+ SpeedSurface::validate, fpm.hpp:81-91): the
 * surface is nn x nm samples, row-major in n (samples[i*nm + j].x must equal
 * m_values[j]); out receives the nm samples of row fixed_n and
 * *out_unit_cells = fixed_n * unit_cells. */
int imb_slice_surface(int64_t unit_cells, int64_t granularity, const int64_t* n_values, int nn,
                      const int64_t* m_values, int nm, const imb_speed_sample* samples,
                      int64_t fixed_n, imb_speed_sample* out, int64_t* out_unit_cells);

/* ---- partitioner: partition.hpp:17-72 ----------------------------------
 * shares/per_time hold `p` values; *offset = -1 when absent. */
int imb_predict_makespan(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                         int ns, const int64_t* shares, int p, double* per_time,
                         double* makespan); /* partition.hpp:37 */
int imb_partition_paired(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                         int ns, int64_t total, int p, int allow_idle, int64_t* shares,
                         double* per_time, double* makespan,
                         int64_t* offset); /* partition.hpp:45, Algorithm 1 */
int imb_partition_general(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                          int ns, int64_t total, int p, int allow_idle, int64_t* shares,
                          double* per_time, double* makespan,
                          int64_t* offset); /* partition.hpp:51 */
int imb_brute_force_oracle(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                           int ns, int64_t total, int p, int allow_idle, int64_t cap,
                           int64_t* shares, double* per_time, double* makespan,
                           int64_t* offset); /* partition.hpp:56 */
int imb_improvement_search(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                           int ns, int64_t balanced, int* found, int64_t* delta, double* gain,
                           int64_t pair[2]); /* partition.hpp:69 */

/* ---- stats: stats.hpp:8-33 (Boost-free) -------------------------------- */
double imb_t_quantile_975(int df);
int imb_summarize(const double* xs, int n, double* mean, double* stddev, double* ci_halfwidth);

#ifdef __cplusplus
}
#endif
#endif
