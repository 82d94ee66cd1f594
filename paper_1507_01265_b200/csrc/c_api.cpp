// The C-ABI boundary (include/imb_mpdata.h): extern "C" entry points over the
// imb:: host API and the GPU team runtime. Exceptions never cross it: every
// imb::Error becomes its numeric status (errors.hpp mapping) and the message
// is kept thread-locally for imb_last_error().
#include "imb_mpdata.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <sstream>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "imbalance/errors.hpp"
#include "imbalance/fpm.hpp"
#include "imbalance/partition.hpp"
#include "imbalance/stats.hpp"
#include "imbalance/workload.hpp"
#include "team.hpp"

namespace imb::rt {
void nccl_unique_id(unsigned char* out);
}

struct imb_team {
  std::unique_ptr<imb::rt::Team> t;
  bool owned = true;  // false for teams owned by a group
};

struct imb_group {
  std::vector<std::unique_ptr<imb::rt::Team>> teams;
  std::vector<imb_team> handles;
  int sync = 0;  // IMB_GROUP_SYNC_EVENTS / IMB_GROUP_SYNC_FLAGS
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    return IMB_OK;
  } catch (const imb::Error& e) {
    g_last_error = e.what();
    return e.code();
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return IMB_E_NOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return IMB_E_INTERNAL;
  } catch (...) {
    g_last_error = "unknown failure";
    return IMB_E_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw imb::ContractError(std::string(what) + " must not be NULL");
}

imb::SpeedFunction model(std::int64_t unit, std::int64_t g, const imb_speed_sample* s, int ns) {
  if (ns < 0) throw imb::ContractError("sample count must be >= 0");
  if (ns > 0) need(s, "samples");
  std::vector<imb::SpeedSample> v(static_cast<std::size_t>(ns));
  for (int q = 0; q < ns; ++q) v[static_cast<std::size_t>(q)] = {s[q].x, s[q].speed, s[q].ci_halfwidth, s[q].repetitions};
  return imb::SpeedFunction(unit, g, std::move(v), "c-abi");
}

imb::rt::Options opts_of(const imb_opts* o) {
  need(o, "opts");
  if (o->precision != IMB_FP64 && o->precision != IMB_FP32)
    throw imb::ConfigError("precision must be IMB_FP64 or IMB_FP32");
  return imb::rt::Options{o->iord, o->nonos ? 1 : 0, o->precision == IMB_FP64};
}

void put(const imb::Partition& p, std::int64_t* shares, double* per_time, double* makespan,
         std::int64_t* offset) {
  for (std::size_t q = 0; q < p.shares.size(); ++q) {
    if (shares) shares[q] = p.shares[q];
    if (per_time) per_time[q] = p.per_time[q];
  }
  if (makespan) *makespan = p.makespan;
  if (offset) *offset = p.offset ? *p.offset : -1;
}

imb::StencilDomain dom(const imb_domain* d) {
  need(d, "domain");
  imb::StencilDomain s{d->n, d->m, d->l, d->halo};
  s.validate();
  return s;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw imb::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

imb::rt::Team& team_of(imb_team* t) {
  need(t, "team");
  return *t->t;
}

}  // namespace

extern "C" {

const char* imb_last_error(void) { return g_last_error.c_str(); }
const char* imb_version(void) { return "0.1.0-b200"; }

int imb_step_radius(const imb_opts* opts) {
  imb::rt::Options o;
  int r = -1;
  const int st = guard([&] {
    o = opts_of(opts);
    r = imb::rt::step_radius(o);
  });
  return st == IMB_OK ? r : -st;
}

// ---- teams -------------------------------------------------------------------
int imb_team_create(const imb_domain* global, const imb_opts* opts, int device, int64_t i0,
                    int64_t ni, imb_team** out) {
  return guard([&] {
    need(global, "global");
    need(out, "out");
    *out = nullptr;
    auto h = std::make_unique<imb_team>();
    h->t = std::make_unique<imb::rt::Team>(global->n, global->m, global->l, opts_of(opts), device,
                                           i0, ni);
    *out = h.release();
  });
}

int imb_team_destroy(imb_team* t) {
  return guard([&] {
    if (t && t->owned) delete t;
  });
}

int imb_team_init_recipe(imb_team* t, int recipe, uint64_t seed) {
  return guard([&] { team_of(t).init_recipe(recipe, seed); });
}

int imb_team_upload(imb_team* t, int field, const void* host, size_t bytes) {
  return guard([&] {
    need(host, "host");
    team_of(t).upload(field, host, bytes);
  });
}

int imb_team_download(imb_team* t, int field, void* host, size_t bytes) {
  return guard([&] {
    need(host, "host");
    team_of(t).download(field, host, bytes);
  });
}

int imb_team_reset(imb_team* t) {
  return guard([&] { team_of(t).reset(); });
}

int imb_team_run(imb_team* t, int steps, double* compute_s, double* wall_s) {
  return guard([&] { team_of(t).run(steps, compute_s, wall_s); });
}

int imb_team_step_host(imb_team* t, const void* x_in, void* x_out) {
  return guard([&] {
    need(x_in, "x_in");
    need(x_out, "x_out");
    team_of(t).step_host(x_in, x_out);
  });
}

int imb_team_checksum(imb_team* t, uint64_t* out) {
  return guard([&] {
    need(out, "out");
    *out = team_of(t).checksum();
  });
}

int64_t imb_team_launch_count(const imb_team* t) { return (t && t->t) ? t->t->launches() : -1; }

int imb_nccl_unique_id(unsigned char id[IMB_NCCL_ID_BYTES]) {
  return guard([&] {
    need(id, "id");
    imb::rt::nccl_unique_id(id);
  });
}

int imb_team_connect_nccl(imb_team* t, const unsigned char id[IMB_NCCL_ID_BYTES], int nranks,
                          int rank) {
  return guard([&] {
    need(id, "id");
    team_of(t).connect_nccl(id, nranks, rank);
  });
}

int imb_team_ipc_export(imb_team* t, unsigned char blob[IMB_IPC_BLOB_BYTES]) {
  return guard([&] {
    need(blob, "blob");
    team_of(t).ipc_export(blob);
  });
}

int imb_team_connect_ipc(imb_team* t, const unsigned char left[IMB_IPC_BLOB_BYTES],
                         const unsigned char right[IMB_IPC_BLOB_BYTES], int nranks, int rank) {
  return guard([&] {
    need(left, "left");
    need(right, "right");
    team_of(t).connect_ipc(left, right, nranks, rank);
  });
}

int imb_ring_plan(int rank, int nranks, int64_t ni, int64_t R, int* kinds, int* peers,
                  int64_t* first_plane, int64_t* planes) {
  return guard([&] {
    need(kinds, "kinds");
    need(peers, "peers");
    need(first_plane, "first_plane");
    need(planes, "planes");
    imb::rt::RingOp ops[4];
    imb::rt::ring_plan(rank, nranks, ni, R, ops);
    for (int q = 0; q < 4; ++q) {
      kinds[q] = ops[q].kind;
      peers[q] = ops[q].peer;
      first_plane[q] = ops[q].first_plane;
      planes[q] = ops[q].planes;
    }
  });
}

int imb_slab_offsets(const int64_t* shares, int p, int64_t* offsets) {
  return guard([&] {
    need(shares, "shares");
    need(offsets, "offsets");
    if (p < 1) throw imb::ContractError("share list is empty");
    const std::vector<std::int64_t> off =
        imb::slab_offsets(std::span<const std::int64_t>(shares, static_cast<std::size_t>(p)));
    std::copy(off.begin(), off.end(), offsets);
  });
}

// ---- groups ------------------------------------------------------------------
int imb_group_create(const imb_domain* global, const imb_opts* opts, int nteams,
                     const int* devices, const int64_t* shares, imb_group** out) {
  return guard([&] {
    need(global, "global");
    need(devices, "devices");
    need(shares, "shares");
    need(out, "out");
    *out = nullptr;
    if (nteams < 1) throw imb::ContractError("a group needs at least one team");
    std::int64_t sum = 0;
    for (int g = 0; g < nteams; ++g) sum += shares[g];
    if (sum != global->n)
      throw imb::ContractError("shares sum to " + std::to_string(sum) + ", grid has n=" +
                               std::to_string(global->n));
    const std::vector<std::int64_t> off =
        imb::slab_offsets(std::span<const std::int64_t>(shares, static_cast<std::size_t>(nteams)));
    const imb::rt::Options o = opts_of(opts);
    auto grp = std::make_unique<imb_group>();
    for (int g = 0; g < nteams; ++g)
      grp->teams.push_back(std::make_unique<imb::rt::Team>(global->n, global->m, global->l, o,
                                                           devices[g], off[static_cast<std::size_t>(g)],
                                                           shares[g]));
    for (int g = 0; g < nteams; ++g) {
      imb::rt::Team* left = grp->teams[static_cast<std::size_t>((g + nteams - 1) % nteams)].get();
      imb::rt::Team* right = grp->teams[static_cast<std::size_t>((g + 1) % nteams)].get();
      grp->teams[static_cast<std::size_t>(g)]->set_ring(left, right);
      for (imb::rt::Team* nb : {left, right}) {
        if (nb->device() == devices[g]) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices[g], nb->device());
        if (!can) {  // the kernel cannot store into that device: pull with peer copies
          grp->teams[static_cast<std::size_t>(g)]->set_push_ok(false);
          continue;
        }
        cudaSetDevice(devices[g]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(nb->device(), 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else if (e != cudaSuccess) {
          cudaGetLastError();
          grp->teams[static_cast<std::size_t>(g)]->set_push_ok(false);
        }
      }
    }
    grp->handles.resize(static_cast<std::size_t>(nteams));
    for (int g = 0; g < nteams; ++g) {
      grp->handles[static_cast<std::size_t>(g)].owned = false;
    }
    *out = grp.release();
  });
}

int imb_group_destroy(imb_group* g) {
  return guard([&] {
    if (!g) return;
    for (imb_team& h : g->handles) (void)h.t.release();  // non-owning views
    delete g;
  });
}

int imb_group_team(imb_group* g, int index, imb_team** out) {
  return guard([&] {
    need(g, "group");
    need(out, "out");
    if (index < 0 || index >= static_cast<int>(g->teams.size()))
      throw imb::ContractError("team index out of range");
    imb_team& h = g->handles[static_cast<std::size_t>(index)];
    if (!h.t) h.t.reset(g->teams[static_cast<std::size_t>(index)].get());
    *out = &h;
  });
}

int imb_group_set_sync(imb_group* g, int mode) {
  return guard([&] {
    need(g, "group");
    if (mode != IMB_GROUP_SYNC_EVENTS && mode != IMB_GROUP_SYNC_FLAGS)
      throw imb::ConfigError("unknown group sync mode " + std::to_string(mode));
    g->sync = mode;
  });
}

int imb_group_init_recipe(imb_group* g, int recipe, uint64_t seed) {
  return guard([&] {
    need(g, "group");
    for (auto& t : g->teams) t->init_recipe(recipe, seed);
  });
}

int imb_group_run(imb_group* g, int steps, double* per_team_s, double* wall_s) {
  return guard([&] {
    need(g, "group");
    if (steps < 0) throw imb::ContractError("steps must be >= 0");
    const std::size_t nt = g->teams.size();
    std::vector<cudaEvent_t> t0(nt, nullptr), t1(nt, nullptr);
    struct Events {  // destroyed on every exit path, including a throw
      std::vector<imb::rt::Team*> teams;
      std::vector<cudaEvent_t>* evs[2];
      ~Events() {
        for (auto* v : evs)
          for (std::size_t q = 0; q < v->size(); ++q)
            if ((*v)[q]) {
              cudaSetDevice(teams[q]->device());
              cudaEventDestroy((*v)[q]);
            }
      }
    } guard_ev{{}, {&t0, &t1}};
    for (auto& t : g->teams) guard_ev.teams.push_back(t.get());
    for (std::size_t q = 0; q < nt; ++q) {
      cuda_ok(cudaSetDevice(g->teams[q]->device()), "cudaSetDevice");
      cuda_ok(cudaEventCreate(&t0[q]), "cudaEventCreate");
      cuda_ok(cudaEventCreate(&t1[q]), "cudaEventCreate");
      g->teams[q]->take_compute_seconds();
      cuda_ok(cudaEventRecord(t0[q], g->teams[q]->stream()), "cudaEventRecord");
    }
    // The flag protocol needs fused slabs that push into each other and the
    // stream memory operations; when it is usable, event steps keep the flag
    // words in step too, so imb_group_set_sync may switch modes at any time.
    bool can_flag = imb::rt::stream_memops_available();
    for (auto& t : g->teams) can_flag = can_flag && t->fused() && t->push_ok();
    const bool flags = can_flag && g->sync == IMB_GROUP_SYNC_FLAGS;
    for (int s = 0; s < steps; ++s) {
      bool ready = flags;
      for (auto& t : g->teams) ready = ready && t->halos_ready();
      if (ready) {
        for (auto& t : g->teams) t->group_flag_step();
        continue;
      }
      // event-synchronised step (always the first one after init/upload)
      for (auto& t : g->teams) t->group_mark_ready();
      for (auto& t : g->teams) t->group_pull();
      for (auto& t : g->teams) t->group_compute();
      for (auto& t : g->teams) t->group_finish(can_flag);
    }
    double wall = 0.0;
    for (std::size_t q = 0; q < nt; ++q) {
      cuda_ok(cudaSetDevice(g->teams[q]->device()), "cudaSetDevice");
      cuda_ok(cudaEventRecord(t1[q], g->teams[q]->stream()), "cudaEventRecord");
      cuda_ok(cudaEventSynchronize(t1[q]), "cudaEventSynchronize");
      float ms = 0.f;
      cuda_ok(cudaEventElapsedTime(&ms, t0[q], t1[q]), "cudaEventElapsedTime");
      wall = std::max(wall, static_cast<double>(ms) * 1e-3);
      const double c = g->teams[q]->take_compute_seconds();
      if (per_team_s) per_team_s[q] = c;
    }
    cuda_ok(cudaGetLastError(), "group step");
    if (wall_s) *wall_s = wall;
  });
}

// ---- reference stage ops on padded fields -------------------------------------
int imb_fill_halo_clamped(const imb_domain* d, double* field) {
  return guard([&] {
    need(field, "field");
    imb::StencilDomain s = dom(d);
    imb::GridField g(s);
    std::copy(field, field + s.storage(), g.data());
    imb::fill_halo_clamped(g);
    std::copy(g.data(), g.data() + s.storage(), field);
  });
}

static int stage7_c(const imb_domain* d, const double* in, double* out, bool is_max) {
  return guard([&] {
    need(in, "in");
    need(out, "out");
    imb::StencilDomain s = dom(d);
    imb::GridField gi(s), go(s);
    std::copy(in, in + s.storage(), gi.data());
    std::copy(out, out + s.storage(), go.data());
    gi.halo_valid = true;
    if (is_max)
      imb::stage_max7(gi, go);
    else
      imb::stage_min7(gi, go);
    std::copy(go.data(), go.data() + s.storage(), out);
  });
}

int imb_stage_max7(const imb_domain* d, const double* in, double* out) { return stage7_c(d, in, out, true); }
int imb_stage_min7(const imb_domain* d, const double* in, double* out) { return stage7_c(d, in, out, false); }

int imb_checksum_padded(const imb_domain* d, const double* field, uint64_t* out) {
  return guard([&] {
    need(field, "field");
    need(out, "out");
    imb::StencilDomain s = dom(d);
    imb::GridField g(s);
    std::copy(field, field + s.storage(), g.data());
    *out = imb::checksum(g);
  });
}

// ---- FPM ---------------------------------------------------------------------
int imb_speed_validate(int64_t unit, int64_t g, const imb_speed_sample* s, int ns) {
  return guard([&] { (void)model(unit, g, s, ns); });
}

int imb_eval_speed(int64_t unit, int64_t g, const imb_speed_sample* s, int ns, double x, double* out) {
  return guard([&] {
    need(out, "out");
    *out = imb::eval_speed(model(unit, g, s, ns), x);
  });
}

int imb_eval_time(int64_t unit, int64_t g, const imb_speed_sample* s, int ns, double x, double* out) {
  return guard([&] {
    need(out, "out");
    *out = imb::eval_time(model(unit, g, s, ns), x);
  });
}

int imb_check_condition(int64_t unit, int64_t g, const imb_speed_sample* s, int ns, int* satisfied,
                        int64_t* viol, int cap, int* nviol, int64_t max_gain_pair[2]) {
  return guard([&] {
    need(satisfied, "satisfied");
    need(nviol, "nviol");
    need(max_gain_pair, "max_gain_pair");
    const imb::ConditionReport r = imb::check_condition(model(unit, g, s, ns));
    *satisfied = r.satisfied ? 1 : 0;
    *nviol = static_cast<int>(r.violations.size());
    for (int q = 0; q < *nviol && q < cap && viol; ++q) {
      viol[2 * q] = r.violations[static_cast<std::size_t>(q)].first;
      viol[2 * q + 1] = r.violations[static_cast<std::size_t>(q)].second;
    }
    max_gain_pair[0] = r.max_gain_pair ? r.max_gain_pair->first : -1;
    max_gain_pair[1] = r.max_gain_pair ? r.max_gain_pair->second : -1;
  });
}

int imb_classify_shape(int64_t unit, int64_t g, const imb_speed_sample* s, int ns, int* cls,
                       int64_t* peak_x) {
  return guard([&] {
    need(cls, "cls");
    need(peak_x, "peak_x");
    const imb::ShapeReport r = imb::classify_shape(model(unit, g, s, ns));
    *cls = static_cast<int>(r.classification);
    *peak_x = r.peak_x ? *r.peak_x : -1;
  });
}

int imb_average(int64_t unit, int64_t g, const imb_speed_sample* s, int nf, int ns,
                imb_speed_sample* out) {
  return guard([&] {
    need(out, "out");
    std::vector<imb::SpeedFunction> fs;
    for (int f = 0; f < nf; ++f) fs.push_back(model(unit, g, s + static_cast<std::ptrdiff_t>(f) * ns, ns));
    const imb::SpeedFunction a = imb::average(fs);
    for (int q = 0; q < ns; ++q) {
      const imb::SpeedSample& v = a.samples()[static_cast<std::size_t>(q)];
      out[q] = imb_speed_sample{v.x, v.speed, v.ci_halfwidth, v.repetitions};
    }
  });
}

int imb_scaled(int64_t unit, int64_t g, const imb_speed_sample* s, int ns, double factor,
               imb_speed_sample* out) {
  return guard([&] {
    need(out, "out");
    const imb::SpeedFunction a = imb::scaled(model(unit, g, s, ns), factor);
    for (int q = 0; q < ns; ++q) {
      const imb::SpeedSample& v = a.samples()[static_cast<std::size_t>(q)];
      out[q] = imb_speed_sample{v.x, v.speed, v.ci_halfwidth, v.repetitions};
    }
  });
}

int imb_speed_csv_parse(const char* text, size_t len, int64_t* unit_cells, int64_t* granularity,
                        imb_speed_sample* out, int cap, int* ns, char* label, size_t label_cap,
                        int* err_line) {
  if (err_line) *err_line = 0;
  try {
    need(text, "text");
    need(ns, "ns");
    std::istringstream is(std::string(text, len));
    const imb::SpeedFunction f = imb::read_speed_function_csv(is);
    const auto& sm = f.samples();
    *ns = static_cast<int>(sm.size());
    if (cap > 0) need(out, "out");
    for (int q = 0; q < cap && q < *ns; ++q)
      out[q] = imb_speed_sample{sm[q].x, sm[q].speed, sm[q].ci_halfwidth, sm[q].repetitions};
    if (unit_cells) *unit_cells = f.unit_cells();
    if (granularity) *granularity = f.granularity();
    if (label && label_cap > 0) {
      const std::size_t n = std::min(label_cap - 1, f.label().size());
      std::memcpy(label, f.label().data(), n);
      label[n] = '\0';
    }
    return IMB_OK;
  } catch (const imb::ParseError& e) {
    if (err_line) *err_line = e.line;
    return guard([&] { throw; });
  } catch (...) {
    return guard([&] { throw; });
  }
}

int imb_speed_csv_format(int64_t unit_cells, int64_t granularity, const imb_speed_sample* s,
                         int ns, const char* label, char* out, size_t cap, size_t* len) {
  return guard([&] {
    need(len, "len");
    std::vector<imb::SpeedSample> v;
    if (ns > 0) need(s, "samples");
    for (int q = 0; q < ns; ++q) v.push_back({s[q].x, s[q].speed, s[q].ci_halfwidth, s[q].repetitions});
    const imb::SpeedFunction f(unit_cells, granularity, std::move(v), label ? label : "");
    std::ostringstream os;
    imb::write_speed_function_csv(os, f);
    const std::string t = os.str();
    *len = t.size();
    if (cap < t.size() + 1) throw imb::RangeError("output buffer too small for the CSV text");
    need(out, "out");
    std::memcpy(out, t.data(), t.size());
    out[t.size()] = '\0';
  });
}

int imb_slice_surface(int64_t unit, int64_t g, const int64_t* n_values, int nn,
                      const int64_t* m_values, int nm, const imb_speed_sample* samples,
                      int64_t fixed_n, imb_speed_sample* out, int64_t* out_unit_cells) {
  return guard([&] {
    need(out, "out");
    need(out_unit_cells, "out_unit_cells");
    if (nn < 0 || nm < 0) throw imb::ContractError("surface extents must be >= 0");
    if (nn > 0) need(n_values, "n_values");
    if (nm > 0) need(m_values, "m_values");
    if (nn * nm > 0) need(samples, "samples");
    imb::SpeedSurface srf;
    srf.unit_cells = unit;
    srf.granularity = g;
    srf.label = "c-abi";
    srf.n_values.assign(n_values, n_values + nn);
    srf.m_values.assign(m_values, m_values + nm);
    for (int q = 0; q < nn * nm; ++q)
      srf.samples.push_back({samples[q].x, samples[q].speed, samples[q].ci_halfwidth,
                             samples[q].repetitions});
    const imb::SpeedFunction f = imb::slice_surface(srf, fixed_n);
    for (std::size_t q = 0; q < f.samples().size(); ++q) {
      const imb::SpeedSample& v = f.samples()[q];
      out[q] = imb_speed_sample{v.x, v.speed, v.ci_halfwidth, v.repetitions};
    }
    *out_unit_cells = f.unit_cells();
  });
}

// ---- partitioner -------------------------------------------------------------
int imb_predict_makespan(int64_t unit, int64_t g, const imb_speed_sample* s, int ns,
                         const int64_t* shares, int p, double* per_time, double* makespan) {
  return guard([&] {
    if (p > 0) need(shares, "shares");
    const imb::Partition r = imb::predict_makespan(
        model(unit, g, s, ns), std::span<const std::int64_t>(shares, static_cast<std::size_t>(std::max(p, 0))));
    put(r, nullptr, per_time, makespan, nullptr);
  });
}

static int partition_c(int kind, int64_t unit, int64_t g, const imb_speed_sample* s, int ns,
                       int64_t total, int p, int allow_idle, int64_t cap, int64_t* shares,
                       double* per_time, double* makespan, int64_t* offset) {
  return guard([&] {
    imb::PartitionProblem pr{total, p, model(unit, g, s, ns), allow_idle != 0};
    const imb::Partition r = kind == 0   ? imb::partition_paired(pr)
                             : kind == 1 ? imb::partition_general(pr)
                                         : imb::brute_force_oracle(pr, cap);
    put(r, shares, per_time, makespan, offset);
  });
}

int imb_partition_paired(int64_t unit, int64_t g, const imb_speed_sample* s, int ns, int64_t total,
                         int p, int allow_idle, int64_t* shares, double* per_time, double* makespan,
                         int64_t* offset) {
  return partition_c(0, unit, g, s, ns, total, p, allow_idle, 0, shares, per_time, makespan, offset);
}

int imb_partition_general(int64_t unit, int64_t g, const imb_speed_sample* s, int ns, int64_t total,
                          int p, int allow_idle, int64_t* shares, double* per_time, double* makespan,
                          int64_t* offset) {
  return partition_c(1, unit, g, s, ns, total, p, allow_idle, 0, shares, per_time, makespan, offset);
}

int imb_brute_force_oracle(int64_t unit, int64_t g, const imb_speed_sample* s, int ns,
                           int64_t total, int p, int allow_idle, int64_t cap, int64_t* shares,
                           double* per_time, double* makespan, int64_t* offset) {
  return partition_c(2, unit, g, s, ns, total, p, allow_idle, cap, shares, per_time, makespan, offset);
}

int imb_improvement_search(int64_t unit, int64_t g, const imb_speed_sample* s, int ns,
                           int64_t balanced, int* found, int64_t* delta, double* gain,
                           int64_t pair[2]) {
  return guard([&] {
    need(found, "found");
    const auto r = imb::improvement_search(model(unit, g, s, ns), balanced);
    *found = r ? 1 : 0;
    if (delta) *delta = r ? r->delta : 0;
    if (gain) *gain = r ? r->gain_s : 0.0;
    if (pair) {
      pair[0] = r ? r->violating_pair.first : -1;
      pair[1] = r ? r->violating_pair.second : -1;
    }
  });
}

// ---- stats -------------------------------------------------------------------
double imb_t_quantile_975(int df) {
  double v = -1.0;
  if (guard([&] { v = imb::t_quantile_975(df); }) != IMB_OK) return -1.0;
  return v;
}

int imb_summarize(const double* xs, int n, double* mean, double* stddev, double* ci) {
  return guard([&] {
    if (n > 0) need(xs, "xs");
    const imb::Summary r =
        imb::summarize(std::span<const double>(xs, static_cast<std::size_t>(std::max(n, 0))));
    if (mean) *mean = r.mean;
    if (stddev) *stddev = r.stddev;
    if (ci) *ci = r.ci_halfwidth;
  });
}

}  // extern "C"
