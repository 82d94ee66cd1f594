/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the MPDATA step.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this code, and only as the checker or the
 * timed CPU baseline. The product (paper_1507_01265_b200/) never links it.
 *
 * PARITY UNPINNED BY THE REFERENCE: the reference declares the MPDATA step
 * API (/root/reference/proj/include/imbalance/workload.hpp:14-133) but ships
 * no implementation, no golden checksum and no fixture.
 * This file restates the published MPDATA scheme (Smolarkiewicz 1984;
 * Smolarkiewicz & Grabowski 1990) as plain scalar C,
 * compiled with -ffp-contract=off. It is pinned instead by analytic
 * properties (tests/test_oracle_props.py) and by golden checksums it
 * generated itself (tests/golden/, with the generating script committed).
 *
 * Layout: a global n x m x l grid, i outermost, k contiguous, matching the
 * interior order of GridField::index (workload.hpp:40-43). All axes periodic.
 */
#ifndef IMB_MPDATA_ORACLE_H
#define IMB_MPDATA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_RECIPE_UNIFORM = 0, ORC_RECIPE_GAUSS = 1, ORC_RECIPE_ROTCUBE = 2 };

/* Seeded fields of the global n x m x l grid for the i-planes [i0, i0+ni)
 * (global i taken modulo n, so halo planes wrap). Each value is a pure
 * function of (seed, field, i, j, k) — workload.hpp:61-63. */
int orc_init_f64(int recipe, int64_t n, int64_t m, int64_t l, uint64_t seed, int64_t i0,
                 int64_t ni, double* x, double* u, double* v, double* w, double* h);
int orc_init_f32(int recipe, int64_t n, int64_t m, int64_t l, uint64_t seed, int64_t i0,
                 int64_t ni, float* x, float* u, float* v, float* w, float* h);

/* `steps` MPDATA steps in place on x (periodic global grid), IORD passes,
 * optional nonoscillatory limiter, `threads` workers over contiguous
 * j-slabs (the TeamRunner m-slab split, workload.hpp:91-93). */
int orc_run_f64(int iord, int nonos, int64_t n, int64_t m, int64_t l, double* x,
                const double* u, const double* v, const double* w, const double* h, int steps,
                int threads);
int orc_run_f32(int iord, int nonos, int64_t n, int64_t m, int64_t l, float* x, const float* u,
                const float* v, const float* w, const float* h, int steps, int threads);

/* FNV-1a 64 over the little-endian bytes of each value, in storage order
 * (workload.hpp:82-83; byte granularity pinned in SURVEY.md App. C #6). */
uint64_t orc_checksum_f64(const double* x, size_t count);
uint64_t orc_checksum_f32(const float* x, size_t count);

/* Reference surrogate stage ops on the padded GridField layout
 * ((n+2h)(m+2h)(l+2h), workload.hpp:40-43): fill_halo_clamped
 * (workload.hpp:66-67) and stage_max7 / stage_min7 (workload.hpp:69-74). */
void orc_fill_halo_clamped(double* f, int64_t n, int64_t m, int64_t l, int64_t halo);
void orc_stage_max7(const double* in, double* out, int64_t n, int64_t m, int64_t l, int64_t halo);
void orc_stage_min7(const double* in, double* out, int64_t n, int64_t m, int64_t l, int64_t halo);

double orc_eps(void);

#ifdef __cplusplus
}
#endif
#endif
