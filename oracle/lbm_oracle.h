/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker of the parity suite.
 *
 * lbm_oracle: a plain-C, single-threaded, FP64 restatement of the reference
 * hot path (/root/reference/proj/src: lattice, collision, solver, boundary,
 * ib, runner step order) for ONE region.  Operation order follows the
 * reference expression by expression and the file is compiled with
 * -ffp-contract=off, so its fields are bit-identical to the compiled
 * reference (pinned by tests/test_oracle.py against oracle/_ref and against
 * the committed golden vectors in tests/golden/).
 *
 * Never linked into the product; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.
 */
#ifndef LBM_ORACLE_H
#define LBM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/lbmg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_state orc_state;

/* Lattice / model tables (lattice.cpp:8-46, collision.cpp:18-47). */
void orc_lattice(int* c /*27*3*/, double* w, int* opposite, int* row_exponents /*27*3*/);
int orc_make_rates(const lbmg_scene_config* cfg, double* rates);
void orc_equilibrium(double rho, const double* u, double* feq);
/* collide (collision.cpp:176-212) on n nodes. */
int orc_collide_batch(const lbmg_scene_config* cfg, size_t n, const double* f, const double* rho,
                      const double* u, double* omega);

/* Integer helpers: morton3 (ib.cpp:13-25), reorder permutation
 * (ib.cpp:231-292), split_domain (decomp.cpp:5-18), face ownership
 * (boundary.cpp:28-40) as an owner table n_nodes*27 (255 = streams). */
uint64_t orc_morton3(uint32_t x, uint32_t y, uint32_t z);
int orc_reorder_permutation(size_t n, const double* pos, const uint32_t* src, int ell, uint32_t* perm);
int orc_split_domain(int nz, int m, int* z0z1);
void orc_face_owner(const lbmg_scene_config* cfg, uint8_t* out);
/* kernel_support (ib.cpp:294-308): returns inside; base[3]; w[6]. */
int orc_kernel_support(const double* pos, int nx, int ny, int nz, int* base, double* w);

/* Single-region Runner (runner.cpp:22-230 with m = 1).  Solids are given as
 * sample sets in storage order (positions, reference positions, source ids);
 * motion comes from cfg->solids[s]. */
orc_state* orc_create(const lbmg_scene_config* cfg, const size_t* counts, const double* const* pos,
                      const double* const* ref, const uint32_t* const* src);
void orc_destroy(orc_state* s);
int orc_advance(orc_state* s, long steps, lbmg_status* st);
long orc_step_count(const orc_state* s);
/* what: 0 rho, 1 u, 2 f (canonical AoS FP64). */
void orc_gather(const orc_state* s, int what, double* out);
size_t orc_totals_count(const orc_state* s);
void orc_totals(const orc_state* s, double* out);
void orc_samples(const orc_state* s, int solid, double* pos, double* ub, double* force, double* sampled,
                 uint8_t* flagged);
/* Raw state access for phase-level tests: f / f_star (AoS, n*27). */
double* orc_f(orc_state* s);
double* orc_f_star(orc_state* s);

#ifdef __cplusplus
}
#endif
#endif
