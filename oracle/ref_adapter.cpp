// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI adapter over the UNMODIFIED reference library (/root/reference/proj),
// compiled with -Dlbm=lbm_ref so its symbols cannot collide with the product.
// Built by oracle/Makefile into oracle/_ref/libref_adapter.so.  Used by
// tests/ (parity checker) and bench.py --impl reference / cpu_baseline.
//
// Scene input uses the product's lbmg_scene_config struct (include/lbmg.h)
// so both sides are driven from the same POD description.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <algorithm>

#include "lbm/autotune.hpp"
#include "lbm/io.hpp"
#include "lbm/boundary.hpp"
#include "lbm/collision.hpp"
#include "lbm/decomp.hpp"
#include "lbm/ib.hpp"
#include "lbm/runner.hpp"
#include "lbm/scene.hpp"
#include "lbm/solver.hpp"
#include "lbm/tracer.hpp"
#include "lbmg.h"
#include "oracles.hpp"

using namespace lbm;  // == lbm_ref via -Dlbm=lbm_ref

namespace {

thread_local std::string g_err;

Vec3 v3(const double* p) { return {p[0], p[1], p[2]}; }

SceneConfig to_cfg(const lbmg_scene_config* c) {
    SceneConfig cfg;
    cfg.dims = {c->nx, c->ny, c->nz};
    cfg.viscosity = c->viscosity;
    cfg.kind = static_cast<CollisionKind>(c->kind);
    cfg.high_order_rate = c->high_order_rate;
    cfg.policy = static_cast<RatePolicy>(c->policy);
    cfg.policy_eps0 = c->policy_eps0;
    if (c->has_explicit_rates) {
        std::array<double, 27> r;
        for (int i = 0; i < 27; ++i) r[i] = c->rates[i];
        cfg.explicit_rates = r;
    }
    for (int f = 0; f < 6; ++f) {
        cfg.boundary.faces[f].condition = static_cast<FaceCondition>(c->faces[f].condition);
        cfg.boundary.faces[f].inlet_velocity = v3(c->faces[f].velocity);
    }
    cfg.body_force = v3(c->body_force);
    for (int s = 0; s < c->n_solids; ++s) {
        const lbmg_solid_config& sc = c->solids[s];
        SolidConfig o;
        o.mesh.type = static_cast<MeshConfig::Type>(sc.mesh.type);
        o.mesh.center = v3(sc.mesh.center);
        o.mesh.lo = v3(sc.mesh.lo);
        o.mesh.hi = v3(sc.mesh.hi);
        o.mesh.origin = v3(sc.mesh.origin);
        o.mesh.radius = sc.mesh.radius;
        o.mesh.subdivisions = sc.mesh.subdivisions;
        o.mesh.fins = sc.mesh.fins;
        o.mesh.fin_length = sc.mesh.fin_length;
        o.mesh.fin_height = sc.mesh.fin_height;
        o.mesh.fin_spacing = sc.mesh.fin_spacing;
        o.mesh.size = sc.mesh.size;
        o.mesh.plane_z = sc.mesh.plane_z;
        o.poisson_radius = sc.poisson_radius;
        o.sampling = static_cast<SamplingMethod>(sc.sampling);
        if (sc.has_motion) {
            RigidMotion m;
            m.linear_velocity = v3(sc.linear_velocity);
            m.angular_velocity = v3(sc.angular_velocity);
            m.center = v3(sc.center);
            o.motion = m;
        }
        cfg.solids.push_back(o);
    }
    cfg.init = static_cast<InitKind>(c->init);
    cfg.init_density = c->init_density;
    cfg.init_velocity = v3(c->init_velocity);
    cfg.tg_u_max = c->tg_u_max;
    cfg.regions = c->regions;
    cfg.threads_per_region = c->threads_per_region;
    cfg.alpha = c->alpha;
    cfg.block_edge = c->block_edge;
    cfg.ib_mode = static_cast<AccumulationMode>(c->ib_mode);
    cfg.seed = c->seed;
    return cfg;
}

void put_status(const StepStatus& s, lbmg_status* o) {
    if (!o) return;
    o->ok = s.ok ? 1 : 0;
    o->mach_warning = s.mach_warning ? 1 : 0;
    o->step = s.step;
    std::snprintf(o->reason, sizeof o->reason, "%s", s.reason.c_str());
}

struct RefRunner {
    Scene scene;
    std::unique_ptr<Runner> runner;
};

template <class Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return LBMG_ERR_CONFIG;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LBMG_ERR_STATE;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Scene + Runner(scene, regions, threads) in one call.
int ref_runner_create(const lbmg_scene_config* c, int regions, unsigned threads, void** out) {
    return guard([&] {
        auto rr = new RefRunner;
        rr->scene = build_scene(to_cfg(c));
        rr->runner = std::make_unique<Runner>(rr->scene, regions, threads);
        *out = rr;
    });
}

// Same but the caller provides the sample sets (positions/ref/source, stored
// order) instead of the reference's own sampling.
int ref_runner_create_with_samples(const lbmg_scene_config* c, int regions, unsigned threads,
                                   const size_t* counts, const double* const* positions,
                                   const double* const* refs, const uint32_t* const* sources,
                                   void** out) {
    return guard([&] {
        auto rr = new RefRunner;
        SceneConfig cfg = to_cfg(c);
        rr->scene = build_scene(cfg);
        for (std::size_t s = 0; s < rr->scene.solids.size(); ++s) {
            SolidSampleSet& set = rr->scene.solids[s].samples;
            const std::size_t n = counts[s];
            set.positions.resize(n);
            set.reference_positions.resize(n);
            set.boundary_velocity.assign(n, Vec3{});
            set.penalty_force.assign(n, Vec3{});
            set.sampled_velocity.assign(n, Vec3{});
            set.flagged.assign(n, 0);
            set.source_id.resize(n);
            for (std::size_t k = 0; k < n; ++k) {
                set.positions[k] = v3(positions[s] + 3 * k);
                set.reference_positions[k] = v3(refs[s] + 3 * k);
                set.source_id[k] = sources[s][k];
            }
        }
        rr->runner = std::make_unique<Runner>(rr->scene, regions, threads);
        *out = rr;
    });
}

void ref_runner_destroy(void* h) { delete static_cast<RefRunner*>(h); }

// Scene with tracer emitters (SceneConfig::emitters) + Runner.
int ref_runner_create_tracers(const lbmg_scene_config* c, int regions, unsigned threads, int n_emitters,
                              const lbmg_emitter* em, void** out) {
    return guard([&] {
        SceneConfig cfg = to_cfg(c);
        for (int k = 0; k < n_emitters; ++k) {
            TracerEmitter e;
            e.lo = v3(em[k].lo);
            e.hi = v3(em[k].hi);
            e.rate = em[k].rate;
            cfg.emitters.push_back(e);
        }
        auto rr = new RefRunner;
        rr->scene = build_scene(cfg);
        rr->runner = std::make_unique<Runner>(rr->scene, regions, threads);
        *out = rr;
    });
}

size_t ref_runner_tracer_count(void* h) { return static_cast<RefRunner*>(h)->runner->tracers().size(); }

void ref_runner_tracers(void* h, double* pos, int64_t* birth) {
    const TracerCloud& c = static_cast<RefRunner*>(h)->runner->tracers();
    for (std::size_t k = 0; k < c.size(); ++k) {
        pos[3 * k] = c.positions[k].x;
        pos[3 * k + 1] = c.positions[k].y;
        pos[3 * k + 2] = c.positions[k].z;
        birth[k] = c.birth_step[k];
    }
}

// emit_tracers of one step into an empty cloud: E positions (AoS).
size_t ref_emit_tracers(int n_emitters, const lbmg_emitter* em, long step, uint64_t seed, double* pos) {
    std::vector<TracerEmitter> es;
    for (int k = 0; k < n_emitters; ++k) {
        TracerEmitter e;
        e.lo = v3(em[k].lo);
        e.hi = v3(em[k].hi);
        e.rate = em[k].rate;
        es.push_back(e);
    }
    TracerCloud c;
    emit_tracers(c, es, step, seed);
    for (std::size_t k = 0; k < c.size(); ++k) {
        pos[3 * k] = c.positions[k].x;
        pos[3 * k + 1] = c.positions[k].y;
        pos[3 * k + 2] = c.positions[k].z;
    }
    return c.size();
}

void ref_rasterize_density(size_t n, const double* pos, int nx, int ny, int nz, double* vol) {
    TracerCloud c;
    for (size_t k = 0; k < n; ++k) {
        c.positions.push_back(v3(pos + 3 * k));
        c.birth_step.push_back(0);
    }
    const std::vector<double> v = rasterize_density(c, GridDims{nx, ny, nz});
    std::copy(v.begin(), v.end(), vol);
}

int ref_runner_advance(void* h, long steps, lbmg_status* st) {
    return guard([&] {
        auto* rr = static_cast<RefRunner*>(h);
        put_status(rr->runner->advance(steps), st);
    });
}

// advance with per-phase timing rows: phases[k] (24 chars), seconds[k].
int ref_runner_advance_timed(void* h, long steps, lbmg_status* st, lbmg_timing_row* rows,
                             size_t cap, size_t* n) {
    return guard([&] {
        auto* rr = static_cast<RefRunner*>(h);
        std::vector<TimingRow> t;
        put_status(rr->runner->advance(steps, &t), st);
        std::size_t k = 0;
        for (; k < t.size() && k < cap; ++k) {
            std::snprintf(rows[k].phase, sizeof rows[k].phase, "%s", t[k].phase.c_str());
            rows[k].step = t[k].step;
            rows[k].seconds = t[k].seconds;
        }
        *n = k;
    });
}

long ref_runner_step_count(void* h) { return static_cast<RefRunner*>(h)->runner->step_count(); }

int ref_runner_set_layout(void* h, int ell, size_t alpha) {
    return guard([&] { static_cast<RefRunner*>(h)->runner->set_layout(ell, alpha); });
}

static void copy_store(const FieldStore& fs, double* out) {
    for (std::size_t k = 0; k < fs.n_nodes(); ++k)
        for (std::size_t i = 0; i < fs.beta(); ++i) out[k * fs.beta() + i] = fs.get(k, i);
}

void ref_runner_gather_rho(void* h, double* out) {
    copy_store(static_cast<RefRunner*>(h)->runner->gather_rho(), out);
}
void ref_runner_gather_u(void* h, double* out) {
    copy_store(static_cast<RefRunner*>(h)->runner->gather_u(), out);
}
void ref_runner_gather_f(void* h, double* out) {
    copy_store(static_cast<RefRunner*>(h)->runner->gather_f(), out);
}

size_t ref_runner_totals_count(void* h) {
    return static_cast<RefRunner*>(h)->runner->totals_log().size();
}
void ref_runner_totals(void* h, double* out) {
    const auto& log = static_cast<RefRunner*>(h)->runner->totals_log();
    for (std::size_t s = 0; s < log.size(); ++s) {
        for (int a = 0; a < 3; ++a) out[6 * s + a] = log[s].force[a];
        for (int a = 0; a < 3; ++a) out[6 * s + 3 + a] = log[s].torque[a];
    }
}

int ref_runner_solid_count(void* h) {
    return static_cast<int>(static_cast<RefRunner*>(h)->scene.solids.size());
}

size_t ref_runner_sample_count(void* h, int region, int solid) {
    return static_cast<RefRunner*>(h)->runner->region_solids()[region][solid].size();
}

// Any pointer may be NULL.
void ref_runner_samples(void* h, int region, int solid, double* pos, double* ub, double* force,
                        double* sampled, double* refpos, uint32_t* src, uint8_t* flagged) {
    const SolidSampleSet& s = static_cast<RefRunner*>(h)->runner->region_solids()[region][solid];
    for (std::size_t k = 0; k < s.size(); ++k) {
        for (int a = 0; a < 3; ++a) {
            if (pos) pos[3 * k + a] = s.positions[k][a];
            if (ub) ub[3 * k + a] = s.boundary_velocity[k][a];
            if (force) force[3 * k + a] = s.penalty_force[k][a];
            if (sampled) sampled[3 * k + a] = s.sampled_velocity[k][a];
            if (refpos) refpos[3 * k + a] = s.reference_positions[k][a];
        }
        if (src) src[k] = s.source_id[k];
        if (flagged) flagged[k] = s.flagged[k];
    }
}

// Scene-level sample set (build_scene output) + sampling report.
size_t ref_scene_sample_count(void* h, int solid) {
    return static_cast<RefRunner*>(h)->scene.solids[solid].samples.size();
}
void ref_scene_samples(void* h, int solid, double* pos, double* refpos, uint32_t* src,
                       double* bbox6, int* ell, double* report6) {
    const SolidInstance& si = static_cast<RefRunner*>(h)->scene.solids[solid];
    const SolidSampleSet& s = si.samples;
    for (std::size_t k = 0; k < s.size(); ++k) {
        for (int a = 0; a < 3; ++a) {
            if (pos) pos[3 * k + a] = s.positions[k][a];
            if (refpos) refpos[3 * k + a] = s.reference_positions[k][a];
        }
        if (src) src[k] = s.source_id[k];
    }
    if (bbox6)
        for (int a = 0; a < 3; ++a) {
            bbox6[a] = s.bbox_lo[a];
            bbox6[3 + a] = s.bbox_hi[a];
        }
    if (ell) *ell = s.block_edge;
    if (report6) {
        report6[0] = static_cast<double>(si.report.n_samples);
        report6[1] = static_cast<double>(si.report.occupied_cells);
        report6[2] = si.report.density_min;
        report6[3] = si.report.density_mean;
        report6[4] = si.report.density_max;
        report6[5] = static_cast<double>(si.report.attempts);
    }
}

// ---- kernel-level reference functions ------------------------------------

int ref_make_rates(const lbmg_scene_config* c, double* rates) {
    return guard([&] {
        CollisionModel m = to_cfg(c).make_model();
        for (int r = 0; r < 27; ++r) rates[r] = m.rates[r];
    });
}

// collide() over n nodes (collision.cpp:207-212).
int ref_collide_batch(const lbmg_scene_config* c, size_t n, const double* f, const double* rho,
                      const double* u, double* omega) {
    return guard([&] {
        CollisionModel m = to_cfg(c).make_model();
        for (std::size_t k = 0; k < n; ++k) {
            std::array<double, 27> fk;
            for (int i = 0; i < 27; ++i) fk[i] = f[27 * k + i];
            auto o = collide(fk, rho[k], {u[3 * k], u[3 * k + 1], u[3 * k + 2]}, m);
            for (int i = 0; i < 27; ++i) omega[27 * k + i] = o[i];
        }
    });
}

// Dense M^-1 D M oracle (tests/oracles.hpp:74-94).
int ref_dense_collide_batch(const lbmg_scene_config* c, size_t n, const double* f,
                            const double* rho, const double* u, double* omega) {
    return guard([&] {
        CollisionModel m = to_cfg(c).make_model();
        for (std::size_t k = 0; k < n; ++k) {
            std::array<double, 27> fk;
            for (int i = 0; i < 27; ++i) fk[i] = f[27 * k + i];
            auto o = oracle::dense_collide(fk, rho[k], {u[3 * k], u[3 * k + 1], u[3 * k + 2]}, m);
            for (int i = 0; i < 27; ++i) omega[27 * k + i] = o[i];
        }
    });
}

void ref_equilibrium(double rho, const double* u, double* feq) {
    auto e = equilibrium(rho, v3(u));
    for (int i = 0; i < 27; ++i) feq[i] = e[i];
}

void ref_lattice(int* c, double* w, int* opposite) {
    const auto& lat = LatticeD3Q27::instance();
    for (int i = 0; i < 27; ++i) {
        for (int a = 0; a < 3; ++a) c[3 * i + a] = lat.c[i][a];
        w[i] = lat.w[i];
        opposite[i] = lat.opposite[i];
    }
}

void ref_moment_exponents(int* q, int* degree) {
    const auto& e = moment_exponents();
    for (int r = 0; r < 27; ++r) {
        for (int a = 0; a < 3; ++a) q[3 * r + a] = e[r][a];
        degree[r] = moment_degree(r);
    }
}

uint64_t ref_morton3(uint32_t x, uint32_t y, uint32_t z) { return morton3(x, y, z); }

int ref_split_domain(int nz, int m, int* z0z1) {
    return guard([&] {
        auto s = split_domain({1, 1, nz}, m);
        for (int r = 0; r < m; ++r) {
            z0z1[2 * r] = s[r].z0;
            z0z1[2 * r + 1] = s[r].z1;
        }
    });
}

// Owner face per (node, direction) via face_owns_direction (boundary.cpp:28-40):
// out[k*27+i] = face or 255.
void ref_face_owner(const lbmg_scene_config* c, uint8_t* out) {
    SceneConfig cfg = to_cfg(c);
    const GridDims g = cfg.dims;
    for (int z = 0; z < g.nz; ++z)
        for (int y = 0; y < g.ny; ++y)
            for (int x = 0; x < g.nx; ++x) {
                std::size_t k = node_index(x, y, z, g);
                for (int i = 0; i < 27; ++i) {
                    uint8_t owner = 255;
                    for (int f = 0; f < 6; ++f)
                        if (face_owns_direction(g, cfg.boundary, x, y, z, i, f)) {
                            owner = static_cast<uint8_t>(f);
                            break;
                        }
                    out[k * 27 + i] = owner;
                }
            }
}

// reorder_samples (ib.cpp:231-292): perm[new] = old index.
int ref_reorder_permutation(size_t n, const double* positions, const uint32_t* source_id, int ell,
                            uint32_t* perm) {
    return guard([&] {
        SolidSampleSet set;
        set.positions.resize(n);
        set.boundary_velocity.assign(n, Vec3{});
        set.penalty_force.assign(n, Vec3{});
        set.sampled_velocity.assign(n, Vec3{});
        set.reference_positions.resize(n);
        set.flagged.assign(n, 0);
        set.source_id.resize(n);
        for (std::size_t k = 0; k < n; ++k) {
            set.positions[k] = v3(positions + 3 * k);
            // tag the original index in the reference position
            set.reference_positions[k] = {static_cast<double>(k), 0, 0};
            set.source_id[k] = source_id[k];
        }
        SolidSampleSet out = reorder_samples(set, ell);
        for (std::size_t k = 0; k < n; ++k)
            perm[k] = static_cast<uint32_t>(out.reference_positions[k].x);
    });
}

// kernel_support (ib.cpp:294-308): base[3], w[6] (wx0,wx1,wy0,wy1,wz0,wz1), inside.
int ref_kernel_support(const double* pos, int nx, int ny, int nz, int* base, double* w) {
    KernelSupport ks = kernel_support(v3(pos), {nx, ny, nz});
    for (int a = 0; a < 3; ++a) base[a] = ks.base[a];
    w[0] = ks.wx[0];
    w[1] = ks.wx[1];
    w[2] = ks.wy[0];
    w[3] = ks.wy[1];
    w[4] = ks.wz[0];
    w[5] = ks.wz[1];
    return ks.inside ? 1 : 0;
}

// Single-region phase-level step with an explicit f/f_star state (for the
// stale-outflow semantic tests): AoS FP64 arrays over dims.
int ref_stream_and_faces(const lbmg_scene_config* c, const double* f_prev, double* f_star) {
    return guard([&] {
        SceneConfig cfg = to_cfg(c);
        const GridDims g = cfg.dims;
        const std::size_t n = g.n_nodes();
        FieldStore fp(LayoutParams::make(1, 27, n)), fs(LayoutParams::make(1, 27, n));
        std::memcpy(fp.data(), f_prev, n * 27 * sizeof(double));
        std::memcpy(fs.data(), f_star, n * 27 * sizeof(double));
        DomainContext ctx = DomainContext::single(g, cfg.boundary.axis_periodic(0),
                                                  cfg.boundary.axis_periodic(1),
                                                  cfg.boundary.axis_periodic(2));
        ThreadPool pool(1);
        stream(fp, fs, ctx, pool);
        apply_domain_boundaries(fs, fp, cfg.boundary, ctx, pool);
        std::memcpy(f_star, fs.data(), n * 27 * sizeof(double));
    });
}

// step(SimState&, ...) (solver.hpp:82-83, solver.cpp:181-191) on an explicit
// single-region state without solids: f, f_star (AoS FP64, nodes*27) in,
// `steps` steps, then f(t+steps), rho*, u* of the last step out.
int ref_step(const lbmg_scene_config* c, const double* f, const double* f_star, long t, long steps,
             double* f_out, double* rho_out, double* u_out, lbmg_status* st) {
    return guard([&] {
        SceneConfig cfg = to_cfg(c);
        const GridDims g = cfg.dims;
        const std::size_t n = g.n_nodes();
        SimState s = SimState::make(g, 1);
        std::memcpy(s.f.data(), f, n * 27 * sizeof(double));
        std::memcpy(s.f_star.data(), f_star, n * 27 * sizeof(double));
        s.t = t;
        DomainContext ctx = DomainContext::single(g, cfg.boundary.axis_periodic(0), cfg.boundary.axis_periodic(1),
                                                  cfg.boundary.axis_periodic(2));
        const CollisionModel model = cfg.make_model();
        ThreadPool pool(1);
        StepStatus status;
        for (long k = 0; k < steps; ++k) {
            status = step(s, model, cfg.boundary, cfg.body_force, ctx, pool);
            if (!status.ok) break;
        }
        std::memcpy(f_out, s.f.data(), n * 27 * sizeof(double));
        std::memcpy(rho_out, s.rho.data(), n * sizeof(double));
        std::memcpy(u_out, s.u.data(), n * 3 * sizeof(double));
        put_status(status, st);
    });
}

namespace {
SolidSampleSet make_set(size_t n, const double* pos, const double* ub, const double* sampled, const double* force,
                        const uint8_t* flagged) {
    SolidSampleSet set;
    set.positions.resize(n);
    set.reference_positions.assign(n, Vec3{});
    set.boundary_velocity.assign(n, Vec3{});
    set.sampled_velocity.assign(n, Vec3{});
    set.penalty_force.assign(n, Vec3{});
    set.flagged.assign(n, 0);
    set.source_id.assign(n, 0);
    for (std::size_t k = 0; k < n; ++k) {
        set.positions[k] = v3(pos + 3 * k);
        if (ub) set.boundary_velocity[k] = v3(ub + 3 * k);
        if (sampled) set.sampled_velocity[k] = v3(sampled + 3 * k);
        if (force) set.penalty_force[k] = v3(force + 3 * k);
        if (flagged) set.flagged[k] = flagged[k];
    }
    return set;
}
FieldStore field(const double* v, std::size_t nodes, int beta) {
    FieldStore fs(LayoutParams::make(1, beta, nodes));
    std::memcpy(fs.data(), v, nodes * beta * sizeof(double));
    return fs;
}
}  // namespace

// The IB free functions (ib.hpp:96-128) on a single-region context; fields are
// canonical AoS FP64 over the grid, sample arrays AoS Vec3.
int ref_ib_interpolate_velocity(size_t n, const double* pos, const double* u, int nx, int ny, int nz,
                                double* sampled, uint8_t* flagged) {
    return guard([&] {
        GridDims d{nx, ny, nz};
        SolidSampleSet set = make_set(n, pos, nullptr, nullptr, nullptr, nullptr);
        FieldStore fu = field(u, d.n_nodes(), 3);
        DomainContext ctx = DomainContext::single(d, false, false, false);
        ThreadPool pool(1);
        interpolate_velocity(set, fu, ctx, pool);
        for (std::size_t k = 0; k < n; ++k) {
            for (int a = 0; a < 3; ++a) sampled[3 * k + a] = set.sampled_velocity[k][a];
            flagged[k] = set.flagged[k];
        }
    });
}

int ref_ib_penalty_forces(size_t n, const double* pos, const double* ub, const double* sampled,
                          const uint8_t* flagged, const double* rho, int nx, int ny, int nz, double* force) {
    return guard([&] {
        GridDims d{nx, ny, nz};
        SolidSampleSet set = make_set(n, pos, ub, sampled, nullptr, flagged);
        FieldStore fr = field(rho, d.n_nodes(), 1);
        DomainContext ctx = DomainContext::single(d, false, false, false);
        ThreadPool pool(1);
        penalty_forces(set, fr, ctx, pool);
        for (std::size_t k = 0; k < n; ++k)
            for (int a = 0; a < 3; ++a) force[3 * k + a] = set.penalty_force[k][a];
    });
}

int ref_ib_spread_forces(size_t n, const double* pos, const double* force, const uint8_t* flagged, int nx,
                         int ny, int nz, int deterministic, double* g) {
    return guard([&] {
        GridDims d{nx, ny, nz};
        SolidSampleSet set = make_set(n, pos, nullptr, nullptr, force, flagged);
        FieldStore fg = field(g, d.n_nodes(), 3);
        DomainContext ctx = DomainContext::single(d, false, false, false);
        ThreadPool pool(1);
        spread_forces(set, fg, ctx, deterministic ? AccumulationMode::Deterministic : AccumulationMode::Atomic, pool);
        std::memcpy(g, fg.data(), d.n_nodes() * 3 * sizeof(double));
    });
}

int ref_ib_update_rigid_motion(size_t n, const double* ref, const double* v, const double* w, const double* c,
                               long t, int nx, int ny, int nz, double* pos, double* ub, uint8_t* flagged) {
    return guard([&] {
        SolidSampleSet set = make_set(n, ref, nullptr, nullptr, nullptr, nullptr);
        for (std::size_t k = 0; k < n; ++k) set.reference_positions[k] = v3(ref + 3 * k);
        RigidMotion m;
        m.linear_velocity = v3(v);
        m.angular_velocity = v3(w);
        m.center = v3(c);
        ThreadPool pool(1);
        update_rigid_motion(set, m, t, {nx, ny, nz}, pool);
        for (std::size_t k = 0; k < n; ++k) {
            for (int a = 0; a < 3; ++a) {
                pos[3 * k + a] = set.positions[k][a];
                ub[3 * k + a] = set.boundary_velocity[k][a];
            }
            flagged[k] = set.flagged[k];
        }
    });
}

int ref_ib_reaction_totals(size_t n, const double* pos, const double* force, const double* center, int z0, int z1,
                           double* out6) {
    return guard([&] {
        SolidSampleSet set = make_set(n, pos, nullptr, nullptr, force, nullptr);
        ReactionTotals r = reaction_totals(set, v3(center), z0, z1);
        for (int a = 0; a < 3; ++a) {
            out6[a] = r.force[a];
            out6[3 + a] = r.torque[a];
        }
    });
}

// Gathering oracle (tests/oracles.hpp:121-168) on a sample set with given
// penalty forces: g (n_nodes*3), loops (n_nodes).
int ref_gather_forces(size_t n, const double* pos, const double* force, const uint8_t* flagged,
                      int nx, int ny, int nz, double* g, uint32_t* loops) {
    return guard([&] {
        SolidSampleSet set;
        set.positions.resize(n);
        set.penalty_force.resize(n);
        set.flagged.resize(n);
        for (std::size_t k = 0; k < n; ++k) {
            set.positions[k] = v3(pos + 3 * k);
            set.penalty_force[k] = v3(force + 3 * k);
            set.flagged[k] = flagged ? flagged[k] : 0;
        }
        GridDims d{nx, ny, nz};
        auto r = oracle::gather_forces(set, d);
        for (std::size_t k = 0; k < d.n_nodes(); ++k) {
            for (int a = 0; a < 3; ++a) g[3 * k + a] = r.g[k][a];
            loops[k] = r.loops[k];
        }
    });
}

// TuneSpec::from_scene (autotune.cpp:9-27) of a runner's scene: ell range and
// the alpha list (cap entries at most; returns the count).
int ref_tune_spec(void* h, int n_steps, int warmup, int* ell_min, int* ell_max, size_t* alphas, size_t cap,
                  size_t* n_alphas) {
    return guard([&] {
        auto* rr = static_cast<RefRunner*>(h);
        const TuneSpec spec = TuneSpec::from_scene(rr->scene, n_steps, warmup);
        *ell_min = spec.ell_min;
        *ell_max = spec.ell_max;
        *n_alphas = spec.alphas.size();
        for (std::size_t k = 0; k < spec.alphas.size() && k < cap; ++k) alphas[k] = spec.alphas[k];
    });
}

// search_with_cost (autotune.cpp:38-60) over an injected cost table
// cost[(ell - ell_min) * n_alphas + k] (SPEC autotune example: fake cost fn).
int ref_search_with_cost(int ell_min, int ell_max, const size_t* alphas, size_t n_alphas, const double* cost,
                         int* ell, size_t* alpha, double* best) {
    return guard([&] {
        TuneSpec spec;
        spec.ell_min = ell_min;
        spec.ell_max = ell_max;
        spec.alphas.assign(alphas, alphas + n_alphas);
        std::vector<std::size_t> idx(alphas, alphas + n_alphas);
        const TuneOutcome o = search_with_cost(spec, [&](int l, std::size_t a) {
            std::size_t k = std::find(idx.begin(), idx.end(), a) - idx.begin();
            return cost[std::size_t(l - ell_min) * n_alphas + k];
        });
        *ell = o.ell;
        *alpha = o.alpha;
        *best = o.cost;
    });
}

// io.cpp:34-87: dump_field (canonical) and load_field of the reference.
int ref_dump_field(const char* path, int nx, int ny, int nz, int beta, const double* aos) {
    return guard([&] {
        GridDims d;
        d.nx = nx;
        d.ny = ny;
        d.nz = nz;
        FieldStore fs(LayoutParams::make(1, std::size_t(beta), d.n_nodes()));
        for (std::size_t k = 0; k < d.n_nodes(); ++k)
            for (int i = 0; i < beta; ++i) fs.set(k, std::size_t(i), aos[k * beta + i]);
        dump_field(fs, d, path, true);
    });
}

int ref_load_field(const char* path, int* dims, int* beta, double* out, size_t cap) {
    return guard([&] {
        const LoadedField lf = load_field(path);
        dims[0] = lf.dims.nx;
        dims[1] = lf.dims.ny;
        dims[2] = lf.dims.nz;
        *beta = int(lf.field.beta());
        const std::size_t n = lf.field.n_nodes();
        for (std::size_t k = 0; k < n; ++k)
            for (std::size_t i = 0; i < lf.field.beta(); ++i)
                if (k * lf.field.beta() + i < cap) out[k * lf.field.beta() + i] = lf.field.get(k, i);
    });
}

}  // extern "C"
