// lbm_b200.hpp — C++ mirror of the reference solver API
// (/root/reference/proj/include/lbm: scene.hpp, runner.hpp, solver.hpp,
// ib.hpp, core.hpp) over the C ABI in lbmg.h.  A reference client switches by
// including this header instead of "lbm/runner.hpp"/"lbm/scene.hpp" and
// linking _build/liblbmg.so; type and member names are the reference's.
//
// Header-only; exceptions: lbm::ConfigError / lbm::IoError as in core.hpp:50-58,
// lbm::DeviceError for CUDA failures.  Divergence is reported in StepStatus.
#pragma once

#include <array>
#include <cmath>
#include <functional>
#include <limits>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbmg.h"

namespace lbm {

struct Vec3 {  // core.hpp:14-32 (value type subset)
    double x = 0.0, y = 0.0, z = 0.0;
    double operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
};

struct GridDims {  // core.hpp:36-47
    int nx = 0, ny = 0, nz = 0;
    std::size_t n_nodes() const { return std::size_t(nx) * std::size_t(ny) * std::size_t(nz); }
};

class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class IoError : public std::runtime_error {
public:
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
class DeviceError : public std::runtime_error {
public:
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

namespace detail {
inline void check(int code) {
    if (code == LBMG_OK) return;
    const std::string msg = lbmg_last_error();
    if (code == LBMG_ERR_CONFIG) throw ConfigError(msg);
    if (code == LBMG_ERR_IO) throw IoError(msg);
    throw DeviceError(msg);
}
inline void put3(double* d, const Vec3& v) {
    d[0] = v.x;
    d[1] = v.y;
    d[2] = v.z;
}
}  // namespace detail

enum class CollisionKind { BGK, RawMomentMRT, CentralMomentMRT };          // collision.hpp:23
enum class RatePolicy { Constant, RelaxTowardOne };                        // collision.hpp:25
enum class FaceCondition { NoSlip, VelocityInlet, Outflow, Periodic };     // boundary.hpp:22
enum class AccumulationMode { Atomic, Deterministic };                      // ib.hpp:33
enum class SamplingMethod { DartThrowing, SampleElimination };             // ib.hpp:35
enum class InitKind { Uniform, TaylorGreen };                              // scene.hpp:43

struct FaceSpec {  // boundary.hpp:24-27
    FaceCondition condition = FaceCondition::NoSlip;
    Vec3 inlet_velocity;
};
struct BoundarySet {  // boundary.hpp:33-42
    std::array<FaceSpec, 6> faces;
};

struct MeshConfig {  // scene.hpp:22-33 (no File meshes)
    enum class Type { Sphere, Box, FinComb, Quad } type = Type::Sphere;
    Vec3 center, lo, hi, origin;
    double radius = 1.0;
    int subdivisions = 3;
    int fins = 8;
    double fin_length = 8, fin_height = 6, fin_spacing = 2;
    double size = 1.0, plane_z = 0.0;
};

struct RigidMotion {  // ib.hpp:111-115
    Vec3 linear_velocity, angular_velocity, center;
};

struct SolidConfig {  // scene.hpp:35-40
    MeshConfig mesh;
    double poisson_radius = 0.5;
    SamplingMethod sampling = SamplingMethod::DartThrowing;
    std::optional<RigidMotion> motion;
};

struct TracerEmitter {  // tracer.hpp:14-17
    Vec3 lo, hi;
    int rate = 0;
};

struct TracerCloud {  // tracer.hpp:19-25
    std::vector<Vec3> positions;
    std::vector<long> birth_step;
    std::size_t size() const { return positions.size(); }
};

struct SceneConfig {  // scene.hpp:49-78 (hot-path fields)
    GridDims dims;
    double viscosity = 0.05;
    CollisionKind kind = CollisionKind::BGK;
    double high_order_rate = 1.0;
    RatePolicy policy = RatePolicy::Constant;
    double policy_eps0 = 0.01;
    std::optional<std::array<double, 27>> explicit_rates;
    BoundarySet boundary;
    Vec3 body_force;
    std::vector<SolidConfig> solids;
    std::vector<TracerEmitter> emitters;
    InitKind init = InitKind::Uniform;
    double init_density = 1.0;
    Vec3 init_velocity;
    double tg_u_max = 0.02;
    int regions = 1;
    unsigned threads_per_region = 0;
    std::size_t alpha = 1;
    int block_edge = 1;
    AccumulationMode ib_mode = AccumulationMode::Atomic;
    std::uint64_t seed = 1;
};

struct StepStatus {  // solver.hpp:47-52
    bool ok = true;
    bool mach_warning = false;
    long step = -1;
    std::string reason;
};

struct TimingRow {  // io.hpp:50-54
    std::string phase;
    long step = 0;
    double seconds = 0.0;
};

struct ReactionTotals {  // ib.hpp:124-127
    Vec3 force, torque;
};

// Canonical AoS FP64 field (the layout gather_* returns, runner.cpp:260-295).
class FieldStore {
public:
    FieldStore() = default;
    FieldStore(std::size_t n, std::size_t beta) : n_(n), beta_(beta), data_(n * beta) {}
    std::size_t n_nodes() const { return n_; }
    std::size_t beta() const { return beta_; }
    double get(std::size_t k, std::size_t i) const { return data_[k * beta_ + i]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    std::size_t size() const { return data_.size(); }

private:
    std::size_t n_ = 0, beta_ = 1;
    std::vector<double> data_;
};

class Runner;

// Scene (scene.hpp:92-96): owns the sampled, ordered solids.
class Scene {
public:
    Scene() = default;
    Scene(const Scene&) = delete;
    Scene& operator=(const Scene&) = delete;
    Scene(Scene&& o) noexcept : cfg(std::move(o.cfg)), h_(o.h_) { o.h_ = nullptr; }
    ~Scene() { lbmg_scene_destroy(h_); }
    SceneConfig cfg;
    std::size_t sample_count(int solid) const { return lbmg_scene_sample_count(h_, solid); }

private:
    friend Scene build_scene(const SceneConfig&);
    friend class Runner;
    lbmg_scene* h_ = nullptr;
};

inline lbmg_scene_config to_c(const SceneConfig& c, std::vector<lbmg_solid_config>& solids) {
    lbmg_scene_config o;
    lbmg_scene_config_default(&o);
    o.nx = c.dims.nx;
    o.ny = c.dims.ny;
    o.nz = c.dims.nz;
    o.viscosity = c.viscosity;
    o.kind = int(c.kind);
    o.high_order_rate = c.high_order_rate;
    o.policy = int(c.policy);
    o.policy_eps0 = c.policy_eps0;
    if (c.explicit_rates) {
        o.has_explicit_rates = 1;
        for (int r = 0; r < 27; ++r) o.rates[r] = (*c.explicit_rates)[r];
    }
    for (int f = 0; f < 6; ++f) {
        o.faces[f].condition = int(c.boundary.faces[f].condition);
        detail::put3(o.faces[f].velocity, c.boundary.faces[f].inlet_velocity);
    }
    detail::put3(o.body_force, c.body_force);
    solids.clear();
    for (const auto& s : c.solids) {
        lbmg_solid_config sc{};
        sc.mesh.type = int(s.mesh.type);
        detail::put3(sc.mesh.center, s.mesh.center);
        detail::put3(sc.mesh.lo, s.mesh.lo);
        detail::put3(sc.mesh.hi, s.mesh.hi);
        detail::put3(sc.mesh.origin, s.mesh.origin);
        sc.mesh.radius = s.mesh.radius;
        sc.mesh.subdivisions = s.mesh.subdivisions;
        sc.mesh.fins = s.mesh.fins;
        sc.mesh.fin_length = s.mesh.fin_length;
        sc.mesh.fin_height = s.mesh.fin_height;
        sc.mesh.fin_spacing = s.mesh.fin_spacing;
        sc.mesh.size = s.mesh.size;
        sc.mesh.plane_z = s.mesh.plane_z;
        sc.poisson_radius = s.poisson_radius;
        sc.sampling = int(s.sampling);
        if (s.motion) {
            sc.has_motion = 1;
            detail::put3(sc.linear_velocity, s.motion->linear_velocity);
            detail::put3(sc.angular_velocity, s.motion->angular_velocity);
            detail::put3(sc.center, s.motion->center);
        }
        solids.push_back(sc);
    }
    o.n_solids = int(solids.size());
    o.solids = solids.empty() ? nullptr : solids.data();
    o.init = int(c.init);
    o.init_density = c.init_density;
    detail::put3(o.init_velocity, c.init_velocity);
    o.tg_u_max = c.tg_u_max;
    o.regions = c.regions;
    o.threads_per_region = c.threads_per_region;
    o.alpha = c.alpha;
    o.block_edge = c.block_edge;
    o.ib_mode = int(c.ib_mode);
    o.seed = c.seed;
    return o;
}

// build_scene, scene.hpp:100.
inline Scene build_scene(const SceneConfig& cfg) {
    std::vector<lbmg_solid_config> solids;
    const lbmg_scene_config c = to_c(cfg, solids);
    Scene s;
    s.cfg = cfg;
    detail::check(lbmg_scene_build(&c, &s.h_));
    if (!cfg.emitters.empty()) {
        std::vector<lbmg_emitter> em(cfg.emitters.size());
        for (std::size_t k = 0; k < em.size(); ++k) {
            detail::put3(em[k].lo, cfg.emitters[k].lo);
            detail::put3(em[k].hi, cfg.emitters[k].hi);
            em[k].rate = cfg.emitters[k].rate;
        }
        detail::check(lbmg_scene_set_emitters(s.h_, int(em.size()), em.data()));
    }
    return s;
}

// Runner, runner.hpp:25-83, on the B200 engine.
class Runner {
public:
    explicit Runner(const Scene& scene, int device = 0) : Runner(scene, scene.cfg.regions, 0, device) {}
    Runner(const Scene& scene, int regions, unsigned /*threads_per_region*/, int device = 0) {
        detail::check(lbmg_runner_create(scene.h_, regions, device, &h_));
    }
    // Runner(scene, regions, threads) with region r on devices[r % size]
    // (lbmg_runner_create_devices: halos by NVLink peer stores)
    Runner(const Scene& scene, int regions, const std::vector<int>& devices) {
        detail::check(lbmg_runner_create_devices(scene.h_, regions, int(devices.size()), devices.data(), &h_));
    }
    Runner(const Runner&) = delete;
    Runner& operator=(const Runner&) = delete;
    Runner(Runner&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~Runner() { lbmg_runner_destroy(h_); }

    StepStatus advance(long steps, std::vector<TimingRow>* timings = nullptr) {
        lbmg_status st;
        if (!timings) {
            detail::check(lbmg_runner_advance(h_, steps, &st, nullptr, 0, nullptr));
        } else {
            std::vector<lbmg_timing_row> rows(std::size_t(steps > 0 ? steps : 1) * 5);  // <= 5 phases per step
            std::size_t n = 0;
            detail::check(lbmg_runner_advance(h_, steps, &st, rows.data(), rows.size(), &n));
            for (std::size_t k = 0; k < n; ++k) timings->push_back({rows[k].phase, rows[k].step, rows[k].seconds});
        }
        return {st.ok != 0, st.mach_warning != 0, st.step, st.reason};
    }
    long step_count() const { return lbmg_runner_step_count(h_); }
    StepStatus status() const {
        lbmg_status st;
        detail::check(lbmg_runner_status(h_, &st));
        return {st.ok != 0, st.mach_warning != 0, st.step, st.reason};
    }
    GridDims dims() const {
        GridDims d;
        detail::check(lbmg_runner_dims(h_, &d.nx, &d.ny, &d.nz));
        return d;
    }
    int region_count() const { return lbmg_runner_region_count(h_); }
    void set_layout(int block_edge, std::size_t alpha) { detail::check(lbmg_runner_set_layout(h_, block_edge, alpha)); }
    std::size_t alpha() const { return lbmg_runner_alpha(h_); }
    int block_edge() const { return lbmg_runner_block_edge(h_); }

    FieldStore gather_rho() const { return gather(1, lbmg_runner_gather_rho); }
    FieldStore gather_u() const { return gather(3, lbmg_runner_gather_u); }
    FieldStore gather_f() const { return gather(27, lbmg_runner_gather_f); }

    std::vector<ReactionTotals> totals_log() const {
        const std::size_t n = lbmg_runner_totals_count(h_);
        std::vector<double> raw(6 * n);
        if (n) detail::check(lbmg_runner_totals(h_, raw.data(), n));
        std::vector<ReactionTotals> out(n);
        for (std::size_t s = 0; s < n; ++s) {
            out[s].force = {raw[6 * s], raw[6 * s + 1], raw[6 * s + 2]};
            out[s].torque = {raw[6 * s + 3], raw[6 * s + 4], raw[6 * s + 5]};
        }
        return out;
    }

    Runner clone() const {
        Runner c;
        detail::check(lbmg_runner_clone(h_, &c.h_));
        return c;
    }

    // Kernel variants (the tuner's launch-split dimension, lbmg.h).
    void set_variant(int fluid, int ib) { detail::check(lbmg_runner_set_variant(h_, fluid, ib)); }
    std::array<int, 2> variant() const {
        std::array<int, 2> v{};
        detail::check(lbmg_runner_variant(h_, &v[0], &v[1]));
        return v;
    }
    // CTA shape of the staged fluid kernel (512 / 256 / 128 threads, 0 = default).
    void set_cta(int threads) { detail::check(lbmg_runner_set_cta(h_, threads)); }
    int cta() const { return lbmg_runner_cta(h_); }
    std::uint64_t layout_key(std::size_t alpha) const {
        std::uint64_t k = 0;
        detail::check(lbmg_runner_layout_key(h_, alpha, &k));
        return k;
    }

    // Asynchronous rho*, u* snapshot (driver.cpp:45-59 without the stall).
    void snapshot_begin() { detail::check(lbmg_runner_snapshot_begin(h_)); }
    long snapshot_wait(FieldStore& rho, FieldStore& u) {
        const GridDims d = dims();
        rho = FieldStore(d.n_nodes(), 1);
        u = FieldStore(d.n_nodes(), 3);
        long t = 0;
        detail::check(lbmg_runner_snapshot_wait(h_, rho.data(), u.data(), &t));
        return t;
    }

    // Runner::tracers (runner.hpp:54): the live cloud after the last step.
    TracerCloud tracers() const {
        const std::size_t n = lbmg_runner_tracer_count(h_);
        std::vector<double> pos(3 * n);
        std::vector<std::int64_t> birth(n);
        detail::check(lbmg_runner_tracers(h_, pos.data(), birth.data()));
        TracerCloud c;
        for (std::size_t k = 0; k < n; ++k) {
            c.positions.push_back({pos[3 * k], pos[3 * k + 1], pos[3 * k + 2]});
            c.birth_step.push_back(long(birth[k]));
        }
        return c;
    }
    // rasterize_density(tracers(), dims()) from the device-resident cloud.
    std::vector<double> tracer_density() const {
        std::vector<double> vol(dims().n_nodes());
        detail::check(lbmg_runner_tracer_density(h_, vol.data()));
        return vol;
    }

    int region_device(int region) const { return lbmg_runner_region_device(h_, region); }

    // SimState (solver.hpp:29-45) of a single-region runner without solids:
    // f(t), the face-pass scratch f* (empty: f) and t
    void load_state(const FieldStore& f, const FieldStore& f_star, long t) {
        detail::check(lbmg_runner_load_state(h_, f.data(), f_star.size() ? f_star.data() : nullptr, t));
    }

    lbmg_runner* handle() { return h_; }

private:
    Runner() = default;
    template <class F>
    FieldStore gather(std::size_t beta, F fn) const {
        const GridDims d = dims();
        FieldStore out(d.n_nodes(), beta);
        detail::check(fn(h_, out.data()));
        return out;
    }
    lbmg_runner* h_ = nullptr;
};

// step(SimState&, ...) (solver.hpp:82-83): one single-region step on the
// state the runner holds (load_state / the last advance).
inline StepStatus step(Runner& runner) {
    lbmg_status st;
    detail::check(lbmg_step(runner.handle(), &st));
    return {st.ok != 0, st.mach_warning != 0, st.step, st.reason};
}

// ---- IB free functions (ib.hpp:47-128) on the device, host arrays in/out ----

struct SolidSampleSet {  // ib.hpp:47-60 (per-sample arrays)
    std::vector<Vec3> positions, boundary_velocity, penalty_force, sampled_velocity, reference_positions;
    std::vector<std::uint32_t> source_id;
    std::vector<std::uint8_t> flagged;
    std::size_t size() const { return positions.size(); }
};

struct KernelSupport {  // ib.hpp:75-82
    int base[3] = {0, 0, 0};
    double wx[2] = {0, 0}, wy[2] = {0, 0}, wz[2] = {0, 0};
    bool inside = true;
    double weight(int ox, int oy, int oz) const { return wx[ox] * wy[oy] * wz[oz]; }
};

// The slab a call owns (DomainContext::global + owned planes, domain.hpp:17-24).
struct SlabContext {
    GridDims global;
    int z0 = 0, z1 = -1;  // owned global planes [z0, z1); z1 < 0: the whole grid
    int end() const { return z1 < 0 ? global.nz : z1; }
};

namespace detail {
inline std::vector<double> flat3(const std::vector<Vec3>& v) {
    std::vector<double> o(3 * v.size());
    for (std::size_t k = 0; k < v.size(); ++k) put3(&o[3 * k], v[k]);
    return o;
}
inline void unflat3(const std::vector<double>& o, std::vector<Vec3>& v) {
    v.resize(o.size() / 3);
    for (std::size_t k = 0; k < v.size(); ++k) v[k] = {o[3 * k], o[3 * k + 1], o[3 * k + 2]};
}
}  // namespace detail

inline KernelSupport kernel_support(const Vec3& pos, const GridDims& global) {  // ib.cpp:294-308
    double p[3];
    detail::put3(p, pos);
    int base[3];
    double w[6];
    std::uint8_t inside = 0;
    detail::check(lbmg_ib_kernel_support(1, p, global.nx, global.ny, global.nz, base, w, &inside));
    KernelSupport ks;
    for (int a = 0; a < 3; ++a) ks.base[a] = base[a];
    ks.wx[0] = w[0], ks.wx[1] = w[1], ks.wy[0] = w[2], ks.wy[1] = w[3], ks.wz[0] = w[4], ks.wz[1] = w[5];
    ks.inside = inside != 0;
    return ks;
}

inline void interpolate_velocity(SolidSampleSet& set, const FieldStore& u, const SlabContext& ctx) {  // ib.cpp:321-343
    const auto pos = detail::flat3(set.positions);
    std::vector<double> sampled(pos.size());
    set.flagged.resize(set.size());
    detail::check(lbmg_ib_interpolate_velocity(set.size(), pos.data(), u.data(), ctx.global.nx, ctx.global.ny,
                                               ctx.global.nz, ctx.z0, ctx.end(), sampled.data(), set.flagged.data()));
    detail::unflat3(sampled, set.sampled_velocity);
}

inline void penalty_forces(SolidSampleSet& set, const FieldStore& rho, const SlabContext& ctx) {  // ib.cpp:345-365
    const auto pos = detail::flat3(set.positions), ub = detail::flat3(set.boundary_velocity),
               us = detail::flat3(set.sampled_velocity);
    std::vector<double> force(pos.size());
    detail::check(lbmg_ib_penalty_forces(set.size(), pos.data(), ub.data(), us.data(),
                                         set.flagged.empty() ? nullptr : set.flagged.data(), rho.data(),
                                         ctx.global.nx, ctx.global.ny, ctx.global.nz, ctx.z0, ctx.end(),
                                         force.data()));
    detail::unflat3(force, set.penalty_force);
}

inline void spread_forces(const SolidSampleSet& set, FieldStore& g, const SlabContext& ctx) {  // ib.cpp:369-454
    const auto pos = detail::flat3(set.positions), force = detail::flat3(set.penalty_force);
    detail::check(lbmg_ib_spread_forces(set.size(), pos.data(), force.data(),
                                        set.flagged.empty() ? nullptr : set.flagged.data(), ctx.global.nx,
                                        ctx.global.ny, ctx.global.nz, ctx.z0, ctx.end(), g.data()));
}

inline void update_rigid_motion(SolidSampleSet& set, const RigidMotion& m, long t, const GridDims& global) {
    // ib.cpp:456-489
    const auto ref = detail::flat3(set.reference_positions);
    double v[3], w[3], c[3];
    detail::put3(v, m.linear_velocity);
    detail::put3(w, m.angular_velocity);
    detail::put3(c, m.center);
    std::vector<double> pos(ref.size()), ub(ref.size());
    set.flagged.resize(ref.size() / 3);
    detail::check(lbmg_ib_update_rigid_motion(ref.size() / 3, ref.data(), v, w, c, t, global.nx, global.ny,
                                              global.nz, pos.data(), ub.data(), set.flagged.data()));
    detail::unflat3(pos, set.positions);
    detail::unflat3(ub, set.boundary_velocity);
}

inline ReactionTotals reaction_totals(const SolidSampleSet& set, const Vec3& center, int z0, int z1) {
    // ib.cpp:491-501
    const auto pos = detail::flat3(set.positions), force = detail::flat3(set.penalty_force);
    double c[3], out[6];
    detail::put3(c, center);
    detail::check(lbmg_ib_reaction_totals(set.size(), pos.data(), force.data(), c, z0, z1, out));
    return {{out[0], out[1], out[2]}, {out[3], out[4], out[5]}};
}

// rasterize_density (tracer.hpp:43, tracer.cpp:67-92) on device 0.
inline std::vector<double> rasterize_density(const TracerCloud& cloud, const GridDims& dims) {
    std::vector<double> pos(3 * cloud.size()), vol(dims.n_nodes());
    for (std::size_t k = 0; k < cloud.size(); ++k) detail::put3(&pos[3 * k], cloud.positions[k]);
    detail::check(lbmg_rasterize_density(cloud.size(), pos.data(), dims.nx, dims.ny, dims.nz, 0, vol.data()));
    return vol;
}

// dump_field (io.hpp:19-20, canonical = true): LBF1 file readable by load_field.
inline void dump_field(const FieldStore& field, const GridDims& dims, const std::string& path) {
    detail::check(lbmg_dump_field(path.c_str(), dims.nx, dims.ny, dims.nz, int(field.beta()), field.data()));
}

// ---- auto-tuner (autotune.hpp; Eq. 10), device-timed costs -------------------

struct TuneSpec {  // autotune.hpp:18-35 (+ the kernel-variant dimension)
    int ell_min = 1;
    int ell_max = 1;
    std::vector<std::size_t> alphas;
    int n_steps = 10;
    int warmup = 5;
    std::vector<std::array<int, 2>> variants{{0, 0}};
    std::size_t candidate_count() const {
        return std::size_t(ell_max - ell_min + 1) * alphas.size() * variants.size();
    }
};

struct TuneRow {
    int ell;
    std::size_t alpha;
    double seconds;
    std::array<int, 2> variant;
};

struct TuneOutcome {  // autotune.hpp:37-42
    int ell = 0;
    std::size_t alpha = 0;
    double cost = std::numeric_limits<double>::infinity();
    std::array<int, 2> variant{0, 0};
    std::vector<TuneRow> rows;
};

// measure_cost (autotune.cpp:29-36): mean device seconds per step, inf on divergence.
inline double measure_cost(Runner& runner, int ell, std::size_t alpha, const TuneSpec& spec) {
    double sec = 0.0;
    detail::check(lbmg_runner_measure_cost(runner.handle(), ell, alpha, spec.warmup, spec.n_steps, &sec));
    return sec;
}

using CostFn = std::function<double(int ell, std::size_t alpha, std::array<int, 2> variant)>;

// search_with_cost (autotune.cpp:38-60): ascending enumeration, strict <.
inline TuneOutcome search_with_cost(const TuneSpec& spec, const CostFn& cost) {
    TuneOutcome out;
    for (const auto& v : spec.variants)
        for (int ell = spec.ell_min; ell <= spec.ell_max; ++ell)
            for (std::size_t a : spec.alphas) {
                const double c = cost(ell, a, v);
                out.rows.push_back({ell, a, c, v});
                if (c < out.cost) {
                    out.cost = c;
                    out.ell = ell;
                    out.alpha = a;
                    out.variant = v;
                }
            }
    if (!std::isfinite(out.cost)) throw ConfigError("tune: every candidate was invalid");
    return out;
}

// search (autotune.cpp:62-70): on a clone; equal device layouts measured once.
inline TuneOutcome search(const Runner& base, const TuneSpec& spec) {
    Runner probe = base.clone();
    struct Seen {
        std::array<int, 2> v;
        int ell;
        std::uint64_t key;
        double cost;
    };
    std::vector<Seen> seen;
    return search_with_cost(spec, [&](int ell, std::size_t alpha, std::array<int, 2> v) {
        if (probe.variant() != v) probe.set_variant(v[0], v[1]);
        const std::uint64_t key = probe.layout_key(alpha);
        for (const auto& s : seen)
            if (s.v == v && s.ell == ell && s.key == key) return s.cost;
        const double c = measure_cost(probe, ell, alpha, spec);
        seen.push_back({v, ell, key, c});
        return c;
    });
}

}  // namespace lbm
