// extern "C" surface (include/lbmg.h).  Exceptions never cross the ABI:
// each entry point maps them to an LBMG_ERR_* code + lbmg_last_error().
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <exception>
#include <thread>
#include <vector>
#include <cstring>
#include <string>

#include "lbmg.h"
#include "runner.hpp"
#include "scene.hpp"

using namespace lbmg;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return LBMG_OK;
    } catch (const lbmg::ConfigError& e) {
        g_err = e.what();
        return LBMG_ERR_CONFIG;
    } catch (const OomError& e) {
        g_err = e.what();
        return LBMG_ERR_OOM;
    } catch (const IoError& e) {
        g_err = e.what();
        return LBMG_ERR_IO;
    } catch (const CudaError& e) {
        g_err = e.what();
        return LBMG_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LBMG_ERR_STATE;
    }
}

void put_status(const Status& s, lbmg_status* o) {
    if (!o) return;
    o->ok = s.ok ? 1 : 0;
    o->mach_warning = s.mach_warning ? 1 : 0;
    o->step = s.step;
    std::snprintf(o->reason, sizeof o->reason, "%s", s.reason.c_str());
}

Runner& R(lbmg_runner* r) {
    if (!r || !r->impl) throw StateError("null runner");
    return *r->impl;
}
const Runner& R(const lbmg_runner* r) {
    if (!r || !r->impl) throw StateError("null runner");
    return *r->impl;
}

}  // namespace

extern "C" {

int lbmg_abi_version(void) { return LBMG_ABI_VERSION; }
const char* lbmg_last_error(void) { return g_err.c_str(); }

int lbmg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void lbmg_scene_config_default(lbmg_scene_config* c) {
    std::memset(c, 0, sizeof *c);
    c->viscosity = 0.05;
    c->kind = LBMG_BGK;
    c->high_order_rate = 1.0;
    c->policy = LBMG_POLICY_CONSTANT;
    c->policy_eps0 = 0.01;
    for (int f = 0; f < 6; ++f) c->faces[f].condition = LBMG_NOSLIP;
    c->init = LBMG_INIT_UNIFORM;
    c->init_density = 1.0;
    c->tg_u_max = 0.02;
    c->regions = 1;
    c->alpha = 1;
    c->block_edge = 1;
    c->ib_mode = LBMG_IB_ATOMIC;
    c->seed = 1;
}

int lbmg_validate_config(const lbmg_scene_config* cfg, double* rates) {
    return guarded([&] {
        validate_config(*cfg);
        if (rates) {
            auto r = make_rates(*cfg);
            for (int i = 0; i < 27; ++i) rates[i] = r[i];
        }
    });
}

// build_scene, scene.cpp:341-366.
int lbmg_scene_build(const lbmg_scene_config* cfg, lbmg_scene** out) {
    return guarded([&] {
        validate_config(*cfg);
        auto* s = new lbmg_scene;
        try {
            s->cfg = *cfg;
            s->solid_cfgs.assign(cfg->solids, cfg->solids + cfg->n_solids);
            s->cfg.solids = s->solid_cfgs.empty() ? nullptr : s->solid_cfgs.data();
            // build_scene (scene.cpp:341-366): solid i is sampled with seed
            // cfg.seed + i, independently of the others -> the solids of a
            // large scene (C4: ~3.7 M samples over many boxes) are sampled on
            // all host cores, bit-identical to the sequential order.
            const size_t ns = s->solid_cfgs.size();
            std::vector<SolidInstance> built(ns);
            std::vector<std::exception_ptr> errs(ns);
            std::atomic<size_t> next{0};
            auto work = [&] {
                for (size_t i = next++; i < ns; i = next++) {
                    try {
                        const auto& sc = s->solid_cfgs[i];
                        SolidInstance& inst = built[i];
                        inst.cfg = sc;
                        const TriMesh mesh = build_mesh(sc.mesh);
                        inst.samples = sample_surface(mesh, sc.poisson_radius, cfg->seed + i, sc.sampling, &inst.report);
                        if (sc.has_motion) {
                            inst.moving = true;
                            inst.linear_velocity = v3(sc.linear_velocity);
                            inst.angular_velocity = v3(sc.angular_velocity);
                            inst.center = v3(sc.center);
                            for (size_t k = 0; k < inst.samples.size(); ++k)
                                inst.samples.reference_positions[k] = inst.samples.positions[k] - inst.center;
                        } else {
                            inst.samples.reference_positions = inst.samples.positions;
                        }
                        reorder_samples(inst.samples, cfg->block_edge);
                    } catch (...) {
                        errs[i] = std::current_exception();
                    }
                }
            };
            const size_t nt = std::min<size_t>(ns, std::max(1u, std::thread::hardware_concurrency()));
            std::vector<std::thread> pool;
            for (size_t t = 1; t < nt; ++t) pool.emplace_back(work);
            work();
            for (auto& t : pool) t.join();
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
            for (auto& inst : built) s->solids.push_back(std::move(inst));
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

void lbmg_scene_destroy(lbmg_scene* s) { delete s; }

int lbmg_scene_solid_count(const lbmg_scene* s) { return s ? int(s->solids.size()) : 0; }

size_t lbmg_scene_sample_count(const lbmg_scene* s, int solid) {
    if (!s || solid < 0 || solid >= int(s->solids.size())) return 0;
    return s->solids[solid].samples.size();
}

int lbmg_scene_samples(const lbmg_scene* s, int solid, double* pos, double* refpos, uint32_t* src,
                       uint8_t* flagged, double* bbox, int* ell) {
    return guarded([&] {
        if (!s || solid < 0 || solid >= int(s->solids.size())) throw StateError("solid index out of range");
        const SampleSet& set = s->solids[solid].samples;
        for (size_t k = 0; k < set.size(); ++k) {
            for (int a = 0; a < 3; ++a) {
                if (pos) pos[3 * k + a] = set.positions[k][a];
                if (refpos) refpos[3 * k + a] = set.reference_positions[k][a];
            }
            if (src) src[k] = set.source_id[k];
            if (flagged) flagged[k] = 0;
        }
        if (bbox)
            for (int a = 0; a < 3; ++a) {
                bbox[a] = set.bbox_lo[a];
                bbox[3 + a] = set.bbox_hi[a];
            }
        if (ell) *ell = set.block_edge;
    });
}

int lbmg_scene_set_samples(lbmg_scene* s, int solid, size_t n, const double* pos, const double* refpos,
                           const uint32_t* src) {
    return guarded([&] {
        if (!s || solid < 0 || solid >= int(s->solids.size())) throw StateError("solid index out of range");
        SampleSet& set = s->solids[solid].samples;
        set.positions.resize(n);
        set.reference_positions.resize(n);
        set.source_id.resize(n);
        set.bbox_lo = {1e300, 1e300, 1e300};
        set.bbox_hi = {-1e300, -1e300, -1e300};
        for (size_t k = 0; k < n; ++k) {
            set.positions[k] = v3(pos + 3 * k);
            set.reference_positions[k] = v3(refpos + 3 * k);
            set.source_id[k] = src[k];
            for (int a = 0; a < 3; ++a) {
                set.bbox_lo[a] = std::min(set.bbox_lo[a], set.positions[k][a]);
                set.bbox_hi[a] = std::max(set.bbox_hi[a], set.positions[k][a]);
            }
        }
    });
}

uint64_t lbmg_morton3(uint32_t x, uint32_t y, uint32_t z) { return morton3(x, y, z); }

int lbmg_reorder_permutation(size_t n, const double* positions, const uint32_t* source_id, int ell,
                             uint32_t* perm) {
    return guarded([&] {
        std::vector<V3> p(n);
        for (size_t k = 0; k < n; ++k) p[k] = v3(positions + 3 * k);
        auto out = reorder_permutation(p, std::vector<uint32_t>(source_id, source_id + n), ell);
        std::memcpy(perm, out.data(), n * sizeof(uint32_t));
    });
}

int lbmg_split_domain(int nz, int m, int* z0z1) {
    return guarded([&] {
        auto s = split_domain(nz, m);
        for (int r = 0; r < m; ++r) {
            z0z1[2 * r] = s[r][0];
            z0z1[2 * r + 1] = s[r][1];
        }
    });
}

int lbmg_runner_create(const lbmg_scene* scene, int regions, int device, lbmg_runner** out) {
    return guarded([&] {
        if (!scene) throw StateError("null scene");
        auto* r = new lbmg_runner;
        try {
            r->impl = std::make_unique<Runner>(*scene, regions, device, 0, 0);
        } catch (...) {
            delete r;
            throw;
        }
        *out = r;
    });
}

int lbmg_runner_create_devices(const lbmg_scene* scene, int regions, int n_devices, const int* devices,
                               lbmg_runner** out) {
    return guarded([&] {
        if (!scene || !out) throw lbmg::ConfigError("runner: scene and out are required");
        if (n_devices < 1 || !devices) throw lbmg::ConfigError("devices: at least one device");
        std::vector<int> devs(devices, devices + n_devices);
        auto r = new lbmg_runner;
        try {
            r->impl = std::make_unique<Runner>(*scene, regions, devs[0], 0, 0, devs);
        } catch (...) {
            delete r;
            throw;
        }
        *out = r;
    });
}

int lbmg_runner_region_device(const lbmg_runner* r, int region) {
    if (!r || !r->impl || region < 0 || region >= r->impl->region_count()) return -1;
    return r->impl->region_device(region);
}

int lbmg_runner_create_rank(const lbmg_scene* scene, int world, int rank, int device, lbmg_runner** out) {
    return guarded([&] {
        if (!scene) throw StateError("null scene");
        if (world < 1) throw lbmg::ConfigError("world must be >= 1");
        auto* r = new lbmg_runner;
        try {
            r->impl = std::make_unique<Runner>(*scene, 1, device, world, rank);
        } catch (...) {
            delete r;
            throw;
        }
        *out = r;
    });
}

void lbmg_runner_destroy(lbmg_runner* r) { delete r; }

int lbmg_runner_clone(const lbmg_runner* r, lbmg_runner** out) {
    return guarded([&] {
        auto* c = new lbmg_runner;
        try {
            c->impl = R(r).clone();
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int lbmg_runner_set_stream(lbmg_runner* r, void* stream) {
    return guarded([&] { R(r).set_stream(static_cast<cudaStream_t>(stream)); });
}

int lbmg_runner_advance(lbmg_runner* r, long steps, lbmg_status* status, lbmg_timing_row* rows, size_t cap,
                        size_t* n_rows) {
    return guarded([&] {
        std::vector<Timing> t;
        Status st = R(r).advance(steps, rows ? &t : nullptr);
        put_status(st, status);
        if (rows) {
            size_t k = 0;
            for (; k < t.size() && k < cap; ++k) {
                std::snprintf(rows[k].phase, sizeof rows[k].phase, "%s", t[k].phase.c_str());
                rows[k].step = t[k].step;
                rows[k].seconds = t[k].seconds;
            }
            if (n_rows) *n_rows = k;
        }
    });
}

long lbmg_runner_step_count(const lbmg_runner* r) { return r && r->impl ? r->impl->step_count() : -1; }

int lbmg_runner_status(const lbmg_runner* r, lbmg_status* status) {
    return guarded([&] { put_status(R(r).status(), status); });
}

int lbmg_runner_dims(const lbmg_runner* r, int* nx, int* ny, int* nz) {
    return guarded([&] {
        *nx = R(r).nx();
        *ny = R(r).ny();
        *nz = R(r).nz();
    });
}

int lbmg_runner_region_count(const lbmg_runner* r) { return r && r->impl ? r->impl->region_count() : 0; }

int lbmg_runner_set_layout(lbmg_runner* r, int block_edge, size_t alpha) {
    return guarded([&] { R(r).set_layout(block_edge, alpha); });
}

int lbmg_runner_set_variant(lbmg_runner* r, int fluid, int ib) {
    return guarded([&] { R(r).set_variant(fluid, ib); });
}

int lbmg_runner_variant(const lbmg_runner* r, int* fluid, int* ib) {
    return guarded([&] {
        if (fluid) *fluid = R(r).fluid_variant();
        if (ib) *ib = R(r).ib_variant();
    });
}

int lbmg_runner_measure_cost(lbmg_runner* r, int block_edge, size_t alpha, int warmup, int n_steps,
                             double* seconds) {
    return guarded([&] { *seconds = R(r).measure_cost(block_edge, alpha, warmup, n_steps); });
}

int lbmg_runner_layout_key(const lbmg_runner* r, size_t alpha, uint64_t* key) {
    return guarded([&] { *key = R(r).layout_key(alpha); });
}

size_t lbmg_runner_alpha(const lbmg_runner* r) { return r && r->impl ? r->impl->alpha() : 0; }
int lbmg_runner_block_edge(const lbmg_runner* r) { return r && r->impl ? r->impl->block_edge() : 0; }

int lbmg_runner_gather_rho(const lbmg_runner* r, double* out) {
    return guarded([&] { R(r).gather(0, out); });
}
int lbmg_runner_gather_u(const lbmg_runner* r, double* out) {
    return guarded([&] { R(r).gather(1, out); });
}
int lbmg_runner_snapshot_begin(lbmg_runner* r) {
    return guarded([&] { R(r).snapshot_begin(); });
}

int lbmg_runner_snapshot_wait(lbmg_runner* r, double* rho, double* u, long* step) {
    return guarded([&] {
        const long t = R(r).snapshot_wait(rho, u);
        if (step) *step = t;
    });
}

// LBF1 field dump, canonical order (io.cpp:34-55 with canonical = true):
// magic, endian probe, nx, ny, nz, beta (u32), alpha = 0 (u64), width (u32),
// n_nodes (u64), then n_nodes * beta doubles node-major.
int lbmg_dump_field(const char* path, int nx, int ny, int nz, int beta, const double* aos) {
    return guarded([&] {
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw IoError(std::string("cannot write field dump: ") + path);
        const char magic[4] = {'L', 'B', 'F', '1'};
        const uint32_t probe = 0x01020304u, dims[4] = {uint32_t(nx), uint32_t(ny), uint32_t(nz), uint32_t(beta)};
        const uint64_t alpha = 0, n = uint64_t(nx) * uint64_t(ny) * uint64_t(nz);
        const uint32_t width = sizeof(double);
        bool ok = std::fwrite(magic, 1, 4, f) == 4 && std::fwrite(&probe, 4, 1, f) == 1 &&
                  std::fwrite(dims, 4, 4, f) == 4 && std::fwrite(&alpha, 8, 1, f) == 1 &&
                  std::fwrite(&width, 4, 1, f) == 1 && std::fwrite(&n, 8, 1, f) == 1 &&
                  std::fwrite(aos, sizeof(double), n * uint64_t(beta), f) == n * uint64_t(beta);
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) throw IoError(std::string("short write: ") + path);
    });
}

int lbmg_runner_gather_f(const lbmg_runner* r, double* out) {
    return guarded([&] { R(r).gather(2, out); });
}
int lbmg_runner_slab(const lbmg_runner* r, int* z0, int* z1) {
    return guarded([&] { R(r).slab(z0, z1); });
}

size_t lbmg_runner_totals_count(const lbmg_runner* r) {
    return r && r->impl ? r->impl->totals_log().size() : 0;
}

int lbmg_runner_totals(const lbmg_runner* r, double* out, size_t cap) {
    return guarded([&] {
        const auto& log = R(r).totals_log();
        for (size_t s = 0; s < log.size() && s < cap; ++s)
            for (int a = 0; a < 6; ++a) out[6 * s + a] = log[s][a];
    });
}

size_t lbmg_runner_sample_count(const lbmg_runner* r, int region, int solid) {
    try {
        return R(r).sample_count(region, solid);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    }
}

int lbmg_runner_samples(const lbmg_runner* r, int region, int solid, double* pos, double* ub, double* force,
                        double* sampled, uint32_t* src, uint8_t* flagged) {
    return guarded([&] { R(r).samples(region, solid, pos, ub, force, sampled, src, flagged); });
}

int lbmg_runner_set_cta(lbmg_runner* r, int threads) {
    return guarded([&] { R(r).set_cta(threads); });
}

int lbmg_runner_cta(const lbmg_runner* r) {
    try {
        return R(r).cta();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int lbmg_runner_cell_flags(const lbmg_runner* r, uint8_t* out) {
    return guarded([&] { R(r).cell_flags(out); });
}

// ---- tracers -------------------------------------------------------------

int lbmg_scene_set_emitters(lbmg_scene* s, int n, const lbmg_emitter* emitters) {
    return guarded([&] {
        if (!s) throw StateError("null scene");
        if (n < 0 || (n > 0 && !emitters)) throw lbmg::ConfigError("tracers: bad emitter list");
        for (int k = 0; k < n; ++k)  // scene.cpp:251-257: rate in [0, 1e6]
            if (emitters[k].rate < 0 || emitters[k].rate > 1000000)
                throw lbmg::ConfigError("$.tracers[" + std::to_string(k) + "].rate: out of range [0, 1000000]");
        s->emitters.assign(emitters, emitters + n);
    });
}

int lbmg_emit_tracers(int n, const lbmg_emitter* emitters, long step, uint64_t seed, double* positions) {
    return guarded([&] {
        if (n < 0 || (n > 0 && !emitters)) throw lbmg::ConfigError("tracers: bad emitter list");
        emit_positions(std::vector<lbmg_emitter>(emitters, emitters + n), step, seed, positions);
    });
}

size_t lbmg_runner_tracer_count(const lbmg_runner* r) {
    try {
        return R(r).tracer_count();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    }
}

int lbmg_runner_tracers(const lbmg_runner* r, double* positions, int64_t* birth_step) {
    return guarded([&] { R(r).tracers(positions, birth_step); });
}

int lbmg_runner_tracer_density(const lbmg_runner* r, double* vol) {
    return guarded([&] { R(r).tracer_density(vol); });
}

int lbmg_rasterize_density(size_t n, const double* positions, int nx, int ny, int nz, int device, double* vol) {
    return guarded([&] {
        if (nx < 2 || ny < 2 || nz < 2) throw lbmg::ConfigError("rasterize_density: every extent must be >= 2");
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        const size_t nn = size_t(nx) * ny * nz;
        double *dp = nullptr, *dv = nullptr;
        cuda_check(cudaMalloc(&dv, sizeof(double) * nn), "cudaMalloc(vol)");
        if (n && cudaMalloc(&dp, sizeof(double) * 3 * n) != cudaSuccess) {
            cudaFree(dv);
            throw OomError("rasterize_density: position upload allocation failed");
        }
        cuda_check(cudaMemset(dv, 0, sizeof(double) * nn), "cudaMemset");
        if (n) {
            cuda_check(cudaMemcpy(dp, positions, sizeof(double) * 3 * n, cudaMemcpyHostToDevice), "upload");
            launch_rasterize(dp, dp + 1, dp + 2, 3, nullptr, n, nx, ny, nz, dv, nullptr);
        }
        cuda_check(cudaMemcpy(vol, dv, sizeof(double) * nn, cudaMemcpyDeviceToHost), "download");
        cudaFree(dp);
        cudaFree(dv);
    });
}

int lbmg_runner_halo_f(lbmg_runner* r, int parity, void** sl, void** sh, void** rl, void** rh, size_t* b) {
    return guarded([&] { R(r).halo_f(parity, sl, sh, rl, rh, b); });
}

int lbmg_runner_halo_macro(lbmg_runner* r, void** sl, void** sh, void** rl, void** rh, size_t* b) {
    return guarded([&] { R(r).halo_macro(sl, sh, rl, rh, b); });
}

int lbmg_runner_phase(lbmg_runner* r, int phase, int write_macro) {
    return guarded([&] { R(r).phase(phase, write_macro); });
}

int lbmg_runner_sync(lbmg_runner* r, lbmg_status* status) {
    return guarded([&] { put_status(R(r).sync_external(), status); });
}

long lbmg_runner_sync_interval(const lbmg_runner* r) {
    return r && r->impl ? r->impl->chunk_cap() : 0;
}

long lbmg_runner_kernel_launches(const lbmg_runner* r) {
    return r && r->impl ? r->impl->kernel_launches() : 0;
}

long lbmg_runner_kernels_per_step(const lbmg_runner* r) {
    return r && r->impl ? r->impl->kernels_per_step_ : 0;
}

int lbmg_step(lbmg_runner* r, lbmg_status* status) {
    return guarded([&] { put_status(R(r).step_once(), status); });
}

int lbmg_runner_load_state(lbmg_runner* r, const double* f, const double* f_star, long t) {
    return guarded([&] {
        if (!f) throw lbmg::ConfigError("load_state: f is required");
        R(r).load_state(f, f_star, t);
    });
}

extern "C++" {
namespace {

// Device scratch for the IB free functions: every buffer on one stream,
// freed on scope exit; uploads/downloads complete before returning.
struct Scratch {
    cudaStream_t st = nullptr;
    std::vector<void*> bufs;
    explicit Scratch(int device) {
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    ~Scratch() {
        if (st) cudaStreamSynchronize(st);
        for (void* p : bufs) cudaFree(p);
        if (st) cudaStreamDestroy(st);
    }
    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        if (cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)) != cudaSuccess) {
            cudaGetLastError();
            throw OomError("IB free function: device allocation failed");
        }
        bufs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* up(const T* h, size_t count) {
        T* d = alloc<T>(count);
        if (count) cuda_check(cudaMemcpyAsync(d, h, sizeof(T) * count, cudaMemcpyHostToDevice, st), "upload");
        return d;
    }
    template <class T>
    void down(T* h, const T* d, size_t count) {
        if (count) cuda_check(cudaMemcpyAsync(h, d, sizeof(T) * count, cudaMemcpyDeviceToHost, st), "download");
    }
    void sync() {
        cuda_check(cudaGetLastError(), "IB free function launch");
        cuda_check(cudaStreamSynchronize(st), "IB free function");
    }
};

void check_grid(int nx, int ny, int nz) {
    if (nx < 2 || ny < 2 || nz < 2) throw lbmg::ConfigError("grid: every extent must be >= 2");
}

void check_slab(int nz, int z0, int z1) {
    if (z0 < 0 || z1 > nz || z0 >= z1) throw lbmg::ConfigError("slab: 0 <= z0 < z1 <= nz");
}

}  // namespace
}  // extern "C++"


int lbmg_ib_kernel_support(size_t n, const double* pos, int nx, int ny, int nz, int* base, double* w,
                           uint8_t* inside) {
    return guarded([&] {
        check_grid(nx, ny, nz);
        Scratch S(0);
        const double* dp = S.up(pos, 3 * n);
        int* db = S.alloc<int>(3 * n);
        double* dw = S.alloc<double>(6 * n);
        unsigned char* di = S.alloc<unsigned char>(n);
        launch_ib_support_batch(n, dp, nx, ny, nz, db, dw, di, S.st);
        if (base) S.down(base, db, 3 * n);
        if (w) S.down(w, dw, 6 * n);
        if (inside) S.down(inside, di, n);
        S.sync();
    });
}

int lbmg_ib_interpolate_velocity(size_t n, const double* pos, const double* u, int nx, int ny, int nz, int z0,
                                 int z1, double* sampled, uint8_t* flagged) {
    return guarded([&] {
        check_grid(nx, ny, nz);
        check_slab(nz, z0, z1);
        const size_t nodes = size_t(nx) * ny * nz;
        Scratch S(0);
        const double* dp = S.up(pos, 3 * n);
        const double* du = S.up(u, 3 * nodes);
        double* ds = S.alloc<double>(3 * n);
        unsigned char* df = S.alloc<unsigned char>(n);
        launch_ib_interp_batch(n, dp, du, nx, ny, nz, z0, z1, ds, df, S.st);
        S.down(sampled, ds, 3 * n);
        if (flagged) S.down(flagged, df, n);
        S.sync();
    });
}

int lbmg_ib_penalty_forces(size_t n, const double* pos, const double* boundary_velocity,
                           const double* sampled_velocity, const uint8_t* flagged, const double* rho, int nx, int ny,
                           int nz, int z0, int z1, double* penalty_force) {
    return guarded([&] {
        check_grid(nx, ny, nz);
        check_slab(nz, z0, z1);
        const size_t nodes = size_t(nx) * ny * nz;
        Scratch S(0);
        const double* dp = S.up(pos, 3 * n);
        const double* dub = S.up(boundary_velocity, 3 * n);
        const double* dsa = S.up(sampled_velocity, 3 * n);
        std::vector<unsigned char> zeros;
        if (!flagged) zeros.assign(n, 0);
        const unsigned char* dfl = S.up(flagged ? flagged : zeros.data(), n);
        const double* dr = S.up(rho, nodes);
        double* dfo = S.alloc<double>(3 * n);
        launch_ib_penalty_batch(n, dp, dub, dsa, dfl, dr, nx, ny, nz, z0, z1, dfo, S.st);
        S.down(penalty_force, dfo, 3 * n);
        S.sync();
    });
}

int lbmg_ib_spread_forces(size_t n, const double* pos, const double* penalty_force, const uint8_t* flagged, int nx,
                          int ny, int nz, int z0, int z1, double* g) {
    return guarded([&] {
        check_grid(nx, ny, nz);
        check_slab(nz, z0, z1);
        const size_t nodes = size_t(nx) * ny * nz;
        Scratch S(0);
        const double* dp = S.up(pos, 3 * n);
        const double* dfo = S.up(penalty_force, 3 * n);
        std::vector<unsigned char> zeros;
        if (!flagged) zeros.assign(n, 0);
        const unsigned char* dfl = S.up(flagged ? flagged : zeros.data(), n);
        double* dg = S.up(g, 3 * nodes);
        launch_ib_spread_batch(n, dp, dfo, dfl, nx, ny, nz, z0, z1, dg, S.st);
        S.down(g, dg, 3 * nodes);
        S.sync();
    });
}

int lbmg_ib_update_rigid_motion(size_t n, const double* reference_positions, const double* linear_velocity,
                                const double* angular_velocity, const double* center, long t, int nx, int ny, int nz,
                                double* pos, double* boundary_velocity, uint8_t* flagged) {
    return guarded([&] {
        check_grid(nx, ny, nz);
        // centre(t) and Rodrigues R(t) on the host with the reference's
        // expressions (ib.cpp:456-475, glibc cos/sin): bit-exact positions
        const V3 v{linear_velocity[0], linear_velocity[1], linear_velocity[2]};
        const V3 w{angular_velocity[0], angular_velocity[1], angular_velocity[2]};
        const V3 c0{center[0], center[1], center[2]};
        double row[kMotionRow];
        motion_table_row(v, w, c0, t, row);
        Scratch S(0);
        const double* dref = S.up(reference_positions, 3 * n);
        const double* drow = S.up(row, kMotionRow);
        double* dp = S.alloc<double>(3 * n);
        double* dub = S.alloc<double>(3 * n);
        unsigned char* dfl = S.alloc<unsigned char>(n);
        launch_ib_motion_batch(n, dref, drow, nx, ny, nz, dp, dub, dfl, S.st);
        S.down(pos, dp, 3 * n);
        S.down(boundary_velocity, dub, 3 * n);
        if (flagged) S.down(flagged, dfl, n);
        S.sync();
    });
}

int lbmg_ib_reaction_totals(size_t n, const double* pos, const double* penalty_force, const double* center, int z0,
                            int z1, double* force_torque) {
    return guarded([&] {
        Scratch S(0);
        const double* dp = S.up(pos, 3 * n);
        const double* dfo = S.up(penalty_force, 3 * n);
        double* partial = S.alloc<double>(6 * size_t(ib_totals_batch_blocks(n)));
        double* dout = S.alloc<double>(6);
        launch_ib_totals_batch(n, dp, dfo, center, z0, z1, partial, dout, S.st);
        S.down(force_torque, dout, 6);
        S.sync();
    });
}

int lbmg_collide_batch(const lbmg_scene_config* cfg, size_t n, const double* f, const double* rho,
                       const double* u, double* omega) {
    return guarded([&] {
        const auto rates = make_rates(*cfg);
        const auto& T = model_tables();
        ModelConst m{};
        m.kind = cfg->kind;
        m.policy = cfg->kind == LBMG_CENTRAL_MRT ? cfg->policy : LBMG_POLICY_CONSTANT;
        m.omega = float(1.0 / (3.0 * cfg->viscosity + 0.5));
        m.eps0 = float(cfg->policy_eps0);
        for (int mu = 0; mu < 27; ++mu) m.rate[mu] = float(rates[T.mu_to_row[mu]]);
        double *df = nullptr, *dr = nullptr, *du = nullptr, *dom = nullptr;
        auto cleanup = [&] {
            cudaFree(df);
            cudaFree(dr);
            cudaFree(du);
            cudaFree(dom);
        };
        try {
            cuda_check(cudaMalloc(&df, n * 27 * 8 + 8), "cudaMalloc");
            cuda_check(cudaMalloc(&dr, n * 8 + 8), "cudaMalloc");
            cuda_check(cudaMalloc(&du, n * 24 + 8), "cudaMalloc");
            cuda_check(cudaMalloc(&dom, n * 27 * 8 + 8), "cudaMalloc");
            cuda_check(cudaMemcpy(df, f, n * 27 * 8, cudaMemcpyHostToDevice), "H2D f");
            cuda_check(cudaMemcpy(dr, rho, n * 8, cudaMemcpyHostToDevice), "H2D rho");
            cuda_check(cudaMemcpy(du, u, n * 24, cudaMemcpyHostToDevice), "H2D u");
            launch_collide_batch(m, unsigned(n), df, dr, du, dom, nullptr);
            cuda_check(cudaGetLastError(), "collide_batch launch");
            cuda_check(cudaMemcpy(omega, dom, n * 27 * 8, cudaMemcpyDeviceToHost), "D2H omega");
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
