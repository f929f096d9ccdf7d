// Device-engine Runner: the GPU counterpart of lbm::Runner
// (runner.hpp:25-83 / runner.cpp).  Owns every device allocation; host-side
// results (status, step count, totals log) mirror the reference semantics.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"
#include "scene.hpp"
#include "tracers.hpp"

namespace lbmg {

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct OomError : std::runtime_error {
    explicit OomError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
    explicit StateError(const std::string& m) : std::runtime_error(m) {}
};

void cuda_check(cudaError_t e, const char* what);

struct Status {
    bool ok = true;
    bool mach_warning = false;
    long step = -1;
    std::string reason;
};

struct Timing {
    std::string phase;
    long step;
    double seconds;
};

struct Layout {
    size_t alpha_req = 1;  // API value (Runner::alpha)
    int la = 5;            // effective device group log2 (31 = SoA)
    bool soa = false;
};

class Runner {
public:
    // world/rank: rank mode (one slab of `world`, external halo exchange).
    // world == 0: in-process mode with `regions` slabs, on `device`, or —
    // when `devices` is given — region r on devices[r % devices.size()]
    // (peer access between neighbouring slabs' devices: the halo stores and
    // the IB seam reads go over NVLink; one stream per region, cross-device
    // events per step).
    Runner(const lbmg_scene& scene, int regions, int device, int world, int rank,
           const std::vector<int>& devices = {});
    ~Runner();
    Runner(const Runner&) = delete;
    Runner& operator=(const Runner&) = delete;

    std::unique_ptr<Runner> clone() const;

    Status advance(long steps, std::vector<Timing>* timings);
    // step(SimState&, ...) (solver.hpp:82-83): one single-region step without
    // solids, on the state load_state set (or the one advance left)
    Status step_once();
    // SimState of a single-region runner without solids (solver.hpp:29-45):
    // f(t) and the face-pass scratch f_star (its face entries seed the
    // persistent face slots the stale outflow reads use; nullptr: f) as
    // canonical AoS FP64, and the step counter t
    void load_state(const double* f, const double* f_star, long t);
    long step_count() const { return t_; }
    const Status& status() const { return status_; }
    int region_count() const { return int(regions_.size()); }
    int global_regions() const { return m_global_; }
    void set_layout(int ell, size_t alpha);
    // Kernel variants (the launch-split dimension of the tuner): fluid 0 =
    // TMA-staged kernel on the ghost layout (needs nx % 4 == 0), 1 =
    // register-direct kernels on the compact layout; ib 0 = fused single-region
    // IB kernel, 1 = mark / band / spread / totals pipeline.
    void set_variant(int fluid, int ib);
    long kernel_launches() const { return launches_; }
    int fluid_variant() const { return variant_fluid_; }
    // CTA size of the staged fluid kernel (512 / 256 / 128 threads = 1024 /
    // 512 / 256-slot tiles; 0 = LBMG_GHOST_THREADS or 512): results are
    // identical, only the tile period changes — the tuner's CTA-shape dimension
    void set_cta(int threads);
    int cta() const { return cta_; }
    int ib_variant() const { return variant_ib_; }
    // Eq. 10 cost of one candidate (autotune.cpp:29-36): set_layout, warm-up,
    // mean device seconds per step over n_steps (CUDA events around advance);
    // +inf when the run diverges.
    double measure_cost(int ell, size_t alpha, int warmup, int n_steps);
    // identity of the device layout alpha maps to (ghost, log2 block, block)
    unsigned long long layout_key(size_t alpha) const;
    size_t alpha() const { return layout_.alpha_req; }
    int block_edge() const { return ell_; }
    int nx() const { return nx_; }
    int ny() const { return ny_; }
    int nz() const { return nz_; }
    void slab(int* z0, int* z1) const;

    void gather(int what, double* out) const;  // 0 rho, 1 u, 2 f
    // Asynchronous rho*/u* snapshot (driver.cpp:45-59 without stalling the
    // step loop): device conversion + D2H into pinned memory on a copy
    // stream; the next advance only waits for it before rho/u are rewritten.
    void snapshot_begin();
    long snapshot_wait(double* rho, double* u);  // returns the snapshot's step
    const std::vector<std::array<double, 6>>& totals_log() const { return totals_; }
    size_t sample_count(int region, int solid) const;
    void samples(int region, int solid, double* pos, double* ub, double* force, double* sampled,
                 uint32_t* src, uint8_t* flagged) const;
    void cell_flags(uint8_t* out) const;
    // smoke tracers (Runner::tracers, runner.hpp:54; tracers.cu)
    size_t tracer_count() const { return size_t(tn_ - tdead_); }
    void tracers(double* pos, int64_t* birth) const;
    void tracer_density(double* vol) const;
    void set_stream(cudaStream_t s) { ext_stream_ = s; invalidate_graphs(); }
    int region_device(int r) const { return regions_.at(size_t(r)).dev; }
    bool multi_device() const { return multi_dev_; }
    cudaStream_t stream() const { return ext_stream_ ? ext_stream_ : stream_; }

    // rank mode
    void halo_f(int parity, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi, size_t* bytes);
    void halo_macro(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi, size_t* bytes);
    void phase(int ph, int write_macro);
    Status sync_external();
    long chunk_cap() const { return cap_; }

private:
    struct SolidDev {
        IbSolidDev d;
    };
    struct Region {
        int z0 = 0, z1 = 0;
        int dev = 0;                       // CUDA device of the slab
        cudaStream_t st = nullptr;         // its stream (multi-device mode)
        cudaEvent_t ev_fill = nullptr, ev_fluid = nullptr;
        bool has_lo = false, has_hi = false;
        RegionGeo geo{};
        RegionPtrs ptr{};
        FillRec* plan[2] = {nullptr, nullptr};  // per-step ghost fill programs (fill_ghosts_full)
        unsigned plan_cap = 0;
        unsigned plan_eoff = 0;
        unsigned* plan_count = nullptr;
        float* inlet_g = nullptr;
        unsigned* sband = nullptr;   // IB band path: sorted unique support-node slots of the static solids
        unsigned sband_n = 0;
        float* sband_m = nullptr;    // 4 floats per band node, written each step
        float* f[3] = {nullptr, nullptr, nullptr};
        float* recv_lo[2] = {nullptr, nullptr};
        float* recv_hi[2] = {nullptr, nullptr};
        float* own_send_lo[2] = {nullptr, nullptr};  // rank mode only
        float* own_send_hi[2] = {nullptr, nullptr};
        float* mrecv_lo = nullptr;
        float* mrecv_hi = nullptr;
        float* own_msend_lo = nullptr;
        float* own_msend_hi = nullptr;
        unsigned* stamp = nullptr;
        unsigned* band = nullptr;
        double* partial = nullptr;
        double* fused_partial = nullptr;  // fused IB: per-block totals
        IbSolidDev* batch_solids = nullptr;  // device copy of `solids` (the fused kernel's batch)
        unsigned* batch_start = nullptr;
        unsigned* batch_block_solid = nullptr;  // solid index per fused-IB block
        int* batch_moving = nullptr;
        unsigned batch_blocks = 0;
        std::vector<IbSolidDev> solids;
        FluidParams params() const;
    };

    void* dalloc(size_t bytes, bool zero = true, int dev = -1);
    cudaStream_t rst(const Region& r) const { return multi_dev_ ? r.st : stream(); }
    cudaStream_t dev_stream(int dev) const;
    void enqueue_step_multi(bool write_macro);
    cudaError_t copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) const;
    void dfree(void* p);
    void build_regions(int device);
    void compute_geo(Region& r) const;
    void alloc_f(Region& r);
    void link_halos();
    void init_fields();
    void upload_solids();
    void build_active_lists();
    void fill_motion_table(long t0, long rows, bool sync);
    void motion_row(int solid, long t, double* row) const;
    void enqueue_step(bool write_macro, std::vector<cudaEvent_t>* ev, bool publish = true);
    void enqueue_ib_pre();
    void enqueue_ib_mid();
    bool fused_ib() const;
    static bool overlap_off();
    void fill_ghosts_full();
    void build_fill_plan(Region& r);
    void refresh_active_pu();
    void set_ib_totals(FluidParams& P, int ri) const;
    void build_band_lists();
    bool band_path() const;
    void enqueue_fluid(bool write_macro, int part);
    void invalidate_graphs();
    void ensure_graphs();
    void finish_chunk(long t0, long requested);
    void copy_state_from(const Runner& o);
    void tracer_reserve(unsigned long long need);
    void tracer_prepare_chunk(long t0, long chunk);

    lbmg_scene scene_;
    int nx_ = 0, ny_ = 0, nz_ = 0;
    int m_global_ = 1;  // total slabs (regions, or world in rank mode)
    bool rank_mode_ = false;
    int rank_ = 0;
    int device_ = 0;
    int sm_count_ = 148;
    std::vector<Region> regions_;
    Layout layout_;
    int ell_ = 1;
    int variant_fluid_ = 0, variant_ib_ = 0;
    int cta_ = 0;
    FaceTable faces_{};
    ModelConst model_{};
    bool has_solids_ = false;
    std::vector<char> moving_;
    bool any_moving_ = false;
    bool no_write_value_ = false;  // stream write-value unavailable: chunk start by H2D copy
    bool motion_static_done_ = false;  // static solids: motion table uploaded once
    static constexpr size_t kCtrBytes = 256;  // DevCounters slot ahead of the totals
    size_t total_samples_ = 0;

    DevCounters* ctr_ = nullptr;
    double* motion_tab_ = nullptr;  // [cap+1][nsolid][kMotionRow]
    double* totals_dev_ = nullptr;  // [cap][regions][nsolid][6]
    long cap_ = 256;
    std::vector<void*> allocs_;

    cudaStream_t stream_ = nullptr;
    cudaStream_t ext_stream_ = nullptr;
    cudaStream_t side_ = nullptr;             // ghost fill concurrent with the fused IB kernel
    cudaEvent_t fork_ = nullptr, join_ = nullptr;
    bool ib_overlap_ok_ = false;
    double* pinned_up_ = nullptr;      // chunk_t0 + motion rows (host -> device)
    char* pinned_down_ = nullptr;      // counters + totals (device -> host)
    char* pinned_down_dev_ = nullptr;  // its device alias (mapped): the zero-copy results
    bool zc_steps_ = false;            // the step graphs publish the results zero-copy
    size_t pinned_down_bytes_ = 0;
    bool downloaded_ = false;
    // rho*/u* of the last advanced step are produced on demand: the step
    // graphs do not store them (16 B/node less on the last step of every
    // advance); macro_kernel recomputes them bit-identically from f(t) of
    // that step (still resident in its A/B buffer) when something reads them
    mutable bool macro_pending_ = false;
    long macro_t_ = 0;
    void ensure_macro() const;
    static bool lazy_macro();
    cudaStream_t copy_ = nullptr;
    cudaEvent_t snap_ready_ = nullptr, snap_done_ = nullptr;
    double* snap_dev_ = nullptr;   // rho (n) then u (3n), canonical order of this runner's slabs
    double* snap_host_ = nullptr;  // pinned
    bool snap_pending_ = false;
    long snap_step_ = 0;
    static constexpr int kMultiSteps = 8;
    cudaGraphExec_t graph_[3] = {nullptr, nullptr, nullptr};
    bool multi_dev_ = false;          // regions on their own streams (and devices)
    std::vector<int> devices_;        // as given to the constructor (clone)
    cudaEvent_t ev_step_ = nullptr;   // home stream: step inputs / previous step end
    long graph_kernels_[3] = {0, 0, 0};  // kernel nodes per graph launch
    long launches_ = 0;                  // engine kernels launched by advance()

    long t_ = 0;
    Status status_;
    std::vector<std::array<double, 6>> totals_;
    long ext_chunk_t0_ = 0;
    long t_ext_ = 0;  // rank mode: steps enqueued through phase(END)

    // tracers: cloud SoA in HBM with tombstones (tracers.cu)
    bool has_tracers_ = false;
    unsigned long long temit_ = 0;  // particles emitted per step
    unsigned long long tcap_ = 0, tn_ = 0, tdead_ = 0;
    TracerDev tdev_{};
    TracerRegion* treg_dev_ = nullptr;
    std::vector<TracerRegion> treg_host_;
    double* temit_dev_ = nullptr;             // [cap][E][3]
    double* pinned_temit_ = nullptr;          // same, host staging
    unsigned long long* pinned_tstate_ = nullptr;  // rank mode: start of the externally driven chunk

public:
    long kernels_per_step_ = 0;  // kernel nodes of the captured step graph
};

}  // namespace lbmg

struct lbmg_runner {
    std::unique_ptr<lbmg::Runner> impl;
};
