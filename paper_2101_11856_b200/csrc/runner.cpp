// Runner orchestration on the device (runner.cpp:22-319 of the reference,
// re-designed: one fused kernel per region per step, device-side step
// counter, CUDA-graph replay, in-process or NCCL-driven halo exchange).
#include "runner.hpp"

#include <cuda.h>  // driver types only: cuStreamWriteValue64 is fetched at run time (no libcuda link)

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <type_traits>
#include <string>

namespace lbmg {

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw OomError(std::string(what) + ": " + cudaGetErrorString(e));
    }
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(x) cuda_check((x), #x)

namespace {

unsigned round_up(unsigned n, unsigned a) { return (n + a - 1) / a * a; }

// A 64-bit value written into device memory in stream order by the stream's
// front end (cuStreamWriteValue64): no copy-engine transfer for the 8-byte
// chunk start of every advance() call.  Falls back to a pinned H2D copy when
// the driver entry point or 64-bit stream memory operations are unavailable.
using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WriteValue64Fn write_value64() {
    static const WriteValue64Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return WriteValue64Fn(nullptr);
        }
        return reinterpret_cast<WriteValue64Fn>(p);
    }();
    return fn;
}

size_t next_pow2(size_t v) {
    size_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

int log2i(size_t v) {
    int s = 0;
    while ((size_t(1) << s) < v) ++s;
    return s;
}

// Current-device guard: regions may live on different devices.
struct DevGuard {
    int prev = -1, want;
    explicit DevGuard(int d) : want(d) {
        cudaGetDevice(&prev);
        if (prev != want) cuda_check(cudaSetDevice(want), "cudaSetDevice");
    }
    ~DevGuard() {
        if (prev >= 0 && prev != want) cudaSetDevice(prev);
    }
};

// equilibrium, collision.cpp:148-157 (FP64, reference operation order).
double feq(int i, double rho, const double u[3]) {
    const double usq = 1.5 * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    const double cu = cx(i) * u[0] + cy(i) * u[1] + cz(i) * u[2];
    return weight_d(i) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - usq);
}

}  // namespace

// Every host-side copy of the runner goes through its own (non-blocking)
// stream and completes before returning: a plain cudaMemcpy runs on the
// legacy default stream, which non-blocking streams do not wait for, and a
// device-to-device (or pageable host-to-device) cudaMemcpy may return before
// the data has landed.
cudaError_t Runner::copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) const {
    int dev = device_;
    if (multi_dev_) {  // the stream of the device that holds the device side
        cudaPointerAttributes a{};
        const void* dside = kind == cudaMemcpyHostToDevice ? dst : src;
        if (cudaPointerGetAttributes(&a, dside) == cudaSuccess && a.type == cudaMemoryTypeDevice) dev = a.device;
        cudaGetLastError();
    }
    DevGuard g(dev);
    cudaStream_t st = dev_stream(dev);
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
}

cudaStream_t Runner::dev_stream(int dev) const {
    if (dev == device_ || !multi_dev_) return stream();
    for (const auto& r : regions_)
        if (r.dev == dev && r.st) return r.st;
    return stream();
}

FluidParams Runner::Region::params() const { return FluidParams{geo, {}, {}, ptr, nullptr}; }

void* Runner::dalloc(size_t bytes, bool zero, int dev) {
    if (bytes == 0) bytes = 16;
    if (dev < 0) dev = device_;
    DevGuard g(dev);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw OomError("device allocation of " + std::to_string(bytes) + " bytes failed: " +
                       cudaGetErrorString(e));
    }
    if (zero) {  // on the runner's stream (non-blocking streams skip the legacy one), complete on return
        cudaStream_t zs = dev_stream(dev);
        CK(cudaMemsetAsync(p, 0, bytes, zs));
        CK(cudaStreamSynchronize(zs));
    }
    allocs_.push_back(p);
    return p;
}

void Runner::dfree(void* p) {
    if (!p) return;
    auto it = std::find(allocs_.begin(), allocs_.end(), p);
    if (it != allocs_.end()) allocs_.erase(it);
    cudaFree(p);
}

Runner::Runner(const lbmg_scene& scene, int regions, int device, int world, int rank,
               const std::vector<int>& devices) {
    scene_ = scene;
    scene_.cfg.solids = scene_.solid_cfgs.empty() ? nullptr : scene_.solid_cfgs.data();
    scene_.cfg.n_solids = int(scene_.solid_cfgs.size());
    const lbmg_scene_config& c = scene_.cfg;
    validate_config(c);
    nx_ = c.nx;
    ny_ = c.ny;
    nz_ = c.nz;
    if (int64_t(nx_) * ny_ * nz_ >= (int64_t(1) << 31) && world == 0 && regions == 1)
        throw ConfigError("grid: a single slab must hold fewer than 2^31 nodes; use more regions");
    rank_mode_ = world > 0;
    m_global_ = rank_mode_ ? world : regions;
    rank_ = rank_mode_ ? rank : 0;
    if (m_global_ < 1 || m_global_ > nz_)
        throw ConfigError("decomp: region count must satisfy 1 <= m <= nz (got m=" +
                          std::to_string(m_global_) + ", nz=" + std::to_string(nz_) + ")");
    if (rank_mode_ && (rank < 0 || rank >= world)) throw ConfigError("rank out of range");
    const auto slabs = split_domain(nz_, m_global_);
    // runner.cpp:32-37: z outflow reads one plane into the slab interior
    for (int f = 4; f < 6; ++f)
        if (c.faces[f].condition == LBMG_OUTFLOW && m_global_ > 1)
            for (const auto& s : slabs)
                if (s[1] - s[0] < 2) throw ConfigError("decomp: z outflow needs slabs at least 2 planes thick");

    const auto rates = make_rates(c);
    const auto& T = model_tables();
    model_.kind = c.kind;
    // only cm-mrt carries the rate policy (scene.cpp:33-37: raw_mrt/bgk are Constant)
    model_.policy = c.kind == LBMG_CENTRAL_MRT ? c.policy : LBMG_POLICY_CONSTANT;
    model_.omega = float(1.0 / (3.0 * c.viscosity + 0.5));
    model_.eps0 = float(c.policy_eps0);
    for (int mu = 0; mu < 27; ++mu) model_.rate[mu] = float(rates[T.mu_to_row[mu]]);
    for (int a = 0; a < 3; ++a) model_.body[a] = float(c.body_force[a]);
    for (int f = 0; f < 6; ++f) {
        faces_.cond[f] = c.faces[f].condition;
        for (int i = 0; i < 27; ++i)
            faces_.inlet[f][i] = float(feq(i, 1.0, c.faces[f].velocity) - weight_d(i));
    }
    has_solids_ = !scene_.solids.empty();
    for (const auto& s : scene_.solids) {
        moving_.push_back(s.moving ? 1 : 0);
        any_moving_ = any_moving_ || s.moving;
        total_samples_ += s.samples.size();
    }
    ell_ = c.block_edge;
    layout_.alpha_req = c.alpha;
    // The fused IB kernel reads f* of its support nodes as plain pulls; if no
    // support node can lie on a domain face, none of those pulls touches a
    // ghost slot and the ghost fill may run concurrently with the IB kernel.
    // Static solids: their sample positions; moving ones: the sphere of their
    // largest reference radius around a fixed centre (no linear motion).
    ib_overlap_ok_ = has_solids_;
    for (const auto& s : scene_.solids) {
        V3 lo{1e300, 1e300, 1e300}, hi{-1e300, -1e300, -1e300};
        if (s.moving) {
            if (dot(s.linear_velocity, s.linear_velocity) != 0.0) ib_overlap_ok_ = false;
            double r2 = 0.0;
            for (const auto& q : s.samples.reference_positions) r2 = std::max(r2, dot(q, q));
            const double r = std::sqrt(r2) + 1e-6;
            lo = s.center + V3{-r, -r, -r};
            hi = s.center + V3{r, r, r};
        } else {
            for (const auto& q : s.samples.positions)
                for (int a = 0; a < 3; ++a) {
                    lo[a] = std::min(lo[a], q[a]);
                    hi[a] = std::max(hi[a], q[a]);
                }
        }
        const int n[3] = {nx_, ny_, nz_};
        for (int a = 0; a < 3; ++a)  // support nodes floor(p) .. floor(p)+1 strictly inside
            if (!(std::floor(lo[a]) >= 1.0 && std::floor(hi[a]) + 1.0 <= double(n[a] - 2))) ib_overlap_ok_ = false;
    }

    device_ = device;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming));

    const int first = rank_mode_ ? rank_ : 0;
    const int count = rank_mode_ ? 1 : m_global_;
    regions_.resize(count);
    devices_ = devices;
    if (!devices.empty()) {
        if (rank_mode_) throw ConfigError("devices: rank mode places its one slab with `device`");
        if (!scene_.emitters.empty())
            throw ConfigError("tracers: emitters need a single-stream runner (no per-region devices)");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        for (int d : devices)
            if (d < 0 || d >= ndev) throw ConfigError("devices: no CUDA device " + std::to_string(d));
        if (!scene_.solids.empty() && !(nx_ % 4 == 0 && ghost_layout_enabled()))
            throw ConfigError("devices: solids on several devices need the ghost layout (nx % 4 == 0)");
        multi_dev_ = true;
        device_ = devices[0];
        CK(cudaSetDevice(device_));
    }
    for (int r = 0; r < count; ++r) {
        Region& R = regions_[r];
        R.dev = multi_dev_ ? devices[size_t(r) % devices.size()] : device_;
        if (multi_dev_) {
            DevGuard g(R.dev);
            CK(cudaStreamCreateWithFlags(&R.st, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&R.ev_fill, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&R.ev_fluid, cudaEventDisableTiming));
        }
    }
    if (multi_dev_) {
        CK(cudaEventCreateWithFlags(&ev_step_, cudaEventDisableTiming));
        // peer access: neighbouring slabs (halo stores, IB seam reads) and
        // every slab with the home device (step counters, motion and totals)
        auto peer = [](int a, int b) {
            if (a == b) return;
            int ok = 0;
            CK(cudaDeviceCanAccessPeer(&ok, a, b));
            if (!ok)
                throw ConfigError("devices: no peer access between devices " + std::to_string(a) + " and " +
                                  std::to_string(b));
            DevGuard g(a);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else CK(e);
        };
        for (int r = 0; r < count; ++r) {
            const int lo = r > 0 ? r - 1 : count - 1, hi = r + 1 < count ? r + 1 : 0;
            for (int q : {lo, hi}) {
                peer(regions_[r].dev, regions_[q].dev);
                peer(regions_[q].dev, regions_[r].dev);
            }
            peer(regions_[r].dev, device_);
            peer(device_, regions_[r].dev);
        }
    }
    for (int r = 0; r < count; ++r) {
        regions_[r].z0 = slabs[first + r][0];
        regions_[r].z1 = slabs[first + r][1];
        const int g = first + r;
        regions_[r].has_lo = g > 0 || c.faces[4].condition == LBMG_PERIODIC;
        regions_[r].has_hi = g + 1 < m_global_ || c.faces[4].condition == LBMG_PERIODIC;
    }
    build_regions(device);
    link_halos();
    // counters and the chunk's reaction totals share one allocation (totals at
    // kCtrBytes) so a chunk's results come back in one D2H copy
    static_assert(sizeof(DevCounters) <= kCtrBytes, "DevCounters outgrew its slot");
    const size_t tot_bytes = has_solids_ ? sizeof(double) * cap_ * regions_.size() * scene_.solids.size() * 6 : 0;
    char* ctr_block = static_cast<char*>(dalloc(kCtrBytes + tot_bytes));
    ctr_ = reinterpret_cast<DevCounters*>(ctr_block);
    if (has_solids_) {
        const size_t ns = scene_.solids.size();
        motion_tab_ = static_cast<double*>(dalloc(sizeof(double) * (cap_ + 2) * ns * kMotionRow));
        totals_dev_ = reinterpret_cast<double*>(ctr_block + kCtrBytes);
    }
    {
        const size_t ns = scene_.solids.size();
        CK(cudaMallocHost(&pinned_up_, sizeof(double) * (1 + (cap_ + 2) * std::max<size_t>(ns, 1) * kMotionRow)));
        pinned_down_bytes_ = kCtrBytes + sizeof(double) * cap_ * regions_.size() * std::max<size_t>(ns, 1) * 6;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&pinned_down_), pinned_down_bytes_,
                         cudaHostAllocMapped | cudaHostAllocPortable));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&pinned_down_dev_), pinned_down_, 0));
    }
    upload_solids();
    init_fields();
    if (rank_mode_ && has_solids_) fill_motion_table(0, cap_ + 1, true);
    for (const auto& e : scene_.emitters) {
        if (e.rate < 0) throw ConfigError("tracers: rate must be >= 0");
        temit_ += (unsigned long long)e.rate;
    }
    has_tracers_ = !scene_.emitters.empty();
    if (has_tracers_ && rank_mode_)
        throw ConfigError("tracers: emitters need an in-process runner (rank mode samples one slab only)");
    if (has_tracers_) {
        treg_dev_ = static_cast<TracerRegion*>(dalloc(sizeof(TracerRegion) * regions_.size()));
        tdev_.state = static_cast<unsigned long long*>(dalloc(2 * sizeof(unsigned long long)));
        temit_dev_ = static_cast<double*>(dalloc(sizeof(double) * 3 * std::max<unsigned long long>(temit_, 1) * cap_, false));
        CK(cudaMallocHost(&pinned_temit_, sizeof(double) * 3 * std::max<unsigned long long>(temit_, 1) * cap_));
        CK(cudaMallocHost(&pinned_tstate_, 2 * sizeof(unsigned long long)));
        tdev_.emit = temit_dev_;
        tdev_.E = temit_;
        tdev_.reg = treg_dev_;
        tdev_.m = int(regions_.size());
        tdev_.nx = nx_;
        tdev_.ny = ny_;
        tdev_.nz = nz_;
        tracer_reserve(4096);
    }
    CK(cudaStreamSynchronize(stream_));
}

Runner::~Runner() {
    invalidate_graphs();
    if (snap_pending_ && snap_done_) cudaEventSynchronize(snap_done_);
    if (snap_host_) cudaFreeHost(snap_host_);
    if (copy_) cudaStreamDestroy(copy_);
    if (snap_ready_) cudaEventDestroy(snap_ready_);
    if (snap_done_) cudaEventDestroy(snap_done_);
    if (pinned_up_) cudaFreeHost(pinned_up_);
    if (pinned_down_) cudaFreeHost(pinned_down_);  // (cudaHostAlloc)
    if (pinned_temit_) cudaFreeHost(pinned_temit_);
    if (pinned_tstate_) cudaFreeHost(pinned_tstate_);
    for (auto& r : regions_) {
        if (r.st) cudaStreamSynchronize(r.st);
    }
    for (void* p : allocs_) cudaFree(p);
    allocs_.clear();
    for (auto& r : regions_) {
        if (r.st) cudaStreamDestroy(r.st);
        if (r.ev_fill) cudaEventDestroy(r.ev_fill);
        if (r.ev_fluid) cudaEventDestroy(r.ev_fluid);
    }
    if (ev_step_) cudaEventDestroy(ev_step_);
    if (stream_) cudaStreamDestroy(stream_);
    if (side_) cudaStreamDestroy(side_);
    if (fork_) cudaEventDestroy(fork_);
    if (join_) cudaEventDestroy(join_);
}

void Runner::invalidate_graphs() {
    for (auto& g : graph_)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
}

void Runner::compute_geo(Region& r) const {
    RegionGeo& g = r.geo;
    g.cta = cta_;
    g.nx = nx_;
    g.ny = ny_;
    g.nzl = r.z1 - r.z0;
    g.NZ = nz_;
    g.gz0 = r.z0;
    for (int a = 0; a < 3; ++a) g.per[a] = scene_.cfg.faces[2 * a].condition == LBMG_PERIODIC;
    g.plane = unsigned(nx_) * unsigned(ny_);
    g.n = g.plane * unsigned(g.nzl);
    g.ns = round_up(g.n, 32);
    // alpha below one warp (incl. the reference default 1 = AoS) has no
    // coalesced device equivalent: store SoA, the alpha -> infinity limit of
    // Eq. 9 (results are layout-invariant bit for bit, tests/test_gpu_parity.py)
    const size_t a = next_pow2(std::max<size_t>(layout_.alpha_req, 32));
    if (layout_.alpha_req < 32 || a >= g.n) {  // SoA: one group of n_pad nodes
        g.la = 31;
        g.amask = 0x7fffffffu;
        g.n_pad = round_up(g.n, 32);
        g.A = g.n_pad;
    } else {
        g.la = log2i(a);
        g.amask = unsigned(a - 1);
        g.n_pad = round_up(g.n, unsigned(a));
        g.A = unsigned(a);
    }
    g.div_nx = FastDiv(unsigned(nx_));
    g.div_ny = FastDiv(unsigned(ny_));
    g.ghost = 0;
    g.nbuf = 2;
    if (nx_ % 4 == 0 && ghost_layout_enabled() && variant_fluid_ == 0) {
        // ghost-layer layout (device_common.cuh): pitch nx+4, ny+1 rows,
        // planes -1..nzl, CSoA blocks of alpha >= 256 slots (one staged tile
        // writes one contiguous 27 KB block); alpha >= slots is SoA
        g.ghost = 1;
        g.PX = unsigned(nx_) + 4u;
        g.PY = unsigned(ny_) + 1u;
        g.PP = g.PX * g.PY;
        g.zwrap = g.per[2] && regions_.size() == 1 && !rank_mode_;
        g.has_outflow = 0;
        for (int f = 0; f < 6; ++f)
            if (scene_.cfg.faces[f].condition == LBMG_OUTFLOW) g.has_outflow = 1;
        g.div_px = FastDiv(g.PX);
        g.div_py = FastDiv(g.PY);
        // a tile (<= 1024 slots, aligned down from the first owned plane) reads
        // windows reaching off_max + 3 = PP + PX + 4 slots below its first slot
        // and kWin - 1 - off_min above its last one
        g.base = round_up(g.PX + 1040u, 256u);
        unsigned slots = round_up(g.base + unsigned(g.nzl + 2) * g.PP + g.PX + 2080u, 256u);
        size_t areq = layout_.alpha_req;
        if (const char* e = std::getenv("LBMG_GHOST_ALPHA")) areq = std::strtoull(e, nullptr, 10);  // layout probes
        // alpha below one 256-slot tile (incl. the reference default 1) has no
        // device benefit: SoA; otherwise Eq. 9 blocks of next_pow2(alpha)
        const size_t ga = next_pow2(std::max<size_t>(areq, 256));
        if (areq < 256 || ga >= slots) {
            g.la = 31;
            g.amask = 0x7fffffffu;
            g.n_pad = slots;
            g.A = slots;
        } else {
            g.la = log2i(ga);
            g.amask = unsigned(ga - 1);
            g.n_pad = round_up(slots, unsigned(ga));
            g.A = unsigned(ga);
        }
    }
}

void Runner::alloc_f(Region& r) {
    for (int p = 0; p < r.geo.nbuf; ++p) {
        r.f[p] = static_cast<float*>(dalloc(sizeof(float) * f_alloc_floats(r.geo), false, r.dev));
        r.ptr.f[p] = r.f[p];
    }
}

void Runner::build_regions(int) {
    for (auto& r : regions_) {
        compute_geo(r);
        RegionGeo& g = r.geo;
        alloc_f(r);
        r.ptr.queue = static_cast<unsigned*>(dalloc(sizeof(unsigned) * 8, true, r.dev));
        r.ptr.rho = static_cast<float*>(dalloc(sizeof(float) * g.ns, true, r.dev));
        r.ptr.u = static_cast<float*>(dalloc(sizeof(float) * 3ull * g.ns, true, r.dev));
        if (has_solids_) {
            r.ptr.gib = static_cast<float*>(dalloc(sizeof(float) * 3ull * g.ns, true, r.dev));
            r.ptr.tflag = static_cast<unsigned char*>(dalloc(g.ns + 64, true, r.dev));
            {  // per 64-slot chunk of the ghost layout (upper bound of its slot count, any alpha)
                const size_t px = size_t(nx_) + 4, pp = px * (size_t(ny_) + 1);
                const size_t slots = px + 1040 + 256 + size_t(g.nzl + 2) * pp + px + 2080 + 256;
                r.ptr.cflag = static_cast<unsigned char*>(dalloc((slots >> 6) + 64, true, r.dev));
            }
            r.stamp = static_cast<unsigned*>(dalloc(sizeof(unsigned) * g.ns, true, r.dev));
            const size_t cap = std::max<size_t>(1, std::min<size_t>(g.n, 8 * total_samples_));
            r.band = static_cast<unsigned*>(dalloc(sizeof(unsigned) * cap, true, r.dev));
            r.ptr.band_count = static_cast<unsigned*>(dalloc(sizeof(unsigned), true, r.dev));
            r.partial = static_cast<double*>(dalloc(sizeof(double) * 6 * 256, true, r.dev));
            size_t blocks = 1;
            for (const auto& so : scene_.solids) blocks += size_t(std::max(1, fused_blocks(so.samples.size())));
            r.fused_partial = static_cast<double*>(dalloc(sizeof(double) * 6 * blocks, true, r.dev));
        }
        for (int f = 0; f < 6; ++f) {
            const int a = face_axis(f);
            bool present = scene_.cfg.faces[f].condition != LBMG_PERIODIC;
            if (a == 2) present = present && ((f == 4 && r.z0 == 0) || (f == 5 && r.z1 == nz_));
            for (int p = 0; p < 2; ++p)
                r.ptr.slot[p][f] =
                    present ? static_cast<float*>(dalloc(sizeof(float) * 9ull * g.slot_plane(f), true, r.dev)) : nullptr;
        }
        const size_t hb = sizeof(float) * 9ull * g.plane;
        for (int p = 0; p < 2; ++p) {
            if (r.has_lo) r.recv_lo[p] = static_cast<float*>(dalloc(hb, true, r.dev));
            if (r.has_hi) r.recv_hi[p] = static_cast<float*>(dalloc(hb, true, r.dev));
            r.ptr.recv_lo[p] = r.recv_lo[p];
            r.ptr.recv_hi[p] = r.recv_hi[p];
            if (rank_mode_) {
                if (r.has_lo) r.own_send_lo[p] = static_cast<float*>(dalloc(hb, true, r.dev));
                if (r.has_hi) r.own_send_hi[p] = static_cast<float*>(dalloc(hb, true, r.dev));
            }
        }
        if (has_solids_) {
            const size_t mb = sizeof(float) * 4ull * g.plane;
            if (r.has_lo) r.mrecv_lo = static_cast<float*>(dalloc(mb, true, r.dev));
            if (r.has_hi) r.mrecv_hi = static_cast<float*>(dalloc(mb, true, r.dev));
            if (rank_mode_) {
                if (r.has_lo) r.own_msend_lo = static_cast<float*>(dalloc(mb, true, r.dev));
                if (r.has_hi) r.own_msend_hi = static_cast<float*>(dalloc(mb, true, r.dev));
            }
            r.ptr.mrecv_lo = r.mrecv_lo;
            r.ptr.mrecv_hi = r.mrecv_hi;
        }
    }
}

// In-process: a region's outgoing halo IS the neighbour's incoming buffer
// (region r's send_hi == region r+1's recv_lo; periodic z wraps, a single
// periodic slab feeds itself).  Rank mode: own send buffers, moved by NCCL.
void Runner::link_halos() {
    const int m = int(regions_.size());
    for (int r = 0; r < m; ++r) {
        Region& R = regions_[r];
        if (rank_mode_) {
            for (int p = 0; p < 2; ++p) {
                R.ptr.send_lo[p] = R.own_send_lo[p];
                R.ptr.send_hi[p] = R.own_send_hi[p];
            }
            R.ptr.msend_lo = R.own_msend_lo;
            R.ptr.msend_hi = R.own_msend_hi;
            continue;
        }
        const int lo = r > 0 ? r - 1 : m - 1;
        const int hi = r + 1 < m ? r + 1 : 0;
        for (int p = 0; p < 2; ++p) {
            R.ptr.send_lo[p] = R.has_lo ? regions_[lo].recv_hi[p] : nullptr;
            R.ptr.send_hi[p] = R.has_hi ? regions_[hi].recv_lo[p] : nullptr;
        }
        R.ptr.msend_lo = R.has_lo && has_solids_ ? regions_[lo].mrecv_hi : nullptr;
        R.ptr.msend_hi = R.has_hi && has_solids_ ? regions_[hi].mrecv_lo : nullptr;
    }
}

void Runner::upload_solids() {
    for (auto& r : regions_) {
        r.solids.clear();
        for (const auto& s : scene_.solids) {
            IbSolidDev d{};
            const size_t n = s.samples.size();
            d.n = unsigned(n);
            d.pos = static_cast<double*>(dalloc(sizeof(double) * 3 * n, true, r.dev));
            d.ref = static_cast<double*>(dalloc(sizeof(double) * 3 * n, true, r.dev));
            d.ub = static_cast<double*>(dalloc(sizeof(double) * 3 * n, true, r.dev));
            d.force = static_cast<double*>(dalloc(sizeof(double) * 3 * kIbHalves * n, true, r.dev));  // parts (ib_half)
            d.sampled = static_cast<double*>(dalloc(sizeof(double) * 3 * kIbHalves * n, true, r.dev));
            d.nbuf = r.geo.nbuf;
            d.source = static_cast<unsigned*>(dalloc(sizeof(unsigned) * n, true, r.dev));
            d.flagged = static_cast<unsigned char*>(dalloc(n, true, r.dev));
            if (scene_.cfg.ib_mode == LBMG_IB_DETERMINISTIC && n) {
                d.rec_key = static_cast<unsigned*>(dalloc(sizeof(unsigned) * 8 * n, true, r.dev));
                d.rec_idx = static_cast<unsigned*>(dalloc(sizeof(unsigned) * 8 * n, true, r.dev));
                d.key_sorted = static_cast<unsigned*>(dalloc(sizeof(unsigned) * 8 * n, true, r.dev));
                d.idx_sorted = static_cast<unsigned*>(dalloc(sizeof(unsigned) * 8 * n, true, r.dev));
                d.rec_val = static_cast<double*>(dalloc(sizeof(double) * 24 * n, true, r.dev));
                d.sort_temp_bytes = ib_det_temp_bytes(unsigned(n));
                d.sort_temp = dalloc(d.sort_temp_bytes, true, r.dev);
            }
            std::vector<double> pos(3 * n), ref(3 * n);
            for (size_t k = 0; k < n; ++k)
                for (int a = 0; a < 3; ++a) {
                    pos[3 * k + a] = s.samples.positions[k][a];
                    ref[3 * k + a] = s.samples.reference_positions[k][a];
                }
            if (n) {
                CK(copy_sync(d.pos, pos.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
                CK(copy_sync(d.ref, ref.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
                CK(copy_sync(d.source, s.samples.source_id.data(), sizeof(unsigned) * n,
                              cudaMemcpyHostToDevice));
            }
            r.solids.push_back(d);
        }
        const size_t ns = r.solids.size();
        if (ns) {
            std::vector<int> mv(ns);
            for (size_t k = 0; k < ns; ++k) mv[k] = moving_[k] ? 1 : 0;
            r.batch_solids = static_cast<IbSolidDev*>(dalloc(sizeof(IbSolidDev) * ns, true, r.dev));
            r.batch_start = static_cast<unsigned*>(dalloc(sizeof(unsigned) * (ns + 1), true, r.dev));
            r.batch_moving = static_cast<int*>(dalloc(sizeof(int) * ns, true, r.dev));
            CK(copy_sync(r.batch_moving, mv.data(), sizeof(int) * ns, cudaMemcpyHostToDevice));
        }
    }
    build_active_lists();
}

// The fused IB kernel's batch of each region (every solid in one launch):
// a static solid runs over the samples whose support lies inside the grid
// and touches the region's slab (kernel_support / sample_active,
// ib.cpp:294-317: fixed for a static set, so the slabs partition the work
// instead of every region replaying every sample); a moving one, and every
// solid in deterministic mode (its records are indexed by sample), over all.
// The inactive samples' outputs stay zero, as the reference writes them.
void Runner::build_active_lists() {
    if (!has_solids_) return;
    const bool det = scene_.cfg.ib_mode == LBMG_IB_DETERMINISTIC;
    for (auto& r : regions_) {
        const size_t ns = r.solids.size();
        std::vector<unsigned> start(ns + 1, 0);
        for (size_t k = 0; k < ns; ++k) {
            IbSolidDev& d = r.solids[k];
            if (d.active) {
                dfree(d.active);
                d.active = nullptr;
            }
            if (d.act_pu) {
                dfree(d.act_pu);
                d.act_pu = nullptr;
            }
            if (d.corner_band) {
                dfree(d.corner_band);
                d.corner_band = nullptr;
            }
            d.n_active = 0;
            if (!moving_[k] && !det && d.n) {
                std::vector<double> pos(3 * size_t(d.n));
                CK(copy_sync(pos.data(), d.pos, sizeof(double) * pos.size(), cudaMemcpyDeviceToHost));
                std::vector<unsigned> act;
                const int n3[3] = {nx_, ny_, nz_};
                for (unsigned q = 0; q < d.n; ++q) {
                    bool inside = true;
                    for (int a = 0; a < 3; ++a)
                        if (pos[3 * q + a] < 0.0 || pos[3 * q + a] > double(n3[a] - 1)) inside = false;
                    const int bz = std::max(0, std::min(int(std::floor(pos[3 * q + 2])), nz_ - 2));
                    if (inside && bz + 1 >= r.z0 && bz < r.z1) act.push_back(q);
                }
                d.active = static_cast<unsigned*>(dalloc(sizeof(unsigned) * std::max<size_t>(act.size(), 1), false, r.dev));
                if (!act.empty())
                    CK(copy_sync(d.active, act.data(), sizeof(unsigned) * act.size(), cudaMemcpyHostToDevice));
                d.n_active = unsigned(act.size());
                d.act_pu = static_cast<double*>(dalloc(sizeof(double) * 6 * std::max<size_t>(act.size(), 1), false, r.dev));
            }
            // (at least one block: it writes the solid's totals row of the region)
            start[k + 1] = start[k] + unsigned(std::max(1, fused_blocks(d.active ? d.n_active : d.n)));
        }
        if (ns) {
            CK(copy_sync(r.batch_solids, r.solids.data(), sizeof(IbSolidDev) * ns, cudaMemcpyHostToDevice));
            CK(copy_sync(r.batch_start, start.data(), sizeof(unsigned) * (ns + 1), cudaMemcpyHostToDevice));
            std::vector<unsigned> bs(std::max<unsigned>(start[ns], 1u), 0u);
            for (size_t k = 0; k < ns; ++k)
                for (unsigned b = start[k]; b < start[k + 1]; ++b) bs[b] = unsigned(k);
            if (r.batch_block_solid) dfree(r.batch_block_solid);
            r.batch_block_solid = static_cast<unsigned*>(dalloc(sizeof(unsigned) * bs.size(), false, r.dev));
            CK(copy_sync(r.batch_block_solid, bs.data(), sizeof(unsigned) * bs.size(), cudaMemcpyHostToDevice));
        }
        r.batch_blocks = start[ns];
    }
    refresh_active_pu();
}

// (pos, u_b) of the static solids' active samples in run order (the fused
// kernel's copy); after every change of the static positions (init's
// update_rigid_motion(0), a re-sort), same buffers so captured graphs stay valid.
void Runner::refresh_active_pu() {
    for (auto& r : regions_)
        for (auto& d : r.solids) {
            if (!d.act_pu || !d.active || !d.n_active) continue;
            std::vector<double> pos(3 * size_t(d.n)), ub(3 * size_t(d.n)), pu(6 * size_t(d.n_active));
            std::vector<unsigned> act(d.n_active);
            CK(copy_sync(pos.data(), d.pos, sizeof(double) * pos.size(), cudaMemcpyDeviceToHost));
            CK(copy_sync(ub.data(), d.ub, sizeof(double) * ub.size(), cudaMemcpyDeviceToHost));
            CK(copy_sync(act.data(), d.active, sizeof(unsigned) * act.size(), cudaMemcpyDeviceToHost));
            for (size_t j = 0; j < act.size(); ++j)
                for (int a = 0; a < 3; ++a) {
                    pu[6 * j + a] = pos[3 * size_t(act[j]) + a];
                    pu[6 * j + 3 + a] = ub[3 * size_t(act[j]) + a];
                }
            CK(copy_sync(d.act_pu, pu.data(), sizeof(double) * pu.size(), cudaMemcpyHostToDevice));
        }
    build_band_lists();
}

// Band path of the fused IB kernel: one region, atomic mode, static solids
// with at least kBandMin active samples in total (LBMG_IB_BAND=1 / 0 forces
// it on / off).  Below that the per-corner gathers of the fused kernel are
// cheaper than an extra launch on the step's critical path.
bool Runner::band_path() const {
    static const int env = [] {
        const char* e = std::getenv("LBMG_IB_BAND");
        return e ? std::atoi(e) : -1;
    }();
    constexpr size_t kBandMin = 65536;
    if (env == 0 || regions_.size() != 1 || multi_dev_ || rank_mode_ || !has_solids_ ||
        scene_.cfg.ib_mode == LBMG_IB_DETERMINISTIC || !regions_[0].geo.ghost)
        return false;
    size_t n = 0;
    for (const auto& d : regions_[0].solids)
        if (d.act_pu) n += d.n_active;
    return n > 0 && (env == 1 || n >= kBandMin);
}

void Runner::build_band_lists() {
    for (auto& r : regions_) {
        if (r.sband) {
            dfree(r.sband);
            dfree(r.sband_m);
            r.sband = nullptr;
            r.sband_m = nullptr;
            r.sband_n = 0;
        }
        for (auto& d : r.solids)
            if (d.corner_band) {
                dfree(d.corner_band);
                d.corner_band = nullptr;
            }
    }
    if (!band_path()) return;
    Region& r = regions_[0];
    DevGuard dg(r.dev);
    size_t total = 0;
    for (auto& d : r.solids)
        if (d.act_pu && d.n_active) {
            d.corner_band = static_cast<unsigned*>(dalloc(sizeof(unsigned) * 8 * size_t(d.n_active), false, r.dev));
            total += 8 * size_t(d.n_active);
        }
    unsigned* band = static_cast<unsigned*>(dalloc(sizeof(unsigned) * std::max<size_t>(total, 1), false, r.dev));
    FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
    const unsigned n = build_ib_band(P, r.solids.data(), r.solids.size(), band, rst(r));
    r.sband = band;
    r.sband_n = n;
    r.sband_m = static_cast<float*>(dalloc(sizeof(float) * 4 * std::max<size_t>(n, 1), false, r.dev));
    if (r.batch_solids)
        CK(copy_sync(r.batch_solids, r.solids.data(), sizeof(IbSolidDev) * r.solids.size(), cudaMemcpyHostToDevice));
}

// Rigid motion row at step t (ib.cpp:456-475): centre(t) and Rodrigues R(t)
// computed on the host with the reference's expressions (glibc cos/sin).
void Runner::motion_row(int solid, long t, double* row) const {
    const SolidInstance& s = scene_.solids[solid];
    motion_table_row(s.linear_velocity, s.angular_velocity, s.center, t, row);
}

// Motion rows of steps t0 .. t0+rows-1, solid-major ([solid][step][row]: the
// kernels index (t - chunk_t0) * kMotionRow within a per-solid view), staged
// in pinned memory and uploaded asynchronously on the runner's stream (the
// caller synchronises once per advance chunk, after the step graphs).
void Runner::fill_motion_table(long t0, long rows, bool sync) {
    const size_t ns = scene_.solids.size();
    double* tab = pinned_up_ + 1;
    for (size_t s = 0; s < ns; ++s)
        for (long j = 0; j < rows; ++j) motion_row(int(s), t0 + j, &tab[(s * (cap_ + 2) + j) * kMotionRow]);
    // one strided copy for every solid's rows
    const size_t pitch = sizeof(double) * size_t(cap_ + 2) * kMotionRow;
    CK(cudaMemcpy2DAsync(motion_tab_, pitch, tab, pitch, sizeof(double) * size_t(rows) * kMotionRow, ns,
                         cudaMemcpyHostToDevice, stream()));
    if (sync) CK(cudaStreamSynchronize(stream()));
}

void Runner::init_fields() {
    const lbmg_scene_config& c = scene_.cfg;
    InitParams ip{};
    ip.kind = c.init;
    ip.rho0 = c.init_density;
    for (int a = 0; a < 3; ++a) ip.u0[a] = c.init_velocity[a];
    ip.tg_u = c.tg_u_max;
    ip.NX = nx_;
    ip.NY = ny_;
    for (auto& r : regions_) {
        DevGuard dg(r.dev);
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        launch_init(P, ip, rst(r));
        CK(cudaStreamSynchronize(rst(r)));  // (init writes the neighbours' halo inputs)
    }
    fill_ghosts_full();
    CK(cudaGetLastError());
    // update_rigid_motion(t=0) for every solid (runner.cpp:104-106)
    if (has_solids_) {
        double* row = static_cast<double*>(dalloc(sizeof(double) * kMotionRow));
        for (size_t s = 0; s < scene_.solids.size(); ++s) {
            double h[kMotionRow];
            motion_row(int(s), 0, h);
            CK(copy_sync(row, h, sizeof h, cudaMemcpyHostToDevice));
            for (auto& r : regions_) {
                DevGuard dg(r.dev);
                launch_ib_motion_once(r.solids[s], row, nx_, ny_, nz_, rst(r));
                CK(cudaStreamSynchronize(rst(r)));
            }
        }
        dfree(row);
        refresh_active_pu();
    }
    CK(cudaStreamSynchronize(stream()));
}

void Runner::enqueue_ib_pre() {
    cudaStream_t st = stream();
    for (auto& r : regions_) CK(cudaMemsetAsync(r.ptr.band_count, 0, sizeof(unsigned), st));
    for (auto& r : regions_) {
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        for (auto& s : r.solids) launch_ib_mark(P, s, r.stamp, r.band, st);
    }
    for (auto& r : regions_) {
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        launch_ib_band(P, r.band, sm_count_, st);
    }
    if (m_global_ > 1)
        for (auto& r : regions_) {
            FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
            launch_macro_pack(P, st);
        }
}

void Runner::enqueue_ib_mid() {
    cudaStream_t st = stream();
    const int ns = int(scene_.solids.size());
    const int m = int(regions_.size());
    for (auto& r : regions_) {
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        for (auto& s : r.solids) launch_ib_spread(P, s, st, scene_.cfg.ib_mode == LBMG_IB_DETERMINISTIC);
    }
    for (int ri = 0; ri < m; ++ri) {
        Region& r = regions_[ri];
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        for (int s = 0; s < ns; ++s)
            launch_ib_totals(P, r.solids[s], motion_tab_ + size_t(s) * (cap_ + 2) * kMotionRow, r.partial,
                             totals_dev_ + size_t(ri * ns + s) * 6, m * ns * 6, st);
    }
    for (auto& r : regions_)
        for (int s = 0; s < ns; ++s)
            if (moving_[s])
                launch_ib_motion(ctr_, r.solids[s], motion_tab_ + size_t(s) * (cap_ + 2) * kMotionRow, nx_, ny_,
                                 nz_, st);
}

// part: 0 all planes, 1 boundary planes only, 2 interior planes only.
void Runner::enqueue_fluid(bool write_macro, int part) {
    cudaStream_t st = stream();
    for (auto& r : regions_) {
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        launch_fluid(P, part, write_macro, st);
    }
}

// Every ghost slot of the current step's input buffer (the fluid kernel only
// pushes the next step's values; state set up outside the step loop needs
// all of them).
void Runner::fill_ghosts_full() {
    for (auto& r : regions_)
        if (r.geo.ghost) {
            DevGuard dg(r.dev);
            FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
            launch_ghost_fill(P, rst(r), true);
            if (multi_dev_) CK(cudaStreamSynchronize(r.st));
            build_fill_plan(r);
        }
}

// The per-step ghost fill of each step parity as a copy program: resolved
// once here (geometry, layout and buffers are fixed until the next full
// fill), replayed by ghost_copy_kernel every step (LBMG_FILL_PLAN=0: the
// general per-entry kernel, for A/B).
void Runner::build_fill_plan(Region& r) {
    static const bool off = [] {
        const char* e = std::getenv("LBMG_FILL_PLAN");
        return e && std::string(e) == "0";
    }();
    r.ptr.fill_plan[0] = r.ptr.fill_plan[1] = nullptr;
    r.ptr.fill_n[0] = r.ptr.fill_n[1] = r.ptr.fill_runs[0] = r.ptr.fill_runs[1] = 0;
    if (off || !r.geo.ghost || r.geo.nbuf != 2) return;
    DevGuard dg(r.dev);
    cudaStream_t st = rst(r);
    if (!r.inlet_g) {
        r.inlet_g = static_cast<float*>(dalloc(sizeof(float) * 6 * 27, false, r.dev));
        CK(cudaMemcpyAsync(r.inlet_g, &faces_.inlet[0][0], sizeof(float) * 6 * 27, cudaMemcpyHostToDevice, st));
        r.plan_count = static_cast<unsigned*>(dalloc(2 * sizeof(unsigned), true, r.dev));
    }
    r.ptr.inlet_g = r.inlet_g;
    FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
    {  // counts first: how many rows form runs depends on the layout (Eq. 9 block edges)
        unsigned c[2][2];
        for (int p = 0; p < 2; ++p) launch_fill_plan(P, p, nullptr, 0, r.plan_count, c[p], st);
        const unsigned eoff = std::max(c[0][0], c[1][0]), cap = eoff + std::max(c[0][1], c[1][1]);
        if (!r.plan[0] || cap > r.plan_cap) {  // (callers re-capture their step graphs after a full fill)
            for (int p = 0; p < 2; ++p) {
                if (r.plan[p]) dfree(r.plan[p]);
                r.plan[p] = static_cast<FillRec*>(dalloc(sizeof(FillRec) * std::max(cap, 1u), false, r.dev));
            }
            r.plan_cap = cap;
        }
        r.plan_eoff = eoff;
    }
    unsigned c[2][2];
    for (int p = 0; p < 2; ++p) {
        launch_fill_plan(P, p, r.plan[p], r.plan_eoff, r.plan_count, c[p], st);
        if (c[p][0] > r.plan_eoff || r.plan_eoff + c[p][1] > r.plan_cap)
            throw std::runtime_error("fill plan: record count changed between passes");
    }
    for (int p = 0; p < 2; ++p) {
        r.ptr.fill_plan[p] = r.plan[p];
        r.ptr.fill_runs[p] = c[p][0];
        r.ptr.fill_n[p] = c[p][1];
    }
    r.ptr.fill_eoff = r.plan_eoff;
}

// The fused IB kernel leaves per-block partials; the region's fluid kernel
// of the same step sums them into the totals row (RegionPtrs::ib_partial).
void Runner::set_ib_totals(FluidParams& P, int ri) const {
    if (!fused_ib()) return;
    const Region& r = regions_[size_t(ri)];
    const int ns = int(scene_.solids.size()), m = int(regions_.size());
    P.p.ib_partial = r.fused_partial;
    P.p.ib_start = r.batch_start;
    P.p.ib_solids = unsigned(ns);
    P.p.ib_out = totals_dev_ + size_t(ri) * ns * 6;
    P.p.ib_stride = m * ns * 6;
}

bool Runner::overlap_off() {
    static const bool off = [] {
        const char* e = std::getenv("LBMG_IB_OVERLAP");
        return e && std::string(e) == "0";
    }();
    return off;
}

// In-process regions on the ghost layout: the ghost fills first, then one
// fused IB kernel per region (every solid; support nodes across a seam are
// read from the neighbour slab's buffers on the same device), then the fluid
// kernels.  Rank mode (one slab per process) keeps the split pipeline and its
// macro halo.
bool Runner::fused_ib() const {
    static const bool off = [] {
        const char* e = std::getenv("LBMG_IB_FUSED");
        return e && std::string(e) == "0";
    }();
    if (!has_solids_ || off || variant_ib_ != 0 || rank_mode_) return false;
    for (const auto& r : regions_)
        if (!r.geo.ghost) return false;
    return true;
}

// One step on the runner's stream.  Timing events (advance with timings):
// [0] boundary = ghost fill (the six face passes, wraps, halos) [1] ib [2]
// fluid = the fused stream/moments/collision kernel [3] step end [4].
// One step with every region on its own stream (and device): the home stream
// orders the step (chunk inputs, then step_end after every region's fluid
// kernel); each region waits for it, fills its ghost slots, waits for its
// neighbours' fills (its IB reads their f* across the seams), runs the fused
// IB and the fluid kernel, whose boundary planes store straight into the
// neighbours' halo buffers (peer memory).
void Runner::enqueue_step_multi(bool write_macro) {
    cudaStream_t hs = stream();
    const int m = int(regions_.size());
    {
        DevGuard dg(device_);
        CK(cudaEventRecord(ev_step_, hs));
    }
    for (auto& r : regions_) {
        DevGuard dg(r.dev);
        CK(cudaStreamWaitEvent(r.st, ev_step_, 0));
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        if (r.geo.ghost) launch_ghost_fill(P, r.st);
        CK(cudaEventRecord(r.ev_fill, r.st));
    }
    if (has_solids_) {
        const int ns = int(scene_.solids.size());
        auto slab = [&](const Region& q) {
            IbSlab sl{};
            sl.g = q.geo;
            for (int b = 0; b < 3; ++b) sl.f[b] = q.ptr.f[b];
            return sl;
        };
        for (int ri = 0; ri < m; ++ri) {
            Region& r = regions_[ri];
            DevGuard dg(r.dev);
            if (ri > 0) CK(cudaStreamWaitEvent(r.st, regions_[ri - 1].ev_fill, 0));
            if (ri + 1 < m) CK(cudaStreamWaitEvent(r.st, regions_[ri + 1].ev_fill, 0));
            FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
            IbBatch B{};
            B.own = slab(r);
            B.lo = ri > 0 ? slab(regions_[ri - 1]) : B.own;
            B.hi = ri + 1 < m ? slab(regions_[ri + 1]) : B.own;
            B.solids = r.batch_solids;
            B.block_start = r.batch_start;
            B.block_solid = r.batch_block_solid;
            B.moving = r.batch_moving;
            B.n_solids = unsigned(ns);
            if (ns == 1) B.solo = r.solids[0];
            B.table = motion_tab_;
            B.table_stride = size_t(cap_ + 2) * kMotionRow;
            B.partial = r.fused_partial;
            launch_ib_fused(P, B, r.batch_blocks, r.solids.data(), r.st,
                            scene_.cfg.ib_mode == LBMG_IB_DETERMINISTIC);
        }
    }
    for (auto& r : regions_) {
        DevGuard dg(r.dev);
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        set_ib_totals(P, int(&r - regions_.data()));
        launch_fluid(P, 0, write_macro, r.st, false, false);
        CK(cudaEventRecord(r.ev_fluid, r.st));
    }
    DevGuard dg(device_);
    for (auto& r : regions_) CK(cudaStreamWaitEvent(hs, r.ev_fluid, 0));
    launch_step_end(ctr_, hs);
}

void Runner::enqueue_step(bool write_macro, std::vector<cudaEvent_t>* ev, bool publish) {
    if (multi_dev_) {
        enqueue_step_multi(write_macro);
        return;
    }
    cudaStream_t st = stream();
    write_macro = write_macro || has_tracers_;  // the tracers sample u* of every step
    if (ev) CK(cudaEventRecord((*ev)[0], st));
    // ghost fill || fused IB when no IB support node can touch a ghost slot
    // (a fork/join inside the captured graph); timed runs keep them serial
    // (the band path's moments kernel reads the filled f*: fill, band moments, IB in order)
    const bool band = fused_ib() && regions_[0].sband_n > 0;
    const bool overlap = !ev && fused_ib() && regions_.size() == 1 && ib_overlap_ok_ && !overlap_off() && !band;
    // ... and with a fill program in atomic mode, both in ONE launch (the
    // fill records as extra blocks of the IB kernel: no fork/join, one launch
    // gap less; LBMG_IB_MERGE=0 keeps the fork/join)
    static const bool merge_off = [] {
        const char* e = std::getenv("LBMG_IB_MERGE");
        return e && std::string(e) == "0";
    }();
    const bool merged = overlap && !merge_off && scene_.cfg.ib_mode != LBMG_IB_DETERMINISTIC &&
                        regions_[0].ptr.fill_plan[0] != nullptr;
    cudaStream_t fst = st;
    if (overlap && !merged) {
        CK(cudaEventRecord(fork_, st));
        CK(cudaStreamWaitEvent(side_, fork_, 0));
        fst = side_;
    }
    for (auto& r : regions_)
        if (r.geo.ghost && !merged) {
            FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
            launch_ghost_fill(P, fst);
        }
    if (overlap && !merged) CK(cudaEventRecord(join_, side_));
    if (ev) CK(cudaEventRecord((*ev)[1], st));
    if (fused_ib()) {
        const int ns = int(scene_.solids.size()), m = int(regions_.size());
        auto slab = [&](const Region& q) {
            IbSlab sl{};
            sl.g = q.geo;
            for (int b = 0; b < 3; ++b) sl.f[b] = q.ptr.f[b];
            return sl;
        };
        for (int ri = 0; ri < m; ++ri) {
            Region& r = regions_[ri];
            FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
            IbBatch B{};
            B.own = slab(r);
            B.lo = ri > 0 ? slab(regions_[ri - 1]) : B.own;  // (support never wraps: kernel_support clamps)
            B.hi = ri + 1 < m ? slab(regions_[ri + 1]) : B.own;
            B.solids = r.batch_solids;
            B.block_start = r.batch_start;
            B.block_solid = r.batch_block_solid;
            B.moving = r.batch_moving;
            B.n_solids = unsigned(ns);
            if (ns == 1) B.solo = r.solids[0];
            B.table = motion_tab_;
            B.table_stride = size_t(cap_ + 2) * kMotionRow;
            B.partial = r.fused_partial;
            if (band) {
                launch_ib_band_moments(P, r.sband, r.sband_n, r.sband_m, st);
                B.band_m = r.sband_m;
            }
            if (merged) launch_ib_fused_fill(P, B, r.batch_blocks, st);
            else launch_ib_fused(P, B, r.batch_blocks, r.solids.data(), st, scene_.cfg.ib_mode == LBMG_IB_DETERMINISTIC);
        }
    } else if (has_solids_) {
        enqueue_ib_pre();
        enqueue_ib_mid();
    }
    if (overlap && !merged) CK(cudaStreamWaitEvent(st, join_, 0));
    if (ev) CK(cudaEventRecord((*ev)[2], st));
    bool ended = false;
    for (auto& r : regions_) {
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        set_ib_totals(P, int(&r - regions_.data()));
        // one region whose fluid kernel ends the step: results zero-copy
        const bool zc = regions_.size() == 1 && !has_tracers_ && (!has_solids_ || fused_ib());
        if (zc) {
            // the counters only from the last step of an advance (a kernel that
            // writes host memory last waits for that write before it completes);
            // the totals rows every step (written early in the kernel)
            if (publish) P.p.ctr_host = reinterpret_cast<DevCounters*>(pinned_down_dev_);
            if (P.p.ib_out) P.p.ib_out_host = reinterpret_cast<double*>(pinned_down_dev_ + kCtrBytes);
        }
        ended = launch_fluid(P, 0, write_macro, st, false, regions_.size() == 1 && !has_tracers_);
        zc_steps_ = zc && ended;
    }
    if (ev) CK(cudaEventRecord((*ev)[3], st));
    // emit + advect after collision, before the step counter moves (runner.cpp:213-223)
    if (has_tracers_) launch_tracer_step(tdev_, ctr_, sm_count_, st);
    if (!ended) launch_step_end(ctr_, st);
    if (ev) CK(cudaEventRecord((*ev)[4], st));
}

// Step graphs: [0] one step, [1] the last step of an advance (writes
// rho*/u*), [2] kMultiSteps steps (fewer graph launches and inter-graph gaps).
// All three are captured and instantiated together on first use.
void Runner::ensure_graphs() {
    cudaStream_t st = stream();
    for (int which = 0; which < 3; ++which) {
        cudaGraphExec_t& g = graph_[which];
        if (g) continue;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        const int n = which == 2 ? kMultiSteps : 1;
        // [1] = the last step of an advance: publishes the counters, stores
        // rho*/u* unless they are produced on demand
        for (int q = 0; q < n; ++q) enqueue_step(which == 1 && !lazy_macro(), nullptr, which == 1);
        CK(cudaStreamEndCapture(st, &graph));
        size_t nn = 0;
        CK(cudaGraphGetNodes(graph, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
        long kernels = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty == cudaGraphNodeTypeKernel) ++kernels;
        }
        if (which == 0) kernels_per_step_ = kernels;
        graph_kernels_[which] = kernels;
        CK(cudaGraphInstantiate(&g, graph, 0));
        CK(cudaGraphDestroy(graph));
        // upload now: the first launch of a fresh executable graph pays it otherwise
        CK(cudaGraphUpload(g, st));
    }
}

bool Runner::lazy_macro() {
    static const bool on = [] {
        const char* e = std::getenv("LBMG_LAZY_MACRO");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// The moments-phase rho*, u* of step macro_t_ from f(macro_t_) (the A/B
// buffer the step read, the ghost slots and face slots it used): the same
// values the fluid kernel computed in that step, bit for bit (scalar and
// packed moments are identical per node).
void Runner::ensure_macro() const {
    if (!macro_pending_) return;
    macro_pending_ = false;
    for (const auto& r : regions_) {
        DevGuard dg(r.dev);
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        launch_macro(P, macro_t_, rst(r));
        CK(cudaStreamSynchronize(rst(r)));
    }
}

Status Runner::advance(long steps, std::vector<Timing>* timings) {
    if (!status_.ok || steps <= 0) return status_;
    cudaStream_t st = stream();
    CK(cudaSetDevice(device_));
    // the step graphs' last step stores rho*/u* unless they are produced on demand
    const bool lazy = lazy_macro() && !has_tracers_ && !multi_dev_ && !timings;
    macro_pending_ = false;  // superseded: readers see this advance's last step
    long done = 0;
    while (done < steps) {
        const long chunk = std::min(cap_, steps - done);
        const long t0 = t_;
        // an in-flight snapshot reads rho/u: the split IB pipeline rewrites
        // them at band nodes every step, the fluid kernel on the last step
        // (on every step when tracers sample u*)
        if (snap_pending_ && (has_tracers_ || (has_solids_ && !fused_ib())))
            CK(cudaStreamWaitEvent(st, snap_done_, 0));
        // inputs of the chunk (pinned, async, ordered before the step graphs)
        // static solids: every row is the same, the table is uploaded once
        if (has_solids_ && (any_moving_ || !motion_static_done_)) {
            fill_motion_table(t0, any_moving_ ? chunk + 1 : cap_ + 1, false);
            motion_static_done_ = true;
        }
        if (has_tracers_) tracer_prepare_chunk(t0, chunk);
        *reinterpret_cast<long long*>(pinned_up_) = t0;
        bool written = false;
        if (!no_write_value_) {
            if (auto wv = write_value64())
                written = wv(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(&ctr_->chunk_t0),
                             cuuint64_t(t0), 0) == CUDA_SUCCESS;
            if (!written) no_write_value_ = true;
        }
        if (!written)
            CK(cudaMemcpyAsync(&ctr_->chunk_t0, pinned_up_, sizeof(long long), cudaMemcpyHostToDevice, st));
        std::vector<std::array<cudaEvent_t, 5>> evs;
        // every step graph is captured and instantiated before the first one
        // runs, so no later advance() pays a capture inside its own time
        if (!timings && !multi_dev_) ensure_graphs();
        for (long j = 0; j < chunk;) {
            const bool last = done + j == steps - 1;
            if (last && snap_pending_) CK(cudaStreamWaitEvent(st, snap_done_, 0));
            if (multi_dev_) {  // eager launches: the step spans several streams and devices
                enqueue_step_multi(last);
                launches_ += long(regions_.size()) * (has_solids_ ? 3 : 2) + 1;
                ++j;
            } else if (timings) {
                std::vector<cudaEvent_t> e(5);
                for (auto& x : e) CK(cudaEventCreate(&x));
                enqueue_step(last, &e);
                launches_ += kernels_per_step_;
                evs.push_back({e[0], e[1], e[2], e[3], e[4]});
                ++j;
            } else if (!last && j + kMultiSteps < chunk && done + j + kMultiSteps < steps) {
                CK(cudaGraphLaunch(graph_[2], st));
                launches_ += graph_kernels_[2];
                j += kMultiSteps;
            } else {
                // the last step of every chunk publishes the counters its
                // results are read from (zero-copy); [2] never ends a chunk
                const int which = last || j == chunk - 1 ? 1 : 0;
                CK(cudaGraphLaunch(graph_[which], st));
                launches_ += graph_kernels_[which];
                ++j;
            }
        }
        // results of the chunk (counters + reaction totals), one sync
        const size_t tot_now = has_solids_ ? sizeof(double) * size_t(chunk) * regions_.size() * scene_.solids.size() * 6 : 0;
        // (graph steps whose fluid kernel published them zero-copy need no copy)
        if (!(zc_steps_ && !timings && !multi_dev_))
            CK(cudaMemcpyAsync(pinned_down_, ctr_, (has_solids_ ? kCtrBytes : sizeof(DevCounters)) + tot_now,
                               cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaGetLastError());
        downloaded_ = true;
        if (timings) {
            for (size_t j = 0; j < evs.size(); ++j) {
                float seg[4] = {0, 0, 0, 0};
                for (int q = 0; q < 4; ++q) CK(cudaEventElapsedTime(&seg[q], evs[j][q], evs[j][q + 1]));
                const long step = t0 + long(j);
                if (seg[0] > 0.f) timings->push_back({"boundary", step, seg[0] * 1e-3});
                if (has_solids_) timings->push_back({"ib", step, seg[1] * 1e-3});
                timings->push_back({"fluid", step, seg[2] * 1e-3});
                if (has_tracers_) timings->push_back({"tracers", step, seg[3] * 1e-3});
                timings->push_back({"total", step, (seg[0] + seg[1] + seg[2] + seg[3]) * 1e-3});
                for (auto x : evs[j]) cudaEventDestroy(x);
            }
        }
        finish_chunk(t0, chunk);
        if (!status_.ok) break;
        done += chunk;
    }
    if (lazy && status_.ok && t_ > 0) {
        macro_pending_ = true;
        macro_t_ = t_ - 1;
    }
    return status_;
}

void Runner::finish_chunk(long t0, long) {
    // advance() downloads counters + totals asynchronously with its final
    // sync; other callers (rank mode) read them here
    const bool pre = downloaded_;
    downloaded_ = false;
    DevCounters h{};
    if (pre) std::memcpy(&h, pinned_down_, sizeof h);
    else CK(copy_sync(&h, ctr_, sizeof h, cudaMemcpyDeviceToHost));
    const long completed = long(h.t) - t0;
    if (has_solids_ && completed > 0) {
        const size_t ns = scene_.solids.size(), m = regions_.size();
        std::vector<double> tot(size_t(completed) * m * ns * 6);
        if (pre) std::memcpy(tot.data(), pinned_down_ + kCtrBytes, sizeof(double) * tot.size());
        else CK(copy_sync(tot.data(), totals_dev_, sizeof(double) * tot.size(), cudaMemcpyDeviceToHost));
        for (long j = 0; j < completed; ++j) {
            std::array<double, 6> sum{};
            for (size_t r = 0; r < m; ++r)
                for (size_t s = 0; s < ns; ++s)
                    for (int a = 0; a < 6; ++a) sum[a] += tot[((size_t(j) * m + r) * ns + s) * 6 + a];
            totals_.push_back(sum);
        }
    }
    if (has_tracers_ && completed > 0) {
        tn_ += temit_ * (unsigned long long)completed;
        unsigned long long ts[2];
        CK(copy_sync(ts, tdev_.state, sizeof ts, cudaMemcpyDeviceToHost));
        tdead_ = ts[1];
    }
    t_ = long(h.t);
    if (h.mach) status_.mach_warning = true;
    if (h.diverged && status_.ok) {
        status_.ok = false;
        status_.step = long(h.t);  // the counter stops at the diverging step (both paths)
        status_.reason = "divergence: non-positive or non-finite density";
        // rho*/u* of the diverging step from f(t) (solver.cpp:113-122)
        for (auto& r : regions_) {
            DevGuard dg(r.dev);
            FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
            launch_macro(P, t_, rst(r));
            CK(cudaStreamSynchronize(rst(r)));
        }
        // the reference returns before update_rigid_motion(t+1)
        if (has_solids_) {
            double* row = static_cast<double*>(dalloc(sizeof(double) * kMotionRow));
            for (size_t s = 0; s < scene_.solids.size(); ++s) {
                if (!moving_[s]) continue;
                double hrow[kMotionRow];
                motion_row(int(s), t_, hrow);
                CK(copy_sync(row, hrow, sizeof hrow, cudaMemcpyHostToDevice));
                for (auto& r : regions_) {
                    DevGuard dg(r.dev);
                    launch_ib_motion_once(r.solids[s], row, nx_, ny_, nz_, rst(r));
                    CK(cudaStreamSynchronize(rst(r)));
                }
            }
            dfree(row);
        }
        CK(cudaStreamSynchronize(stream()));
    }
}

Status Runner::step_once() {
    if (regions_.size() != 1 || rank_mode_ || has_solids_)
        throw StateError("step(): a single region without solids (solver.hpp:82-83; the Runner orchestrates the rest)");
    return advance(1, nullptr);
}

void Runner::load_state(const double* f, const double* f_star, long t) {
    ensure_macro();
    if (regions_.size() != 1 || rank_mode_ || has_solids_ || has_tracers_)
        throw StateError("load_state: a single in-process region without solids or tracers");
    if (t < 0) throw ConfigError("load_state: the step counter must be >= 0");
    CK(cudaSetDevice(device_));
    Region& r = regions_[0];
    DevGuard dg(r.dev);
    const size_t bytes = sizeof(double) * 27 * size_t(r.geo.n);
    double* d = static_cast<double*>(dalloc(bytes, false, r.dev));
    try {
        DevCounters h{};
        h.t = t;
        CK(copy_sync(ctr_, &h, sizeof h, cudaMemcpyHostToDevice));
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        CK(copy_sync(d, f_star ? f_star : f, bytes, cudaMemcpyHostToDevice));
        for (int p = 0; p < 2; ++p) launch_write_slots(P, p, d, rst(r));
        CK(cudaStreamSynchronize(rst(r)));
        CK(copy_sync(d, f, bytes, cudaMemcpyHostToDevice));
        launch_write_f(P, fcur(r.geo, t), int(t & 1), d, rst(r));
        CK(cudaStreamSynchronize(rst(r)));
    } catch (...) {
        dfree(d);
        throw;
    }
    dfree(d);
    t_ = t;
    status_ = Status{};
    totals_.clear();
    fill_ghosts_full();
    CK(cudaStreamSynchronize(stream()));
    CK(cudaGetLastError());
}

void Runner::slab(int* z0, int* z1) const {
    *z0 = regions_.front().z0;
    *z1 = regions_.back().z1;
}

void Runner::gather(int what, double* out) const {
    if (what != 2) ensure_macro();
    const size_t beta = what == 0 ? 1 : (what == 1 ? 3 : 27);
    const unsigned chunk = 1u << 20;
    const size_t base_plane = size_t(regions_.front().z0) * regions_.front().geo.plane;
    for (const auto& r : regions_) {
        DevGuard dg(r.dev);
        cudaStream_t st = rst(r);
        double* stage = nullptr;
        CK(cudaMalloc(&stage, sizeof(double) * beta * chunk));
        try {
            FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
            const size_t off = size_t(r.z0) * r.geo.plane - base_plane;
            for (unsigned k0 = 0; k0 < r.geo.n; k0 += chunk) {
                const unsigned k1 = std::min(r.geo.n, k0 + chunk);
                if (what == 2) launch_read_f(P, fcur(r.geo, t_), k0, k1, stage, st);
                else launch_read_macro(P, k0, k1, what == 0 ? stage : nullptr, what == 1 ? stage : nullptr, st);
                CK(cudaGetLastError());
                CK(cudaMemcpyAsync(out + (off + k0) * beta, stage, sizeof(double) * beta * (k1 - k0),
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
            }
        } catch (...) {
            cudaFree(stage);
            throw;
        }
        cudaFree(stage);
    }
}

void Runner::snapshot_begin() {
    ensure_macro();
    CK(cudaSetDevice(device_));
    if (snap_pending_) CK(cudaEventSynchronize(snap_done_));
    size_t n = 0;
    for (const auto& r : regions_) n += r.geo.n;
    if (multi_dev_) {  // slabs on several devices: a synchronous gather into pinned memory
        if (!snap_host_) {
            CK(cudaMallocHost(&snap_host_, sizeof(double) * 4 * n));
            CK(cudaEventCreateWithFlags(&snap_done_, cudaEventDisableTiming));
        }
        for (auto& r : regions_) CK(cudaStreamSynchronize(r.st));
        gather(0, snap_host_);
        gather(1, snap_host_ + n);
        CK(cudaEventRecord(snap_done_, stream()));
        snap_pending_ = true;
        snap_step_ = t_;
        return;
    }
    if (!snap_dev_) {
        snap_dev_ = static_cast<double*>(dalloc(sizeof(double) * 4 * n, false));
        CK(cudaMallocHost(&snap_host_, sizeof(double) * 4 * n));
        CK(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&snap_ready_, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&snap_done_, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(snap_ready_, stream()));
    CK(cudaStreamWaitEvent(copy_, snap_ready_, 0));
    const size_t base_plane = size_t(regions_.front().z0) * regions_.front().geo.plane;
    for (const auto& r : regions_) {
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        const size_t off = size_t(r.z0) * r.geo.plane - base_plane;
        launch_read_macro(P, 0, r.geo.n, snap_dev_ + off, snap_dev_ + n + 3 * off, copy_);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(snap_host_, snap_dev_, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, copy_));
    CK(cudaEventRecord(snap_done_, copy_));
    snap_pending_ = true;
    snap_step_ = t_;
}

long Runner::snapshot_wait(double* rho, double* u) {
    if (!snap_pending_ && !snap_host_) throw StateError("snapshot_wait: no snapshot was started");
    CK(cudaEventSynchronize(snap_done_));
    snap_pending_ = false;
    size_t n = 0;
    for (const auto& r : regions_) n += r.geo.n;
    if (rho) std::memcpy(rho, snap_host_, sizeof(double) * n);
    if (u) std::memcpy(u, snap_host_ + n, sizeof(double) * 3 * n);
    return snap_step_;
}

size_t Runner::sample_count(int region, int solid) const {
    if (region < 0 || region >= int(regions_.size()) || solid < 0 || solid >= int(scene_.solids.size()))
        throw StateError("region/solid index out of range");
    return regions_[region].solids[solid].n;
}

void Runner::samples(int region, int solid, double* pos, double* ub, double* force, double* sampled,
                     uint32_t* src, uint8_t* flagged) const {
    const IbSolidDev& d = regions_[region].solids[sample_count(region, solid) >= 0 ? solid : 0];
    const size_t n = d.n;
    if (n == 0) return;
    CK(cudaStreamSynchronize(stream()));
    if (pos) CK(copy_sync(pos, d.pos, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (ub) CK(copy_sync(ub, d.ub, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    const size_t half = ib_half(d, t_ - 1);  // the last step whose IB phase ran
    if (force) CK(copy_sync(force, d.force + half, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (sampled) CK(copy_sync(sampled, d.sampled + half, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (src) CK(copy_sync(src, d.source, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
    if (flagged) CK(copy_sync(flagged, d.flagged, n, cudaMemcpyDeviceToHost));
}

void Runner::cell_flags(uint8_t* out) const {
    const size_t base_plane = size_t(regions_.front().z0) * regions_.front().geo.plane;
    for (const auto& r : regions_) {
        DevGuard dg(r.dev);
        unsigned char* d = nullptr;
        CK(cudaMalloc(&d, size_t(r.geo.n) * 27));
        FluidParams P{r.geo, faces_, model_, r.ptr, ctr_};
        launch_cell_flags(P, 0, r.geo.n, d, rst(r));
        CK(cudaStreamSynchronize(rst(r)));
        const size_t off = size_t(r.z0) * r.geo.plane - base_plane;
        cudaError_t e = copy_sync(out + off * 27, d, size_t(r.geo.n) * 27, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
    }
}

// Runner::set_layout (runner.cpp:252-258): permute f into the new Eq. 9
// layout and re-sort every sample replica by the new block edge.
void Runner::set_layout(int ell, size_t alpha) {
    ensure_macro();
    if (ell < 1) throw ConfigError("reorder_samples: block edge must be >= 1");
    if (alpha < 1) throw ConfigError("layout: alpha and beta must be >= 1");
    CK(cudaSetDevice(device_));
    CK(cudaStreamSynchronize(stream()));
    for (auto& r : regions_)
        if (r.st) CK(cudaStreamSynchronize(r.st));
    const Layout old = layout_;
    layout_.alpha_req = alpha;
    for (auto& r : regions_) {
        const RegionGeo go = r.geo;
        compute_geo(r);
        const RegionGeo gn = r.geo;
        if (gn.la == go.la && gn.A == go.A && gn.n_pad == go.n_pad && gn.ghost == go.ghost && gn.nbuf == go.nbuf)
            continue;
        // f(t) is the population state: permute it into every buffer of the
        // new layout (the one holding step t first)
        float* nf[3] = {nullptr, nullptr, nullptr};
        const int src = fcur(go, t_);
        DevGuard dg(r.dev);
        for (int b = 0; b < gn.nbuf; ++b) {
            nf[b] = static_cast<float*>(dalloc(sizeof(float) * f_alloc_floats(gn), false, r.dev));
            launch_relayout(r.f[src], nf[b], go, gn, rst(r));
        }
        CK(cudaStreamSynchronize(rst(r)));
        for (int b = 0; b < 3; ++b) {
            if (b < go.nbuf) dfree(r.f[b]);
            r.f[b] = nf[b];
            r.ptr.f[b] = nf[b];
        }
        if (gn.nbuf != go.nbuf) {  // per-step IB parts: move the readback part
            for (auto& d : r.solids) {
                if (d.n) {
                    IbSolidDev o = d;
                    o.nbuf = go.nbuf;
                    const size_t from = ib_half(o, t_ - 1);
                    d.nbuf = gn.nbuf;
                    const size_t to = ib_half(d, t_ - 1);
                    CK(copy_sync(d.force + to, d.force + from, 24 * d.n, cudaMemcpyDeviceToDevice));
                    CK(copy_sync(d.sampled + to, d.sampled + from, 24 * d.n, cudaMemcpyDeviceToDevice));
                }
                d.nbuf = gn.nbuf;
            }
            if (r.batch_solids)
                CK(copy_sync(r.batch_solids, r.solids.data(), sizeof(IbSolidDev) * r.solids.size(),
                              cudaMemcpyHostToDevice));
        }
    }
    (void)old;
    fill_ghosts_full();
    CK(cudaStreamSynchronize(stream()));
    for (auto& r : regions_)
        for (auto& d : r.solids) {
            const size_t n = d.n;
            if (n == 0) continue;
            std::vector<double> pos(3 * n), ref(3 * n), ub(3 * n), fo(3 * kIbHalves * n), sa(3 * kIbHalves * n);
            std::vector<unsigned> src(n);
            std::vector<unsigned char> fl(n);
            CK(copy_sync(pos.data(), d.pos, 24 * n, cudaMemcpyDeviceToHost));
            CK(copy_sync(ref.data(), d.ref, 24 * n, cudaMemcpyDeviceToHost));
            CK(copy_sync(ub.data(), d.ub, 24 * n, cudaMemcpyDeviceToHost));
            CK(copy_sync(fo.data(), d.force, fo.size() * 8, cudaMemcpyDeviceToHost));
            CK(copy_sync(sa.data(), d.sampled, sa.size() * 8, cudaMemcpyDeviceToHost));
            CK(copy_sync(src.data(), d.source, 4 * n, cudaMemcpyDeviceToHost));
            CK(copy_sync(fl.data(), d.flagged, n, cudaMemcpyDeviceToHost));
            std::vector<V3> p3(n);
            for (size_t k = 0; k < n; ++k) p3[k] = v3(&pos[3 * k]);
            const auto perm = reorder_permutation(p3, std::vector<uint32_t>(src.begin(), src.end()), ell);
            auto permute3 = [&](std::vector<double>& v) {  // every 3n half
                std::vector<double> o(v.size());
                for (size_t h = 0; h < v.size(); h += 3 * n)
                    for (size_t k = 0; k < n; ++k)
                        for (int a = 0; a < 3; ++a) o[h + 3 * k + a] = v[h + 3 * perm[k] + a];
                v.swap(o);
            };
            permute3(pos);
            permute3(ref);
            permute3(ub);
            permute3(fo);
            permute3(sa);
            std::vector<unsigned> s2(n);
            std::vector<unsigned char> f2(n);
            for (size_t k = 0; k < n; ++k) {
                s2[k] = src[perm[k]];
                f2[k] = fl[perm[k]];
            }
            CK(copy_sync(d.pos, pos.data(), 24 * n, cudaMemcpyHostToDevice));
            CK(copy_sync(d.ref, ref.data(), 24 * n, cudaMemcpyHostToDevice));
            CK(copy_sync(d.ub, ub.data(), 24 * n, cudaMemcpyHostToDevice));
            CK(copy_sync(d.force, fo.data(), fo.size() * 8, cudaMemcpyHostToDevice));
            CK(copy_sync(d.sampled, sa.data(), sa.size() * 8, cudaMemcpyHostToDevice));
            CK(copy_sync(d.source, s2.data(), 4 * n, cudaMemcpyHostToDevice));
            CK(copy_sync(d.flagged, f2.data(), n, cudaMemcpyHostToDevice));
        }
    ell_ = ell;
    build_active_lists();  // the sample order changed
    invalidate_graphs();
}

void Runner::set_variant(int fluid, int ib) {
    if (fluid < 0 || fluid > 1 || ib < 0 || ib > 1) throw ConfigError("set_variant: fluid and ib variants are 0 or 1");
    if (multi_dev_ && has_solids_ && (ib != 0 || fluid != 0))
        throw ConfigError("set_variant: slabs on several devices run the staged fluid kernel and the fused IB kernel");
    variant_ib_ = ib;
    if (fluid != variant_fluid_) {
        variant_fluid_ = fluid;
        set_layout(ell_, layout_.alpha_req);  // re-lays the populations out (ghost <-> compact)
    }
    invalidate_graphs();
}

void Runner::set_cta(int threads) {
    if (threads != 0 && threads != 128 && threads != 256 && threads != 512)
        throw ConfigError("set_cta: the staged fluid kernel runs 128, 256 or 512 threads per CTA (0 = default)");
    cta_ = threads;
    for (auto& r : regions_) r.geo.cta = threads;
    invalidate_graphs();
}

unsigned long long Runner::layout_key(size_t alpha) const {
    Runner* self = const_cast<Runner*>(this);
    const size_t keep = layout_.alpha_req;
    self->layout_.alpha_req = alpha;
    Region r = regions_.front();
    compute_geo(r);
    self->layout_.alpha_req = keep;
    return (static_cast<unsigned long long>(r.geo.ghost) << 40) | (static_cast<unsigned long long>(r.geo.la) << 32) |
           r.geo.A;
}

double Runner::measure_cost(int ell, size_t alpha, int warmup, int n_steps) {
    if (n_steps < 1) throw ConfigError("tune: n_steps must be >= 1");
    set_layout(ell, alpha);
    if (warmup > 0 && !advance(warmup, nullptr).ok) return std::numeric_limits<double>::infinity();
    if (!status_.ok) return std::numeric_limits<double>::infinity();
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, stream()));
    const Status st = advance(n_steps, nullptr);
    CK(cudaEventRecord(e1, stream()));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (!st.ok) return std::numeric_limits<double>::infinity();
    return double(ms) * 1e-3 / n_steps;
}

std::unique_ptr<Runner> Runner::clone() const {
    auto c = std::make_unique<Runner>(scene_, rank_mode_ ? 1 : m_global_, device_, rank_mode_ ? m_global_ : 0,
                                      rank_, devices_);
    c->variant_ib_ = variant_ib_;
    if (cta_) c->set_cta(cta_);
    if (variant_fluid_ != c->variant_fluid_) c->set_variant(variant_fluid_, variant_ib_);
    if (layout_.alpha_req != c->layout_.alpha_req || ell_ != c->ell_) c->set_layout(ell_, layout_.alpha_req);
    c->copy_state_from(*this);
    return c;
}

void Runner::copy_state_from(const Runner& o) {
    o.ensure_macro();
    CK(cudaStreamSynchronize(o.stream()));
    for (const auto& r : o.regions_)
        if (r.st) CK(cudaStreamSynchronize(r.st));
    cudaStream_t st = stream();
    auto cp = [&st](void* d, const void* s, size_t b) {
        if (d && s && b) CK(cudaMemcpyAsync(d, s, b, cudaMemcpyDefault, st));
    };
    for (size_t ri = 0; ri < regions_.size(); ++ri) {
        Region& d = regions_[ri];
        const Region& s = o.regions_[ri];
        const RegionGeo& g = d.geo;
        DevGuard dg(d.dev);
        st = rst(d);
        for (int b = 0; b < g.nbuf; ++b) cp(d.f[b], s.f[b], sizeof(float) * 27ull * g.n_pad);
        for (int p = 0; p < 2; ++p) {
            cp(d.recv_lo[p], s.recv_lo[p], sizeof(float) * 9ull * g.plane);
            cp(d.recv_hi[p], s.recv_hi[p], sizeof(float) * 9ull * g.plane);
            cp(d.own_send_lo[p], s.own_send_lo[p], sizeof(float) * 9ull * g.plane);
            cp(d.own_send_hi[p], s.own_send_hi[p], sizeof(float) * 9ull * g.plane);
            for (int f = 0; f < 6; ++f) cp(d.ptr.slot[p][f], s.ptr.slot[p][f], sizeof(float) * 9ull * g.slot_plane(f));
        }
        cp(d.ptr.rho, s.ptr.rho, sizeof(float) * g.ns);
        cp(d.ptr.u, s.ptr.u, sizeof(float) * 3ull * g.ns);
        if (has_solids_) {
            cp(d.stamp, s.stamp, sizeof(unsigned) * g.ns);
            cp(d.mrecv_lo, s.mrecv_lo, sizeof(float) * 4ull * g.plane);
            cp(d.mrecv_hi, s.mrecv_hi, sizeof(float) * 4ull * g.plane);
            for (size_t k = 0; k < d.solids.size(); ++k) {
                const IbSolidDev &a = d.solids[k], &b = s.solids[k];
                const size_t n = a.n;
                cp(a.pos, b.pos, 24 * n);
                cp(a.ref, b.ref, 24 * n);
                cp(a.ub, b.ub, 24 * n);
                cp(a.force, b.force, 24 * kIbHalves * n);
                cp(a.sampled, b.sampled, 24 * kIbHalves * n);
                cp(a.source, b.source, 4 * n);
                cp(a.flagged, b.flagged, n);
            }
        }
        CK(cudaStreamSynchronize(st));
    }
    CK(cudaSetDevice(device_));
    st = stream();
    cp(ctr_, o.ctr_, sizeof(DevCounters));
    if (has_tracers_) {
        tracer_reserve(o.tn_);
        cp(tdev_.x, o.tdev_.x, sizeof(double) * o.tn_);
        cp(tdev_.y, o.tdev_.y, sizeof(double) * o.tn_);
        cp(tdev_.z, o.tdev_.z, sizeof(double) * o.tn_);
        cp(tdev_.birth, o.tdev_.birth, sizeof(long long) * o.tn_);
        cp(tdev_.state, o.tdev_.state, 2 * sizeof(unsigned long long));
        tn_ = o.tn_;
        tdead_ = o.tdead_;
    }
    CK(cudaStreamSynchronize(st));
    t_ = o.t_;
    ext_chunk_t0_ = o.ext_chunk_t0_;
    t_ext_ = o.t_ext_;
    if (rank_mode_ && has_solids_) fill_motion_table(ext_chunk_t0_, cap_ + 1, true);
    status_ = o.status_;
    totals_ = o.totals_;
}

// ---- tracers ---------------------------------------------------------------

void Runner::tracer_reserve(unsigned long long need) {
    if (need <= tcap_) return;
    const unsigned long long cap = std::max<unsigned long long>({need, 2 * tcap_, 4096ull});
    auto grow = [&](auto*& p, size_t elem) {
        using T = std::remove_reference_t<decltype(*p)>;
        T* q = static_cast<T*>(dalloc(elem * cap, false));
        if (p) {
            if (tn_) CK(cudaMemcpyAsync(q, p, elem * tn_, cudaMemcpyDeviceToDevice, stream()));
            CK(cudaStreamSynchronize(stream()));
            dfree(p);
        }
        p = q;
    };
    grow(tdev_.x, sizeof(double));
    grow(tdev_.y, sizeof(double));
    grow(tdev_.z, sizeof(double));
    grow(tdev_.birth, sizeof(long long));
    tcap_ = cap;
    invalidate_graphs();  // the step graphs hold the cloud pointers
}

// Inputs of a chunk: compaction once half the entries are tombstones, room
// for the chunk's emissions, the emission batch itself (host mt19937_64, the
// reference's stream), the region table and the entry count at chunk start.
void Runner::tracer_prepare_chunk(long t0, long chunk) {
    cudaStream_t st = stream();
    if (tdead_ > 0 && 2 * tdead_ >= tn_) {
        double* sx = static_cast<double*>(dalloc(sizeof(double) * tn_, false));
        double* sy = static_cast<double*>(dalloc(sizeof(double) * tn_, false));
        double* sz = static_cast<double*>(dalloc(sizeof(double) * tn_, false));
        long long* sb = static_cast<long long*>(dalloc(sizeof(long long) * tn_, false));
        tn_ = tracer_compact(tdev_, tn_, sx, sy, sz, sb, st);
        dfree(sx);
        dfree(sy);
        dfree(sz);
        dfree(sb);
        tdead_ = 0;
    }
    tracer_reserve(tn_ + temit_ * (unsigned long long)chunk);
    std::vector<TracerRegion> reg;
    for (const auto& r : regions_) reg.push_back({r.ptr.u, r.z0, r.z1, r.geo.ns});
    bool same = reg.size() == treg_host_.size();
    for (size_t k = 0; same && k < reg.size(); ++k)
        same = reg[k].u == treg_host_[k].u && reg[k].z0 == treg_host_[k].z0 && reg[k].ns == treg_host_[k].ns;
    if (!same) {
        CK(copy_sync(treg_dev_, reg.data(), sizeof(TracerRegion) * reg.size(), cudaMemcpyHostToDevice));
        treg_host_ = reg;
    }
    if (temit_) {
        for (long j = 0; j < chunk; ++j)
            emit_positions(scene_.emitters, t0 + j, scene_.cfg.seed, pinned_temit_ + 3 * temit_ * size_t(j));
        CK(cudaMemcpyAsync(temit_dev_, pinned_temit_, sizeof(double) * 3 * temit_ * size_t(chunk),
                           cudaMemcpyHostToDevice, st));
    }
    pinned_tstate_[0] = tn_;
    pinned_tstate_[1] = tdead_;
    CK(cudaMemcpyAsync(tdev_.state, pinned_tstate_, 2 * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
}

void Runner::tracers(double* pos, int64_t* birth) const {
    CK(cudaStreamSynchronize(stream()));
    if (!has_tracers_ || tn_ == 0) return;
    std::vector<double> x(tn_), y(tn_), z(tn_);
    std::vector<long long> b(tn_);
    CK(copy_sync(x.data(), tdev_.x, sizeof(double) * tn_, cudaMemcpyDeviceToHost));
    CK(copy_sync(y.data(), tdev_.y, sizeof(double) * tn_, cudaMemcpyDeviceToHost));
    CK(copy_sync(z.data(), tdev_.z, sizeof(double) * tn_, cudaMemcpyDeviceToHost));
    CK(copy_sync(b.data(), tdev_.birth, sizeof(long long) * tn_, cudaMemcpyDeviceToHost));
    size_t w = 0;
    for (size_t p = 0; p < tn_; ++p) {
        if (b[p] < 0) continue;  // tombstone: retired (advect_tracers removes it, order kept)
        if (pos) {
            pos[3 * w] = x[p];
            pos[3 * w + 1] = y[p];
            pos[3 * w + 2] = z[p];
        }
        if (birth) birth[w] = b[p];
        ++w;
    }
}

void Runner::tracer_density(double* vol) const {
    const size_t n = size_t(nx_) * ny_ * nz_;
    double* d = nullptr;
    if (cudaMalloc(&d, sizeof(double) * n) != cudaSuccess) {
        cudaGetLastError();
        throw OomError("tracer density volume allocation failed");
    }
    cudaStream_t st = stream();
    CK(cudaMemsetAsync(d, 0, sizeof(double) * n, st));
    if (has_tracers_) launch_rasterize(tdev_.x, tdev_.y, tdev_.z, 1, tdev_.birth, tn_, nx_, ny_, nz_, d, st);
    CK(cudaMemcpyAsync(vol, d, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(d);
}

// ---- rank mode -----------------------------------------------------------

void Runner::halo_f(int parity, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                    size_t* bytes) {
    const int p = parity & 1;
    const Region& r = regions_.front();
    *send_lo = r.ptr.send_lo[p];
    *send_hi = r.ptr.send_hi[p];
    *recv_lo = const_cast<float*>(r.ptr.recv_lo[p]);
    *recv_hi = const_cast<float*>(r.ptr.recv_hi[p]);
    *bytes = sizeof(float) * 9ull * r.geo.plane;
}

void Runner::halo_macro(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi, size_t* bytes) {
    const Region& r = regions_.front();
    *send_lo = r.ptr.msend_lo;
    *send_hi = r.ptr.msend_hi;
    *recv_lo = const_cast<float*>(r.ptr.mrecv_lo);
    *recv_hi = const_cast<float*>(r.ptr.mrecv_hi);
    *bytes = sizeof(float) * 4ull * r.geo.plane;
}

void Runner::phase(int ph, int write_macro) {
    if (!rank_mode_) throw StateError("phase(): only valid for a rank-mode runner");
    CK(cudaSetDevice(device_));
    // an in-flight snapshot reads rho/u, which the IB band pass and the fluid
    // phases (write_macro) rewrite
    if (snap_pending_) CK(cudaStreamWaitEvent(stream(), snap_done_, 0));
    // the device motion / totals tables hold cap_ steps from the chunk start
    if (ph == LBMG_PHASE_PRE && t_ext_ - ext_chunk_t0_ >= cap_)
        throw StateError("phase(): " + std::to_string(cap_) +
                         " steps since the last sync(); call lbmg_runner_sync at least that often");
    switch (ph) {
        case LBMG_PHASE_PRE:
            // the motion/totals tables cover cap_ steps: call sync() at least
            // that often (lbmg_runner_sync)
            if (has_solids_) enqueue_ib_pre();
            break;
        case LBMG_PHASE_MID:
            if (has_solids_) enqueue_ib_mid();
            break;
        case LBMG_PHASE_FLUID_EDGE: enqueue_fluid(write_macro != 0, 1); break;
        case LBMG_PHASE_FLUID_BULK: enqueue_fluid(write_macro != 0, 2); break;
        case LBMG_PHASE_END:
            launch_step_end(ctr_, stream());
            ++t_ext_;
            break;
        default: throw StateError("unknown phase");
    }
    CK(cudaGetLastError());
}

Status Runner::sync_external() {
    CK(cudaStreamSynchronize(stream()));
    finish_chunk(ext_chunk_t0_, 0);
    ext_chunk_t0_ = t_;
    t_ext_ = t_;
    if (has_solids_) {
        fill_motion_table(t_, cap_ + 1, true);
        long long t0d = t_;
        CK(copy_sync(&ctr_->chunk_t0, &t0d, sizeof t0d, cudaMemcpyHostToDevice));
    }
    return status_;
}

}  // namespace lbmg
