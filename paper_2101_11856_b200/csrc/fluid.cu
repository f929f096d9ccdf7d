// The fused fluid step of one region (stream + six face passes + moments +
// CM-MRT/ACM collision + forcing, runner.cpp:135-208).
//
// Ghost-layer layout (RegionGeo::ghost):
//  ghost_fill_kernel   the face passes, periodic wraps and z halos of this
//                      step, written into the ghost slots the face nodes pull
//                      from (+ the persistent face slots).
//  fluid_ghost_kernel  every owned node: TMA-staged plain shifted pulls,
//                      moments, packed (FFMA2) collision, forcing; persistent
//                      CTAs on an in-order device tile queue.
// Compact layout (nx % 4 != 0, or the register-direct tuner variant):
//  fluid_bulk_kernel   interior nodes, two x-nodes per thread, LDG.64 + SHFL.
//  fluid_shell_kernel  the boundary layers: per-direction ownership, bounce-
//                      back / inlet / outflow (incl. the stale edge read),
//                      halo sends, face slots.
// All paths share collision.cuh and are bit-identical per node.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "collision.cuh"
#include "device_common.cuh"
#include "engine.hpp"
#include "fluid_dev.cuh"
#include "tma.cuh"

namespace lbmg {

namespace {

// f*_i at (x,y,lz) once face pass `owner` has run this step (apply_face,
// boundary.cpp:42-118).  Outflow copies f*_i of the interior neighbour as it
// stands at that point of the pass sequence: the streamed value, an earlier
// face's fresh reconstruction (followed), or — when a later face owns it —
// the previous step's slot value (the stale edge read).
__device__ __forceinline__ float reconstruct(const FluidParams& P, const StepView& v, int x, int y, int lz, int i,
                                         int owner) {
    const RegionGeo& g = P.g;
    const FaceTable& ft = P.faces;
    int f = owner;
    for (int guard = 0; guard < 7; ++guard) {
        const int cond = ft.cond[f];
        if (cond == kNoSlip) return v.fin[g.at(x, y, lz, opposite(i))];
        if (cond == kInlet) return ft.inlet[f][i];
        const int a = face_axis(f), s = face_side(f);
        if (a == 0) x -= s;
        else if (a == 1) y -= s;
        else lz -= s;
        const int fn = owner_face(g, x, y, g.gz0 + lz, i);
        if (fn == kNoOwner) return pull_rt(g, v, x, y, lz, i);
        if (fn > f) return P.p.slot[v.p][fn][g.slot_index(fn, x, y, lz, i)];
        f = fn;
    }
    return 0.0f;  // unreachable: the owner strictly decreases along the chain
}

// f~* (post-stream, post-face-pass) of one node.
template <bool WRITE_SLOTS>
__device__ __forceinline__ void gather_node(const FluidParams& P, const StepView& v, float* const* slot_cur,
                                            unsigned k, int x, int y, int lz, float (&fs)[27]) {
    const RegionGeo& g = P.g;
    const bool interior = x >= 1 && x <= g.nx - 2 && y >= 1 && y <= g.ny - 2 && lz >= 1 && lz <= g.nzl - 2;
    if (interior) {
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            fs[i] = __ldg(&v.fin[g.at(x - cx(i), y - cy(i), lz - cz(i), i)]);
        });
        return;
    }
    const int gz = g.gz0 + lz;
    // 1) every pull's address, branch-free (wrap in x/y, halo planes in z; a
    //    missing pull points at the node itself) -> 27 independent loads
    unsigned miss = 0;
    static_for<0, 27>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int own = owner_face_c<i>(g, x, y, gz);
        int sx = x - cx(i), sy = y - cy(i);
        sx = sx < 0 ? sx + g.nx : (sx >= g.nx ? sx - g.nx : sx);
        sy = sy < 0 ? sy + g.ny : (sy >= g.ny ? sy - g.ny : sy);
        const int lzs = lz - cz(i);
        const unsigned hp = cross9(i, 2) * g.plane + unsigned(sy) * g.nx + unsigned(sx);
        const float* src;
        if constexpr (cz(i) == 1) src = lzs < 0 ? v.halo_lo + hp : v.fin + g.at(sx, sy, lzs, i);
        else if constexpr (cz(i) == -1) src = lzs >= g.nzl ? v.halo_hi + hp : v.fin + g.at(sx, sy, lzs, i);
        else src = v.fin + g.at(sx, sy, lzs, i);
        if (own != kNoOwner) {
            src = v.fin + g.at(x, y, lz, i);
            miss |= 1u << i;
        }
        fs[i] = __ldg(src);
    });
    // 2) the missing populations (face passes, boundary.cpp:42-125)
    if (miss) {
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if (miss & (1u << i)) {
                const int own = owner_face_c<i>(g, x, y, gz);
                const float val = reconstruct(P, v, x, y, lz, i, own);
                fs[i] = val;
                if constexpr (WRITE_SLOTS) slot_cur[own][g.slot_index(own, x, y, lz, i)] = val;
            }
        });
    }
}


// Shell enumeration: planes lz=0 and lz=nzl-1 first (the "edge" part that
// feeds the halos), then per interior plane the rows y=0, y=ny-1 and the
// columns x=0, x=nx-1.
__device__ __forceinline__ void shell_decode(const RegionGeo& g, unsigned s, int& x, int& y, int& lz) {
    const unsigned zplanes = g.nzl >= 2 ? 2u : 1u;
    if (s < zplanes * g.plane) {
        const unsigned q = s >= g.plane ? s - g.plane : s;
        lz = s >= g.plane ? g.nzl - 1 : 0;
        const unsigned yy = g.div_nx.div(q);
        y = int(yy);
        x = int(q - yy * unsigned(g.nx));
        return;
    }
    const unsigned r0 = s - zplanes * g.plane;
    const unsigned cnt = 2u * g.nx + 2u * (g.ny - 2);
    const unsigned pl = r0 / cnt;
    unsigned r = r0 - pl * cnt;
    lz = 1 + int(pl);
    if (r < unsigned(g.nx)) {
        y = 0;
        x = int(r);
    } else if (r < 2u * g.nx) {
        y = g.ny - 1;
        x = int(r - g.nx);
    } else {
        r -= 2u * g.nx;
        y = 1 + int(r >> 1);
        x = (r & 1u) ? g.nx - 1 : 0;
    }
}

}  // namespace

// Collision output form shared by every fluid kernel of a run (bitwise
// identical per node across kernels): 0 = f* - t' with f* in registers,
// 1 = the same with the bulk kernel's f* in shared memory, 2 = feq + t''.
template <int FORM, class V>
using StashFor = typename std::conditional<FORM == 2, NoStash<V>, RegStash<V>>::type;

// ---------------------------------------------------------------------------
// Shell (and generic all-node) kernel: one node per thread, general path.
template <int KIND, int POLICY, bool STD, int FORM>
__global__ void __launch_bounds__(128) fluid_shell_kernel(const FluidParams P, unsigned s0, unsigned s1,
                                                          int write_macro, int all_nodes) {
    DevCounters* ctr = P.ctr;
    if (ctr->diverged) return;
    const unsigned s = s0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= s1) return;
    const RegionGeo& g = P.g;
    int x, y, lz;
    if (all_nodes) decode(g, s, x, y, lz);
    else shell_decode(g, s, x, y, lz);
    const unsigned k = g.node(x, y, lz);
    const long long t = ctr->t;
    const int p = int(t & 1);
    const unsigned char epoch = ib_epoch(t);  // IB force flags of this step
    const StepView v = make_view(P, t);

    float fs[27];
    gather_node<true>(P, v, P.p.slot[p ^ 1], k, x, y, lz, fs);
    const MacroV<float> mc = moments_v<float>(fs);
    if (mc.bad[0]) {
        flag_divergence(ctr);
        return;
    }
    if (mc.mach[0]) raise_mach(ctr);
    if (write_macro) {
        P.p.rho[k] = mc.rho;
        P.p.u[k] = mc.ux;
        P.p.u[k + g.ns] = mc.uy;
        P.p.u[k + 2u * g.ns] = mc.uz;
    }
    float gx = P.m.body[0], gy = P.m.body[1], gz = P.m.body[2];
    if (P.p.tflag != nullptr && P.p.tflag[k] == epoch) {
        float* gib = P.p.gib;
        gx = __fadd_rn(gx, gib[k]);
        gy = __fadd_rn(gy, gib[k + g.ns]);
        gz = __fadd_rn(gz, gib[k + 2u * g.ns]);
        gib[k] = 0.f;
        gib[k + g.ns] = 0.f;
        gib[k + 2u * g.ns] = 0.f;
    }
    StashFor<FORM, float> stash;
    collide_v<KIND, POLICY, STD, float>(fs, mc, gx, gy, gz, gx != 0.f || gy != 0.f || gz != 0.f, P.m, stash);

    float* fout = P.p.f[fnext(g, t)];
    static_for<0, 27>([&](auto I) {
        constexpr int i = decltype(I)::value;
        fout[g.idx(k, i)] = fs[i];
    });
    // crossing populations of the boundary planes -> neighbour halos
    const unsigned hp = unsigned(y) * g.nx + x;
    if (lz == 0) {
        float* sd = P.p.send_lo[p ^ 1];
        if (sd)
            static_for<1, 10>([&](auto I) {
                constexpr int i = decltype(I)::value;
                sd[cross9(i, 2) * g.plane + hp] = fs[i];
            });
    }
    if (lz == g.nzl - 1) {
        float* sd = P.p.send_hi[p ^ 1];
        if (sd)
            static_for<18, 27>([&](auto I) {
                constexpr int i = decltype(I)::value;
                sd[cross9(i, 2) * g.plane + hp] = fs[i];
            });
    }
}

// f* of the bulk kernel's node pairs parked in shared memory during the
// moment transform ([direction][thread], 27.6 KB per 128-thread CTA).
constexpr int kBulkThreads = 128;
struct SmemStash {
    static constexpr bool kFeqOut = false;
    __device__ __forceinline__ float2* base() const {
        __shared__ float2 sm[27][kBulkThreads];
        return &sm[0][threadIdx.x];
    }
    __device__ __forceinline__ void put(int i, float2 x) { base()[i * kBulkThreads] = x; }
    __device__ __forceinline__ float2 get(int i) const { return base()[i * kBulkThreads]; }
};

// ---------------------------------------------------------------------------
// Bulk kernel: nodes [kb, ke) = local planes 1..nzl-2, two nodes per thread.
template <int KIND, int POLICY, bool STD, bool SOA, int FORM>
__global__ void __launch_bounds__(kBulkThreads, FORM == 2 ? 4 : 3) fluid_bulk_kernel(const FluidParams P, unsigned kb, unsigned ke,
                                                         int write_macro) {
    DevCounters* ctr = P.ctr;
    if (ctr->diverged) return;
    const RegionGeo& g = P.g;
    const unsigned ln = threadIdx.x & 31u;
    const unsigned kw = kb + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 64u;
    if (kw >= ke) return;  // warp-uniform
    unsigned k = kw + 2u * ln;
    const bool inr = k < ke;
    int x, y, lz;
    decode(g, inr ? k : kb, x, y, lz);
    const bool yok = inr && y >= 1 && y <= g.ny - 2;
    const bool v0 = yok && x >= 1;
    const bool v1 = yok && x + 1 <= g.nx - 2;
    if (!__any_sync(kFull, v0 || v1)) return;
    // lanes without a valid node load from a safe interior pair instead
    const unsigned kl = (v0 || v1) ? k : g.plane + unsigned(g.nx) + 2u;

    const long long t = ctr->t;
    const unsigned char epoch = ib_epoch(t);  // IB force flags of this step
    const float* __restrict__ fin = P.p.f[fcur(g, t)];
    float2 fs[27];
    static_for<0, 27>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const unsigned ks = kl - unsigned(g.nx * cy(i) + int(g.plane) * cz(i));
        const float* src = SOA ? fin + size_t(i) * g.A + ks : fin + g.idx(ks, i);
        const float2 pr = __ldg(reinterpret_cast<const float2*>(src));
        if constexpr (cx(i) == 0) {
            fs[i] = pr;
        } else if constexpr (cx(i) == 1) {  // source x-1
            float left = __shfl_up_sync(kFull, pr.y, 1);
            if (ln == 0 && v0) left = SOA ? __ldg(src - 1) : __ldg(fin + g.idx(ks - 1, i));
            fs[i] = make_float2(left, pr.x);
        } else {  // source x+1
            float right = __shfl_down_sync(kFull, pr.x, 1);
            if (ln == 31 && v1) right = SOA ? __ldg(src + 2) : __ldg(fin + g.idx(ks + 2, i));
            fs[i] = make_float2(pr.y, right);
        }
    });
    if (!(v0 || v1)) return;  // (after the shuffles)

    const MacroV<float2> mc = moments_v<float2>(fs);
    if ((v0 && mc.bad[0]) || (v1 && mc.bad[1])) {
        flag_divergence(ctr);
        return;
    }
    if ((v0 && mc.mach[0]) || (v1 && mc.mach[1])) raise_mach(ctr);
    const bool both = v0 && v1;
    if (write_macro) {
        const float2 r = mc.rho, ux = mc.ux, uy = mc.uy, uz = mc.uz;
        if (both) {
            *reinterpret_cast<float2*>(P.p.rho + k) = r;
            *reinterpret_cast<float2*>(P.p.u + k) = ux;
            *reinterpret_cast<float2*>(P.p.u + k + g.ns) = uy;
            *reinterpret_cast<float2*>(P.p.u + k + 2u * g.ns) = uz;
        } else {
            const unsigned kk = v0 ? k : k + 1;
            const int j = v0 ? 0 : 1;
            P.p.rho[kk] = lane(r, j);
            P.p.u[kk] = lane(ux, j);
            P.p.u[kk + g.ns] = lane(uy, j);
            P.p.u[kk + 2u * g.ns] = lane(uz, j);
        }
    }
    float2 gx = make_float2(P.m.body[0], P.m.body[0]);
    float2 gy = make_float2(P.m.body[1], P.m.body[1]);
    float2 gz = make_float2(P.m.body[2], P.m.body[2]);
    if (P.p.tflag != nullptr && (P.p.tflag[k] == epoch || P.p.tflag[k + 1] == epoch)) {
        float* gib = P.p.gib;
        float2 a = *reinterpret_cast<const float2*>(gib + k);
        float2 b = *reinterpret_cast<const float2*>(gib + k + g.ns);
        float2 c = *reinterpret_cast<const float2*>(gib + k + 2u * g.ns);
        // only this kernel's nodes: a shell node's force is consumed there
        if (!v0) a.x = b.x = c.x = 0.f;
        if (!v1) a.y = b.y = c.y = 0.f;
        gx = __fadd2_rn(gx, a);
        gy = __fadd2_rn(gy, b);
        gz = __fadd2_rn(gz, c);
        if (v0) gib[k] = gib[k + g.ns] = gib[k + 2u * g.ns] = 0.f;
        if (v1) gib[k + 1] = gib[k + 1 + g.ns] = gib[k + 1 + 2u * g.ns] = 0.f;
    }
    const bool any_force = gx.x != 0.f || gx.y != 0.f || gy.x != 0.f || gy.y != 0.f || gz.x != 0.f || gz.y != 0.f;
    typename std::conditional<FORM == 1, SmemStash, StashFor<FORM, float2>>::type stash;
    collide_v<KIND, POLICY, STD, float2>(fs, mc, gx, gy, gz, any_force, P.m, stash);

    float* __restrict__ fout = P.p.f[fnext(g, t)];
    if (both) {
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            float* dst = SOA ? fout + size_t(i) * g.A + k : fout + g.idx(k, i);
            *reinterpret_cast<float2*>(dst) = fs[i];
        });
    } else {
        const unsigned kk = v0 ? k : k + 1;
        const int j = v0 ? 0 : 1;
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            float* dst = SOA ? fout + size_t(i) * g.A + kk : fout + g.idx(kk, i);
            *dst = lane(fs[i], j);
        });
    }
}

// ---------------------------------------------------------------------------
// Ghost-layer path (RegionGeo::ghost, SoA with nx % 4 == 0).
//
//  ghost_fill_kernel   the six face passes of this step (apply_face,
//                      boundary.cpp:42-125), periodic wraps and z halos:
//                      for every node on a face of the slab and each of the
//                      9 directions crossing that face, f*_i(node) is written
//                      into the ghost slot the node pulls from,
//                      s(node) - off_i.  Afterwards every pull of every owned
//                      node is a plain shifted read.
//  fluid_ghost_kernel  persistent CTAs walk contiguous chunks of kTile
//                      storage slots.  Per tile one elected thread issues 27
//                      one-dimensional TMA bulk copies — each direction's
//                      window, shifted by off_i and widened to 16-byte
//                      alignment — into a ring of kStages shared-memory stages
//                      completed on mbarriers, so the next tile is in flight
//                      while the CTA computes the current one (two nodes per
//                      thread, packed FFMA2 collision, 64-bit stores).  Lanes on
//                      ghost/pad slots compute but do not store.
// 1-D grid over the concatenated entry list: faces 0..5 in order, each
// 9 direction slots x the face's nodes (no idle blocks for the smaller faces)
__global__ void __launch_bounds__(256) ghost_fill_kernel(const __grid_constant__ FluidParams P, int full) {
    DevCounters* ctr = P.ctr;
    if (ctr->diverged) return;
    const RegionGeo& g = P.g;
    unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned FX = unsigned(g.ny) * g.nzl, FY = unsigned(g.nx) * g.nzl, FZ = g.plane;
    int f = 0;
    unsigned F = FX;
    for (; f < 6; ++f) {
        F = f < 2 ? FX : (f < 4 ? FY : FZ);
        if (e < 9u * F) break;
        e -= 9u * F;
    }
    if (f == 6) return;
    const unsigned j = e / F, q = e - j * F;
    const long long t = ctr->t;
    const bool fl = full != 0;
    switch (f) {
        case 0: ghost_fill_entry<0>(P, t, q, j, fl); break;
        case 1: ghost_fill_entry<1>(P, t, q, j, fl); break;
        case 2: ghost_fill_entry<2>(P, t, q, j, fl); break;
        case 3: ghost_fill_entry<3>(P, t, q, j, fl); break;
        case 4: ghost_fill_entry<4>(P, t, q, j, fl); break;
        default: ghost_fill_entry<5>(P, t, q, j, fl); break;
    }
}

// The fill program of step parity p: same enumeration as ghost_fill_kernel.
// A warp whose 32 entries each give one record, consecutive in source and
// destination (a y/z face row), becomes one run at out[count[0]++]; other
// records are appended per warp at out[eoff + count[1]++] (out == null:
// count only).
__global__ void __launch_bounds__(256) ghost_plan_kernel(const __grid_constant__ FluidParams P, int p, FillRec* out,
                                                         unsigned eoff, unsigned* count) {
    const RegionGeo& g = P.g;
    unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned FX = unsigned(g.ny) * g.nzl, FY = unsigned(g.nx) * g.nzl, FZ = g.plane;
    int f = 0;
    unsigned F = FX;
    for (; f < 6; ++f) {
        F = f < 2 ? FX : (f < 4 ? FY : FZ);
        if (e < 9u * F) break;
        e -= 9u * F;
    }
    FillRec rec[2];
    int n = 0;
    if (f < 6) {
        const unsigned j = e / F, q = e - j * F;
        switch (f) {
            case 0: n = ghost_plan_entry<0>(P, p, q, j, rec); break;
            case 1: n = ghost_plan_entry<1>(P, p, q, j, rec); break;
            case 2: n = ghost_plan_entry<2>(P, p, q, j, rec); break;
            case 3: n = ghost_plan_entry<3>(P, p, q, j, rec); break;
            case 4: n = ghost_plan_entry<4>(P, p, q, j, rec); break;
            default: n = ghost_plan_entry<5>(P, p, q, j, rec); break;
        }
    }
    const unsigned lane = threadIdx.x & 31u;
    const unsigned b0 = __ballot_sync(kFull, n > 0), b1 = __ballot_sync(kFull, n == 1);
    const unsigned b2 = __ballot_sync(kFull, n > 1);
    // the record that fills the ghost slot is rec[n - 1]; a run needs one
    // record per lane (no face-slot copy) at consecutive addresses
    const FillRec last = n > 0 ? rec[n - 1] : FillRec{nullptr, nullptr};
    const unsigned long long s0 = __shfl_sync(kFull, (unsigned long long)last.src, 0);
    const unsigned long long d0 = __shfl_sync(kFull, (unsigned long long)last.dst, 0);
    const bool run = b1 == kFull && __all_sync(kFull, (unsigned long long)last.src == s0 + 4ull * lane &&
                                                       (unsigned long long)last.dst == d0 + 4ull * lane);
    if (run) {
        if (lane == 0) {
            const unsigned at = atomicAdd(&count[0], 1u);
            if (out != nullptr && at < eoff) out[at] = last;
        }
        return;
    }
    const unsigned total = __popc(b0) + __popc(b2);
    unsigned base = 0;
    if (lane == 0 && total) base = atomicAdd(&count[1], total);
    base = __shfl_sync(kFull, base, 0);
    if (out == nullptr) return;
    out += eoff;
    // all first records of the warp in lane order, then the second ones
    const unsigned pos0 = base + __popc(b0 & ((1u << lane) - 1u));
    const unsigned pos1 = base + __popc(b0) + __popc(b2 & ((1u << lane) - 1u));
    if (n > 0) out[pos0] = rec[0];
    if (n > 1) out[pos1] = rec[1];
}

// Per-step ghost fill through the program of this step's parity (no decode,
// no ownership logic; fill_copy_block).
__global__ void __launch_bounds__(256) ghost_copy_kernel(const __grid_constant__ FluidParams P) {
    if (P.ctr->diverged) return;
    fill_copy_block(P, blockIdx.x, threadIdx.x, blockDim.x);
}

// The step's counters into the mapped host block (RegionPtrs::ctr_host), by
// the last CTA of the launch that ends the step (after every CTA's updates).
__device__ __forceinline__ void publish_counters(const FluidParams& P) {
    DevCounters* h = P.p.ctr_host;
    if (h == nullptr) return;
    const DevCounters* c = P.ctr;
    h->t = __ldcg(&c->t);
    h->diverged = __ldcg(&c->diverged);
    h->mach = __ldcg(&c->mach);
    h->diverged_step = __ldcg(&c->diverged_step);
    h->chunk_t0 = __ldcg(&c->chunk_t0);
}

template <int KIND, int POLICY, bool STD, int T>
__global__ void __launch_bounds__(T, 512 / T)
    fluid_ghost_kernel(const __grid_constant__ FluidParams P, int z_a, int z_b, int slot, int write_macro, int dbg,
                       int pf, int end_step) {
    constexpr int kTile = GhostTile<T>::kTile, kWin = GhostTile<T>::kWin;
    constexpr unsigned kStageBytes = GhostTile<T>::kStageBytes;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* const stage0 = reinterpret_cast<float*>(smem_raw);
    uint64_t* const full = reinterpret_cast<uint64_t*>(smem_raw + kStages * kStageBytes);
    DevCounters* ctr = P.ctr;
    if (ctr->diverged) {  // CTA-uniform; still counted for the queue rewind
        if (threadIdx.x == 0 && atomicAdd(&P.p.queue[4 + slot], 1u) == gridDim.x - 1) {
            P.p.queue[slot] = 0u;
            P.p.queue[4 + slot] = 0u;
            if (end_step) publish_counters(P);
        }
        return;
    }
    const RegionGeo& g = P.g;
    const long long t = ctr->t;
    const int p = int(t & 1);
    const unsigned char epoch = ib_epoch(t);  // IB force flags of this step
    const float* __restrict__ fin = P.p.f[fcur(g, t)];
    float* __restrict__ fout = P.p.f[fnext(g, t)];
    const unsigned tid = threadIdx.x;
    // slots of planes [z_a, z_b); tiles are kTile-aligned (CSoA blocks are
    // multiples of kTile), lanes outside [sb, se) do not store
    const unsigned sb = g.base + unsigned(z_a + 1) * g.PP, se = g.base + unsigned(z_b + 1) * g.PP;
    const unsigned org = (sb / kTile) * kTile - (dbg >> 8);  // tile origin (probe: LBMG_GHOST_DBG >> 8 shift)
    const unsigned ntiles = (se - org + kTile - 1) / kTile;
    // Tiles are handed out in order by a device counter (reset by the ghost
    // fill of this step): all CTAs sweep the arrays together, so DRAM pages
    // stay open across CTAs and the window edges two neighbouring tiles share
    // are fetched once and hit in L2 for the other.
    unsigned* const next_tile = &P.p.queue[slot];
    // tile id per (stage, phase parity): the refill for phase k+1 writes the
    // other parity slot than the one phase-k readers use (no WAR hazard)
    __shared__ unsigned stage_tile[kStages][2];
    __shared__ unsigned reads_done[kStages];
    // the tile's IB force-chunk epochs (cflag), bulk-copied with its windows
    __shared__ __align__(16) unsigned char force_s[kStages][16];
    const unsigned char* const cflag = P.p.cflag;

    // claim the next tile into stage s (elected thread); past the end the
    // stage's phase completes empty so the consumers see the end marker
    auto refill = [&](int s, unsigned phase) {
        const unsigned tile = atomicAdd(next_tile, 1u);
        stage_tile[s][phase & 1u] = tile;
        if (tile >= ntiles) {
            mbar_arrive(&full[s]);
            return;
        }
        const long long k0 = (long long)org + (long long)tile * kTile;
        float* dst = stage0 + s * (kStageBytes / 4);
        mbar_arrive_expect_tx(&full[s], kStageBytes + (cflag != nullptr ? 16u : 0u));
        if (cflag != nullptr)  // the 16 chunk bytes around the tile's (a tile spans <= 16 aligned chunks)
            tma_load_1d(force_s[s], cflag + (((unsigned long long)k0 >> kForceChunkShift) & ~15ull), 16u, &full[s]);
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            // the window may straddle a CSoA block boundary: two segments
            const unsigned long long a0 = (unsigned long long)(k0 - g.soff(i) - win_shift(i));
            const unsigned long long e0 = (a0 | g.amask) + 1ull;
            const unsigned l0 = e0 - a0 < (unsigned long long)kWin ? unsigned(e0 - a0) : unsigned(kWin);
            tma_load_1d(dst + i * kWin, fin + g.gaddr(a0, i), l0 * 4u, &full[s]);
            if (l0 < unsigned(kWin))
                tma_load_1d(dst + i * kWin + l0, fin + g.gaddr(e0, i), (kWin - l0) * 4u, &full[s]);
        });
    };
    // consumer release: the last warp to finish reading a stage refills it
    // (no CTA-wide barrier per tile: warps never wait for the slowest one)
    // the fused IB kernel's reaction totals of this step (RegionPtrs::ib_partial):
    // shared memory of the not yet filled stages as scratch, before the first refill
    for (unsigned k = blockIdx.x; k < P.p.ib_solids; k += gridDim.x) {
        double* tree = reinterpret_cast<double*>(stage0);  // [6][128]
        const unsigned b0 = P.p.ib_start[k], nblk = P.p.ib_start[k + 1] - b0;
        if (tid < 128) {
            double acc[6] = {0, 0, 0, 0, 0, 0};
            for (unsigned b = tid; b < nblk; b += 128)
                for (int a = 0; a < 6; ++a) acc[a] += __ldcg(&P.p.ib_partial[size_t(b0 + b) * 6 + a]);
            for (int a = 0; a < 6; ++a) tree[a * 128 + tid] = acc[a];
        }
        __syncthreads();
        for (unsigned off = 64; off > 0; off >>= 1) {
            if (tid < off)
                for (int a = 0; a < 6; ++a) tree[a * 128 + tid] += tree[a * 128 + tid + off];
            __syncthreads();
        }
        if (tid < 6) {
            const long long at = (t - ctr->chunk_t0) * P.p.ib_stride + 6 * k + tid;
            P.p.ib_out[at] = tree[tid * 128];
            if (P.p.ib_out_host != nullptr) P.p.ib_out_host[at] = tree[tid * 128];  // (zero-copy row)
        }
        __syncthreads();
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            reads_done[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        // the totals scratch above was written through the generic proxy:
        // order it before the bulk copies (async proxy) into the same stage
        if (blockIdx.x < P.p.ib_solids) fence_proxy_async_smem();
        for (int s = 0; s < kStages; ++s) refill(s, 0u);
    }

    for (unsigned it = 0;; ++it) {
        const int s = int(it % kStages);
        const float* const st = stage0 + s * (kStageBytes / 4);
        mbar_wait_parity(&full[s], (it / kStages) & 1u);
        const unsigned tile = stage_tile[s][(it / kStages) & 1u];
        if (tile >= ntiles) break;
        // Tiles are claimed in order by all CTAs, so tile + pf will be claimed
        // about pf / (stages * grid) tile periods from now: pull its windows
        // into L2 already (deeper pipeline at no shared-memory cost; issued
        // here, before the tile is read into registers)
        if (pf > 0 && tid == 0 && tile + unsigned(pf) < ntiles) {
            const long long k1 = (long long)org + (long long)(tile + unsigned(pf)) * kTile;
            static_for<0, 27>([&](auto I) {
                constexpr int i = decltype(I)::value;
                const unsigned long long a1 = (unsigned long long)(k1 - g.soff(i) - win_shift(i));
                const unsigned long long e1 = (a1 | g.amask) + 1ull;
                const unsigned l1 = e1 - a1 < (unsigned long long)kWin ? unsigned(e1 - a1) : unsigned(kWin);
                prefetch_l2(fin + g.gaddr(a1, i), l1 * 4u);
            });
        }
        const unsigned m = 2u * tid;
        const unsigned sl = org + tile * kTile + m;  // storage slot of the pair's first node
        const unsigned row = g.div_px.div(sl - g.base);
        const int col = int(sl - g.base - row * g.PX);
        const unsigned pl = g.div_py.div(row);
        const int r = int(row - pl * g.PY);
        const int x = col - 2, y = r - 1, lz = int(pl) - 1;
        // pairs are all-ghost or all-owned (nx, PX even)
        const bool valid = sl >= sb && sl < se && x >= 0 && x < g.nx && y >= 0;
        // IB force epoch of the pair's storage chunk (staged with the tile:
        // read before this warp releases the stage)
        const bool forced = cflag != nullptr && force_s[s][(sl >> kForceChunkShift) & 15u] == epoch;
        float2 fs[27];
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int d = win_shift(i);
            const float* w = st + i * kWin + m + d;
            if constexpr (d % 2 == 0) fs[i] = *reinterpret_cast<const float2*>(w);
            else fs[i] = make_float2(w[0], w[1]);
        });
        // ptxas sinks the gib loads next to their use (the collision epilogue:
        // 127 live registers), so a forced warp would wait a full DRAM round
        // trip there; pulling the lines into L2 here — before the stage
        // release branch, which the scheduler does not move them across —
        // turns that into an L2 hit
        if (forced && valid) {
            const unsigned kp = (unsigned(lz) * g.ny + unsigned(y)) * g.nx + unsigned(x);
            prefetch_l2_line(P.p.gib + kp);
            prefetch_l2_line(P.p.gib + kp + g.ns);
            prefetch_l2_line(P.p.gib + kp + 2u * g.ns);
        }
        __syncwarp();
        if ((tid & 31u) == 0) {
            __threadfence_block();  // this warp's reads of stage s are done
            if (atomicAdd(&reads_done[s], 1u) == T / 32 - 1) {
                reads_done[s] = 0;
                __threadfence_block();  // (acquire: every warp's reads of stage s precede the refill)
                fence_proxy_async_smem();
                refill(s, it / kStages + 1u);
            }
        }
        if (!valid) continue;
        const unsigned k = (unsigned(lz) * g.ny + unsigned(y)) * g.nx + unsigned(x);  // compact node index
        // body force + this step's IB force (loads issued before the moments:
        // their latency hides behind them; consumed at the end of collide)
        float2 gx = make_float2(P.m.body[0], P.m.body[0]);
        float2 gy = make_float2(P.m.body[1], P.m.body[1]);
        float2 gz = make_float2(P.m.body[2], P.m.body[2]);
        // (gib is zero wherever the IB did not scatter this step: every
        // scattered node is zeroed here when consumed, so a forced chunk's
        // other nodes add +0 and need no store)
        if (forced) {
            float* gib = P.p.gib;
            const float2 a = __ldcg(reinterpret_cast<const float2*>(gib + k));
            const float2 b = __ldcg(reinterpret_cast<const float2*>(gib + k + g.ns));
            const float2 c = __ldcg(reinterpret_cast<const float2*>(gib + k + 2u * g.ns));
            gx = __fadd2_rn(gx, a);
            gy = __fadd2_rn(gy, b);
            gz = __fadd2_rn(gz, c);
            if (a.x != 0.f || a.y != 0.f || b.x != 0.f || b.y != 0.f || c.x != 0.f || c.y != 0.f) {
                *reinterpret_cast<float2*>(gib + k) = make_float2(0.f, 0.f);
                *reinterpret_cast<float2*>(gib + k + g.ns) = make_float2(0.f, 0.f);
                *reinterpret_cast<float2*>(gib + k + 2u * g.ns) = make_float2(0.f, 0.f);
            }
        }
        if (dbg & 3) {  // bandwidth probes: 1 = staged loads only, 2 = loads + stores (no collision)
            if ((dbg & 3) == 2)
                static_for<0, 27>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    *reinterpret_cast<float2*>(fout + g.gaddr(sl, i)) = fs[i];
                });
            else if (fs[0].x == 12345.f)
                fout[sl] = fs[26].y;
            continue;
        }

        const MacroV<float2> mc = moments_v<float2>(fs);
        if (mc.bad[0] || mc.bad[1]) {
            flag_divergence(ctr);
            continue;
        }
        if (mc.mach[0] || mc.mach[1]) raise_mach(ctr);
        if (write_macro) {
            *reinterpret_cast<float2*>(P.p.rho + k) = mc.rho;
            *reinterpret_cast<float2*>(P.p.u + k) = mc.ux;
            *reinterpret_cast<float2*>(P.p.u + k + g.ns) = mc.uy;
            *reinterpret_cast<float2*>(P.p.u + k + 2u * g.ns) = mc.uz;
        }
        const bool any_force = gx.x != 0.f || gx.y != 0.f || gy.x != 0.f || gy.y != 0.f || gz.x != 0.f || gz.y != 0.f;
        NoStash<float2> stash;
        collide_v<KIND, POLICY, STD, float2>(fs, mc, gx, gy, gz, any_force, P.m, stash);
        float* const ob = fout + g.gaddr(sl, 0);  // a tile never straddles a CSoA block
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            *reinterpret_cast<float2*>(ob + size_t(i) * g.A) = fs[i];
        });
        // crossing populations of the slab's boundary planes -> neighbour halos
        const unsigned hp = unsigned(y) * g.nx + unsigned(x);
        if (lz == 0 && P.p.send_lo[p ^ 1] != nullptr) {
            float* sd = P.p.send_lo[p ^ 1];
            static_for<1, 10>([&](auto I) {
                constexpr int i = decltype(I)::value;
                *reinterpret_cast<float2*>(sd + cross9(i, 2) * g.plane + hp) = fs[i];
            });
        }
        if (lz == g.nzl - 1 && P.p.send_hi[p ^ 1] != nullptr) {
            float* sd = P.p.send_hi[p ^ 1];
            static_for<18, 27>([&](auto I) {
                constexpr int i = decltype(I)::value;
                *reinterpret_cast<float2*>(sd + cross9(i, 2) * g.plane + hp) = fs[i];
            });
        }
    }
    // the last CTA out rewinds this launch's tile queue (all of its warps have
    // stopped claiming tiles: barrier first), so every launch starts at 0
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&P.p.queue[4 + slot], 1u) == gridDim.x - 1) {
            P.p.queue[slot] = 0u;
            P.p.queue[4 + slot] = 0u;
            __threadfence();
            if (end_step && !__ldcg(&ctr->diverged)) ctr->t += 1;  // step_end_kernel folded in
            if (end_step) publish_counters(P);
        }
    }
}

// Recompute rho*/u* of the current step from f(t) (after divergence, so the
// readback matches the reference's partially written moments, solver.cpp:113).
__global__ void macro_kernel(const FluidParams P, long long t) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    const RegionGeo& g = P.g;
    if (k >= g.n) return;
    const StepView v = make_view(P, t);
    int x, y, lz;
    decode(g, k, x, y, lz);
    float fs[27];
    gather_node<false>(P, v, nullptr, k, x, y, lz, fs);
    const MacroV<float> mc = moments_v<float>(fs);
    P.p.rho[k] = mc.rho;
    if (!mc.bad[0]) {
        P.p.u[k] = mc.ux;
        P.p.u[k + g.ns] = mc.uy;
        P.p.u[k + 2u * g.ns] = mc.uz;
    }
}

// IB band pre-pass: rho*, u* at the band nodes only.
__global__ void ib_band_kernel(const FluidParams P, const unsigned* band) {
    DevCounters* ctr = P.ctr;
    if (ctr->diverged) return;
    const unsigned count = *P.p.band_count;
    const RegionGeo& g = P.g;
    const StepView v = make_view(P, ctr->t);
    for (unsigned j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
        const unsigned k = band[j];
        int x, y, lz;
        decode(g, k, x, y, lz);
        float fs[27];
        gather_node<false>(P, v, nullptr, k, x, y, lz, fs);
        const MacroV<float> mc = moments_v<float>(fs);
        P.p.rho[k] = mc.rho;
        P.p.u[k] = mc.ux;
        P.p.u[k + g.ns] = mc.uy;
        P.p.u[k + 2u * g.ns] = mc.uz;
    }
}

// (rho,u) of the two boundary planes into the neighbours' macro halo.
__global__ void macro_pack_kernel(const FluidParams P) {
    if (P.ctr->diverged) return;
    const RegionGeo& g = P.g;
    const unsigned j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= g.plane) return;
    float* outs[2] = {P.p.msend_lo, P.p.msend_hi};
    const unsigned ks[2] = {j, unsigned(g.nzl - 1) * g.plane + j};
    for (int h = 0; h < 2; ++h) {
        if (!outs[h]) continue;
        const unsigned k = ks[h];
        outs[h][j] = P.p.rho[k];
        outs[h][j + g.plane] = P.p.u[k];
        outs[h][j + 2u * g.plane] = P.p.u[k + g.ns];
        outs[h][j + 3u * g.plane] = P.p.u[k + 2u * g.ns];
    }
}

__global__ void step_end_kernel(DevCounters* ctr) {
    if (!ctr->diverged) ctr->t += 1;
}

// Unit-level collide() on a batch (fp32, same code path): omega = f_out - f*.
template <int KIND, int POLICY, bool STD>
__global__ void collide_batch_kernel(ModelConst m, unsigned n, const double* f, const double* rho,
                                     const double* u, double* omega) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    float fs[27], f0[27];
    for (int i = 0; i < 27; ++i) {
        fs[i] = float(f[size_t(k) * 27 + i] - weight_d(i));
        f0[i] = fs[i];
    }
    MacroV<float> mc;
    mc.rho = float(rho[k]);
    mc.drho = float(rho[k] - 1.0);
    mc.ux = float(u[3 * k]);
    mc.uy = float(u[3 * k + 1]);
    mc.uz = float(u[3 * k + 2]);
    RegStash<float> stash;
    collide_v<KIND, POLICY, STD, float>(fs, mc, 0.f, 0.f, 0.f, false, m, stash);
    for (int i = 0; i < 27; ++i) omega[size_t(k) * 27 + i] = double(fs[i]) - double(f0[i]);
}

// ---------------------------------------------------------------------------
// Host launch wrappers.

namespace {

inline unsigned blocks_for(unsigned long long n, unsigned t) { return unsigned((n + t - 1) / t); }

#define CUDA_OK(x)                                                                                   \
    do {                                                                                             \
        const cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Collision output form (see StashFor; LBMG_FORM overrides, default 2 =
// feq + t'': fewest live registers, fastest measured, profiles/).
int fluid_form() {
    static const int v = [] {
        const char* e = std::getenv("LBMG_FORM");
        const int f = e ? std::atoi(e) : 2;
        return f < 0 || f > 2 ? 2 : f;
    }();
    return v;
}

}  // namespace

// Ghost-layer path availability (LBMG_BULK=ldg forces the compact layout and
// the register-direct kernels, for A/B comparisons).
bool ghost_layout_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("LBMG_BULK");
        return !(e && std::string(e) == "ldg") && fluid_form() == 2;
    }();
    return v;
}

namespace {

thread_local bool t_fill = true;  // launch_fluid(..., fill): the ghost fill is part of this launch
thread_local bool t_end = false;  // launch_fluid(..., end_step): the fluid kernel also ends the step

template <int KIND, int POLICY, bool STD, int T>
void launch_ghost_planes_t(const FluidParams& P, int z_a, int z_b, int slot, int write_macro, cudaStream_t st,
                           int end_step) {
    const RegionGeo& g = P.g;
    constexpr unsigned smem = staged_smem<T>();
    const unsigned ntiles = unsigned(z_b - z_a) * g.PP / GhostTile<T>::kTile + 2;
    // function attributes and occupancy are per device context: cached per device
    constexpr int kMaxDev = 64;
    static int grid_per_sm[kMaxDev] = {}, sms[kMaxDev] = {};
    auto kern = fluid_ghost_kernel<KIND, POLICY, STD, T>;
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    if (dev >= kMaxDev) throw std::runtime_error("fluid kernel: device index beyond the per-device cache");
    if (grid_per_sm[dev] == 0) {
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        CUDA_OK(cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev));
        int nb = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T, smem));
        grid_per_sm[dev] = nb > 0 ? nb : 1;
    }
    const unsigned grid = std::min<unsigned>(ntiles, unsigned(grid_per_sm[dev] * sms[dev]));
    static const int dbg = [] {
        const char* e = std::getenv("LBMG_GHOST_DBG");
        return e ? std::atoi(e) : 0;
    }();
    static const int pf_periods = [] {  // L2 prefetch distance in tile periods (0: off, measured best)
        const char* e = std::getenv("LBMG_L2_PREFETCH");
        return e ? std::atoi(e) : 0;
    }();
    kern<<<grid, T, smem, st>>>(P, z_a, z_b, slot, write_macro, dbg, pf_periods * kStages * int(grid), end_step);
}

// CTA size of the staged kernel (LBMG_GHOST_THREADS, default 512 = 1024-slot
// tiles, one CTA of 16 warps per SM, 2 x 111 KB stages: measured fastest,
// C3 4.92 ms vs 5.31 (256) vs 6.00 (128)); a tile must fit one Eq. 9 block.
template <int KIND, int POLICY, bool STD>
void launch_ghost_planes(const FluidParams& P, int z_a, int z_b, int slot, int write_macro, cudaStream_t st,
                         int end_step = 0) {
    if (z_b <= z_a) return;
    static const int env_threads = [] {
        const char* e = std::getenv("LBMG_GHOST_THREADS");
        return e ? std::atoi(e) : 512;
    }();
    const int threads = P.g.cta > 0 ? P.g.cta : env_threads;  // Runner::set_cta (tuner) wins
    const unsigned block = P.g.amask + 1u;  // Eq. 9 block (slots); SoA: 2^31
    if (threads >= 512 && block >= 1024u)
        launch_ghost_planes_t<KIND, POLICY, STD, 512>(P, z_a, z_b, slot, write_macro, st, end_step);
    else if (threads >= 256 && block >= 512u)
        launch_ghost_planes_t<KIND, POLICY, STD, 256>(P, z_a, z_b, slot, write_macro, st, end_step);
    else
        launch_ghost_planes_t<KIND, POLICY, STD, 128>(P, z_a, z_b, slot, write_macro, st, end_step);
}

// part 0: every plane; 1: ghost fill + the slab's boundary planes (which feed
// the halos); 2: the interior planes.
template <int KIND, int POLICY, bool STD>
void launch_fluid_ghost(const FluidParams& P, int part, int write_macro, cudaStream_t st) {
    const RegionGeo& g = P.g;
    if ((part == 0 || part == 1) && t_fill) launch_ghost_fill(P, st);
    if (part == 0) {
        launch_ghost_planes<KIND, POLICY, STD>(P, 0, g.nzl, 0, write_macro, st, t_end ? 1 : 0);
    } else if (part == 1) {
        launch_ghost_planes<KIND, POLICY, STD>(P, 0, 1, 0, write_macro, st);
        if (g.nzl > 1) launch_ghost_planes<KIND, POLICY, STD>(P, g.nzl - 1, g.nzl, 1, write_macro, st);
    } else {
        launch_ghost_planes<KIND, POLICY, STD>(P, 1, g.nzl - 1, 2, write_macro, st);
    }
}

template <int KIND, int POLICY, bool STD, int FORM>
void launch_fluid_t(const FluidParams& P, int part, int write_macro, cudaStream_t st) {
    const RegionGeo& g = P.g;
    if (g.ghost) {
        if constexpr (FORM == 2) launch_fluid_ghost<KIND, POLICY, STD>(P, part, write_macro, st);
        return;
    }
    const bool bulk_ok = (g.nx % 2 == 0) && g.nx >= 4 && g.ny >= 3 && g.nzl >= 3;
    const unsigned zpart = (g.nzl >= 2 ? 2u : 1u) * g.plane;
    const unsigned shell_total =
        zpart + (g.nzl >= 3 ? unsigned(g.nzl - 2) * (2u * g.nx + 2u * (g.ny - 2)) : 0u);
    if (!bulk_ok) {  // odd nx or thin slabs: general path over every node
        if (part == 1) return;
        fluid_shell_kernel<KIND, POLICY, STD, FORM><<<blocks_for(g.n, 128), 128, 0, st>>>(P, 0, g.n, write_macro, 1);
        return;
    }
    if (part == 0 || part == 2) {
        const unsigned kb = g.plane, ke = g.n - g.plane;
        const unsigned warps = (ke - kb + 63) / 64;
        const unsigned nb = blocks_for(warps, kBulkThreads / 32);
        if (g.la == 31)
            fluid_bulk_kernel<KIND, POLICY, STD, true, FORM><<<nb, kBulkThreads, 0, st>>>(P, kb, ke, write_macro);
        else
            fluid_bulk_kernel<KIND, POLICY, STD, false, FORM><<<nb, kBulkThreads, 0, st>>>(P, kb, ke, write_macro);
    }
    unsigned s0 = 0, s1 = shell_total;
    if (part == 1) s1 = zpart;
    if (part == 2) s0 = zpart;
    if (s1 > s0)
        fluid_shell_kernel<KIND, POLICY, STD, FORM><<<blocks_for(s1 - s0, 128), 128, 0, st>>>(P, s0, s1, write_macro, 0);
}

template <int KIND, int POLICY, int FORM>
void launch_fluid_std(const FluidParams& P, int part, int write_macro, cudaStream_t st) {
    if (rates_standard(P.m.rate)) launch_fluid_t<KIND, POLICY, true, FORM>(P, part, write_macro, st);
    else launch_fluid_t<KIND, POLICY, false, FORM>(P, part, write_macro, st);
}

template <int FORM>
void launch_fluid_form(const FluidParams& P, int part, int write_macro, cudaStream_t st) {
    const int kind = P.m.kind, pol = P.m.policy;
    if (kind == kBGK) launch_fluid_t<kBGK, kPolicyConstant, false, FORM>(P, part, write_macro, st);
    else if (kind == kRawMRT) launch_fluid_std<kRawMRT, kPolicyConstant, FORM>(P, part, write_macro, st);
    else if (pol == kPolicyConstant) launch_fluid_std<kCentralMRT, kPolicyConstant, FORM>(P, part, write_macro, st);
    else launch_fluid_std<kCentralMRT, kPolicyRelax, FORM>(P, part, write_macro, st);
}

}  // namespace

// part: 0 every node, 1 the two halo planes (edge), 2 the rest (bulk).
void launch_ghost_fill(const FluidParams& P, cudaStream_t st, bool full) {
    const RegionGeo& g = P.g;
    if (!full && P.p.fill_plan[0] != nullptr) {
        const unsigned nb = fill_blocks(P.p, 256u);
        if (nb) ghost_copy_kernel<<<nb, 256, 0, st>>>(P);
        return;
    }
    const unsigned long long entries =
        18ull * (unsigned long long)(unsigned(g.ny) * g.nzl + unsigned(g.nx) * g.nzl + g.plane);
    ghost_fill_kernel<<<blocks_for(entries, 256), 256, 0, st>>>(P, full ? 1 : 0);
}

void launch_fill_plan(const FluidParams& P, int p, FillRec* out, unsigned eoff, unsigned* count_dev,
                      unsigned counts[2], cudaStream_t st) {
    const RegionGeo& g = P.g;
    const unsigned long long entries =
        18ull * (unsigned long long)(unsigned(g.ny) * g.nzl + unsigned(g.nx) * g.nzl + g.plane);
    CUDA_OK(cudaMemsetAsync(count_dev, 0, 2 * sizeof(unsigned), st));
    ghost_plan_kernel<<<blocks_for(entries, 256), 256, 0, st>>>(P, p, out, eoff, count_dev);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(counts, count_dev, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
}

bool launch_fluid(const FluidParams& P, int part, int write_macro, cudaStream_t st, bool fill, bool end_step) {
    t_fill = fill;
    t_end = end_step && part == 0 && P.g.ghost && fluid_form() == 2;
    switch (fluid_form()) {
        case 0: launch_fluid_form<0>(P, part, write_macro, st); break;
        case 1: launch_fluid_form<1>(P, part, write_macro, st); break;
        default: launch_fluid_form<2>(P, part, write_macro, st); break;
    }
    return t_end;
}

void launch_macro(const FluidParams& P, long long t, cudaStream_t st) {
    macro_kernel<<<blocks_for(P.g.n, 256), 256, 0, st>>>(P, t);
}

void launch_ib_band(const FluidParams& P, const unsigned* band, int sm_count, cudaStream_t st) {
    ib_band_kernel<<<sm_count * 4, 128, 0, st>>>(P, band);
}

void launch_macro_pack(const FluidParams& P, cudaStream_t st) {
    macro_pack_kernel<<<blocks_for(P.g.plane, 256), 256, 0, st>>>(P);
}

void launch_step_end(DevCounters* ctr, cudaStream_t st) { step_end_kernel<<<1, 1, 0, st>>>(ctr); }

void launch_collide_batch(const ModelConst& m, unsigned n, const double* f, const double* rho, const double* u,
                          double* omega, cudaStream_t st) {
    const unsigned b = blocks_for(n, 128);
    // collide() takes arbitrary (f, rho, u): keep the literal rates (rate 1 on
    // the conserved rows), not the STD shortcut that assumes they are moments of f
    const bool sd = false;
    if (m.kind == kBGK) collide_batch_kernel<kBGK, kPolicyConstant, false><<<b, 128, 0, st>>>(m, n, f, rho, u, omega);
    else if (m.kind == kRawMRT && sd) collide_batch_kernel<kRawMRT, kPolicyConstant, true><<<b, 128, 0, st>>>(m, n, f, rho, u, omega);
    else if (m.kind == kRawMRT) collide_batch_kernel<kRawMRT, kPolicyConstant, false><<<b, 128, 0, st>>>(m, n, f, rho, u, omega);
    else if (m.policy == kPolicyConstant && sd) collide_batch_kernel<kCentralMRT, kPolicyConstant, true><<<b, 128, 0, st>>>(m, n, f, rho, u, omega);
    else if (m.policy == kPolicyConstant) collide_batch_kernel<kCentralMRT, kPolicyConstant, false><<<b, 128, 0, st>>>(m, n, f, rho, u, omega);
    else if (sd) collide_batch_kernel<kCentralMRT, kPolicyRelax, true><<<b, 128, 0, st>>>(m, n, f, rho, u, omega);
    else collide_batch_kernel<kCentralMRT, kPolicyRelax, false><<<b, 128, 0, st>>>(m, n, f, rho, u, omega);
}

}  // namespace lbmg
