// Step pipeline: one persistent launch runs K whole time steps of a single
// ghost-layout region (runner.cpp:121-230 per step: the six face passes,
// IB interpolate/penalty/spread + totals + rigid motion, stream + moments +
// CM-MRT/ACM collision + forcing) as ONE ordered stream of work items:
//
//   FILL(j, w, c)  ghost-fill entries of the face nodes of plane w
//                  (apply_face, boundary.cpp:42-125; chunk c of the plane)
//   IB(j, b)       64 solid samples: f* of the 8 support nodes, trilinear
//                  interpolation, penalty, scatter (ib.cpp:321-454), reaction
//                  totals (ib.cpp:491-501), rigid motion to t+1 (ib.cpp:456-489)
//   TILE(j, k)     1024 storage slots: TMA-staged pulls, moments, collision,
//                  forcing, 64-bit stores of f(t+1)
//
// Tiles are claimed in order (step-major) by each CTA's TMA producer; fill and
// IB items, in their own order (plane by plane, IB after the fill of the
// last IB plane), by each CTA's helper warps; every item waits on per-plane
// completion counters instead of kernel boundaries:
//
//   FILL(j, w)  tiles of step j-1 on planes w-1..w+1 (z-periodic: wrapped)
//   IB(j)       FILL(j) on the IB planes, IB(j-1), all tiles of step j-2
//   TILE(j, k)  FILL(j) on its planes, IB(j) if it touches the IB planes,
//               all tiles of step j-2
//
// (per plane, step j's tiles cannot finish before step j-1's: FILL(j, w)
// waits for them, so cumulative per-plane counters are exact; whole-step
// completion is counted per step)
//
// so step j+1 starts on the low planes while step j finishes the high ones
// (no launch gap, no ramp or tail per step) and the fill / IB of a plane read
// data the previous step wrote a few planes ago — L2 hits.  f rotates through
// three buffers (fcur/fnext, nbuf = 3): step j+1 never writes f(j), so a
// step that diverges leaves f(t) intact, as the reference does
// (runner.cpp:154-161); later items are skipped once it is flagged.
//
// CTA: 4 consumer warpgroups (512 threads, 120 registers each after
// setmaxnreg: tiles only) + 1 producer warpgroup (32 registers): one thread
// claims tiles, waits for their dependencies and issues the 27 TMA window
// copies into a 2-stage shared-memory ring (full/empty mbarriers); 3 helper
// warps claim and run the fill and IB items, so that work overlaps the tiles
// without adding to the consumers' register pressure.  Completion of an item is
// published by the last consumer warp (per-warp gpu fence, CTA counter, then
// one release add on the global counter); a warp publishes its previous item
// when it picks up the next one (before blocking on it, and before the next
// tile's 54 floats go live in registers).  Dependency waits trap after a few seconds
// instead of hanging the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "collision.cuh"
#include "device_common.cuh"
#include "engine.hpp"
#include "fluid_dev.cuh"
#include "ib_dev.cuh"
#include "tma.cuh"

namespace lbmg {

namespace {

constexpr int kPStages = 2;
constexpr unsigned kEndItem = 0xffffffffu;

// Polling uses relaxed loads (an acquire load invalidates the SM's whole L1
// every time: CCTL.IVALL); one acquire fence once the wait is over.
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.global.relaxed.gpu.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acquire.gpu;" ::: "memory"); }
// release-only fence: MEMBAR, no L1 invalidation (__threadfence also invalidates)
__device__ __forceinline__ void fence_release() { asm volatile("fence.release.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned atom_release_add(unsigned* p, unsigned v) {
    unsigned o;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
    return o;
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


// Wait until *p >= target (wrap-safe).  A dependency that never resolves is a
// bug: trap (the launch fails) instead of hanging the device.
__device__ __forceinline__ unsigned spin_ge(const unsigned* p, unsigned target) {
    unsigned ns = 32, spins = 0, v;
    while (int((v = ld_relaxed(p)) - target) < 0) {
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;  // back off: many CTAs poll the same counters
        if (++spins > (1u << 24)) __trap();
    }
    fence_acquire();
    return v;
}


__device__ __forceinline__ unsigned plane_of(const RegionGeo& g, unsigned slot) {
    return g.div_py.div(g.div_px.div(slot - g.base));  // storage plane (lz + 1)
}

// owned planes [wa, wb] covered by tile k (tile = slots per tile)
__device__ __forceinline__ void tile_planes(const RegionGeo& g, unsigned org, unsigned tile, unsigned k, int& wa,
                                            int& wb) {
    const unsigned sb = g.base + g.PP, se = g.base + unsigned(g.nzl + 1) * g.PP;
    const unsigned a = max(org + k * tile, sb);
    const unsigned b = min(org + (k + 1) * tile, se) - 1u;
    wa = int(plane_of(g, a)) - 1;
    wb = int(plane_of(g, b)) - 1;
}

// One ghost-fill entry as (source, destination): the value f*_i of face node
// N that the pull of N reads from ghost slot s(N) - off_i (ghost_fill_entry,
// fluid_dev.cuh).  The source is a population of f(t), a stale face slot or
// a halo plane (src != nullptr, read through L2: other CTAs wrote it in this
// launch), or an inlet constant (cval).
struct FillOp {
    const float* src;
    float cval;
    unsigned long long dst;  // float offset into f[fcur(t)]
    float* slot;             // persistent face slot to refresh, or nullptr
};

__device__ __forceinline__ void pull_plan(const FluidParams& P, long long t, int x, int y, int lz, int i,
                                          const float*& src, float& cval) {
    const RegionGeo& g = P.g;
    const int p = int(t & 1);
    const float* fin = P.p.f[fcur(g, t)];
    auto pull_addr = [&](int xx, int yy, int zz) -> const float* {
        int sx = xx - cx(i), sy = yy - cy(i);
        if (sx < 0) sx += g.nx;
        else if (sx >= g.nx) sx -= g.nx;
        if (sy < 0) sy += g.ny;
        else if (sy >= g.ny) sy -= g.ny;
        const int lzs = zz - cz(i);
        const unsigned hp = cross9(i, 2) * g.plane + unsigned(sy) * g.nx + unsigned(sx);
        if (lzs < 0) return P.p.recv_lo[p] + hp;
        if (lzs >= g.nzl) return P.p.recv_hi[p] + hp;
        return fin + g.at(sx, sy, lzs, i);
    };
    src = nullptr;
    cval = 0.f;
    int f = owner_face(g, x, y, g.gz0 + lz, i);
    if (f == kNoOwner) {
        src = pull_addr(x, y, lz);
        return;
    }
    for (int guard = 0; guard < 7; ++guard) {
        const int cond = P.faces.cond[f];
        if (cond == kNoSlip) {
            src = fin + g.at(x, y, lz, opposite(i));
            return;
        }
        if (cond == kInlet) {
            cval = P.faces.inlet[f][i];
            return;
        }
        const int a = face_axis(f), s = face_side(f);
        if (a == 0) x -= s;
        else if (a == 1) y -= s;
        else lz -= s;
        const int fn = owner_face(g, x, y, g.gz0 + lz, i);
        if (fn == kNoOwner) {
            src = pull_addr(x, y, lz);
            return;
        }
        if (fn > f) {
            src = P.p.slot[p][fn] + g.slot_index(fn, x, y, lz, i);
            return;
        }
        f = fn;
    }
}

// Entry e of plane w's fill list: x faces (2 x 9 x ny), y faces (2 x 9 x nx),
// then the z face entries of the slab's first / last plane (9 x nx x ny each).
__device__ __forceinline__ FillOp fill_plan(const FluidParams& P, long long t, int w, unsigned e) {
    const RegionGeo& g = P.g;
    const unsigned X = 9u * unsigned(g.ny), Y = 9u * unsigned(g.nx), Z = 9u * g.plane;
    int F, x, y, lz = w;
    unsigned j;
    if (e < 2u * X) {
        F = e >= X ? 1 : 0;
        const unsigned r = e - unsigned(F) * X;
        j = g.div_ny.div(r);
        y = int(r - j * unsigned(g.ny));
        x = F == 0 ? 0 : g.nx - 1;
    } else if (e < 2u * X + 2u * Y) {
        const unsigned e2 = e - 2u * X;
        F = e2 >= Y ? 3 : 2;
        const unsigned r = e2 - unsigned(F - 2) * Y;
        j = g.div_nx.div(r);
        x = int(r - j * unsigned(g.nx));
        y = F == 2 ? 0 : g.ny - 1;
    } else {
        unsigned e3 = e - 2u * X - 2u * Y;
        F = (w == 0 && e3 < Z) ? 4 : 5;
        if (F == 5 && w == 0) e3 -= Z;  // nzl == 1: both z faces in plane 0
        const unsigned q = e3 % g.plane;
        j = e3 / g.plane;
        const unsigned yy = g.div_nx.div(q);
        y = int(yy);
        x = int(q - yy * unsigned(g.nx));
    }
    const int A = face_axis(F), S = face_side(F);
    const int ja = int(j % 3u) - 1, jb = int(j / 3u) - 1;
    const int c0 = A == 0 ? -S : ja, c1 = A == 0 ? ja : (A == 1 ? -S : jb), c2 = A == 2 ? -S : jb;
    const int i = tensor_dir((c0 + 1) + 3 * (c1 + 1) + 9 * (c2 + 1));
    FillOp op;
    pull_plan(P, t, x, y, lz, i, op.src, op.cval);
    const unsigned sn = g.sidx(x, y, lz);
    op.dst = g.gaddr((unsigned long long)((long long)sn - g.soff(i)), i);
    op.slot = nullptr;
    const int own = owner_face(g, x, y, g.gz0 + lz, i);
    if (own != kNoOwner && slot_readable(P, x, y, g.gz0 + lz))
        op.slot = P.p.slot[int(t & 1) ^ 1][own] + g.slot_index(own, x, y, lz, i);
    return op;
}

struct Pending {
    unsigned code;  // kEndItem: nothing pending
    unsigned j;
    unsigned s, ph;
};

}  // namespace

__global__ void pipeline_begin_kernel(PipeCounters* pc, DevCounters* ctr, int nzl) {
    for (int k = threadIdx.x; k < 2 * nzl; k += blockDim.x) pc->plane[k] = 0u;
    for (int k = threadIdx.x; k < kPipeMaxSteps; k += blockDim.x) pc->step_tiles[k] = 0u;
    if (threadIdx.x == 0) {
        pc->ticket = 0u;
        pc->ib_done = 0u;
        pc->t_launch = ctr->t;
        pc->div_min = ctr->diverged ? 0ull : ~0ull;
    }
}

namespace {

constexpr int kThreads = 512;  // 16 warps, every one a consumer of every item
constexpr int kWarps = kThreads / 32;
using Tile = GhostTile<kThreads>;  // 1024-slot tiles
constexpr unsigned kParkNone = 0xffffffffu;

__device__ __forceinline__ void named_sync_all() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

// Ghost-fill item: entries [e0, e1) of plane w, four in flight per thread.
__device__ __forceinline__ void pipe_fill_item(const PipeParams& Q, unsigned idx, long long t, unsigned tid) {
    const FluidParams& P = Q.P;
    const RegionGeo& g = P.g;
    const int w = int(__ldg(&Q.fill_desc[3 * idx]));
    const unsigned e0 = __ldg(&Q.fill_desc[3 * idx + 1]), e1 = __ldg(&Q.fill_desc[3 * idx + 2]);
    float* const fin = P.p.f[fcur(g, t)];
    constexpr int kB = 4;
    for (unsigned e = e0 + tid; e < e1; e += kB * kThreads) {
        FillOp op[kB];
        float v[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const unsigned ee = e + unsigned(b) * kThreads;
            if (ee < e1) op[b] = fill_plan(P, t, w, ee);
            else op[b].dst = ~0ull;
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) v[b] = op[b].dst == ~0ull ? 0.f : (op[b].src ? __ldcg(op[b].src) : op[b].cval);
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            if (op[b].dst == ~0ull) continue;
            fin[op[b].dst] = v[b];
            if (op[b].slot) *op[b].slot = v[b];
        }
    }
}

// IB item: 64 samples of one solid, 4 per warp, 8 lanes (the support
// corners) each: f* of the corner node -> rho*, j* (shuffle reduction), FP64
// interpolation and penalty (ib.cpp:321-365), fp32 RED scatter into g with
// the step's force flag (ib.cpp:369-454, atomic mode; single region: every
// support node is owned), reaction totals in a fixed order (ib.cpp:491-501:
// the warp's samples, the warps, the items of the solid) and rigid motion to
// t+1 (ib.cpp:456-489).
__device__ __forceinline__ void pipe_ib_item(const PipeParams& Q, unsigned idx, long long t, unsigned char epoch,
                                             unsigned tid, double (*red)[6]) {
    const FluidParams& P = Q.P;
    const RegionGeo& g = P.g;
    DevCounters* const ctr = P.ctr;
    const unsigned lane = tid & 31u, warp = tid >> 5;
    const IbBatch& B = Q.B;
    unsigned lo = 0, hi = B.n_solids;
    while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        if (__ldg(&Q.ib_item_start[mid]) <= idx) lo = mid;
        else hi = mid;
    }
    const unsigned solid = lo;
    const IbSolidDev S = B.solids[solid];
    const unsigned i0 = __ldg(&Q.ib_item_start[solid]);
    const unsigned nitems = __ldg(&Q.ib_item_start[solid + 1]) - i0;
    const double* row = B.table + size_t(solid) * B.table_stride + (t - ctr->chunk_t0) * kMotionRow;
    const int moving = B.moving[solid];
    const unsigned corner = lane & 7u;
    const int ox = int(corner & 1u), oy = int((corner >> 1) & 1u), oz = int(corner >> 2);
    const unsigned smp = (idx - i0) * kPipeIbSamples + warp * 4u + (lane >> 3);
    const bool have = smp < S.n;
    const unsigned si = have ? smp : 0u;
    const double pos[3] = {__ldcg(&S.pos[3 * si]), __ldcg(&S.pos[3 * si + 1]), __ldcg(&S.pos[3 * si + 2])};
    const Support ks = kernel_support(pos, g.nx, g.ny, g.NZ);
    if (have && corner == 0) S.flagged[smp] = ks.inside ? 0 : 1;
    const bool act = have && ks.inside;
    const int x = act ? ks.base[0] + ox : 0, y = act ? ks.base[1] + oy : 0;
    const int lz = act ? ks.base[2] + oz - g.gz0 : 0;
    const long long sl = g.sidx(x, y, lz);
    const float* fin = P.p.f[fcur(g, t)];
    float v[27];
#pragma unroll
    for (int i = 0; i < 27; ++i) v[i] = __ldcg(&fin[g.gaddr((unsigned long long)(sl - g.soff(i)), i)]);
    float rr = 0.f, jx = 0.f, jy = 0.f, jz = 0.f;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        rr += v[i];
        jx += float(cx(i)) * v[i];
        jy += float(cy(i)) * v[i];
        jz += float(cz(i)) * v[i];
    }
    const float rho = 1.0f + rr;
    const float inv = 1.0f / rho;
    const double wx = ox ? ks.w[0][1] : ks.w[0][0], wy = oy ? ks.w[1][1] : ks.w[1][0];
    const double wz = oz ? ks.w[2][1] : ks.w[2][0];
    const double wgt = __dmul_rn(__dmul_rn(wx, wy), wz);
    double c4[4] = {wgt * double(jx * inv), wgt * double(jy * inv), wgt * double(jz * inv), wgt * double(rho)};
#pragma unroll
    for (int o = 1; o < 8; o <<= 1)
#pragma unroll
        for (int a = 0; a < 4; ++a) c4[a] += __shfl_xor_sync(0xffffffffu, c4[a], o);
    double us[3] = {0.0, 0.0, 0.0}, fg[3] = {0.0, 0.0, 0.0};
    if (act) {
        for (int a = 0; a < 3; ++a) {
            us[a] = c4[a];
            fg[a] = c4[3] * (__ldcg(&S.ub[3 * smp + a]) - us[a]);
        }
        const unsigned k = g.node(x, y, lz);
        atomicAdd(&P.p.gib[k], float(wgt * fg[0]));
        atomicAdd(&P.p.gib[k + g.ns], float(wgt * fg[1]));
        atomicAdd(&P.p.gib[k + 2u * g.ns], float(wgt * fg[2]));
        P.p.tflag[k] = epoch;
    }
    double tot[6] = {0, 0, 0, 0, 0, 0};
    if (have && corner == 0) {
        const size_t po = ib_half(S, t);
        for (int a = 0; a < 3; ++a) {
            S.sampled[po + 3 * smp + a] = us[a];
            S.force[po + 3 * smp + a] = fg[a];
        }
        if (pos[2] >= double(g.gz0) && pos[2] < double(g.gz0 + g.nzl)) {
            const double rv[3] = {pos[0] - row[0], pos[1] - row[1], pos[2] - row[2]};
            tot[0] = -fg[0];
            tot[1] = -fg[1];
            tot[2] = -fg[2];
            tot[3] = -(rv[1] * fg[2] - rv[2] * fg[1]);
            tot[4] = -(rv[2] * fg[0] - rv[0] * fg[2]);
            tot[5] = -(rv[0] * fg[1] - rv[1] * fg[0]);
        }
        if (moving) motion_apply(row + kMotionRow, S, smp, g.nx, g.ny, g.NZ);
    }
#pragma unroll
    for (int a = 0; a < 6; ++a) {
        tot[a] += __shfl_xor_sync(0xffffffffu, tot[a], 8);
        tot[a] += __shfl_xor_sync(0xffffffffu, tot[a], 16);
    }
    if (lane == 0)
        for (int a = 0; a < 6; ++a) red[warp][a] = tot[a];
    named_sync_all();
    if (warp == 0) {
        if (lane < 6) {
            double acc = 0.0;
            for (int w2 = 0; w2 < kWarps; ++w2) acc += red[w2][lane];
            B.partial[size_t(idx) * 6 + lane] = acc;
        }
        fence_release();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) last = atomicAdd(&B.done[solid], 1u) == nitems - 1u ? 1u : 0u;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            fence_acquire();
            double acc[6] = {0, 0, 0, 0, 0, 0};
            for (unsigned b = lane; b < nitems; b += 32)
                for (int a = 0; a < 6; ++a) acc[a] += __ldcg(&B.partial[size_t(i0 + b) * 6 + a]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int a = 0; a < 6; ++a) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], o);
            if (lane == 0) {
                double* out = B.out_base + 6 * solid + (t - ctr->chunk_t0) * B.out_stride;
                for (int a = 0; a < 6; ++a) out[a] = acc[a];
                B.done[solid] = 0u;
            }
        }
    }
}

// Dependencies of item `code` of launch step j (all on items with smaller
// tickets); the counters only grow within a launch.
struct DepView {
    const PipeParams* Q;
    const unsigned* fill_done;
    const unsigned* tile_done;
    int nzl, zwrap;
    unsigned org;
};

template <bool BLOCK>
__device__ __forceinline__ bool ready_ge(const unsigned* p, unsigned target) {
    if constexpr (!BLOCK) return int(ld_relaxed(p) - target) >= 0;
    spin_ge(p, target);
    return true;
}

template <bool BLOCK>
__device__ __forceinline__ bool deps_ready(const DepView& D, unsigned code, unsigned j) {
    const PipeParams& Q = *D.Q;
    const RegionGeo& g = Q.P.g;
    const unsigned type = code >> kPipeTypeShift, idx = code & kPipeIdxMask;
    PipeCounters* const pc = Q.pc;
    if (type == kPipeItemFill) {
        if (j == 0) return true;
        const int w = int(__ldg(&Q.fill_desc[3 * idx]));
        for (int d = -1; d <= 1; ++d) {
            int w2 = w + d;
            if (w2 < 0 || w2 >= D.nzl) {
                if (!D.zwrap) continue;
                w2 = (w2 + D.nzl) % D.nzl;
            }
            if (!ready_ge<BLOCK>(&D.tile_done[w2], j * __ldg(&Q.tile_need[w2]))) return false;
        }
        return true;
    }
    if (type == kPipeItemTile) {
        int wa, wb;
        tile_planes(g, D.org, unsigned(Tile::kTile), idx, wa, wb);
        for (int w = wa; w <= wb; ++w)
            if (!ready_ge<BLOCK>(&D.fill_done[w], (j + 1) * __ldg(&Q.fill_need[w]))) return false;
        if (Q.n_ib && wb >= Q.z0_ib && wa <= Q.z1_ib && !ready_ge<BLOCK>(&pc->ib_done, (j + 1) * Q.n_ib))
            return false;
        if (j >= 2 && !ready_ge<BLOCK>(&pc->step_tiles[j - 2], Q.n_tiles)) return false;
        return true;
    }
    for (int w = Q.z0_ib; w <= Q.z1_ib; ++w)
        if (!ready_ge<BLOCK>(&D.fill_done[w], (j + 1) * __ldg(&Q.fill_need[w]))) return false;
    if (j >= 1 && !ready_ge<BLOCK>(&pc->ib_done, j * Q.n_ib)) return false;
    if (j >= 2 && !ready_ge<BLOCK>(&pc->step_tiles[j - 2], Q.n_tiles)) return false;
    return true;
}

}  // namespace

template <int KIND, int POLICY, bool STD>
__global__ void __launch_bounds__(kThreads, 1) pipeline_kernel(const __grid_constant__ PipeParams Q) {
    constexpr int kWin = Tile::kWin;
    constexpr unsigned kStageBytes = Tile::kStageBytes;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* const stage0 = reinterpret_cast<float*>(smem_raw);
    uint64_t* const full = reinterpret_cast<uint64_t*>(smem_raw + kPStages * kStageBytes);
    __shared__ unsigned stage_item[kPStages];
    __shared__ unsigned stage_step[kPStages];
    __shared__ unsigned parked[kPStages];     // claimed ticket waiting for its dependencies
    __shared__ unsigned reads_done[kPStages];
    __shared__ unsigned work_done[kPStages][2];
    __shared__ double red[kPStages][kWarps][6];
    __shared__ Pending pend_sm[kWarps];
    __shared__ unsigned char step_cur[kPipeMaxSteps], step_next[kPipeMaxSteps], step_epoch[kPipeMaxSteps];

    const FluidParams& P = Q.P;
    const RegionGeo& g = P.g;
    PipeCounters* const pc = Q.pc;
    unsigned* const fill_done = pc->plane;
    unsigned* const tile_done = pc->plane + g.nzl;
    const long long t0 = pc->t_launch;
    const unsigned total = Q.K * Q.n_items;
    const unsigned tid = threadIdx.x;
    const unsigned lane = tid & 31u, warp = tid >> 5;
    DevCounters* const ctr = P.ctr;
    const DepView D{&Q, fill_done, tile_done, g.nzl, g.zwrap, Q.org};

    if (tid == 0) {
        for (int s = 0; s < kPStages; ++s) {
            mbar_init(&full[s], 1);
            parked[s] = kParkNone;
            reads_done[s] = 0u;
            work_done[s][0] = work_done[s][1] = 0u;
        }
        fence_mbar_init();
    }
    if (lane == 0) pend_sm[warp].code = kEndItem;
    if (tid < kPipeMaxSteps) {  // per step: buffer of f(t), of f(t+1), IB epoch (64-bit % once)
        const long long t = t0 + tid;
        step_cur[tid] = (unsigned char)fcur(g, t);
        step_next[tid] = (unsigned char)fnext(g, t);
        step_epoch[tid] = ib_epoch(t);
    }
    __syncthreads();

    // Put item `ticket` into stage s: its descriptor, then the tile's 27 TMA
    // window copies (or a plain arrive).  Called once its dependencies hold.
    auto issue = [&](int s, unsigned ticket) {
        if (ticket >= total) {
            stage_item[s] = kEndItem;
            mbar_arrive(&full[s]);
            return;
        }
        const unsigned j = ticket / Q.n_items;
        unsigned code = __ldg(&Q.pattern[ticket - j * Q.n_items]);
        fence_acquire();  // (the dependency counters were read relaxed)
        // a step that diverged freezes the state: later steps are skipped
        const unsigned long long dmin = *reinterpret_cast<volatile unsigned long long*>(&pc->div_min);
        if (dmin < (unsigned long long)(t0 + (long long)j)) code |= kPipeSkip;
        stage_item[s] = code;
        stage_step[s] = j;
        if ((code >> kPipeTypeShift) == kPipeItemTile && !(code & kPipeSkip)) {
            const float* fin = P.p.f[step_cur[j]];
            const long long k0 = (long long)Q.org + (long long)(code & kPipeIdxMask) * Tile::kTile;
            float* dst = stage0 + s * (kStageBytes / 4);
            asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> async-proxy reads
            mbar_arrive_expect_tx(&full[s], kStageBytes);
            static_for<0, 27>([&](auto I) {
                constexpr int i = decltype(I)::value;
                const unsigned long long a0 = (unsigned long long)(k0 - g.soff(i) - win_shift(i));
                const unsigned long long e0 = (a0 | g.amask) + 1ull;
                const unsigned l0 = e0 - a0 < (unsigned long long)kWin ? unsigned(e0 - a0) : unsigned(kWin);
                tma_load_1d(dst + i * kWin, fin + g.gaddr(a0, i), l0 * 4u, &full[s]);
                if (l0 < unsigned(kWin))
                    tma_load_1d(dst + i * kWin + l0, fin + g.gaddr(e0, i), (kWin - l0) * 4u, &full[s]);
            });
        } else {
            mbar_arrive(&full[s]);
        }
    };
    // Refill (the last warp to release a stage): claim the next ticket; issue
    // it when its dependencies already hold, else park it for whichever warp
    // reaches the stage first (a refilling warp never blocks: it may still
    // owe work on the other stage's item).
    auto refill = [&](int s) {
        fence_proxy_async_smem();  // this CTA's generic reads of stage s before the TMA writes
        const unsigned ticket = atomicAdd(&pc->ticket, 1u);
        if (ticket >= total) {
            issue(s, ticket);
            return;
        }
        const unsigned j = ticket / Q.n_items;
        const unsigned code = __ldg(&Q.pattern[ticket - j * Q.n_items]);
        if (deps_ready<false>(D, code, j)) issue(s, ticket);
        else parked[s] = ticket;
    };

    // publish the completion of this warp's previous item (the last warp of
    // the CTA to do so bumps the counter its dependants wait on)
    auto publish = [&]() {
        const Pending pend = pend_sm[warp];
        if (pend.code == kEndItem) return;
        fence_release();
        __syncwarp();
        if (lane == 0 && atomicAdd(&work_done[pend.s][pend.ph], 1u) == unsigned(kWarps - 1)) {
            work_done[pend.s][pend.ph] = 0u;
            const unsigned type = pend.code >> kPipeTypeShift, idx = pend.code & kPipeIdxMask;
            if (type == kPipeItemTile) {
                int wa, wb;
                tile_planes(g, Q.org, unsigned(Tile::kTile), idx, wa, wb);
                for (int w = wa; w <= wb; ++w) red_release_add(&tile_done[w], 1u);
                const unsigned done = atom_release_add(&pc->step_tiles[pend.j], 1u) + 1u;
                if (done == Q.n_tiles) {  // every tile of step j is in
                    fence_acquire();     // (sees the divergence flags of the step's other tiles)
                    const long long t = t0 + (long long)pend.j;
                    const unsigned long long dmin = *reinterpret_cast<volatile unsigned long long*>(&pc->div_min);
                    if (dmin > (unsigned long long)t) *reinterpret_cast<volatile long long*>(&ctr->t) = t + 1;
                }
            } else if (type == kPipeItemFill) {
                red_release_add(&fill_done[__ldg(&Q.fill_desc[3 * idx])], 1u);
            } else {
                red_release_add(&pc->ib_done, 1u);
            }
        }
        __syncwarp();
        if (lane == 0) pend_sm[warp].code = kEndItem;
        __syncwarp();
    };

    if (tid == 0)
        for (int s = 0; s < kPStages; ++s) refill(s);

#pragma unroll 1
    for (unsigned it = 0;; ++it) {
        const int s = int(it % kPStages);
        const unsigned ph = (it / kPStages) & 1u;
        if (!mbar_test_parity(&full[s], ph)) {
            publish();  // never hold a completion while blocked
            // a parked item: the first warp here waits for its dependencies
            // (it owes nothing else) and issues it
            if (lane == 0 && *reinterpret_cast<volatile unsigned*>(&parked[s]) != kParkNone) {
                const unsigned ticket = atomicExch(&parked[s], kParkNone);
                if (ticket != kParkNone) {
                    const unsigned j = ticket / Q.n_items;
                    deps_ready<true>(D, __ldg(&Q.pattern[ticket - j * Q.n_items]), j);
                    issue(s, ticket);
                }
            }
            __syncwarp();
            mbar_wait_parity_bounded(&full[s], ph);
        }
        const unsigned code = stage_item[s];
        const unsigned j = stage_step[s];
        if (code == kEndItem) break;
        const unsigned type = code >> kPipeTypeShift, idx = code & kPipeIdxMask;
        const bool skip = (code & kPipeSkip) != 0u;
        const long long t = t0 + (long long)j;

        if (type != kPipeItemTile) {
            // ---- fill / IB item: the stage carries only the descriptor
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&reads_done[s], 1u) == unsigned(kWarps - 1)) {
                    reads_done[s] = 0u;
                    __threadfence_block();
                    refill(s);
                }
            }
            publish();
            if (!skip) {
                if (type == kPipeItemFill) pipe_fill_item(Q, idx, t, tid);
                else pipe_ib_item(Q, idx, t, step_epoch[j], tid, red[s]);
            }
        } else {
            // ---- tile
            const float* const st = stage0 + s * (kStageBytes / 4);
            const unsigned m = 2u * tid;
            const unsigned sb = g.base + g.PP, se = g.base + unsigned(g.nzl + 1) * g.PP;
            const unsigned sl = Q.org + idx * unsigned(Tile::kTile) + m;
            const unsigned row = g.div_px.div(sl - g.base);
            const int col = int(sl - g.base - row * g.PX);
            const unsigned pl = g.div_py.div(row);
            const int r = int(row - pl * g.PY);
            const int x = col - 2, y = r - 1, lz = int(pl) - 1;
            const bool valid = !skip && sl >= sb && sl < se && x >= 0 && x < g.nx && y >= 0;
            const unsigned kf = valid ? (unsigned(lz) * g.ny + unsigned(y)) * g.nx + unsigned(x) : 0u;
            const unsigned char epoch = step_epoch[j];
            const unsigned tflag2 =
                P.p.tflag != nullptr ? __ldcg(reinterpret_cast<const unsigned short*>(P.p.tflag + kf)) : 0u;
            float2 fs[27];
            if (!skip)
                static_for<0, 27>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    constexpr int d = win_shift(i);
                    const float* w = st + i * kWin + m + d;
                    if constexpr (d % 2 == 0) fs[i] = *reinterpret_cast<const float2*>(w);
                    else fs[i] = make_float2(w[0], w[1]);
                });
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();  // this warp's reads of stage s are done
                if (atomicAdd(&reads_done[s], 1u) == unsigned(kWarps - 1)) {
                    reads_done[s] = 0u;
                    __threadfence_block();
                    refill(s);
                }
            }
            bool do_store = false;
            if (valid) {
                const unsigned k = kf;
                float2 gx = make_float2(P.m.body[0], P.m.body[0]);
                float2 gy = make_float2(P.m.body[1], P.m.body[1]);
                float2 gz = make_float2(P.m.body[2], P.m.body[2]);
                if (P.p.tflag != nullptr && ((tflag2 & 0xffu) == epoch || (tflag2 >> 8) == epoch)) {
                    float* gib = P.p.gib;
                    gx = __fadd2_rn(gx, __ldcg(reinterpret_cast<const float2*>(gib + k)));
                    gy = __fadd2_rn(gy, __ldcg(reinterpret_cast<const float2*>(gib + k + g.ns)));
                    gz = __fadd2_rn(gz, __ldcg(reinterpret_cast<const float2*>(gib + k + 2u * g.ns)));
                    *reinterpret_cast<float2*>(gib + k) = make_float2(0.f, 0.f);
                    *reinterpret_cast<float2*>(gib + k + g.ns) = make_float2(0.f, 0.f);
                    *reinterpret_cast<float2*>(gib + k + 2u * g.ns) = make_float2(0.f, 0.f);
                }
                const MacroV<float2> mc = moments_v<float2>(fs);
                if (mc.bad[0] || mc.bad[1]) {
                    atomicExch(&ctr->diverged, 1u);
                    atomicMin(&pc->div_min, (unsigned long long)t);
                } else {
                    if (mc.mach[0] || mc.mach[1]) raise_mach(ctr);
                    if (int(j) == Q.macro_j) {
                        *reinterpret_cast<float2*>(P.p.rho + k) = mc.rho;
                        *reinterpret_cast<float2*>(P.p.u + k) = mc.ux;
                        *reinterpret_cast<float2*>(P.p.u + k + g.ns) = mc.uy;
                        *reinterpret_cast<float2*>(P.p.u + k + 2u * g.ns) = mc.uz;
                    }
                    const bool any_force =
                        gx.x != 0.f || gx.y != 0.f || gy.x != 0.f || gy.y != 0.f || gz.x != 0.f || gz.y != 0.f;
                    NoStash<float2> stash;
                    collide_v<KIND, POLICY, STD, float2>(fs, mc, gx, gy, gz, any_force, P.m, stash);
                    do_store = true;
                }
            }
            // the previous item's completion: its stores went out an item
            // ago, so the release fence here costs little; this tile's go next
            publish();
            if (do_store) {
                float* const ob = P.p.f[step_next[j]] + g.gaddr(sl, 0);
                static_for<0, 27>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    *reinterpret_cast<float2*>(ob + size_t(i) * g.A) = fs[i];
                });
                const int p = int(j + unsigned(t0 & 1)) & 1;
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
        }
        __syncwarp();
        if (lane == 0) pend_sm[warp] = Pending{code & ~kPipeSkip, j, unsigned(s), ph};
        __syncwarp();
    }
    publish();
}

// ---------------------------------------------------------------------------
// Host side.

size_t pipe_counter_bytes(const RegionGeo& g) { return sizeof(PipeCounters) + sizeof(unsigned) * 2 * size_t(g.nzl); }

int pipe_tile_slots() { return Tile::kTile; }

PipePlan make_pipe_plan(const RegionGeo& g, unsigned n_ib, int z0_ib, int z1_ib) {
    PipePlan pl;
    const unsigned kT = unsigned(Tile::kTile);
    const unsigned sb = g.base + g.PP, se = g.base + unsigned(g.nzl + 1) * g.PP;
    pl.org = (sb / kT) * kT;
    pl.n_tiles = (se - pl.org + kT - 1) / kT;
    const int nzl = g.nzl;
    auto plane_of_h = [&](unsigned slot) { return int((slot - g.base) / g.PX / g.PY) - 1; };
    auto planes = [&](unsigned k, int& wa, int& wb) {
        const unsigned a = std::max(pl.org + k * kT, sb), b = std::min(pl.org + (k + 1) * kT, se) - 1u;
        wa = plane_of_h(a);
        wb = plane_of_h(b);
    };
    pl.tile_need.assign(nzl, 0u);
    for (unsigned k = 0; k < pl.n_tiles; ++k) {
        int wa, wb;
        planes(k, wa, wb);
        for (int w = wa; w <= wb; ++w) pl.tile_need[w]++;
    }
    const unsigned X = 9u * unsigned(g.ny), Y = 9u * unsigned(g.nx), Z = 9u * g.plane;
    std::vector<std::vector<unsigned>> fills(nzl);
    pl.fill_need.assign(nzl, 0u);
    for (int w = 0; w < nzl; ++w) {
        const unsigned E = 2u * X + 2u * Y + (w == 0 ? Z : 0u) + (w == nzl - 1 ? Z : 0u);
        for (unsigned e0 = 0; e0 < E; e0 += kPipeFillChunk) {
            fills[w].push_back(pl.n_fill++);
            pl.fill_desc.push_back(unsigned(w));
            pl.fill_desc.push_back(e0);
            pl.fill_desc.push_back(std::min(E, e0 + kPipeFillChunk));
        }
        pl.fill_need[w] = unsigned(fills[w].size());
    }
    // one step's order: the fill of a plane kPipeLookahead planes ahead of
    // its tiles, the IB items just before the first tile on an IB plane
    auto code = [](unsigned type, unsigned idx) { return (type << kPipeTypeShift) | idx; };
    int next_fill = 0;
    auto emit_fill = [&](int upto) {
        upto = std::min(upto, nzl - 1);
        for (; next_fill <= upto; ++next_fill)
            for (unsigned f : fills[next_fill]) pl.pattern.push_back(code(kPipeItemFill, f));
    };
    bool ib_emitted = n_ib == 0;
    auto emit_ib = [&]() {
        emit_fill(z1_ib);
        for (unsigned b = 0; b < n_ib; ++b) pl.pattern.push_back(code(kPipeItemIb, b));
        ib_emitted = true;
    };
    for (unsigned k = 0; k < pl.n_tiles; ++k) {
        int wa, wb;
        planes(k, wa, wb);
        emit_fill(wb + kPipeLookahead);
        if (!ib_emitted && wb >= z0_ib && wa <= z1_ib) emit_ib();
        pl.pattern.push_back(code(kPipeItemTile, k));
    }
    emit_fill(nzl - 1);
    if (!ib_emitted) emit_ib();
    return pl;
}

namespace {

#define PIPE_OK(x)                                                                                        \
    do {                                                                                                  \
        const cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <int KIND, int POLICY, bool STD>
void launch_pipeline_t(const PipeParams& Q, int sm_count, cudaStream_t st) {
    constexpr unsigned smem = kPStages * Tile::kStageBytes + 8u * kPStages;
    constexpr int kMaxDev = 64;
    static bool attr_set[kMaxDev] = {};
    auto kern = pipeline_kernel<KIND, POLICY, STD>;
    int dev = 0;
    PIPE_OK(cudaGetDevice(&dev));
    if (dev >= kMaxDev) throw std::runtime_error("pipeline: device index beyond the per-device cache");
    if (!attr_set[dev]) {
        PIPE_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_set[dev] = true;
    }
    pipeline_begin_kernel<<<1, 256, 0, st>>>(Q.pc, Q.P.ctr, Q.P.g.nzl);
    kern<<<sm_count, kThreads, smem, st>>>(Q);
}

template <int KIND, int POLICY>
void launch_pipeline_std(const PipeParams& Q, int sm_count, cudaStream_t st) {
    if (rates_standard(Q.P.m.rate)) launch_pipeline_t<KIND, POLICY, true>(Q, sm_count, st);
    else launch_pipeline_t<KIND, POLICY, false>(Q, sm_count, st);
}

}  // namespace

void launch_pipeline(const PipeParams& Q, int sm_count, cudaStream_t st) {
    const int kind = Q.P.m.kind, pol = Q.P.m.policy;
    if (kind == kBGK) launch_pipeline_t<kBGK, kPolicyConstant, false>(Q, sm_count, st);
    else if (kind == kRawMRT) launch_pipeline_std<kRawMRT, kPolicyConstant>(Q, sm_count, st);
    else if (pol == kPolicyConstant) launch_pipeline_std<kCentralMRT, kPolicyConstant>(Q, sm_count, st);
    else launch_pipeline_std<kCentralMRT, kPolicyRelax>(Q, sm_count, st);
}

}  // namespace lbmg
