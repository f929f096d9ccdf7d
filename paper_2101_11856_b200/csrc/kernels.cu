// sm_100a kernels of the ACM-MRT + IB step.  Every kernel reads the step
// counter from device memory (parity selects the A/B buffers), so one step is
// a fixed launch sequence that replays unchanged inside a CUDA graph.
//
// Step (runner.cpp:121-230, fused):
//   ib_mark      per sample: kernel support, flag, band-node dedup (stamp)
//   ib_band      per band node: pull + face passes + moments -> rho*, u*
//   (macro halo) rho/u of the boundary planes to the neighbour slabs
//   ib_spread    per sample: interpolate, penalty, scatter into g (smem hash)
//   ib_totals    per solid FP64 reaction force/torque (deterministic order)
//   ib_motion    per sample: rigid motion to t+1 (moving solids)
//   fluid        per node: pull-stream + six face passes + moments + CM-MRT
//                (+ adaptive rates) + forcing; writes f(t+1), the crossing
//                populations of the boundary planes into the neighbours' halo,
//                and the face slots
//   step_end     t += 1 unless diverged
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cstdio>
#include <stdexcept>
#include <cstdlib>
#include <string>

#include "device_common.cuh"
#include "engine.hpp"
#include "ib_dev.cuh"

namespace lbmg {

// ---------------------------------------------------------------------------
// Immersed boundary (ib.cpp:294-501).


__global__ void ib_mark_kernel(const FluidParams P, IbSolidDev S, unsigned* stamp, unsigned* band) {
    DevCounters* ctr = P.ctr;
    if (ctr->diverged) return;
    const RegionGeo& g = P.g;
    const unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned ln = threadIdx.x & 31u;
    bool act = s < S.n;
    Support ks{};
    const int z0 = g.gz0, z1 = g.gz0 + g.nzl;
    if (act) {
        const double pos[3] = {S.pos[3 * s], S.pos[3 * s + 1], S.pos[3 * s + 2]};
        ks = kernel_support(pos, g.nx, g.ny, g.NZ);
        S.flagged[s] = ks.inside ? 0 : 1;
        act = ks.inside && sample_active(pos[2], g.NZ, z0, z1);
    }
    const unsigned mark = unsigned(ctr->t) + 1u;
    // each corner: dedup by stamp, then one warp-aggregated append
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int ox = c & 1, oy = (c >> 1) & 1, oz = c >> 2;
        const int gz = ks.base[2] + oz;
        bool fresh = false;
        unsigned k = 0;
        if (act && gz >= z0 && gz < z1) {
            k = g.node(ks.base[0] + ox, ks.base[1] + oy, gz - g.gz0);
            fresh = atomicExch(&stamp[k], mark) != mark;
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, fresh);
        if (ballot == 0u) continue;
        unsigned base = 0;
        if (ln == unsigned(__ffs(ballot) - 1)) base = atomicAdd(P.p.band_count, unsigned(__popc(ballot)));
        base = __shfl_sync(0xffffffffu, base, __ffs(ballot) - 1);
        if (fresh) band[base + __popc(ballot & ((1u << ln) - 1u))] = k;
    }
}

// Interpolate (ib.cpp:321-343), penalty (ib.cpp:345-365) and scatter
// (ib.cpp:369-454, atomic mode) per sample.  Scatter contributions are
// combined in a per-CTA shared-memory hash table (samples are block/Morton
// sorted, so a CTA touches few distinct nodes) and flushed with one global
// atomic per (node, component).
constexpr int kSpreadThreads = 128;
constexpr int kHashSlots = 2048;  // >= 2 * 8 * kSpreadThreads (load <= 0.5), power of two

template <bool SMEM, bool DET = false>
__global__ void __launch_bounds__(kSpreadThreads) ib_spread_kernel(const FluidParams P, IbSolidDev S) {
    __shared__ unsigned hkey[SMEM ? kHashSlots : 1];
    __shared__ float hval[3][SMEM ? kHashSlots : 1];
    DevCounters* ctr = P.ctr;
    if (ctr->diverged) return;
    const RegionGeo& g = P.g;
    if constexpr (SMEM) {
        for (int j = threadIdx.x; j < kHashSlots; j += blockDim.x) {
            hkey[j] = 0xffffffffu;
            hval[0][j] = hval[1][j] = hval[2][j] = 0.f;
        }
        __syncthreads();
    }

    const unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    const int z0 = g.gz0, z1 = g.gz0 + g.nzl;
    if (s < S.n) {
        const double pos[3] = {S.pos[3 * s], S.pos[3 * s + 1], S.pos[3 * s + 2]};
        const Support ks = kernel_support(pos, g.nx, g.ny, g.NZ);
        const bool active = ks.inside && sample_active(pos[2], g.NZ, z0, z1);
        double us[3] = {0.0, 0.0, 0.0};
        double fg[3] = {0.0, 0.0, 0.0};
        if (active) {
            double rs = 0.0;
            for (int oz = 0; oz < 2; ++oz)
                for (int oy = 0; oy < 2; ++oy)
                    for (int ox = 0; ox < 2; ++ox) {
                        const double w = __dmul_rn(__dmul_rn(ks.w[0][ox], ks.w[1][oy]), ks.w[2][oz]);
                        const int x = ks.base[0] + ox, y = ks.base[1] + oy, gz = ks.base[2] + oz;
                        float r, ux, uy, uz;
                        if (gz >= z0 && gz < z1) {
                            const unsigned k = g.node(x, y, gz - g.gz0);
                            r = P.p.rho[k];
                            ux = P.p.u[k];
                            uy = P.p.u[k + g.ns];
                            uz = P.p.u[k + 2u * g.ns];
                        } else {
                            const float* h = gz < z0 ? P.p.mrecv_lo : P.p.mrecv_hi;
                            const unsigned j = unsigned(y) * g.nx + x;
                            r = h[j];
                            ux = h[j + g.plane];
                            uy = h[j + 2u * g.plane];
                            uz = h[j + 3u * g.plane];
                        }
                        us[0] += w * ux;
                        us[1] += w * uy;
                        us[2] += w * uz;
                        rs += w * r;
                    }
            for (int a = 0; a < 3; ++a) fg[a] = rs * (S.ub[3 * s + a] - us[a]);
        }
        // this step's half of the A/B sample outputs (the diverging step's IB
        // results are never read back: runner.cpp:154-161 skips IB there)
        const size_t po = ib_half(S, ctr->t);
        for (int a = 0; a < 3; ++a) {
            S.sampled[po + 3 * s + a] = us[a];
            S.force[po + 3 * s + a] = fg[a];
        }
        if constexpr (DET) {  // one (owned node | ~0u, w g_s) record per corner, sample-major
            for (int c = 0; c < 8; ++c) {
                const int ox = c & 1, oy = (c >> 1) & 1, oz = c >> 2;
                const int gz = ks.base[2] + oz;
                const unsigned rec = s * 8u + unsigned(c);
                const bool own = active && gz >= z0 && gz < z1;
                S.rec_key[rec] = own ? g.node(ks.base[0] + ox, ks.base[1] + oy, gz - g.gz0) : ~0u;
                S.rec_idx[rec] = rec;
                const double w = __dmul_rn(__dmul_rn(ks.w[0][ox], ks.w[1][oy]), ks.w[2][oz]);
                for (int a = 0; a < 3; ++a) S.rec_val[3 * rec + a] = own ? w * fg[a] : 0.0;
            }
        } else if (active) {
            for (int oz = 0; oz < 2; ++oz) {
                const int gz = ks.base[2] + oz;
                if (gz < z0 || gz >= z1) continue;
                for (int oy = 0; oy < 2; ++oy)
                    for (int ox = 0; ox < 2; ++ox) {
                        const double w = __dmul_rn(__dmul_rn(ks.w[0][ox], ks.w[1][oy]), ks.w[2][oz]);
                        const unsigned key = g.node(ks.base[0] + ox, ks.base[1] + oy, gz - g.gz0);
                        if constexpr (!SMEM) {  // direct fire-and-forget reductions in L2
                            atomicAdd(&P.p.gib[key], float(w * fg[0]));
                            atomicAdd(&P.p.gib[key + g.ns], float(w * fg[1]));
                            atomicAdd(&P.p.gib[key + 2u * g.ns], float(w * fg[2]));
                            mark_force(P, key, ib_epoch(P.ctr->t));
                            continue;
                        }
                        unsigned h = (key * 2654435761u) & (kHashSlots - 1);
                        for (;;) {
                            const unsigned prev = atomicCAS(&hkey[h], 0xffffffffu, key);
                            if (prev == 0xffffffffu || prev == key) break;
                            h = (h + 1) & (kHashSlots - 1);
                        }
                        atomicAdd(&hval[0][h], float(w * fg[0]));
                        atomicAdd(&hval[1][h], float(w * fg[1]));
                        atomicAdd(&hval[2][h], float(w * fg[2]));
                    }
            }
        }
    }
    if constexpr (!SMEM) return;
    __syncthreads();
    for (int j = threadIdx.x; j < kHashSlots; j += blockDim.x) {
        const unsigned key = hkey[j];
        if (key == 0xffffffffu) continue;
        atomicAdd(&P.p.gib[key], hval[0][j]);
        atomicAdd(&P.p.gib[key + g.ns], hval[1][j]);
        atomicAdd(&P.p.gib[key + 2u * g.ns], hval[2][j]);
        mark_force(P, key, ib_epoch(P.ctr->t));
    }
}

// Reaction totals (ib.cpp:491-501) over samples with z in [z0, z1):
// per-block FP64 partials, then a fixed-order final sum -> deterministic.
constexpr int kTotThreads = 256;
__global__ void __launch_bounds__(kTotThreads) ib_totals_partial_kernel(const FluidParams P, IbSolidDev S,
                                                                       const double* table,
                                                                       double* partial) {
    if (P.ctr->diverged) return;
    __shared__ double sh[6][kTotThreads];
    const double* motion_row = table + (P.ctr->t - P.ctr->chunk_t0) * kMotionRow;
    const double c[3] = {motion_row[0], motion_row[1], motion_row[2]};
    const double* force = S.force + ib_half(S, P.ctr->t);
    double acc[6] = {0, 0, 0, 0, 0, 0};
    const double z0 = P.g.gz0, z1 = P.g.gz0 + P.g.nzl;
    for (unsigned s = blockIdx.x * blockDim.x + threadIdx.x; s < S.n; s += gridDim.x * blockDim.x) {
        const double pz = S.pos[3 * s + 2];
        if (pz < z0 || pz >= z1) continue;
        const double F[3] = {force[3 * s], force[3 * s + 1], force[3 * s + 2]};
        const double r[3] = {S.pos[3 * s] - c[0], S.pos[3 * s + 1] - c[1], pz - c[2]};
        acc[0] -= F[0];
        acc[1] -= F[1];
        acc[2] -= F[2];
        acc[3] -= r[1] * F[2] - r[2] * F[1];
        acc[4] -= r[2] * F[0] - r[0] * F[2];
        acc[5] -= r[0] * F[1] - r[1] * F[0];
    }
    for (int a = 0; a < 6; ++a) sh[a][threadIdx.x] = acc[a];
    __syncthreads();
    for (int off = kTotThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off)
            for (int a = 0; a < 6; ++a) sh[a][threadIdx.x] += sh[a][threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x < 6) partial[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void ib_totals_final_kernel(const DevCounters* ctr, const double* partial, int nblocks,
                                       double* out_base, int stride) {
    if (ctr->diverged) return;
    const int a = threadIdx.x;
    if (a >= 6) return;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += partial[b * 6 + a];
    out_base[(ctr->t - ctr->chunk_t0) * stride + a] = acc;
}


// update_rigid_motion (ib.cpp:456-489) to step t+1 with host-computed R, c.
// motion table row (per step): c[3], R[9], v[3], w[3].
__global__ void ib_motion_kernel(const DevCounters* ctr, IbSolidDev S, const double* table,
                                 int nx, int ny, int nz) {
    if (ctr->diverged) return;
    const unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S.n) return;
    const double* row = table + (ctr->t + 1 - ctr->chunk_t0) * kMotionRow;
    motion_apply(row, S, s, nx, ny, nz);
}

__global__ void ib_motion_once_kernel(IbSolidDev S, const double* row, int nx, int ny, int nz) {
    const unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S.n) return;
    motion_apply(row, S, s, nx, ny, nz);
}

// ---------------------------------------------------------------------------
// Fused IB step on the ghost layout, after the ghost fill of this region and
// of its neighbour slabs: per sample 8 lanes, one per support corner.  Each
// lane pulls the corner's 27 post-BC populations f* straight from the
// ghost-layer storage of the slab that owns the corner's plane (its own, or
// the in-process neighbour's across a seam: no macro halo) — all 27 loads in
// flight at once — and the lanes reduce rho*, j* by shuffles: the band
// pre-pass without a band list.  Then interpolation (ib.cpp:321-343, FP64),
// penalty (ib.cpp:345-365) for samples whose support touches the slab
// (sample_active, ib.cpp:313-317), the scatter (ib.cpp:369-454, atomic mode:
// one fp32 RED per corner, owned nodes only, ib.cpp:377), the reaction totals
// (ib.cpp:491-501: per-block FP64 partials; the region's fluid kernel sums
// them in block order -> deterministic) and, for moving solids, the rigid motion to t+1
// (ib.cpp:456-489).  Static solids run over the region's active samples only
// (IbSolidDev::active, partitioned once by slab); moving ones over all.
// (Measured alternatives, slower on C2 and configs[3]: 8-warp CTAs with a
// shared-memory pre-aggregated scatter — 2.8 vs 1.9 ms on configs[3] — and a
// per-CTA dedup of support nodes in shared memory — 5.0 ms.)
// rho* - 1 and j* of one node from its 27 pulled f*: the fixed sum order the
// fused kernel's gather and the band kernel share (bit-identical results).
__device__ __forceinline__ void band_sums(const float (&v)[27], float& r, float& jx, float& jy, float& jz) {
    r = jx = jy = jz = 0.f;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        r += v[i];
        jx += float(cx(i)) * v[i];
        jy += float(cy(i)) * v[i];
        jz += float(cz(i)) * v[i];
    }
}

// band path setup: the slot of every (active sample, corner) of a static
// solid on a single region (~0u: sample inactive), as the fused kernel finds it
__global__ void ib_band_keys_kernel(const FluidParams P, IbSolidDev S, unsigned* keys) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 8u * S.n_active) return;
    const unsigned j = e >> 3, c = e & 7u;
    const double* pp = S.act_pu + 6 * size_t(j);
    const double pos[3] = {pp[0], pp[1], pp[2]};
    const RegionGeo& g = P.g;
    const Support ks = kernel_support(pos, g.nx, g.ny, g.NZ);
    const bool act = ks.inside && sample_active(pos[2], g.NZ, g.gz0, g.gz0 + g.nzl);
    const int ox = int(c & 1u), oy = int((c >> 1) & 1u), oz = int(c >> 2);
    keys[e] = act ? g.sidx(ks.base[0] + ox, ks.base[1] + oy, ks.base[2] + oz - g.gz0) : ~0u;
}

__global__ void ib_band_index_kernel(const unsigned* keys, unsigned n_keys, const unsigned* band, unsigned n_band,
                                     unsigned* out) {
    const unsigned e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_keys) return;
    const unsigned key = keys[e];
    unsigned lo = 0, hi = n_band;
    while (lo < hi) {
        const unsigned mid = (lo + hi) >> 1;
        if (band[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    out[e] = key != ~0u && lo < n_band && band[lo] == key ? lo : ~0u;
}

// per step: rho* - 1, j* of every band node (band sorted by slot: consecutive
// threads pull consecutive slots of each direction array)
__global__ void __launch_bounds__(256) ib_band_moments_kernel(const __grid_constant__ FluidParams P,
                                                              const unsigned* __restrict__ band, unsigned n,
                                                              float4* __restrict__ out) {
    if (P.ctr->diverged) return;
    const unsigned b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const RegionGeo& g = P.g;
    const float* fin = P.p.f[fcur(g, P.ctr->t)];
    const long long sl = band[b];
    float v[27];
#pragma unroll
    for (int i = 0; i < 27; ++i) v[i] = __ldcg(&fin[g.gaddr((unsigned long long)(sl - g.soff(i)), i)]);
    float r, jx, jy, jz;
    band_sums(v, r, jx, jy, jz);
    out[b] = make_float4(r, jx, jy, jz);
}

constexpr int kFusedWarps = 4;
constexpr int kLanesPerSample = 8;
constexpr int kFusedSamples = kFusedWarps * 32 / kLanesPerSample;

// All solids of the scene in ONE launch: blocks [block_start[k], block_start[k+1])
// belong to solid k (per-solid totals reductions keep their own counters).
__global__ void __launch_bounds__(kFusedWarps * 32, 8)
    ib_fused_kernel(const __grid_constant__ FluidParams P, const __grid_constant__ IbBatch B, int det) {
    __shared__ double red[kFusedSamples][6];
    DevCounters* ctr = P.ctr;
    if (B.fill_from != 0 && blockIdx.x >= B.fill_from) {  // merged launch: the ghost-fill blocks
        if (ctr->diverged) return;
        fill_copy_block(P, blockIdx.x - B.fill_from, threadIdx.x, blockDim.x);
        return;
    }
    // (the divergence check waits below the sample loads: they are valid
    // either way, and the chain of dependent loads is this kernel's latency)
    const unsigned diverged = ctr->diverged;
    const RegionGeo& g = P.g;
    unsigned lo = 0, hi = B.n_solids;
    if (B.block_solid != nullptr && B.n_solids > 1) {
        lo = B.block_solid[blockIdx.x];
    } else {
        while (hi - lo > 1) {
            const unsigned mid = (lo + hi) >> 1;
            if (B.block_start[mid] <= blockIdx.x) lo = mid;
            else hi = mid;
        }
    }
    const unsigned solid = lo;
    const IbSolidDev S = B.n_solids == 1 ? B.solo : B.solids[solid];  // (one solid: from parameter space)
    const double* table = B.table + size_t(solid) * B.table_stride;
    const int moving = B.moving[solid] | B.probe;
    const unsigned b0 = B.block_start[solid], nblk = B.block_start[solid + 1] - b0;
    double* partial = B.partial + size_t(b0) * 6;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned slot = threadIdx.x / kLanesPerSample;  // sample slot in the block
    const unsigned local = (blockIdx.x - b0) * kFusedSamples + slot;
    const unsigned corner = lane % kLanesPerSample;
    const long long t = ctr->t;
    const double* row = table + (t - ctr->chunk_t0) * kMotionRow;
    double tot[6] = {0, 0, 0, 0, 0, 0};
    const unsigned n_run = S.active ? S.n_active : S.n;
    const bool have = local < n_run;
    const unsigned s = have ? (S.active ? S.active[local] : local) : 0u;
    // band path: the corner's band index, issued with the sample loads (it
    // does not depend on the position)
    const bool band = B.band_m != nullptr && S.corner_band != nullptr;
    const unsigned cb = band && have ? S.corner_band[8u * local + corner] : ~0u;
    // static solids: (pos, u_b) stored in run order, loaded in parallel with s
    const double* pp = S.act_pu != nullptr ? S.act_pu + 6 * size_t(local) : S.pos + 3 * size_t(s);
    const double* up = S.act_pu != nullptr ? pp + 3 : S.ub + 3 * size_t(s);
    const double pos[3] = {have ? pp[0] : 0.0, have ? pp[1] : 0.0, have ? pp[2] : 0.0};
    const double ub[3] = {have ? up[0] : 0.0, have ? up[1] : 0.0, have ? up[2] : 0.0};  // (issued early)
    if (diverged) return;  // block-uniform (set only by the fluid kernel, which runs after)
    const Support ks = kernel_support(pos, g.nx, g.ny, g.NZ);
    if (have && corner == 0) S.flagged[s] = ks.inside ? 0 : 1;
    const int z0 = g.gz0, z1 = g.gz0 + g.nzl;
    const bool act = have && ks.inside && sample_active(pos[2], g.NZ, z0, z1);
    // every lane runs the gather (shuffles need the full warp); inactive
    // lanes read node (0,0,0) of the own slab and discard the result
    const int ox = corner & 1, oy = (corner >> 1) & 1, oz = corner >> 2;
    const int gz = act ? ks.base[2] + oz : z0;
    const IbSlab& R = gz < z0 ? B.lo : (gz >= z1 ? B.hi : B.own);
    const int x = act ? ks.base[0] + ox : 0, y = act ? ks.base[1] + oy : 0;
    float r = 0.f, jx = 0.f, jy = 0.f, jz = 0.f;
    if (band) {  // band path: the corner's moments, one 16-B load
        if (cb != ~0u) {
            const float4 mm = __ldcg(reinterpret_cast<const float4*>(B.band_m) + cb);
            r = mm.x;
            jx = mm.y;
            jy = mm.z;
            jz = mm.w;
        }
    } else {
        const float* fin = R.f[fcur(R.g, t)];
        const long long sl = R.g.sidx(x, y, gz - R.g.gz0);
        float v[27];
#pragma unroll
        for (int i = 0; i < 27; ++i) v[i] = __ldcg(&fin[R.g.gaddr((unsigned long long)(sl - R.g.soff(i)), i)]);
        band_sums(v, r, jx, jy, jz);
    }
    const float rho = 1.0f + r;
    const float inv = 1.0f / rho;
    const double wx = ox ? ks.w[0][1] : ks.w[0][0], wy = oy ? ks.w[1][1] : ks.w[1][0];
    const double wz = oz ? ks.w[2][1] : ks.w[2][0];
    const double w = __dmul_rn(__dmul_rn(wx, wy), wz);
    double c4[4] = {w * double(jx * inv), w * double(jy * inv), w * double(jz * inv), w * double(rho)};
#pragma unroll
    for (int o = 1; o < kLanesPerSample; o <<= 1)
#pragma unroll
        for (int a = 0; a < 4; ++a) c4[a] += __shfl_xor_sync(0xffffffffu, c4[a], o);
    double us[3] = {0.0, 0.0, 0.0}, fg[3] = {0.0, 0.0, 0.0};
    const bool own = act && gz >= z0 && gz < z1;
    const unsigned k = own ? g.node(x, y, gz - z0) : 0u;
    if (act)
        for (int a = 0; a < 3; ++a) {
            us[a] = c4[a];
            fg[a] = c4[3] * (ub[a] - us[a]);
        }
    if (det) {  // deterministic: a (owned node | ~0u, contribution) record per corner
        if (have) {
            const unsigned rec = local * 8u + corner;
            S.rec_key[rec] = own ? k : ~0u;
            S.rec_idx[rec] = rec;
            for (int a = 0; a < 3; ++a) S.rec_val[3 * rec + a] = own ? w * fg[a] : 0.0;
        }
    } else if (own && !(moving & 2)) {
        for (int a = 0; a < 3; ++a) atomicAdd(&P.p.gib[k + a * g.ns], float(w * fg[a]));
        if (!(moving & 4)) mark_force(P, k, x, y, gz - z0, ib_epoch(t));
    }
    if (have && corner == 0) {
        const size_t po = ib_half(S, t);
        for (int a = 0; a < 3; ++a) {
            S.sampled[po + 3 * s + a] = us[a];
            S.force[po + 3 * s + a] = fg[a];
        }
        if (pos[2] >= double(z0) && pos[2] < double(z1)) {
            const double rr[3] = {pos[0] - row[0], pos[1] - row[1], pos[2] - row[2]};
            tot[0] = -fg[0];
            tot[1] = -fg[1];
            tot[2] = -fg[2];
            tot[3] = -(rr[1] * fg[2] - rr[2] * fg[1]);
            tot[4] = -(rr[2] * fg[0] - rr[0] * fg[2]);
            tot[5] = -(rr[0] * fg[1] - rr[1] * fg[0]);
        }
        if (moving & 1) motion_apply(row + kMotionRow, S, s, g.nx, g.ny, g.NZ);
    }
    if (corner == 0)
        for (int a = 0; a < 6; ++a) red[slot][a] = tot[a];
    __syncthreads();
    // this block's partial; the fixed-order sum over the solid's blocks is
    // the fluid kernel's (RegionPtrs::ib_partial): no fence, counter or
    // last-block pass on this kernel's dependency chain
    if (threadIdx.x < 6) {
        double acc = 0.0;
        for (int w2 = 0; w2 < kFusedSamples; ++w2) acc += red[w2][threadIdx.x];
        partial[(blockIdx.x - b0) * 6 + threadIdx.x] = acc;
    }
    (void)nblk;
}

// ---------------------------------------------------------------------------
// init_fields (runner.cpp:60-107): equilibrium f (both the f(0) buffer and
// the face slots, which stand in for the initial f_star), rho, u.

__device__ __forceinline__ void init_state(const InitParams& ip, int x, int y, int gz, double& rho,
                                           double u[3]) {
    if (ip.kind == 0) {
        rho = ip.rho0;
        u[0] = ip.u0[0];
        u[1] = ip.u0[1];
        u[2] = ip.u0[2];
        return;
    }
    const double kx = 2.0 * M_PI / ip.NX, ky = 2.0 * M_PI / ip.NY;
    const double u0 = ip.tg_u;
    u[0] = -u0 * cos(kx * x) * sin(ky * y);
    u[1] = u0 * sin(kx * x) * cos(ky * y);
    u[2] = 0.0;
    const double pr = -0.25 * u0 * u0 * (cos(2.0 * kx * x) + cos(2.0 * ky * y));
    rho = ip.rho0 + 3.0 * pr;
}

__device__ __forceinline__ double feq_shifted(int i, double rho, const double u[3]) {
    const double w = weight_d(i);
    const double usq = 1.5 * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    const double cu = cx(i) * u[0] + cy(i) * u[1] + cz(i) * u[2];
    const double feq = w * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - usq);
    return feq - w;
}

__global__ void init_kernel(const FluidParams P, InitParams ip) {
    const RegionGeo& g = P.g;
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.n) return;
    int x, y, lz;
    decode(g, k, x, y, lz);
    const int gz = g.gz0 + lz;
    double rho, u[3];
    init_state(ip, x, y, gz, rho, u);
    float* f0 = P.p.f[0];
    for (int i = 0; i < 27; ++i) {
        const float v = float(feq_shifted(i, rho, u));
        for (int b = 0; b < g.nbuf; ++b) P.p.f[b][g.idx(k, i)] = v;
    }
    P.p.rho[k] = float(rho);
    P.p.u[k] = float(u[0]);
    P.p.u[k + g.ns] = float(u[1]);
    P.p.u[k + 2u * g.ns] = float(u[2]);
    // face slots (initial f_star = feq, runner.cpp:94) for both parities
    for (int f = 0; f < 6; ++f) {
        float* s0 = P.p.slot[0][f];
        if (!s0) continue;
        const int a = face_axis(f), sd = face_side(f);
        const int coord = a == 0 ? x : (a == 1 ? y : gz);
        const int plane = sd < 0 ? 0 : g.extent(a) - 1;
        if (coord != plane) continue;
        for (int i = 0; i < 27; ++i) {
            if (cc(i, a) != -sd) continue;
            const float v = float(feq_shifted(i, rho, u));
            s0[g.slot_index(f, x, y, lz, i)] = v;
            P.p.slot[1][f][g.slot_index(f, x, y, lz, i)] = v;
        }
    }
    // halos for step 0 (send[0] aliases the neighbour's recv[0] in-process)
    const unsigned hp = unsigned(y) * g.nx + x;
    if (lz == 0 && P.p.send_lo[0])
        for (int i = 1; i <= 9; ++i) P.p.send_lo[0][cross9(i, 2) * g.plane + hp] = f0[g.idx(k, i)];
    if (lz == g.nzl - 1 && P.p.send_hi[0])
        for (int i = 18; i <= 26; ++i) P.p.send_hi[0][cross9(i, 2) * g.plane + hp] = f0[g.idx(k, i)];
}

// Readback: canonical AoS FP64 for local planes [lz0, lz1).
__global__ void read_f_kernel(const FluidParams P, int buffer, unsigned k0, unsigned k1, double* out) {
    const unsigned k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= k1) return;
    const float* f = P.p.f[buffer];
    const RegionGeo& g = P.g;
    for (int i = 0; i < 27; ++i)
        out[size_t(k - k0) * 27 + i] = double(f[g.idx(k, i)]) + weight_d(i);
}

__global__ void read_macro_kernel(const FluidParams P, unsigned k0, unsigned k1, double* rho,
                                  double* u) {
    const unsigned k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= k1) return;
    const RegionGeo& g = P.g;
    if (rho) rho[k - k0] = double(P.p.rho[k]);
    if (u)
        for (int a = 0; a < 3; ++a) u[size_t(k - k0) * 3 + a] = double(P.p.u[k + a * g.ns]);
}

// Canonical AoS FP64 state -> device (Runner::load_state): f of every node
// (DDF-shifted fp32, the readback's inverse) and rho/u as plain moments of f.
__global__ void write_f_kernel(const FluidParams P, int buffer, int parity, const double* f) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    const RegionGeo& g = P.g;
    if (k >= g.n) return;
    float* fb = P.p.f[buffer];
    double r = 0.0, m[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < 27; ++i) {
        const double v = f[size_t(k) * 27 + i];
        fb[g.idx(k, i)] = float(v - weight_d(i));
        r += v;
        m[0] += cx(i) * v;
        m[1] += cy(i) * v;
        m[2] += cz(i) * v;
    }
    P.p.rho[k] = float(r);
    for (int a = 0; a < 3; ++a) P.p.u[k + a * g.ns] = float(m[a] / r);
    // the boundary planes' crossing populations into the halos step t reads
    int x, y, lz;
    decode(g, k, x, y, lz);
    const unsigned hp = unsigned(y) * g.nx + x;
    if (lz == 0 && P.p.send_lo[parity])
        for (int i = 1; i <= 9; ++i) P.p.send_lo[parity][cross9(i, 2) * g.plane + hp] = fb[g.idx(k, i)];
    if (lz == g.nzl - 1 && P.p.send_hi[parity])
        for (int i = 18; i <= 26; ++i) P.p.send_hi[parity][cross9(i, 2) * g.plane + hp] = fb[g.idx(k, i)];
}

// f_star of the face nodes -> the persistent face slots of one parity (the
// values the outflow stale-edge reads see)
__global__ void write_slots_kernel(const FluidParams P, int parity, const double* f_star) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    const RegionGeo& g = P.g;
    if (k >= g.n) return;
    int x, y, lz;
    decode(g, k, x, y, lz);
    const int gz = g.gz0 + lz;
    for (int f = 0; f < 6; ++f) {
        float* sl = P.p.slot[parity][f];
        if (!sl) continue;
        const int a = face_axis(f), sd = face_side(f);
        const int coord = a == 0 ? x : (a == 1 ? y : gz);
        if (coord != (sd < 0 ? 0 : g.extent(a) - 1)) continue;
        for (int i = 0; i < 27; ++i)
            if (cc(i, a) == -sd) sl[g.slot_index(f, x, y, lz, i)] = float(f_star[size_t(k) * 27 + i] - weight_d(i));
    }
}

// Cell flags: owner face per (node, direction).
__global__ void cell_flags_kernel(const FluidParams P, unsigned k0, unsigned k1, unsigned char* out) {
    const unsigned k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= k1) return;
    const RegionGeo& g = P.g;
    int x, y, lz;
    decode(g, k, x, y, lz);
    const int gz = g.gz0 + lz;
    static_for<0, 27>([&](auto I) {
        constexpr int i = decltype(I)::value;
        out[size_t(k - k0) * 27 + i] = (unsigned char)owner_face_c<i>(g, x, y, gz);
    });
}

// Layout change (set_layout, runner.cpp:252-258): pure permutation between
// two Eq. 9 layouts of the same node count.
__global__ void relayout_kernel(const float* src, float* dst, RegionGeo gs, RegionGeo gd) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= gs.n) return;
    for (int i = 0; i < 27; ++i) dst[gd.idx(k, i)] = src[gs.idx(k, i)];
}

// ---------------------------------------------------------------------------
// Host launch wrappers.

namespace {
inline unsigned blocks_for(unsigned long long n, unsigned t) { return unsigned((n + t - 1) / t); }

}  // namespace

void launch_ib_mark(const FluidParams& P, const IbSolidDev& S, unsigned* stamp, unsigned* band, cudaStream_t st) {
    if (S.n == 0) return;
    ib_mark_kernel<<<blocks_for(S.n, 256), 256, 0, st>>>(P, S, stamp, band);
}



// Deterministic accumulation: stable radix sort of the records by node (ties
// keep record = sample order), then one thread per node segment sums its
// contributions in that order in FP64 and adds the fp32 result to g.  The
// sum no longer depends on atomic timing, so runs are bitwise reproducible
// and independent of the region count (SPEC criterion 9; ib.cpp:407-453
// groups by colour instead — same contract, different fixed order).
__global__ void ib_det_segment_kernel(const FluidParams P, IbSolidDev S, unsigned n_rec) {
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rec || P.ctr->diverged) return;
    const unsigned k = S.key_sorted[i];
    if (k == ~0u || (i > 0 && S.key_sorted[i - 1] == k)) return;
    double acc[3] = {0.0, 0.0, 0.0};
    for (unsigned j = i; j < n_rec && S.key_sorted[j] == k; ++j) {
        const unsigned r = S.idx_sorted[j];
        for (int a = 0; a < 3; ++a) acc[a] += S.rec_val[3 * r + a];
    }
    const RegionGeo& g = P.g;
    P.p.gib[k] += float(acc[0]);
    P.p.gib[k + g.ns] += float(acc[1]);
    P.p.gib[k + 2u * g.ns] += float(acc[2]);
    mark_force(P, k, ib_epoch(P.ctr->t));
}

size_t ib_det_temp_bytes(unsigned n_samples) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned*)nullptr, (unsigned*)nullptr,
                                    (const unsigned*)nullptr, (unsigned*)nullptr, int(8u * n_samples));
    return bytes;
}

void launch_ib_det_reduce(const FluidParams& P, const IbSolidDev& S, cudaStream_t st) {
    if (S.n == 0) return;
    const unsigned n_rec = 8u * S.n;
    size_t bytes = S.sort_temp_bytes;
    cub::DeviceRadixSort::SortPairs(S.sort_temp, bytes, S.rec_key, S.key_sorted, S.rec_idx, S.idx_sorted,
                                    int(n_rec), 0, 32, st);
    ib_det_segment_kernel<<<blocks_for(n_rec, 256), 256, 0, st>>>(P, S, n_rec);
}

void launch_ib_spread(const FluidParams& P, const IbSolidDev& S, cudaStream_t st, bool deterministic) {
    if (S.n == 0) return;
    if (deterministic) {
        ib_spread_kernel<false, true><<<blocks_for(S.n, kSpreadThreads), kSpreadThreads, 0, st>>>(P, S);
        launch_ib_det_reduce(P, S, st);
        return;
    }
    static const bool smem = [] {
        const char* e = std::getenv("LBMG_IB_SPREAD");
        return e && std::string(e) == "smem";
    }();
    if (smem) ib_spread_kernel<true><<<blocks_for(S.n, kSpreadThreads), kSpreadThreads, 0, st>>>(P, S);
    else ib_spread_kernel<false><<<blocks_for(S.n, kSpreadThreads), kSpreadThreads, 0, st>>>(P, S);
}

int fused_blocks(size_t n) { return int((n + kFusedSamples - 1) / kFusedSamples); }
void launch_ib_fused(const FluidParams& P, IbBatch B, unsigned total_blocks, const IbSolidDev* host_solids,
                     cudaStream_t st, bool deterministic) {
    if (total_blocks == 0) return;
    static const int probe = [] {  // timing probes: LBMG_IB_NOSCATTER=1 skips the scatter into g,
        const char* e = std::getenv("LBMG_IB_NOSCATTER");  // 2: scatter without force flags
        return e ? (std::atoi(e) == 1 ? 2 : (std::atoi(e) == 2 ? 4 : 0)) : 0;
    }();
    B.probe = probe;
    ib_fused_kernel<<<total_blocks, kFusedWarps * 32, 0, st>>>(P, B, deterministic ? 1 : 0);
    if (deterministic)
        for (unsigned k = 0; k < B.n_solids; ++k) launch_ib_det_reduce(P, host_solids[k], st);
}
void launch_ib_fused_fill(const FluidParams& P, IbBatch B, unsigned total_blocks, cudaStream_t st) {
    B.probe = 0;
    B.fill_from = total_blocks;
    ib_fused_kernel<<<total_blocks + fill_blocks(P.p, kFusedWarps * 32), kFusedWarps * 32, 0, st>>>(P, B, 0);
}
unsigned build_ib_band(const FluidParams& P, IbSolidDev* solids, size_t n_solids, unsigned* band, cudaStream_t st) {
    size_t total = 0;
    for (size_t k = 0; k < n_solids; ++k)
        if (solids[k].corner_band) total += 8ull * solids[k].n_active;
    if (total == 0) return 0;
    unsigned *keys = nullptr, *sorted = nullptr, *count = nullptr;
    void* temp = nullptr;
    size_t tb_sort = 0, tb_uniq = 0;
    auto ok = [](cudaError_t e) {
        if (e != cudaSuccess) throw std::runtime_error(std::string("ib band: ") + cudaGetErrorString(e));
    };
    ok(cudaMalloc(&keys, sizeof(unsigned) * total));
    ok(cudaMalloc(&sorted, sizeof(unsigned) * total));
    ok(cudaMalloc(&count, sizeof(unsigned)));
    size_t off = 0;
    for (size_t k = 0; k < n_solids; ++k) {
        const IbSolidDev& S = solids[k];
        if (!S.corner_band || !S.n_active) continue;
        ib_band_keys_kernel<<<blocks_for(8ull * S.n_active, 256), 256, 0, st>>>(P, S, keys + off);
        off += 8ull * S.n_active;
    }
    cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, keys, sorted, int(total), 0, 32, st);
    cub::DeviceSelect::Unique(nullptr, tb_uniq, sorted, band, count, int(total), st);
    ok(cudaMalloc(&temp, std::max(tb_sort, tb_uniq)));
    cub::DeviceRadixSort::SortKeys(temp, tb_sort, keys, sorted, int(total), 0, 32, st);
    cub::DeviceSelect::Unique(temp, tb_uniq, sorted, band, count, int(total), st);
    unsigned n = 0;
    ok(cudaMemcpyAsync(&n, count, sizeof n, cudaMemcpyDeviceToHost, st));
    ok(cudaStreamSynchronize(st));
    unsigned last = 0;
    if (n) ok(cudaMemcpy(&last, band + n - 1, sizeof last, cudaMemcpyDeviceToHost));
    if (n && last == ~0u) --n;  // inactive corners sort last
    off = 0;
    for (size_t k = 0; k < n_solids; ++k) {
        const IbSolidDev& S = solids[k];
        if (!S.corner_band || !S.n_active) continue;
        ib_band_index_kernel<<<blocks_for(8ull * S.n_active, 256), 256, 0, st>>>(keys + off, 8u * S.n_active, band, n,
                                                                              S.corner_band);
        off += 8ull * S.n_active;
    }
    ok(cudaStreamSynchronize(st));
    ok(cudaGetLastError());
    cudaFree(keys);
    cudaFree(sorted);
    cudaFree(count);
    cudaFree(temp);
    return n;
}

void launch_ib_band_moments(const FluidParams& P, const unsigned* band, unsigned n, float* out, cudaStream_t st) {
    if (n) ib_band_moments_kernel<<<blocks_for(n, 256), 256, 0, st>>>(P, band, n, reinterpret_cast<float4*>(out));
}

int totals_blocks(size_t n) {
    size_t b = (n + kTotThreads - 1) / kTotThreads;
    return int(b < 1 ? 1 : (b > 256 ? 256 : b));
}

void launch_ib_totals(const FluidParams& P, const IbSolidDev& S, const double* table, double* partial,
                      double* out_base, int stride, cudaStream_t st) {
    const int nb = totals_blocks(S.n);
    ib_totals_partial_kernel<<<nb, kTotThreads, 0, st>>>(P, S, table, partial);
    ib_totals_final_kernel<<<1, 32, 0, st>>>(P.ctr, partial, nb, out_base, stride);
}

void launch_ib_motion(const DevCounters* ctr, const IbSolidDev& S, const double* table, int nx, int ny,
                      int nz, cudaStream_t st) {
    if (S.n == 0) return;
    ib_motion_kernel<<<blocks_for(S.n, 256), 256, 0, st>>>(ctr, S, table, nx, ny, nz);
}

void launch_ib_motion_once(const IbSolidDev& S, const double* row, int nx, int ny, int nz, cudaStream_t st) {
    if (S.n == 0) return;
    ib_motion_once_kernel<<<blocks_for(S.n, 256), 256, 0, st>>>(S, row, nx, ny, nz);
}

void launch_init(const FluidParams& P, const InitParams& ip, cudaStream_t st) {
    init_kernel<<<blocks_for(P.g.n, 256), 256, 0, st>>>(P, ip);
}

void launch_read_f(const FluidParams& P, int buffer, unsigned k0, unsigned k1, double* out, cudaStream_t st) {
    if (k1 > k0) read_f_kernel<<<blocks_for(k1 - k0, 256), 256, 0, st>>>(P, buffer, k0, k1, out);
}

void launch_read_macro(const FluidParams& P, unsigned k0, unsigned k1, double* rho, double* u, cudaStream_t st) {
    if (k1 > k0) read_macro_kernel<<<blocks_for(k1 - k0, 256), 256, 0, st>>>(P, k0, k1, rho, u);
}

void launch_write_f(const FluidParams& P, int buffer, int parity, const double* f, cudaStream_t st) {
    write_f_kernel<<<blocks_for(P.g.n, 256), 256, 0, st>>>(P, buffer, parity, f);
}

void launch_write_slots(const FluidParams& P, int parity, const double* f_star, cudaStream_t st) {
    write_slots_kernel<<<blocks_for(P.g.n, 256), 256, 0, st>>>(P, parity, f_star);
}

void launch_cell_flags(const FluidParams& P, unsigned k0, unsigned k1, unsigned char* out, cudaStream_t st) {
    if (k1 > k0) cell_flags_kernel<<<blocks_for(k1 - k0, 256), 256, 0, st>>>(P, k0, k1, out);
}

void launch_relayout(const float* src, float* dst, const RegionGeo& gs, const RegionGeo& gd, cudaStream_t st) {
    relayout_kernel<<<blocks_for(gs.n, 256), 256, 0, st>>>(src, dst, gs, gd);
}


}  // namespace lbmg
