// Device helpers shared by the per-kernel step (fluid.cu) and the persistent
// step pipeline (pipeline.cu): step views of the population / halo buffers,
// the staged-tile geometry, the boundary pull chain (pull_source) and one
// ghost-fill entry (the six face passes, apply_face, boundary.cpp:42-125).
#pragma once

#include <cuda_runtime.h>

#include "device_common.cuh"

namespace lbmg {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Buffers of step parity p (slot pointers stay in kernel-parameter space:
// indexing them by a runtime face id must not spill a copy to local memory).
struct StepView {
    const float* fin;
    const float* halo_lo;
    const float* halo_hi;
    int p;
};

__device__ __forceinline__ StepView make_view(const FluidParams& P, long long t) {
    const int p = int(t & 1);
    return StepView{P.p.f[fcur(P.g, t)], P.p.recv_lo[p], P.p.recv_hi[p], p};
}

// Streamed value f_i(x - c_i) for a pull that is not missing (stream,
// solver.cpp:46-87): periodic wrap in x/y, ghost planes from the halo.
__device__ __forceinline__ float pull_rt(const RegionGeo& g, const StepView& v, int x, int y, int lz, int i) {
    int sx = x - cx(i), sy = y - cy(i);
    if (sx < 0) sx += g.nx;
    else if (sx >= g.nx) sx -= g.nx;
    if (sy < 0) sy += g.ny;
    else if (sy >= g.ny) sy -= g.ny;
    const int lzs = lz - cz(i);
    const unsigned hp = cross9(i, 2) * g.plane + unsigned(sy) * g.nx + unsigned(sx);
    if (lzs < 0) return v.halo_lo[hp];
    if (lzs >= g.nzl) return v.halo_hi[hp];
    return v.fin[g.at(sx, sy, lzs, i)];
}


// Sticky Mach warning (|u|^2 >= 0.16, collision.hpp:55): once set, further
// nodes only read it (L2), so a flow with many fast nodes does not serialise
// every thread on one atomic address.
__device__ __forceinline__ void raise_mach(DevCounters* ctr) {
    if (__ldcg(&ctr->mach) == 0u) atomicOr(&ctr->mach, 1u);
}

__device__ __forceinline__ void flag_divergence(DevCounters* ctr) {
    if (atomicExch(&ctr->diverged, 1u) == 0u) ctr->diverged_step = ctr->t;
}

}  // namespace

// Tile geometry per CTA size T (threads): 2T storage slots per tile.
template <int T>
struct GhostTile {
    static constexpr int kThreads = T;
    static constexpr int kTile = 2 * T;               // storage slots per tile
    static constexpr int kWin = kTile + 4;            // staged floats per direction
    static constexpr unsigned kStageBytes = 27u * kWin * 4u;
};
constexpr int kStages = 2;
template <int T>
constexpr unsigned staged_smem() { return kStages * GhostTile<T>::kStageBytes + 8u * kStages; }

// Window offset of slot 0 of a tile for direction i: tiles start at multiples
// of 4 and PX, PP are multiples of 4, so (tile start - off_i) = -c_x (mod 4).
__host__ __device__ constexpr int win_shift(int i) { return (4 - cx(i)) & 3; }

// Address of f*_i at (x,y,lz) for a pull that does not stream from inside
// the slab: the wrapped / halo source, or — for a missing pull — the value
// face pass `owner` reconstructs (same chain as reconstruct(): bounce-back
// source, inlet constant in kernel-parameter space, stale slot of a later
// face, or the streamed source of the outflow neighbour).  Never a ghost slot.
__device__ __forceinline__ const float* pull_source(const FluidParams& P, long long t, int x, int y, int lz, int i,
                                                   const float* inlet_g = nullptr) {
    const RegionGeo& g = P.g;
    const StepView v = make_view(P, t);
    const int p = v.p;
    auto pull_addr = [&](int xx, int yy, int zz) -> const float* {
        int sx = xx - cx(i), sy = yy - cy(i);
        if (sx < 0) sx += g.nx;
        else if (sx >= g.nx) sx -= g.nx;
        if (sy < 0) sy += g.ny;
        else if (sy >= g.ny) sy -= g.ny;
        const int lzs = zz - cz(i);
        const unsigned hp = cross9(i, 2) * g.plane + unsigned(sy) * g.nx + unsigned(sx);
        if (lzs < 0) return v.halo_lo + hp;
        if (lzs >= g.nzl) return v.halo_hi + hp;
        return v.fin + g.at(sx, sy, lzs, i);
    };
    int f = owner_face(g, x, y, g.gz0 + lz, i);
    if (f == kNoOwner) return pull_addr(x, y, lz);
    for (int guard = 0; guard < 7; ++guard) {
        const int cond = P.faces.cond[f];
        if (cond == kNoSlip) return v.fin + g.at(x, y, lz, opposite(i));
        if (cond == kInlet) return inlet_g != nullptr ? inlet_g + 27 * f + i : &P.faces.inlet[f][i];
        const int a = face_axis(f), s = face_side(f);
        if (a == 0) x -= s;
        else if (a == 1) y -= s;
        else lz -= s;
        const int fn = owner_face(g, x, y, g.gz0 + lz, i);
        if (fn == kNoOwner) return pull_addr(x, y, lz);
        if (fn > f) return P.p.slot[p][fn] + g.slot_index(fn, x, y, lz, i);
        f = fn;
    }
    return &P.faces.inlet[0][0];  // unreachable: the owner strictly decreases along the chain
}

// A persistent face slot is only ever read by an outflow chain (pull_source /
// reconstruct), which reaches a node by stepping one layer inward from an
// outflow face: only slots of nodes on the second layer of some outflow face
// can be read, so the fill stores only those (none without outflow faces).
__device__ __forceinline__ bool slot_readable(const FluidParams& P, int x, int y, int gz) {
    const RegionGeo& g = P.g;
    bool r = false;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        if (P.faces.cond[f] != kOutflow) continue;
        const int a = f >> 1, c = a == 0 ? x : (a == 1 ? y : gz);
        const int n = a == 0 ? g.nx : (a == 1 ? g.ny : g.NZ);
        r |= c == ((f & 1) ? n - 2 : 1);
    }
    return r;
}

// One thread per (slab-face node, crossing direction) entry; faces 0..5 in
// order, direction slot j (the two other velocity components, cross9 order)
// slowest, so consecutive threads walk a face row.  Common rules inline —
// bounce-back (f*_i = f_{i'}(N), boundary.cpp:98-100), inlet
// (feq(1, u_in)_i), periodic wrap / z halo (plain pull) — the outflow chain
// through pull_source().
// Inlet entries are constants (feq(1, u_in)_i): a full fill (init, layout
// change, loaded state) writes their ghost slots in both population buffers;
// the per-step fill only refreshes their (rare) outflow-readable face slots.
template <int F>
__device__ __forceinline__ void ghost_fill_entry(const FluidParams& P, long long t, unsigned q, unsigned j,
                                                 bool full = true) {
    const int p = int(t & 1);
    const RegionGeo& g = P.g;
    constexpr int A = face_axis(F), S = face_side(F);
    int x, y, lz;
    if constexpr (A == 0) {
        const unsigned qq = g.div_ny.div(q);
        y = int(q - qq * unsigned(g.ny));
        lz = int(qq);
        x = S < 0 ? 0 : g.nx - 1;
    } else {
        const unsigned qq = g.div_nx.div(q);
        x = int(q - qq * unsigned(g.nx));
        if constexpr (A == 1) {
            lz = int(qq);
            y = S < 0 ? 0 : g.ny - 1;
        } else {
            y = int(qq);
            lz = S < 0 ? 0 : g.nzl - 1;
        }
    }
    const int ja = int(j % 3u) - 1, jb = int(j / 3u) - 1;
    const int c0 = A == 0 ? -S : ja, c1 = A == 0 ? ja : (A == 1 ? -S : jb), c2 = A == 2 ? -S : jb;
    const int i = tensor_dir((c0 + 1) + 3 * (c1 + 1) + 9 * (c2 + 1));
    const int own = owner_face(g, x, y, g.gz0 + lz, i);
    const unsigned sn = g.sidx(x, y, lz);
    float* fin = P.p.f[fcur(g, t)];
    float val;
    if (own == kNoOwner) {  // periodic wrap in x/y, z halo
        int sx = x - c0, sy = y - c1;
        sx += sx < 0 ? g.nx : (sx >= g.nx ? -g.nx : 0);
        sy += sy < 0 ? g.ny : (sy >= g.ny ? -g.ny : 0);
        const int lzs = lz - c2;
        const unsigned hp = cross9(i, 2) * g.plane + unsigned(sy) * g.nx + unsigned(sx);
        if (lzs < 0) val = P.p.recv_lo[p][hp];
        else if (lzs >= g.nzl) val = P.p.recv_hi[p][hp];
        else val = fin[g.gaddr(g.sidx(sx, sy, lzs), i)];
    } else {
        const int cond = P.faces.cond[own];
        if (cond == kInlet) {
            val = P.faces.inlet[own][i];
            // the face slot of this step stays per step: at t = 0 the stale
            // read of an inlet entry must see the initial f*, later the constant
            if (slot_readable(P, x, y, g.gz0 + lz)) P.p.slot[p ^ 1][own][g.slot_index(own, x, y, lz, i)] = val;
            if (full) {
                const unsigned long long gs = g.gaddr((unsigned long long)((long long)sn - g.soff(i)), i);
                for (int b = 0; b < g.nbuf; ++b) P.p.f[b][gs] = val;
            }
            return;
        }
        if (cond == kNoSlip) val = fin[g.gaddr(sn, 27 - i)];
        else val = *pull_source(P, t, x, y, lz, i);
        if (slot_readable(P, x, y, g.gz0 + lz)) P.p.slot[p ^ 1][own][g.slot_index(own, x, y, lz, i)] = val;
    }
    fin[g.gaddr((unsigned long long)((long long)sn - g.soff(i)), i)] = val;
}

// The per-step (full = false) work of ghost_fill_entry<F> at step parity p as
// copy records (the addresses it would read and write); returns how many (0..2).
template <int F>
__device__ __forceinline__ int ghost_plan_entry(const FluidParams& P, int p, unsigned q, unsigned j, FillRec (&rec)[2]) {
    const RegionGeo& g = P.g;
    constexpr int A = face_axis(F), S = face_side(F);
    int x, y, lz;
    if constexpr (A == 0) {
        const unsigned qq = g.div_ny.div(q);
        y = int(q - qq * unsigned(g.ny));
        lz = int(qq);
        x = S < 0 ? 0 : g.nx - 1;
    } else {
        const unsigned qq = g.div_nx.div(q);
        x = int(q - qq * unsigned(g.nx));
        if constexpr (A == 1) {
            lz = int(qq);
            y = S < 0 ? 0 : g.ny - 1;
        } else {
            y = int(qq);
            lz = S < 0 ? 0 : g.nzl - 1;
        }
    }
    const int ja = int(j % 3u) - 1, jb = int(j / 3u) - 1;
    const int c0 = A == 0 ? -S : ja, c1 = A == 0 ? ja : (A == 1 ? -S : jb), c2 = A == 2 ? -S : jb;
    const int i = tensor_dir((c0 + 1) + 3 * (c1 + 1) + 9 * (c2 + 1));
    const int own = owner_face(g, x, y, g.gz0 + lz, i);
    const unsigned sn = g.sidx(x, y, lz);
    float* fin = P.p.f[fcur(g, p)];
    const float* src;
    int n = 0;
    if (own == kNoOwner) {
        int sx = x - c0, sy = y - c1;
        sx += sx < 0 ? g.nx : (sx >= g.nx ? -g.nx : 0);
        sy += sy < 0 ? g.ny : (sy >= g.ny ? -g.ny : 0);
        const int lzs = lz - c2;
        const unsigned hp = cross9(i, 2) * g.plane + unsigned(sy) * g.nx + unsigned(sx);
        if (lzs < 0) src = P.p.recv_lo[p] + hp;
        else if (lzs >= g.nzl) src = P.p.recv_hi[p] + hp;
        else src = fin + g.gaddr(g.sidx(sx, sy, lzs), i);
    } else {
        const int cond = P.faces.cond[own];
        const bool keep = slot_readable(P, x, y, g.gz0 + lz);
        float* sdst = keep ? P.p.slot[p ^ 1][own] + g.slot_index(own, x, y, lz, i) : nullptr;
        if (cond == kInlet) {  // ghost slots hold the constant since the full fill
            if (keep) rec[n++] = FillRec{P.p.inlet_g + 27 * own + i, sdst};
            return n;
        }
        src = cond == kNoSlip ? fin + g.gaddr(sn, 27 - i) : pull_source(P, p, x, y, lz, i, P.p.inlet_g);
        if (keep) rec[n++] = FillRec{src, sdst};
    }
    rec[n++] = FillRec{src, fin + g.gaddr((unsigned long long)((long long)sn - g.soff(i)), i)};
    return n;
}


}  // namespace lbmg
