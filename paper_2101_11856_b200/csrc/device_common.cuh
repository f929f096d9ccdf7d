// Device-side region description, kernel parameter blocks and the
// boundary-ownership logic shared by the fused fluid kernel and the IB band
// pre-pass.
//
// HBM layout of one region (a z-slab of owned planes):
//   f[2]        27 fp32 populations per node, DDF-shifted (f_i - w_i), in the
//               paper's CSoA layout (Eq. 9, layout.hpp:41-52) with group
//               alpha = 2^la; alpha >= n_pad is plain SoA.  A/B by step parity.
//   rho, u      fp32 rho* and u* (u as 3 SoA planes of stride ns)
//   gib, tflag  fp32 IB force density (3 SoA planes) + one epoch byte per node
//   cflag       (ghost layout) one epoch byte per 64-slot storage chunk
//   slot[2][6]  per-face persistent f* of the 9 populations each face
//               reconstructs (needed for the stale outflow-edge read,
//               SURVEY App. A.3), A/B by parity
//   halo        9 crossing populations of the neighbour's boundary plane
//               (c_z=+1 from below, c_z=-1 from above), A/B by parity
#pragma once

#include <cstdint>

#include "lattice.cuh"

namespace lbmg {

enum : int { kNoSlip = 0, kInlet = 1, kOutflow = 2, kPeriodic = 3 };
enum : int { kBGK = 0, kRawMRT = 1, kCentralMRT = 2 };
enum : int { kPolicyConstant = 0, kPolicyRelax = 1 };
constexpr unsigned char kNoOwner = 255;

// n / d for n < 2^31 with a precomputed magic number (round-up method).
struct FastDiv {
    unsigned d = 1, mul = 0, shift = 0;
    FastDiv() = default;
    explicit FastDiv(unsigned dv) : d(dv) {
        shift = 0;
        while ((1u << shift) < d) ++shift;
        unsigned long long m = ((1ull << 32) * ((1ull << shift) - d)) / d + 1;
        mul = static_cast<unsigned>(m);
    }
    LBMG_HD unsigned div(unsigned n) const {
#ifdef __CUDA_ARCH__
        return (__umulhi(n, mul) + n) >> shift;
#else
        return static_cast<unsigned>(((static_cast<unsigned long long>(n) * mul >> 32) + n) >> shift);
#endif
    }
};

struct RegionGeo {
    int nx, ny, nzl;      // owned local dims
    int NZ;               // global nz
    int gz0;              // global z of local plane 0
    int per[3];           // periodic axes
    unsigned plane;       // nx*ny
    unsigned n;           // owned nodes
    unsigned n_pad;       // padded node count (multiple of alpha, or of 32 for SoA)
    int la;               // log2(alpha); 31 for SoA
    unsigned amask;       // alpha-1; 0x7fffffff for SoA
    unsigned A;           // per-direction stride inside a group: alpha, or n_pad for SoA
    unsigned ns;          // stride of the per-node SoA fields (rho, u, gib): n rounded to 32
    FastDiv div_nx, div_ny;
    // Ghost-layer SoA ("ghost" = 1): each direction array is a padded box
    // with row pitch PX = nx + 4 (column c = x + 2: x = -1 and x = nx are
    // ghost columns, c = 0 and nx + 3 padding), PY = ny + 1 rows per plane
    // (row r = y + 1; row 0 is both the y = -1 ghost row of its plane and the
    // y = ny ghost row of the previous plane: those serve disjoint direction
    // sets, c_y = +1 and c_y = -1) and planes lz = -1 .. nzl.  A pull that
    // does not stream from inside the slab reads the ghost slot
    // s(node) - off_i, which the ghost-fill kernel writes each step.
    // Storage slots are grouped in Eq. 9 CSoA blocks of alpha = 2^la slots
    // (alpha >= 256; alpha >= slots = SoA): gaddr(s, i).  `base` leading
    // slots keep the shifted windows of the first tile inside the buffer.
    int ghost;
    unsigned PX, PY, PP;  // row pitch, rows per plane, PX * PY
    unsigned base;        // leading pad (a multiple of 256 slots)
    int cta;              // staged fluid kernel CTA size (0: LBMG_GHOST_THREADS or 512); a tuner dimension
    int nbuf;             // population buffers (2: the A/B pair)
    int zwrap;            // the slab is its own z neighbour (one periodic region)
    int has_outflow;      // some face is an outflow face (face slots are read)
    FastDiv div_px, div_py;

    LBMG_HD unsigned sidx(int x, int y, int lz) const {
        return base + (unsigned(lz + 1) * PY + unsigned(y + 1)) * PX + unsigned(x + 2);
    }
    LBMG_HD unsigned long long gaddr(unsigned long long s, int i) const {
        return (s >> la) * (27ull * A) + static_cast<unsigned long long>(static_cast<unsigned>(i)) * A + (s & amask);
    }
    // storage offset of one step along c_i in the ghost layout
    LBMG_HD long long soff(int i) const {
        return cx(i) + (long long)PX * cy(i) + (long long)PP * cz(i);
    }

    // Eq. 9 (layout.hpp:41-52): beta*alpha*floor(k/alpha) + alpha*i + k mod alpha
    // (ghost layout: i*A + sidx of the decoded node)
    LBMG_HD unsigned long long idx(unsigned k, int i) const {
        if (ghost) {
            const unsigned q = div_nx.div(k);
            const unsigned q2 = div_ny.div(q);
            return gaddr(sidx(int(k - q * unsigned(nx)), int(q - q2 * unsigned(ny)), int(q2)), i);
        }
        return static_cast<unsigned long long>(k >> la) * (27ull * A) +
               static_cast<unsigned long long>(static_cast<unsigned>(i)) * A + (k & amask);
    }
    // population i of the node at (x, y, lz), 0 <= x < nx, 0 <= y < ny, 0 <= lz < nzl
    LBMG_HD unsigned long long at(int x, int y, int lz, int i) const {
        if (ghost) return gaddr(sidx(x, y, lz), i);
        return idx(node(x, y, lz), i);
    }
    LBMG_HD unsigned node(int x, int y, int lz) const {
        return (static_cast<unsigned>(lz) * static_cast<unsigned>(ny) + static_cast<unsigned>(y)) *
                   static_cast<unsigned>(nx) +
               static_cast<unsigned>(x);
    }
    LBMG_HD int extent(int a) const { return a == 0 ? nx : (a == 1 ? ny : NZ); }
    // Face-plane (slot) extents: x faces (y, lz), y faces (x, lz), z faces (x, y).
    LBMG_HD unsigned slot_plane(int face) const {
        int a = face_axis(face);
        return a == 0 ? unsigned(ny) * nzl : (a == 1 ? unsigned(nx) * nzl : plane);
    }
    LBMG_HD unsigned slot_index(int face, int x, int y, int lz, int i) const {
        int a = face_axis(face);
        unsigned u = a == 0 ? y : x;
        unsigned v = a == 2 ? y : lz;
        unsigned U = a == 0 ? ny : nx;
        return cross9(i, a) * slot_plane(face) + v * U + u;
    }
};

struct FaceTable {
    int cond[6];
    float inlet[6][27];  // feq(1, u_in)_i - w_i per inlet face
};

struct ModelConst {
    int kind;
    int policy;
    float omega;     // BGK rate omega_nu
    float eps0;      // policy epsilon_0
    float rate[27];  // by moment tensor index mu
    float body[3];   // body force
};

// Pointers of one region.  Populations: f[fcur(t)] = f(t) in, f[fnext(t)] =
// f(t+1) out.  The [2] arrays are selected by step parity p=t&1:
// slot[p] = f* slots of step t-1 (read
// for stale outflow), slot[p^1] written; recv[p] = f(t) neighbour halo in;
// send[p^1] = f(t+1) halo out.
struct RegionPtrs {
    float* f[3];  // f(t) lives in f[fcur(t)]
    float* slot[2][6];
    const float* recv_lo[2];
    const float* recv_hi[2];
    float* send_lo[2];
    float* send_hi[2];
    float* rho;
    float* u;    // 3 planes of ns
    float* gib;  // 3 planes of ns, or null without solids
    // per node: ib_epoch(step) (1..255, never the zero of a fresh buffer) when the IB scattered into gib at that
    // step.  Never cleared: a stale byte that happens to match only makes the
    // fluid kernel add a gib it already zeroed (+0), so only the true band
    // nodes of this step pay the gib loads.
    unsigned char* tflag;
    // ghost layout: ib_epoch(step) per 64-slot storage chunk holding a node
    // the IB scattered into at that step (same epoch rule as tflag).  The
    // staged fluid kernel bulk-copies a tile's chunk bytes with its windows,
    // so tiles without IB force never load gib or a per-node flag.
    unsigned char* cflag;
    const float* mrecv_lo;  // (rho,u) of the ghost planes, 4*plane
    const float* mrecv_hi;
    float* msend_lo;
    float* msend_hi;
    unsigned* band_count;  // IB band nodes this step
    unsigned* queue;       // tile queues of the staged fluid launches: counters [4], CTAs done [4]
    // Per-step ghost fill as a copy program (ghost layout): per step parity,
    // fill_n[p] (src, dst) records = what ghost_fill_entry would read and
    // write that step, resolved once (fill_ghosts_full); null: the general kernel
    const float* inlet_g;  // 6 x 27 inlet constants (record sources)
    const struct FillRec* fill_plan[2];
    unsigned fill_runs[2];  // [0, fill_runs[p]): runs of 32 consecutive records (src + k -> dst + k)
    unsigned fill_n[2];     // [fill_eoff, fill_eoff + fill_n[p]): single records
    unsigned fill_eoff;
    // Reaction totals of the fused IB kernel of this step, summed by the
    // fluid kernel (its CTA k, k += grid, before its first tile): solid k's
    // block partials [ib_start[k], ib_start[k+1]) x 6 in the fixed order
    // (thread v of 128 takes blocks v, v + 128, ..., then a tree), row
    // (t - chunk_t0) at ib_out + row * ib_stride + 6k.  ib_solids = 0: none.
    const double* ib_partial;
    const unsigned* ib_start;
    double* ib_out;
    unsigned ib_solids;
    int ib_stride;
    // Zero-copy results (the single-region step the fluid kernel ends): the
    // device aliases of the mapped pinned host block advance() reads after
    // its stream sync — the counters (written by the last CTA) and the
    // totals rows (written next to ib_out) — so no D2H copy follows the step.
    struct DevCounters* ctr_host;
    double* ib_out_host;
};

// One record of the fill program: *dst = *src.
struct FillRec {
    const float* src;
    float* dst;
};

// Physical population buffer of f(t) (the A/B pair: nbuf = 2).
LBMG_HD int fcur(const RegionGeo& g, long long t) { return g.nbuf == 2 ? int(t & 1) : int(t % g.nbuf); }
LBMG_HD int fnext(const RegionGeo& g, long long t) { return fcur(g, t + 1); }

struct DevCounters {
    long long t;               // step counter
    unsigned diverged;         // sticky divergence flag
    unsigned mach;             // sticky Mach warning
    long long diverged_step;   // step at which divergence was detected
    long long chunk_t0;        // first step of the current advance chunk
};

// IB force-flag epoch of step t: 1..255 (a zeroed flag byte never matches)
LBMG_HD unsigned char ib_epoch(long long t) { return (unsigned char)(1 + t % 255); }

struct FluidParams {
    RegionGeo g;
    FaceTable faces;
    ModelConst m;
    RegionPtrs p;
    DevCounters* ctr;
};

// Owner face of the pull of direction i at global (gx, gy, gz): the first
// non-periodic face in pass order whose side the source x - c_i lies beyond,
// or kNoOwner when the pull streams (boundary.cpp:28-40).
template <int I>
LBMG_HD int owner_face_c(const RegionGeo& g, int gx, int gy, int gz) {
    constexpr int c0 = cx(I), c1 = cy(I), c2 = cz(I);
    if constexpr (c0 != 0) {
        if (!g.per[0]) {
            int s = gx - c0;
            if (s < 0) return 0;
            if (s >= g.nx) return 1;
        }
    }
    if constexpr (c1 != 0) {
        if (!g.per[1]) {
            int s = gy - c1;
            if (s < 0) return 2;
            if (s >= g.ny) return 3;
        }
    }
    if constexpr (c2 != 0) {
        if (!g.per[2]) {
            int s = gz - c2;
            if (s < 0) return 4;
            if (s >= g.NZ) return 5;
        }
    }
    return kNoOwner;
}

#ifdef __CUDACC__
// Local node index -> (x, y, lz).
__device__ __forceinline__ void decode(const RegionGeo& g, unsigned k, int& x, int& y, int& lz) {
    const unsigned q = g.div_nx.div(k);
    x = int(k - q * unsigned(g.nx));
    const unsigned q2 = g.div_ny.div(q);
    y = int(q - q2 * unsigned(g.ny));
    lz = int(q2);
}

// Per-step ghost fill through the copy program of this step's parity
// (RegionPtrs::fill_plan), block bid of nthr threads: the first blocks copy
// whole runs (one warp per 32-float run: one broadcast descriptor, coalesced
// 128-byte load and store — the y/z faces), the rest single records
// (x faces, edges, face slots).  kFillPer items per warp / thread with every
// load in flight before the stores.  Shared by ghost_copy_kernel and the
// merged IB + fill launch.
constexpr int kFillPer = 4;
__device__ __forceinline__ unsigned fill_run_blocks(const RegionPtrs& p, unsigned nthr) {
    const unsigned g = p.fill_runs[0] > p.fill_runs[1] ? p.fill_runs[0] : p.fill_runs[1];
    const unsigned per = (nthr / 32u) * kFillPer;
    return (g + per - 1) / per;
}
__device__ __forceinline__ void fill_copy_block(const FluidParams& P, unsigned bid, unsigned tid, unsigned nthr) {
    const int p = int(P.ctr->t & 1);
    const FillRec* __restrict__ rec = P.p.fill_plan[p];
    const unsigned rb = fill_run_blocks(P.p, nthr);
    const float* src[kFillPer];
    float* dst[kFillPer];
    if (bid < rb) {
        const unsigned lane = tid & 31u, w = bid * (nthr / 32u) + tid / 32u, ng = P.p.fill_runs[p];
#pragma unroll
        for (int k = 0; k < kFillPer; ++k) {
            const unsigned e = w * kFillPer + unsigned(k);
            if (e < ng) {
                const ulonglong2 r = __ldg(reinterpret_cast<const ulonglong2*>(rec + e));
                src[k] = reinterpret_cast<const float*>(r.x) + lane;
                dst[k] = reinterpret_cast<float*>(r.y) + lane;
            } else {
                src[k] = nullptr;
                dst[k] = nullptr;
            }
        }
    } else {
        const unsigned first = (bid - rb) * nthr * kFillPer + tid, n = P.p.fill_n[p];
        rec += P.p.fill_eoff;
#pragma unroll
        for (int k = 0; k < kFillPer; ++k) {
            const unsigned e = first + unsigned(k) * nthr;
            if (e < n) {
                const ulonglong2 r = __ldg(reinterpret_cast<const ulonglong2*>(rec + e));
                src[k] = reinterpret_cast<const float*>(r.x);
                dst[k] = reinterpret_cast<float*>(r.y);
            } else {
                src[k] = nullptr;
                dst[k] = nullptr;
            }
        }
    }
    float v[kFillPer];
#pragma unroll
    for (int k = 0; k < kFillPer; ++k) v[k] = src[k] != nullptr ? __ldcg(src[k]) : 0.f;
#pragma unroll
    for (int k = 0; k < kFillPer; ++k)
        if (dst[k] != nullptr) *dst[k] = v[k];
}
// blocks of nthr threads the fill program needs (host side too)
inline unsigned fill_blocks(const RegionPtrs& p, unsigned nthr) {
    const unsigned g = p.fill_runs[0] > p.fill_runs[1] ? p.fill_runs[0] : p.fill_runs[1];
    const unsigned e = p.fill_n[0] > p.fill_n[1] ? p.fill_n[0] : p.fill_n[1];
    const unsigned pr = (nthr / 32u) * kFillPer, pe = nthr * kFillPer;
    return (g + pr - 1) / pr + (e + pe - 1) / pe;
}

// Storage chunk (64 slots: one warp's 32 node pairs of a staged tile) of a
// ghost-layout node: the unit of cflag.  (256-slot chunks — about one grid
// row — made the fluid kernel load and zero 7x more gib than the band needs
// on C2: 207 vs 177 us without force.)
constexpr int kForceChunkShift = 6;

// Mark owned node k = (x, y, lz) as carrying IB force this step: its epoch
// byte (compact-layout kernels) or its storage chunk's (ghost layout).
__device__ __forceinline__ void mark_force(const FluidParams& P, unsigned k, int x, int y, int lz, unsigned char ep) {
    if (P.g.ghost) P.p.cflag[P.g.sidx(x, y, lz) >> kForceChunkShift] = ep;
    else P.p.tflag[k] = ep;
}
__device__ __forceinline__ void mark_force(const FluidParams& P, unsigned k, unsigned char ep) {
    if (P.g.ghost) {
        int x, y, lz;
        decode(P.g, k, x, y, lz);
        P.p.cflag[P.g.sidx(x, y, lz) >> kForceChunkShift] = ep;
    } else {
        P.p.tflag[k] = ep;
    }
}
#endif

// Runtime-direction variant (used on the rare reconstruction chains).
LBMG_HD int owner_face(const RegionGeo& g, int gx, int gy, int gz, int i) {
    const int c[3] = {cx(i), cy(i), cz(i)};
    const int coord[3] = {gx, gy, gz};
    for (int f = 0; f < 6; ++f) {
        int a = face_axis(f);
        if (g.per[a] || c[a] == 0) continue;
        int s = coord[a] - c[a];
        if (face_side(f) < 0 ? s < 0 : s >= g.extent(a)) return f;
    }
    return kNoOwner;
}

}  // namespace lbmg
