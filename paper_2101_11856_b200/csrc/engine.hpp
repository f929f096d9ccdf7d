// Host-visible declarations of the device engine (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "device_common.cuh"

namespace lbmg {

// Device replica of one SolidSampleSet (ib.hpp:47-60), SoA of FP64 Vec3.
struct IbSolidDev {
    unsigned n;
    double* pos;      // n*3
    double* ref;      // n*3
    double* ub;       // n*3
    double* force;    // kIbHalves * n*3: one part per buffered step (ib_half)
    double* sampled;  // kIbHalves * n*3
    int nbuf;         // parts in use: the region's population buffer count
    // samples the fused IB kernel runs over: static solids, the region's
    // active ones (support inside the grid and touching the slab, fixed for a
    // static set); nullptr = all n (moving solids, deterministic mode)
    unsigned* active = nullptr;
    unsigned n_active = 0;
    double* act_pu = nullptr;  // (pos, u_b) of active[j] at 6j: one load level less for the fused kernel
    unsigned* corner_band = nullptr;  // band path: band index of active sample j's corner c at 8j + c (~0u: none)
    unsigned* source;
    unsigned char* flagged;
    // deterministic accumulation (ib_accumulation = deterministic): one
    // record per (sample, support corner) = (owned node | ~0u, w * g_s);
    // sorted by node (stable: sample order), summed per node in FP64
    unsigned* rec_key = nullptr;   // 8n
    unsigned* rec_idx = nullptr;   // 8n
    double* rec_val = nullptr;     // 3 * 8n
    unsigned* key_sorted = nullptr;
    unsigned* idx_sorted = nullptr;
    void* sort_temp = nullptr;
    size_t sort_temp_bytes = 0;
};

// Offset of step t's part of the penalty-force / sampled-velocity arrays
// (nbuf parts, like the population buffers).  Step t writes part t % nbuf;
// the values the reference holds after a run are those of the last step whose
// IB phase ran, t_ - 1, so readback uses part (t_ - 1) % nbuf: a diverging
// step's IB output lands in the other part and is never seen (the reference
// returns before IB, runner.cpp:154-161).
constexpr int kIbHalves = 2;
LBMG_HD size_t ib_half(const IbSolidDev& S, long long t) {
    return size_t(((t % S.nbuf) + S.nbuf) % S.nbuf) * 3 * size_t(S.n);
}

// Motion table row per step: center(t)[3], R(t)[9], v[3], omega[3].
constexpr int kMotionRow = 18;

struct InitParams {
    int kind;  // 0 uniform, 1 Taylor-Green
    double rho0;
    double u0[3];
    double tg_u;
    int NX, NY;
};

// Floats allocated per population buffer: 27 * n_pad plus a tail the bulk
// kernel's staged windows may read past the last direction array (the
// widest window of the last tile ends <= nx + 2 * kBulkTile + 8 floats past
// the owned nodes; never used).
inline unsigned long long f_alloc_floats(const RegionGeo& g) {
    return 27ull * g.n_pad + unsigned(g.nx) + 1024u;
}

bool ghost_layout_enabled();

// part: 0 every node, 1 the two halo planes (edge), 2 everything else (bulk)
// end_step: the (single, part 0, ghost-layout) fluid launch also ends the
// step (t += 1 in its last CTA); returns whether it did, else the caller
// launches step_end_kernel.
bool launch_fluid(const FluidParams& P, int part, int write_macro, cudaStream_t st, bool fill = true,
                  bool end_step = false);
void launch_macro(const FluidParams& P, long long t, cudaStream_t st);  // rho*/u* of step t from f(t)
void launch_ib_mark(const FluidParams& P, const IbSolidDev& S, unsigned* stamp, unsigned* band,
                    cudaStream_t st);
void launch_ib_band(const FluidParams& P, const unsigned* band, int sm_count, cudaStream_t st);
void launch_macro_pack(const FluidParams& P, cudaStream_t st);
void launch_ib_spread(const FluidParams& P, const IbSolidDev& S, cudaStream_t st, bool deterministic = false);
// deterministic accumulation: CUB temp bytes for 8n records; the sort +
// fixed-order per-node FP64 sum into g (after the spread / fused kernel)
size_t ib_det_temp_bytes(unsigned n_samples);
void launch_ib_det_reduce(const FluidParams& P, const IbSolidDev& S, cudaStream_t st);
int totals_blocks(size_t n);
// single-region ghost-layout IB step (interp + penalty + scatter + totals + motion), after launch_ghost_fill
int fused_blocks(size_t n);
// every solid in one launch (device descriptors); totals row of solid k at
// out_base[(t - chunk_t0) * out_stride + 6k]
// A slab whose f the fused IB kernel may read: its geometry and population
// buffers (own region, or an in-process neighbour across a seam).
struct IbSlab {
    RegionGeo g;
    const float* f[3];
};
struct IbBatch {
    IbSlab own, lo, hi;            // the region and its z neighbours (own where absent)
    const IbSolidDev* solids;      // device copy, n_solids
    const unsigned* block_start;   // n_solids + 1 prefix of fused_blocks(samples run)
    const unsigned* block_solid;   // solid of each block (one load instead of a binary search)
    const int* moving;             // n_solids
    unsigned n_solids;
    const double* table;           // motion rows, table_stride doubles per solid
    size_t table_stride;
    double* partial;               // 6 per block
    int probe;
    unsigned fill_from;            // blocks >= fill_from replay the ghost-fill program (0: none)
    const float* band_m;           // band path: (rho* - 1, j*) per band node, 4 floats (null: gathers)
    IbSolidDev solo;               // solids[0] when n_solids == 1 (read from parameter space)
};
void launch_ib_fused(const FluidParams& P, IbBatch B, unsigned total_blocks, const IbSolidDev* host_solids,
                     cudaStream_t st, bool deterministic = false);
// Band path of the fused IB kernel (static solids, one region): the sorted
// unique support-node slots of every active sample (band, sized 8 x the
// active samples) and each (sample, corner)'s band index in corner_band;
// returns the band size.  Per step launch_ib_band_moments writes rho* - 1 and
// j* of every band node (the same 27 pulls and sum order as the fused
// kernel's gather, coalesced along rows), which the fused kernel then reads
// per corner instead of gathering 27 populations.
unsigned build_ib_band(const FluidParams& P, IbSolidDev* solids, size_t n_solids, unsigned* band, cudaStream_t st);
void launch_ib_band_moments(const FluidParams& P, const unsigned* band, unsigned n, float* out, cudaStream_t st);

// The same launch with the ghost-fill program appended as extra blocks (one
// launch instead of a fill || IB fork/join; only when no support node can
// touch a ghost slot and the region has a fill program).  Atomic mode.
void launch_ib_fused_fill(const FluidParams& P, IbBatch B, unsigned total_blocks, cudaStream_t st);

// ghost slots of this step: full = every entry (after init / relayout),
// otherwise only what the previous fluid step did not push
void launch_ghost_fill(const FluidParams& P, cudaStream_t st, bool full = false);
// Resolve the per-step fill of step parity p into copy records: runs at
// out[0..), single records at out[eoff..) (out may be null: count only);
// synchronous, counts = {runs, single records}.
void launch_fill_plan(const FluidParams& P, int p, FillRec* out, unsigned eoff, unsigned* count_dev,
                      unsigned counts[2], cudaStream_t st);
// table: motion rows per step from DevCounters::chunk_t0; stride in doubles per step
void launch_ib_totals(const FluidParams& P, const IbSolidDev& S, const double* table, double* partial,
                      double* out_base, int stride, cudaStream_t st);
void launch_ib_motion(const DevCounters* ctr, const IbSolidDev& S, const double* table, int nx, int ny,
                      int nz, cudaStream_t st);
void launch_ib_motion_once(const IbSolidDev& S, const double* row, int nx, int ny, int nz,
                           cudaStream_t st);
void launch_step_end(DevCounters* ctr, cudaStream_t st);
void launch_init(const FluidParams& P, const InitParams& ip, cudaStream_t st);
void launch_read_f(const FluidParams& P, int buffer, unsigned k0, unsigned k1, double* out,
                   cudaStream_t st);
void launch_read_macro(const FluidParams& P, unsigned k0, unsigned k1, double* rho, double* u,
                       cudaStream_t st);
void launch_cell_flags(const FluidParams& P, unsigned k0, unsigned k1, unsigned char* out,
                       cudaStream_t st);
void launch_relayout(const float* src, float* dst, const RegionGeo& gs, const RegionGeo& gd,
                     cudaStream_t st);
// the IB free functions on sample batches (ib_free.cu)
void launch_ib_support_batch(size_t n, const double* pos, int nx, int ny, int nz, int* base, double* w,
                             unsigned char* inside, cudaStream_t st);
void launch_ib_interp_batch(size_t n, const double* pos, const double* u, int nx, int ny, int nz, int z0, int z1,
                            double* sampled, unsigned char* flagged, cudaStream_t st);
void launch_ib_penalty_batch(size_t n, const double* pos, const double* ub, const double* sampled,
                             const unsigned char* flagged, const double* rho, int nx, int ny, int nz, int z0, int z1,
                             double* force, cudaStream_t st);
void launch_ib_spread_batch(size_t n, const double* pos, const double* force, const unsigned char* flagged, int nx,
                            int ny, int nz, int z0, int z1, double* g, cudaStream_t st);
void launch_ib_motion_batch(size_t n, const double* ref, const double* row, int nx, int ny, int nz, double* pos,
                            double* ub, unsigned char* flagged, cudaStream_t st);
int ib_totals_batch_blocks(size_t n);
void launch_ib_totals_batch(size_t n, const double* pos, const double* force, const double* center, int z0, int z1,
                            double* partial, double* out, cudaStream_t st);
// load a canonical AoS FP64 state: f (nodes*27) into buffer `buffer`, and the
// persistent face slots of parity p from f_star (nodes*27)
void launch_write_f(const FluidParams& P, int buffer, int parity, const double* f, cudaStream_t st);
void launch_write_slots(const FluidParams& P, int parity, const double* f_star, cudaStream_t st);
void launch_collide_batch(const ModelConst& m, unsigned n, const double* f, const double* rho,
                          const double* u, double* omega, cudaStream_t st);

}  // namespace lbmg
