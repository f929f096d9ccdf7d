// Device smoke tracers (tracer.hpp / tracer.cpp; see tracers.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "device_common.cuh"
#include "lbmg.h"

namespace lbmg {

// u* of one z-slab region: compact node index (lz * ny + y) * nx + x,
// component c at + c * ns.
struct TracerRegion {
    const float* u;
    int z0, z1;
    unsigned ns;
};

struct TracerDev {
    double *x, *y, *z;            // cloud, emission order (capacity entries)
    long long* birth;             // birth step, -1 = retired (tombstone)
    const double* emit;           // this chunk's emissions: [step j][E][3]
    unsigned long long* state;    // [0] entries at chunk start, [1] tombstones
    unsigned long long E;         // particles emitted per step (sum of rates)
    const TracerRegion* reg;      // m regions (device array)
    int m;
    int nx, ny, nz;
};

// emit_tracers (tracer.cpp:28-40): the E positions step `step` appends.
void emit_positions(const std::vector<lbmg_emitter>& em, long step, uint64_t seed, double* out);

// One emit + advect + retire step (inside the step graph; after the fluid
// kernel wrote u*, before the step counter advances).
void launch_tracer_step(const TracerDev& T, const DevCounters* ctr, int sm_count, cudaStream_t st);
// Stable compaction of the first n entries (tombstones dropped), in place via
// the scratch arrays; returns the live count (synchronises the stream).
unsigned long long tracer_compact(const TracerDev& T, unsigned long long n, double* sx, double* sy, double* sz,
                                  long long* sb, cudaStream_t st);
// rasterize_density (tracer.cpp:67-92) of n entries (stride between a
// particle's coordinates: 1 for SoA arrays, 3 for AoS), tombstones skipped
// when birth != nullptr; vol (device, nx*ny*nz) is accumulated into.
void launch_rasterize(const double* x, const double* y, const double* z, size_t stride, const long long* birth,
                      unsigned long long n, int nx, int ny, int nz, double* vol, cudaStream_t st);

}  // namespace lbmg
