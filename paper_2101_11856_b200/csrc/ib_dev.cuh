// IB device helpers shared by the IB kernels (kernels.cu) and the step
// pipeline (pipeline.cu): kernel support (ib.cpp:294-308), the seam rule
// (ib.cpp:313-317) and the rigid-motion update of one sample (ib.cpp:456-489).
#pragma once

#include <cuda_runtime.h>

#include "device_common.cuh"
#include "engine.hpp"

namespace lbmg {

namespace {

struct Support {
    int base[3];
    double w[3][2];
    bool inside;
};

// kernel_support (ib.cpp:294-308), FP64, bit-exact flags.
__device__ __forceinline__ Support kernel_support(const double p[3], int nx, int ny, int nz) {
    Support ks;
    ks.inside = true;
    const int n[3] = {nx, ny, nz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (p[a] < 0.0 || p[a] > double(n[a] - 1)) ks.inside = false;
        int b = int(floor(p[a]));
        b = max(0, min(b, n[a] - 2));
        ks.base[a] = b;
        const double t = __dsub_rn(p[a], double(b));
        ks.w[a][0] = __dsub_rn(1.0, t);
        ks.w[a][1] = t;
    }
    return ks;
}

// sample_active (ib.cpp:313-317)
__device__ __forceinline__ bool sample_active(double pz, int NZ, int z0, int z1) {
    int bz = int(floor(pz));
    bz = max(0, min(bz, NZ - 2));
    return bz + 1 >= z0 && bz < z1;
}

}  // namespace

__device__ __forceinline__ void motion_apply(const double* row, IbSolidDev S, unsigned s, int nx, int ny, int nz) {
    const double* c = row;
    const double* R = row + 3;
    const double* v = row + 12;
    const double* w = row + 15;
    const double r0 = S.ref[3 * s], r1 = S.ref[3 * s + 1], r2 = S.ref[3 * s + 2];
    // p = R r, then center + p: same operation order, no contraction
    double p[3];
    for (int a = 0; a < 3; ++a)
        p[a] = __dadd_rn(__dadd_rn(__dmul_rn(R[3 * a], r0), __dmul_rn(R[3 * a + 1], r1)),
                         __dmul_rn(R[3 * a + 2], r2));
    double x[3];
    for (int a = 0; a < 3; ++a) x[a] = __dadd_rn(c[a], p[a]);
    const double d[3] = {__dsub_rn(x[0], c[0]), __dsub_rn(x[1], c[1]), __dsub_rn(x[2], c[2])};
    // omega x d (core.hpp:27-29)
    const double cr[3] = {__dsub_rn(__dmul_rn(w[1], d[2]), __dmul_rn(w[2], d[1])),
                          __dsub_rn(__dmul_rn(w[2], d[0]), __dmul_rn(w[0], d[2])),
                          __dsub_rn(__dmul_rn(w[0], d[1]), __dmul_rn(w[1], d[0]))};
    for (int a = 0; a < 3; ++a) {
        S.pos[3 * s + a] = x[a];
        S.ub[3 * s + a] = __dadd_rn(v[a], cr[a]);
    }
    const Support ks = kernel_support(x, nx, ny, nz);
    S.flagged[s] = ks.inside ? 0 : 1;
}

}  // namespace lbmg
