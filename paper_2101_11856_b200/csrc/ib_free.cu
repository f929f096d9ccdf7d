// The reference's IB free functions (ib.hpp:96-128, ib.cpp:294-501) as batch
// device kernels over host-supplied sample sets and fields: the unit-level
// half of the drop-in surface (the Runner fuses the same arithmetic into its
// step kernels, kernels.cu).  FP64 throughout, reference operation order and
// no contraction, so support, interpolation, penalty and rigid motion are
// bit-identical to the reference; the spreading sums use FP64 atomics (the
// reference's atomic mode) and the reaction totals a fixed-order tree.
//
// Fields are canonical AoS FP64 over the global grid (k = (z ny + y) nx + x);
// the owned slab [z0, z1) applies the seam rule (sample_active,
// ib.cpp:313-317) and restricts spreading to owned planes (ib.cpp:377).
#include <cuda_runtime.h>

#include "engine.hpp"
#include "ib_dev.cuh"

namespace lbmg {

namespace {

inline unsigned blocks_for(size_t n, unsigned t) { return unsigned((n + t - 1) / t); }

__device__ __forceinline__ double weight(const Support& ks, int ox, int oy, int oz) {
    return __dmul_rn(__dmul_rn(ks.w[0][ox], ks.w[1][oy]), ks.w[2][oz]);  // KernelSupport::weight
}

__device__ __forceinline__ size_t gnode(int nx, int ny, int x, int y, int z) {
    return (size_t(z) * size_t(ny) + size_t(y)) * size_t(nx) + size_t(x);
}

__global__ void support_kernel(size_t n, const double* pos, int nx, int ny, int nz, int* base, double* w,
                               unsigned char* inside) {
    const size_t s = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const double p[3] = {pos[3 * s], pos[3 * s + 1], pos[3 * s + 2]};
    const Support ks = kernel_support(p, nx, ny, nz);
    for (int a = 0; a < 3; ++a) {
        base[3 * s + a] = ks.base[a];
        w[6 * s + 2 * a] = ks.w[a][0];
        w[6 * s + 2 * a + 1] = ks.w[a][1];
    }
    inside[s] = ks.inside ? 1 : 0;
}

// interpolate_velocity (ib.cpp:321-343)
__global__ void interp_kernel(size_t n, const double* pos, const double* u, int nx, int ny, int nz, int z0, int z1,
                              double* sampled, unsigned char* flagged) {
    const size_t s = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const double p[3] = {pos[3 * s], pos[3 * s + 1], pos[3 * s + 2]};
    const Support ks = kernel_support(p, nx, ny, nz);
    flagged[s] = ks.inside ? 0 : 1;
    double us[3] = {0.0, 0.0, 0.0};
    if (ks.inside && sample_active(p[2], nz, z0, z1))
        for (int oz = 0; oz < 2; ++oz)
            for (int oy = 0; oy < 2; ++oy)
                for (int ox = 0; ox < 2; ++ox) {
                    const double w = weight(ks, ox, oy, oz);
                    const size_t k = gnode(nx, ny, ks.base[0] + ox, ks.base[1] + oy, ks.base[2] + oz);
                    for (int a = 0; a < 3; ++a) us[a] = __dadd_rn(us[a], __dmul_rn(w, u[3 * k + a]));
                }
    for (int a = 0; a < 3; ++a) sampled[3 * s + a] = us[a];
}

// penalty_forces (ib.cpp:345-365)
__global__ void penalty_kernel(size_t n, const double* pos, const double* ub, const double* sampled,
                               const unsigned char* flagged, const double* rho, int nx, int ny, int nz, int z0,
                               int z1, double* force) {
    const size_t s = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const double p[3] = {pos[3 * s], pos[3 * s + 1], pos[3 * s + 2]};
    if (flagged[s] || !sample_active(p[2], nz, z0, z1)) {
        for (int a = 0; a < 3; ++a) force[3 * s + a] = 0.0;
        return;
    }
    const Support ks = kernel_support(p, nx, ny, nz);
    double rs = 0.0;
    for (int oz = 0; oz < 2; ++oz)
        for (int oy = 0; oy < 2; ++oy)
            for (int ox = 0; ox < 2; ++ox)
                rs = __dadd_rn(rs, __dmul_rn(weight(ks, ox, oy, oz),
                                             rho[gnode(nx, ny, ks.base[0] + ox, ks.base[1] + oy, ks.base[2] + oz)]));
    for (int a = 0; a < 3; ++a) force[3 * s + a] = __dmul_rn(rs, __dsub_rn(ub[3 * s + a], sampled[3 * s + a]));
}

// spread_forces (ib.cpp:369-454, atomic mode): owned planes only
__global__ void spread_kernel(size_t n, const double* pos, const double* force, const unsigned char* flagged, int nx,
                              int ny, int nz, int z0, int z1, double* g) {
    const size_t s = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const double p[3] = {pos[3 * s], pos[3 * s + 1], pos[3 * s + 2]};
    if (flagged[s] || !sample_active(p[2], nz, z0, z1)) return;
    const Support ks = kernel_support(p, nx, ny, nz);
    for (int oz = 0; oz < 2; ++oz) {
        const int gz = ks.base[2] + oz;
        if (gz < z0 || gz >= z1) continue;
        for (int oy = 0; oy < 2; ++oy)
            for (int ox = 0; ox < 2; ++ox) {
                const double w = weight(ks, ox, oy, oz);
                const size_t k = gnode(nx, ny, ks.base[0] + ox, ks.base[1] + oy, gz);
                for (int a = 0; a < 3; ++a) atomicAdd(&g[3 * k + a], __dmul_rn(w, force[3 * s + a]));
            }
    }
}

// update_rigid_motion (ib.cpp:456-489) with R(t), c(t) from the host
__global__ void motion_free_kernel(size_t n, const double* ref, const double* row, int nx, int ny, int nz,
                                   double* pos, double* ub, unsigned char* flagged) {
    const size_t s = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    IbSolidDev S{};
    S.n = unsigned(n);
    S.ref = const_cast<double*>(ref);
    S.pos = pos;
    S.ub = ub;
    S.flagged = flagged;
    motion_apply(row, S, unsigned(s), nx, ny, nz);
}

// reaction_totals (ib.cpp:491-501): per-block partials in thread order, then a
// fixed-order final sum (one block)
constexpr int kRedThreads = 256;
__global__ void totals_free_kernel(size_t n, const double* pos, const double* force, double c0, double c1, double c2,
                                   int z0, int z1, double* partial) {
    __shared__ double sh[6][kRedThreads];
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (size_t s = size_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n; s += size_t(gridDim.x) * blockDim.x) {
        const double z = pos[3 * s + 2];
        if (z < double(z0) || z >= double(z1)) continue;
        const double F[3] = {force[3 * s], force[3 * s + 1], force[3 * s + 2]};
        const double r[3] = {__dsub_rn(pos[3 * s], c0), __dsub_rn(pos[3 * s + 1], c1), __dsub_rn(z, c2)};
        for (int a = 0; a < 3; ++a) acc[a] = __dsub_rn(acc[a], F[a]);
        acc[3] = __dsub_rn(acc[3], __dsub_rn(__dmul_rn(r[1], F[2]), __dmul_rn(r[2], F[1])));
        acc[4] = __dsub_rn(acc[4], __dsub_rn(__dmul_rn(r[2], F[0]), __dmul_rn(r[0], F[2])));
        acc[5] = __dsub_rn(acc[5], __dsub_rn(__dmul_rn(r[0], F[1]), __dmul_rn(r[1], F[0])));
    }
    for (int a = 0; a < 6; ++a) sh[a][threadIdx.x] = acc[a];
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if (int(threadIdx.x) < off)
            for (int a = 0; a < 6; ++a) sh[a][threadIdx.x] = __dadd_rn(sh[a][threadIdx.x], sh[a][threadIdx.x + off]);
        __syncthreads();
    }
    if (threadIdx.x < 6) partial[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void totals_final_kernel(const double* partial, int nblocks, double* out) {
    const int a = threadIdx.x;
    if (a >= 6) return;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc = __dadd_rn(acc, partial[b * 6 + a]);
    out[a] = acc;
}

}  // namespace

void launch_ib_support_batch(size_t n, const double* pos, int nx, int ny, int nz, int* base, double* w,
                             unsigned char* inside, cudaStream_t st) {
    if (n) support_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, nx, ny, nz, base, w, inside);
}

void launch_ib_interp_batch(size_t n, const double* pos, const double* u, int nx, int ny, int nz, int z0, int z1,
                            double* sampled, unsigned char* flagged, cudaStream_t st) {
    if (n) interp_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, u, nx, ny, nz, z0, z1, sampled, flagged);
}

void launch_ib_penalty_batch(size_t n, const double* pos, const double* ub, const double* sampled,
                             const unsigned char* flagged, const double* rho, int nx, int ny, int nz, int z0, int z1,
                             double* force, cudaStream_t st) {
    if (n)
        penalty_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, ub, sampled, flagged, rho, nx, ny, nz, z0, z1,
                                                          force);
}

void launch_ib_spread_batch(size_t n, const double* pos, const double* force, const unsigned char* flagged, int nx,
                            int ny, int nz, int z0, int z1, double* g, cudaStream_t st) {
    if (n) spread_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, pos, force, flagged, nx, ny, nz, z0, z1, g);
}

void launch_ib_motion_batch(size_t n, const double* ref, const double* row, int nx, int ny, int nz, double* pos,
                            double* ub, unsigned char* flagged, cudaStream_t st) {
    if (n) motion_free_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, ref, row, nx, ny, nz, pos, ub, flagged);
}

int ib_totals_batch_blocks(size_t n) {
    const size_t b = (n + kRedThreads - 1) / kRedThreads;
    return int(b < 1 ? 1 : (b > 128 ? 128 : b));
}

void launch_ib_totals_batch(size_t n, const double* pos, const double* force, const double* center, int z0, int z1,
                            double* partial, double* out, cudaStream_t st) {
    const int nb = ib_totals_batch_blocks(n);
    totals_free_kernel<<<nb, kRedThreads, 0, st>>>(n, pos, force, center[0], center[1], center[2], z0, z1, partial);
    totals_final_kernel<<<1, 32, 0, st>>>(partial, nb, out);
}

}  // namespace lbmg
