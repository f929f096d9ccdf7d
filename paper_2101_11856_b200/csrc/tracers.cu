// Smoke tracers on the device (tracer.cpp:28-92, runner.cpp:213-223,
// :232-250): emit -> advect -> retire every step, inside the step graph.
//
// The cloud lives in HBM as FP64 SoA (x, y, z) + int64 birth step in
// emission order.  Retired particles are tombstoned (birth = -1) by the
// advection kernel instead of being compacted every step; the order of the
// live particles is the reference's (emission order, retired removed), and a
// stable compaction (flag -> CUB exclusive scan -> scatter) runs between
// advance chunks once half of the entries are tombstones.  Emission draws
// the reference's mt19937_64 stream on the host (it is an input of the step,
// like the motion table: one batch per chunk, uploaded before the graphs).
#include <cub/cub.cuh>

#include <random>
#include <stdexcept>
#include <string>

#include "tracers.hpp"

namespace lbmg {

void emit_positions(const std::vector<lbmg_emitter>& em, long step, uint64_t seed, double* out) {
    std::mt19937_64 rng(seed ^ (0x9e3779b97f4a7c15ull * static_cast<uint64_t>(step + 1)));
    auto uniform = [&](double lo, double hi) { return lo + (hi - lo) * ((rng() >> 11) * 0x1.0p-53); };
    size_t k = 0;
    for (const auto& e : em)
        for (int p = 0; p < e.rate; ++p) {
            // braced-init order of the reference: x, y, z drawn in sequence
            const double x = uniform(e.lo[0], e.hi[0]);
            const double y = uniform(e.lo[1], e.hi[1]);
            const double z = uniform(e.lo[2], e.hi[2]);
            out[k++] = x;
            out[k++] = y;
            out[k++] = z;
        }
}

namespace {

void tk(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// kernel_support (ib.cpp:294-308): base = clamp(floor(p), 0, n-2), weights
// (1-t, t) with t = p - base, inside <=> 0 <= p <= n-1 on every axis.
struct Support {
    int b[3];
    double w[3][2];
    bool inside;
};

__device__ __forceinline__ Support support_of(const double p[3], const int n[3]) {
    Support s;
    s.inside = true;
    for (int a = 0; a < 3; ++a) {
        if (p[a] < 0.0 || p[a] > double(n[a] - 1)) s.inside = false;
        int b = int(floor(p[a]));
        b = max(0, min(b, n[a] - 2));
        s.b[a] = b;
        const double t = __dsub_rn(p[a], double(b));
        s.w[a][0] = __dsub_rn(1.0, t);
        s.w[a][1] = t;
    }
    return s;
}

__device__ __forceinline__ bool inside_of(const double p[3], const int n[3]) {
    for (int a = 0; a < 3; ++a)
        if (p[a] < 0.0 || p[a] > double(n[a] - 1)) return false;
    return true;
}

// Runner::sample_velocity_region: trilinear u* over the 2x2x2 support, each
// corner read from the region owning its plane (the reference reads the
// base plane's region incl. its exchanged ghost plane: the same values).
// Sum order and rounding as the reference (oz, oy, ox; w = wx*wy*wz; no FMA).
__device__ __forceinline__ void sample_u(const TracerDev& T, const Support& s, double v[3]) {
    v[0] = v[1] = v[2] = 0.0;
    for (int oz = 0; oz < 2; ++oz) {
        const int z = s.b[2] + oz;
        int r = 0;
        while (r + 1 < T.m && z >= T.reg[r].z1) ++r;
        const TracerRegion R = T.reg[r];
        for (int oy = 0; oy < 2; ++oy)
            for (int ox = 0; ox < 2; ++ox) {
                const double w = __dmul_rn(__dmul_rn(s.w[0][ox], s.w[1][oy]), s.w[2][oz]);
                const size_t k =
                    (size_t(z - R.z0) * unsigned(T.ny) + size_t(s.b[1] + oy)) * unsigned(T.nx) + size_t(s.b[0] + ox);
                for (int c = 0; c < 3; ++c)
                    v[c] = __dadd_rn(v[c], __dmul_rn(w, double(__ldg(R.u + k + size_t(c) * R.ns))));
            }
    }
}

// One step of emit_tracers + advect_tracers (tracer.cpp:28-65): entries
// [0, n_prev) are the cloud before this step, [n_prev, n_prev + E) this
// step's emission (batch j = t - chunk_t0 of the uploaded chunk).  A
// particle is retired when its support leaves the grid before or after the
// move (the reference's two sampler calls).
__global__ void __launch_bounds__(256) tracer_step_kernel(TracerDev T, const DevCounters* ctr) {
    if (ctr->diverged) return;  // the reference returns before the tracer phase
    const long long t = ctr->t;
    const unsigned long long j = (unsigned long long)(t - ctr->chunk_t0);
    const unsigned long long n_prev = T.state[0] + T.E * j;
    const unsigned long long total = n_prev + T.E;
    const int n[3] = {T.nx, T.ny, T.nz};
    unsigned dead = 0;
    for (unsigned long long p = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; p < total;
         p += (unsigned long long)gridDim.x * blockDim.x) {
        double q[3];
        long long b;
        if (p >= n_prev) {
            const double* e = T.emit + 3ull * (j * T.E + (p - n_prev));
            q[0] = e[0];
            q[1] = e[1];
            q[2] = e[2];
            b = t;
        } else {
            b = T.birth[p];
            if (b < 0) continue;  // retired earlier
            q[0] = T.x[p];
            q[1] = T.y[p];
            q[2] = T.z[p];
        }
        const Support s = support_of(q, n);
        bool live = s.inside;
        if (live) {
            double v[3];
            sample_u(T, s, v);
            for (int a = 0; a < 3; ++a) q[a] = __dadd_rn(q[a], v[a]);
            live = inside_of(q, n);  // the probe sample after the move
        }
        T.x[p] = q[0];
        T.y[p] = q[1];
        T.z[p] = q[2];
        T.birth[p] = live ? b : -1;
        dead += live ? 0u : 1u;
    }
    // warp-aggregated tombstone count
    for (int o = 16; o > 0; o >>= 1) dead += __shfl_down_sync(0xffffffffu, dead, o);
    if ((threadIdx.x & 31u) == 0 && dead) atomicAdd(&T.state[1], (unsigned long long)dead);
}

__global__ void tracer_flag_kernel(const long long* birth, unsigned long long n, unsigned* flag) {
    for (unsigned long long p = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; p < n;
         p += (unsigned long long)gridDim.x * blockDim.x)
        flag[p] = birth[p] >= 0 ? 1u : 0u;
}

__global__ void tracer_scatter_kernel(TracerDev T, unsigned long long n, const unsigned* idx, double* sx, double* sy,
                                      double* sz, long long* sb) {
    for (unsigned long long p = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; p < n;
         p += (unsigned long long)gridDim.x * blockDim.x) {
        const long long b = T.birth[p];
        if (b < 0) continue;
        const unsigned d = idx[p];
        sx[d] = T.x[p];
        sy[d] = T.y[p];
        sz[d] = T.z[p];
        sb[d] = b;
    }
}

// rasterize_density: cell centres at i + 0.5, clamped offsets (a partition
// of unity at the rim); w = w0 * w1 * w2 as the reference, FP64 atomics
// (the per-cell sum order is not the reference's: agreement to rounding).
__global__ void rasterize_kernel(const double* x, const double* y, const double* z, size_t stride,
                                 const long long* birth, unsigned long long n, int nx, int ny, int nz, double* vol) {
    const int dims[3] = {nx, ny, nz};
    for (unsigned long long p = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; p < n;
         p += (unsigned long long)gridDim.x * blockDim.x) {
        if (birth && birth[p] < 0) continue;
        const double sh[3] = {__dsub_rn(x[p * stride], 0.5), __dsub_rn(y[p * stride], 0.5),
                              __dsub_rn(z[p * stride], 0.5)};
        int base[3];
        double w[3][2];
        for (int a = 0; a < 3; ++a) {
            int b = int(floor(sh[a]));
            b = max(0, min(b, dims[a] - 2));
            double t = __dsub_rn(sh[a], double(b));
            t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
            base[a] = b;
            w[a][0] = __dsub_rn(1.0, t);
            w[a][1] = t;
        }
        for (int oz = 0; oz < 2; ++oz)
            for (int oy = 0; oy < 2; ++oy)
                for (int ox = 0; ox < 2; ++ox) {
                    const size_t k = (size_t(base[2] + oz) * unsigned(ny) + size_t(base[1] + oy)) * unsigned(nx) +
                                     size_t(base[0] + ox);
                    atomicAdd(vol + k, __dmul_rn(__dmul_rn(w[0][ox], w[1][oy]), w[2][oz]));
                }
    }
}

unsigned grid_for(unsigned long long n, int cap) {
    const unsigned long long b = (n + 255) / 256;
    return unsigned(b < 1 ? 1 : (b > (unsigned long long)cap ? cap : b));
}

}  // namespace

void launch_tracer_step(const TracerDev& T, const DevCounters* ctr, int sm_count, cudaStream_t st) {
    // grid-stride over a cloud whose size only the device knows (the graph
    // is replayed across steps): a fixed persistent-style grid
    tracer_step_kernel<<<sm_count * 8, 256, 0, st>>>(T, ctr);
    tk(cudaGetLastError(), "tracer_step_kernel");
}

unsigned long long tracer_compact(const TracerDev& T, unsigned long long n, double* sx, double* sy, double* sz,
                                  long long* sb, cudaStream_t st) {
    if (n == 0) return 0;
    if (n >= (1ull << 32)) throw std::runtime_error("tracer cloud exceeds 2^32 entries");
    unsigned* flag = nullptr;
    unsigned* idx = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    tk(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, flag, idx, int(n), st), "cub scan size");
    tk(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(unsigned) * (n + 1), st), "tracer flags");
    tk(cudaMallocAsync(reinterpret_cast<void**>(&idx), sizeof(unsigned) * (n + 1), st), "tracer index");
    tk(cudaMallocAsync(&temp, temp_bytes, st), "tracer scan temp");
    tracer_flag_kernel<<<grid_for(n, 4096), 256, 0, st>>>(T.birth, n, flag);
    tk(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flag, idx, int(n), st), "cub scan");
    tracer_scatter_kernel<<<grid_for(n, 4096), 256, 0, st>>>(T, n, idx, sx, sy, sz, sb);
    unsigned last_idx = 0, last_flag = 0;
    tk(cudaMemcpyAsync(&last_idx, idx + (n - 1), sizeof(unsigned), cudaMemcpyDeviceToHost, st), "compact count");
    tk(cudaMemcpyAsync(&last_flag, flag + (n - 1), sizeof(unsigned), cudaMemcpyDeviceToHost, st), "compact count");
    tk(cudaStreamSynchronize(st), "compact sync");
    const unsigned long long live = (unsigned long long)last_idx + last_flag;
    tk(cudaMemcpyAsync(T.x, sx, sizeof(double) * live, cudaMemcpyDeviceToDevice, st), "compact copy");
    tk(cudaMemcpyAsync(T.y, sy, sizeof(double) * live, cudaMemcpyDeviceToDevice, st), "compact copy");
    tk(cudaMemcpyAsync(T.z, sz, sizeof(double) * live, cudaMemcpyDeviceToDevice, st), "compact copy");
    tk(cudaMemcpyAsync(T.birth, sb, sizeof(long long) * live, cudaMemcpyDeviceToDevice, st), "compact copy");
    tk(cudaFreeAsync(flag, st), "free");
    tk(cudaFreeAsync(idx, st), "free");
    tk(cudaFreeAsync(temp, st), "free");
    tk(cudaStreamSynchronize(st), "compact sync");
    return live;
}

void launch_rasterize(const double* x, const double* y, const double* z, size_t stride, const long long* birth,
                      unsigned long long n, int nx, int ny, int nz, double* vol, cudaStream_t st) {
    if (n == 0) return;
    rasterize_kernel<<<grid_for(n, 148 * 16), 256, 0, st>>>(x, y, z, stride, birth, n, nx, ny, nz, vol);
    tk(cudaGetLastError(), "rasterize_kernel");
}

}  // namespace lbmg
