// D3Q27 lattice as compile-time tables (host + device).
//
// Canonical direction order follows the reference (lattice.cpp:8-19): index 0
// is rest, 1..26 are lexicographic in (c_z, c_y, c_x).  Everything here is
// constexpr so the unrolled kernels fold all c_i / w_i arithmetic.
//
//  * tensor index  T(i) = (cx+1) + 3(cy+1) + 9(cz+1)   (collision.cpp:38-41)
//  * opposite(i)   = 27 - i for i >= 1               (survey probe `tables`)
//  * c_z = -1  <=>  i in 1..9 ;  c_z = +1  <=>  i in 18..26
//  * moment tensor index mu = qx + 3 qy + 9 qz, degree qx+qy+qz
//    (rows are sorted by degree then (qz,qy,qx), collision.cpp:18-42; the
//     row <-> mu map is computed on the host, see scene.cpp)
#pragma once

#ifndef LBMG_HD
#ifdef __CUDACC__
#define LBMG_HD __host__ __device__ __forceinline__
#else
#define LBMG_HD inline
#endif
#endif

namespace lbmg {

constexpr int Q = 27;

LBMG_HD constexpr int dir_tensor(int i) { return i == 0 ? 13 : (i <= 13 ? i - 1 : i); }
LBMG_HD constexpr int tensor_dir(int t) { return t == 13 ? 0 : (t < 13 ? t + 1 : t); }
LBMG_HD constexpr int cx(int i) { return dir_tensor(i) % 3 - 1; }
LBMG_HD constexpr int cy(int i) { return (dir_tensor(i) / 3) % 3 - 1; }
LBMG_HD constexpr int cz(int i) { return dir_tensor(i) / 9 - 1; }
LBMG_HD constexpr int cc(int i, int a) { return a == 0 ? cx(i) : (a == 1 ? cy(i) : cz(i)); }
LBMG_HD constexpr int opposite(int i) { return i == 0 ? 0 : 27 - i; }
LBMG_HD constexpr int norm2(int i) { return cx(i) * cx(i) + cy(i) * cy(i) + cz(i) * cz(i); }
LBMG_HD constexpr double weight_d(int i) {
    return norm2(i) == 0 ? 8.0 / 27.0
                         : (norm2(i) == 1 ? 2.0 / 27.0 : (norm2(i) == 2 ? 1.0 / 54.0 : 1.0 / 216.0));
}
LBMG_HD constexpr float weight_f(int i) {
    return norm2(i) == 0 ? 8.0f / 27.0f
                         : (norm2(i) == 1 ? 2.0f / 27.0f : (norm2(i) == 2 ? 1.0f / 54.0f : 1.0f / 216.0f));
}
// Moment tensor index -> exponents / degree.
LBMG_HD constexpr int mu_qx(int mu) { return mu % 3; }
LBMG_HD constexpr int mu_qy(int mu) { return (mu / 3) % 3; }
LBMG_HD constexpr int mu_qz(int mu) { return mu / 9; }
LBMG_HD constexpr int mu_degree(int mu) { return mu_qx(mu) + mu_qy(mu) + mu_qz(mu); }

// Index of direction i among the 9 directions that cross a plane normal to
// `axis` (those with c_axis != 0 of a given sign): the two remaining velocity
// components, lower axis fastest.
LBMG_HD constexpr int cross9(int i, int axis) {
    return axis == 0 ? (cy(i) + 1) + 3 * (cz(i) + 1)
                     : (axis == 1 ? (cx(i) + 1) + 3 * (cz(i) + 1) : (cx(i) + 1) + 3 * (cy(i) + 1));
}

// Faces: 0:-x 1:+x 2:-y 3:+y 4:-z 5:+z (boundary.hpp:37-39).
LBMG_HD constexpr int face_axis(int f) { return f / 2; }
LBMG_HD constexpr int face_side(int f) { return f % 2 == 0 ? -1 : +1; }

// Compile-time loop.
template <int N>
struct IntC {
    static constexpr int value = N;
};
template <int B, int E, class F>
LBMG_HD void static_for(F&& f) {
    if constexpr (B < E) {
        f(IntC<B>{});
        static_for<B + 1, E>(f);
    }
}

}  // namespace lbmg
