// Per-node collision + forcing in fp32, exact restatement of
//   collide_range   collision.cpp:176-205  (t = f - feq, forward 3-point
//                   stages per axis, diagonal rates, inverse stages, Omega=-t)
//   equilibrium     collision.cpp:148-157
//   adaptive_rates  collision.cpp:159-174  (relax-toward-one policy)
//   forcing_term    solver.cpp:139-147     (G_i = 3 w_i c_i.g)
//   collide_pass    solver.cpp:149-179     (f_out = f* + Omega + G)
// on DDF-shifted populations (f~ = f - w).  The 3-point stages are rewritten
// in difference form (6 ops forward, 7 inverse per triple) — algebraically the
// reference's Vandermonde / Lagrange products, see DESIGN.md §4.
#pragma once

#include "device_common.cuh"

namespace lbmg {

// c_i . (ax, ay, az) with the velocity components folded at compile time.
template <int I>
__device__ __forceinline__ float cdot(float ax, float ay, float az) {
    constexpr int c0 = cx(I), c1 = cy(I), c2 = cz(I);
    float r;
    if constexpr (c0 == 1) r = ax;
    else if constexpr (c0 == -1) r = -ax;
    if constexpr (c1 != 0) {
        if constexpr (c0 == 0) r = (c1 == 1) ? ay : -ay;
        else r = (c1 == 1) ? r + ay : r - ay;
    }
    if constexpr (c2 != 0) {
        if constexpr (c0 == 0 && c1 == 0) r = (c2 == 1) ? az : -az;
        else r = (c2 == 1) ? r + az : r - az;
    }
    if constexpr (c0 == 0 && c1 == 0 && c2 == 0) r = 0.0f;
    return r;
}

// One forward stage over the 9 triples along the axis with element stride S.
template <int S>
__device__ __forceinline__ void forward_stage(float (&t)[27], float s) {
    static_for<0, 9>([&](auto J) {
        constexpr int j = decltype(J)::value;
        // base of the j-th triple: the two other tensor digits
        constexpr int base = (S == 1) ? 3 * j : ((S == 3) ? (j % 3) + 9 * (j / 3) : j);
        const float v0 = t[base], v1 = t[base + S], v2 = t[base + 2 * S];
        const float d = v2 - v0;
        const float a = v0 + v2;
        const float m0 = a + v1;
        const float m1 = __fmaf_rn(-s, m0, d);
        const float m2 = __fmaf_rn(-s, d + m1, a);
        t[base] = m0;
        t[base + S] = m1;
        t[base + 2 * S] = m2;
    });
}

template <int S>
__device__ __forceinline__ void inverse_stage(float (&t)[27], float s) {
    static_for<0, 9>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr int base = (S == 1) ? 3 * j : ((S == 3) ? (j % 3) + 9 * (j / 3) : j);
        const float m0 = t[base], m1 = t[base + S], m2 = t[base + 2 * S];
        const float D = __fmaf_rn(s, m0, m1);
        const float A = __fmaf_rn(s, m1 + D, m2);
        const float h = 0.5f * A;
        t[base] = __fmaf_rn(-0.5f, D, h);
        t[base + S] = m0 - A;
        t[base + 2 * S] = __fmaf_rn(0.5f, D, h);
    });
}

// fs: f~* by direction on entry, f~(t+1) by direction on exit.
template <int KIND, int POLICY>
__device__ __forceinline__ void collide_node(float (&fs)[27], float rho, float drho, float ux, float uy, float uz,
                          float gx, float gy, float gz, bool has_force, const ModelConst& m) {
    const float usq = 1.5f * (ux * ux + uy * uy + uz * uz);
    float t[27];
    // t = f - feq in tensor order; feq~_i = w_i (drho + rho (3cu + 4.5cu^2 - 1.5u^2))
    static_for<0, 27>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr float w = weight_f(i);
        float feq;
        if constexpr (i == 0) {
            feq = w * __fmaf_rn(-rho, usq, drho);
        } else {
            const float cu = cdot<i>(ux, uy, uz);
            feq = w * __fmaf_rn(rho, __fmaf_rn(cu, __fmaf_rn(4.5f, cu, 3.0f), -usq), drho);
        }
        t[dir_tensor(i)] = fs[i] - feq;
    });

    if constexpr (KIND == kBGK) {
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            fs[i] = __fmaf_rn(-m.omega, t[dir_tensor(i)], fs[i]);
        });
    } else {
        float hi_s = 0.0f;
        if constexpr (POLICY == kPolicyRelax) {
            float eps = 0.0f;
            static_for<0, 27>([&](auto I) { eps += fabsf(t[decltype(I)::value]); });
            eps = eps / fmaxf(rho, 1e-30f);
            hi_s = eps / (eps + m.eps0);
        }
        const float sx = (KIND == kCentralMRT) ? ux : 0.0f;
        const float sy = (KIND == kCentralMRT) ? uy : 0.0f;
        const float sz = (KIND == kCentralMRT) ? uz : 0.0f;
        forward_stage<1>(t, sx);
        forward_stage<3>(t, sy);
        forward_stage<9>(t, sz);
        static_for<0, 27>([&](auto MU) {
            constexpr int mu = decltype(MU)::value;
            float r = m.rate[mu];
            if constexpr (POLICY == kPolicyRelax && mu_degree(mu) >= 3)
                r = fminf(fmaxf(__fmaf_rn(1.0f - r, hi_s, r), 0.05f), 1.95f);
            t[mu] *= r;
        });
        inverse_stage<1>(t, sx);
        inverse_stage<3>(t, sy);
        inverse_stage<9>(t, sz);
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            fs[i] = fs[i] - t[dir_tensor(i)];
        });
    }
    if (has_force) {
        static_for<0, 27>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if constexpr (i != 0) fs[i] = __fmaf_rn(3.0f * weight_f(i), cdot<i>(gx, gy, gz), fs[i]);
        });
    }
}

}  // namespace lbmg
