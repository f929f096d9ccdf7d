// Per-node moments + collision + forcing in fp32 on DDF-shifted populations
// (f~ = f - w), generic over V = float (one node) or float2 (two nodes per
// thread, packed FFMA2/FADD2/FMUL2 on sm_100a).  Every operation is an
// explicit round-to-nearest intrinsic, so the packed and scalar paths are
// bit-identical per node (region/layout invariance stays bitwise).
//
// Restates (exact algebra, fp32 arithmetic):
//   compute_moments  solver.cpp:89-137
//   equilibrium      collision.cpp:148-157
//   collide_range    collision.cpp:176-205   Omega = -M^-1 D M (f - feq)
//   adaptive_rates   collision.cpp:159-174   relax-toward-one policy
//   forcing_term     solver.cpp:139-147      G_i = 3 w_i c_i.g
//   collide_pass     solver.cpp:149-179      f_out = f* + Omega + G
// M factorises into per-axis 3-point stages
// with shift s = u (central) or 0 (raw); the stages are written in
// difference form (6 ops forward, 7 inverse per triple).
#pragma once

#include "device_common.cuh"

namespace lbmg {

template <class V>
struct VOps;

template <>
struct VOps<float> {
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fmaf_rn(b, -1.0f, a); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
    static __device__ __forceinline__ float splat(float x) { return x; }
};

template <>
struct VOps<float2> {
    static __device__ __forceinline__ float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
    static __device__ __forceinline__ float2 sub(float2 a, float2 b) {
        return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a);
    }
    static __device__ __forceinline__ float2 mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
    static __device__ __forceinline__ float2 fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
    static __device__ __forceinline__ float2 splat(float x) { return make_float2(x, x); }
};

// Lane-wise scalar access for the few per-node nonlinear steps.
__device__ __forceinline__ float lane(float v, int) { return v; }
__device__ __forceinline__ float lane(float2 v, int j) { return j ? v.y : v.x; }
__device__ __forceinline__ void set_lane(float& v, int, float x) { v = x; }
__device__ __forceinline__ void set_lane(float2& v, int j, float x) {
    if (j) v.y = x;
    else v.x = x;
}
template <class V>
constexpr int kLanes = 1;
template <>
constexpr int kLanes<float2> = 2;

// c_i . (ax, ay, az), folded at compile time (0-2 adds).
template <int I, class V>
__device__ __forceinline__ V cdot(V ax, V ay, V az) {
    using O = VOps<V>;
    constexpr int c0 = cx(I), c1 = cy(I), c2 = cz(I);
    static_assert(c0 != 0 || c1 != 0 || c2 != 0, "rest direction");
    V r;
    bool have = false;
    auto acc = [&](V a, int c) {
        if (c == 0) return;
        if (!have) {
            r = c > 0 ? a : O::mul(a, O::splat(-1.0f));
            have = true;
        } else {
            r = c > 0 ? O::add(r, a) : O::sub(r, a);
        }
    };
    acc(ax, c0);
    acc(ay, c1);
    acc(az, c2);
    return r;
}

// Moments of one (or two) nodes: grouped by (cy, cz) rows of 3 along x.
template <class V>
struct MacroV {
    V drho, rho, ux, uy, uz;
    bool bad[kLanes<V>];
    bool mach[kLanes<V>];
};

template <class V>
__device__ __forceinline__ MacroV<V> moments_v(const V (&fs)[27]) {
    using O = VOps<V>;
    V s[9], d[9];
    static_for<0, 9>([&](auto G) {
        constexpr int g = decltype(G)::value;  // g = (cy+1) + 3 (cz+1)
        constexpr int t0 = 3 * g;              // tensor of cx = -1
        const V a = fs[tensor_dir(t0)], b = fs[tensor_dir(t0 + 1)], c = fs[tensor_dir(t0 + 2)];
        s[g] = O::add(O::add(a, c), b);
        d[g] = O::sub(c, a);
    });
    MacroV<V> m;
    // rho~ = sum of all 27, j = first moments
    V r = O::add(O::add(s[0], s[1]), s[2]);
    r = O::add(r, O::add(O::add(s[3], s[4]), s[5]));
    r = O::add(r, O::add(O::add(s[6], s[7]), s[8]));
    V jx = O::add(O::add(d[0], d[1]), d[2]);
    jx = O::add(jx, O::add(O::add(d[3], d[4]), d[5]));
    jx = O::add(jx, O::add(O::add(d[6], d[7]), d[8]));
    // cy: g%3 ; cz: g/3
    const V jy = O::sub(O::add(O::add(s[2], s[5]), s[8]), O::add(O::add(s[0], s[3]), s[6]));
    const V jz = O::sub(O::add(O::add(s[6], s[7]), s[8]), O::add(O::add(s[0], s[1]), s[2]));
    m.drho = r;
    m.rho = O::add(r, O::splat(1.0f));
    V inv;
#pragma unroll
    for (int j = 0; j < kLanes<V>; ++j) {
        const float rj = lane(m.rho, j);
        m.bad[j] = !(rj > 0.0f) || !isfinite(rj) || !isfinite(lane(jx, j)) || !isfinite(lane(jy, j)) ||
                   !isfinite(lane(jz, j));
        set_lane(inv, j, __frcp_rn(rj));
    }
    m.ux = O::mul(jx, inv);
    m.uy = O::mul(jy, inv);
    m.uz = O::mul(jz, inv);
    const V u2 = O::fma(m.uz, m.uz, O::fma(m.uy, m.uy, O::mul(m.ux, m.ux)));
#pragma unroll
    for (int j = 0; j < kLanes<V>; ++j) m.mach[j] = lane(u2, j) >= 0.16f;
    return m;
}

template <int S, class V>
__device__ __forceinline__ void forward_stage(V (&t)[27], V s) {
    using O = VOps<V>;
    const V ns = O::mul(s, O::splat(-1.0f));
    static_for<0, 9>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr int base = (S == 1) ? 3 * j : ((S == 3) ? (j % 3) + 9 * (j / 3) : j);
        const V v0 = t[base], v1 = t[base + S], v2 = t[base + 2 * S];
        const V d = O::sub(v2, v0);
        const V a = O::add(v0, v2);
        const V m0 = O::add(a, v1);
        const V m1 = O::fma(ns, m0, d);
        t[base] = m0;
        t[base + S] = m1;
        t[base + 2 * S] = O::fma(ns, O::add(d, m1), a);
    });
}

template <int S, class V>
__device__ __forceinline__ void inverse_stage(V (&t)[27], V s) {
    using O = VOps<V>;
    const V half = O::splat(0.5f), nhalf = O::splat(-0.5f);
    static_for<0, 9>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr int base = (S == 1) ? 3 * j : ((S == 3) ? (j % 3) + 9 * (j / 3) : j);
        const V m0 = t[base], m1 = t[base + S], m2 = t[base + 2 * S];
        const V D = O::fma(s, m0, m1);
        const V A = O::fma(s, O::add(m1, D), m2);
        const V h = O::mul(A, half);
        t[base] = O::fma(nhalf, D, h);
        t[base + S] = O::sub(m0, A);
        t[base + 2 * S] = O::fma(half, D, h);
    });
}

// f* kept across the transform: in registers (scalar path) or in shared
// memory (packed bulk path, keeps the register budget of one 27-vector).
template <class V>
struct RegStash {
    static constexpr bool kFeqOut = false;
    V v[27];
    __device__ __forceinline__ void put(int i, V x) { v[i] = x; }
    __device__ __forceinline__ V get(int i) const { return v[i]; }
};

// No f* kept: the output is rebuilt as feq + G + M^-1((1 - D) M t), exact
// algebra of the same operator; fewer live registers.
template <class V>
struct NoStash {
    static constexpr bool kFeqOut = true;
    __device__ __forceinline__ void put(int, V) {}
    __device__ __forceinline__ V get(int) const { return V{}; }
};

// Collision + forcing of one (two) node(s): f_out = f* - M^-1 D M (f* - feq) + G.
// fs: f~* by direction in, f~(t+1) out.  STD: standard rate pattern
// (deg<2: 1, deg 2: one value, deg>=3: one value).  The conserved moments of
// t = f* - feq vanish in exact arithmetic; with STD their rate is applied as
// 0 so mass and momentum change only by transform round-off instead of by the
// fp32 rounding of feq (bit-for-bit the same as rate 1 in exact arithmetic).
template <int KIND, int POLICY, bool STD, class V, class Stash>
__device__ __forceinline__ void collide_v(V (&fs)[27], const MacroV<V>& mc, V gx, V gy, V gz, bool any_force,
                                          const ModelConst& m, Stash& stash) {
    using O = VOps<V>;
    const V rho = mc.rho, ux = mc.ux, uy = mc.uy, uz = mc.uz;
    const V usq = O::mul(O::splat(1.5f), O::fma(uz, uz, O::fma(uy, uy, O::mul(ux, ux))));
    const V B = O::fma(O::mul(rho, O::splat(-1.0f)), usq, mc.drho);  // drho - 1.5 rho u^2
    const V k45 = O::splat(4.5f), k3 = O::splat(3.0f), km3 = O::splat(-3.0f);

    // t = f* - feq in tensor order; the pair (i, 27-i) shares c.u
    V t[27];
    t[dir_tensor(0)] = O::fma(B, O::splat(-weight_f(0)), fs[0]);
    stash.put(0, fs[0]);
    static_for<1, 14>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int o = opposite(i);
        const V cu = cdot<i>(ux, uy, uz);
        const V q = O::mul(rho, cu);
        const V sym = O::fma(O::mul(q, k45), cu, B);
        const V nw = O::splat(-weight_f(i));
        t[dir_tensor(i)] = O::fma(O::fma(q, k3, sym), nw, fs[i]);
        t[dir_tensor(o)] = O::fma(O::fma(q, km3, sym), nw, fs[o]);
        stash.put(i, fs[i]);
        stash.put(o, fs[o]);
    });

    // FEQ form: relax t by (1 - r) and rebuild f_out = feq + G + t'' at the end
    // (no f* kept); otherwise relax by r and f_out = f* - t' + G.
    constexpr bool FEQ = Stash::kFeqOut;
    auto fac = [](float r) { return FEQ ? __fadd_rn(1.0f, -r) : r; };
    if constexpr (KIND == kBGK) {
        const V om = O::splat(fac(m.omega));
        static_for<0, 27>([&](auto T) { t[decltype(T)::value] = O::mul(t[decltype(T)::value], om); });
    } else {
        V r3v = O::splat(STD ? fac(m.rate[26]) : 0.0f);
        V hi_s = O::splat(0.0f);
        if constexpr (POLICY == kPolicyRelax) {
            // relax-toward-one: eps = sum|f - feq| / rho per node (scalar lanes)
#pragma unroll
            for (int j = 0; j < kLanes<V>; ++j) {
                float e = 0.0f;
                static_for<0, 27>([&](auto T) { e = __fadd_rn(e, fabsf(lane(t[decltype(T)::value], j))); });
                e = __fdiv_rn(e, fmaxf(lane(rho, j), 1e-30f));
                const float s = __fdiv_rn(e, __fadd_rn(e, m.eps0));
                set_lane(hi_s, j, s);
                if constexpr (STD) {
                    const float r = m.rate[26];
                    set_lane(r3v, j, fac(fminf(fmaxf(__fmaf_rn(__fadd_rn(1.0f, -r), s, r), 0.05f), 1.95f)));
                }
            }
        }
        const V sx = KIND == kCentralMRT ? ux : O::splat(0.0f);
        const V sy = KIND == kCentralMRT ? uy : O::splat(0.0f);
        const V sz = KIND == kCentralMRT ? uz : O::splat(0.0f);
        forward_stage<1>(t, sx);
        forward_stage<3>(t, sy);
        forward_stage<9>(t, sz);
        const V r2v = O::splat(fac(m.rate[4]));
        static_for<0, 27>([&](auto MU) {
            constexpr int mu = decltype(MU)::value;
            constexpr int dg = mu_degree(mu);
            if constexpr (STD) {
                t[mu] = O::mul(t[mu], dg < 2 ? O::splat(0.0f) : (dg == 2 ? r2v : r3v));
            } else {
                V r = O::splat(fac(m.rate[mu]));
                if constexpr (POLICY == kPolicyRelax && dg >= 3) {
#pragma unroll
                    for (int j = 0; j < kLanes<V>; ++j) {
                        const float r0 = m.rate[mu];
                        set_lane(r, j,
                                 fac(fminf(fmaxf(__fmaf_rn(__fadd_rn(1.0f, -r0), lane(hi_s, j), r0), 0.05f), 1.95f)));
                    }
                }
                t[mu] = O::mul(t[mu], r);
            }
        });
        inverse_stage<1>(t, sx);
        inverse_stage<3>(t, sy);
        inverse_stage<9>(t, sz);
    }

    if constexpr (FEQ) {
        // f_out = feq + G + t'' = w (B + 3 c.(rho u + g) + 4.5 rho (c.u)^2) + t''
        const V px = O::fma(rho, ux, gx), py = O::fma(rho, uy, gy), pz = O::fma(rho, uz, gz);
        fs[0] = O::fma(B, O::splat(weight_f(0)), t[dir_tensor(0)]);
        static_for<1, 14>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int o = opposite(i);
            const V cu = cdot<i>(ux, uy, uz);
            const V cp = cdot<i>(px, py, pz);
            const V q = O::mul(rho, cu);
            const V sym = O::fma(O::mul(q, k45), cu, B);
            const V w = O::splat(weight_f(i));
            fs[i] = O::fma(O::fma(cp, k3, sym), w, t[dir_tensor(i)]);
            fs[o] = O::fma(O::fma(cp, km3, sym), w, t[dir_tensor(o)]);
        });
        return;
    }
    // f_out = f* - t' (+ G_i = 3 w_i c_i.g)
    static_for<0, 27>([&](auto I) {
        constexpr int i = decltype(I)::value;
        fs[i] = O::sub(stash.get(i), t[dir_tensor(i)]);
    });
    if (any_force) {
        static_for<1, 14>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int o = opposite(i);
            const V cg = cdot<i>(gx, gy, gz);
            const V w3 = O::splat(3.0f * weight_f(i));
            fs[i] = O::fma(w3, cg, fs[i]);
            fs[o] = O::fma(O::mul(w3, O::splat(-1.0f)), cg, fs[o]);
        });
    }
}

// Host-side check that a rate vector (by tensor index) has the STD pattern.
inline bool rates_standard(const float* rate_mu) {
    for (int mu = 0; mu < 27; ++mu) {
        const int d = mu_degree(mu);
        if (d < 2 && rate_mu[mu] != 1.0f) return false;
        if (d == 2 && rate_mu[mu] != rate_mu[4]) return false;
        if (d >= 3 && rate_mu[mu] != rate_mu[26]) return false;
    }
    return true;
}

}  // namespace lbmg
