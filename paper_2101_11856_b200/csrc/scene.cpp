// Host-side scene setup.  Semantics follow the reference (file:line cited per
// function); the implementation is independent.  All FP64 expressions keep
// the reference's operation order and are compiled without FP contraction so
// sample positions come out bit-identical.
#include "scene.hpp"

#include <algorithm>
#include <map>
#include <numeric>
#include <random>
#include <unordered_map>

namespace lbmg {

namespace {

inline double norm(V3 v) { return std::sqrt(dot(v, v)); }
inline double tri_area(V3 a, V3 b, V3 c) { return 0.5 * norm(cross(b - a, c - a)); }  // mesh.cpp:12-14

void add_tri(TriMesh& m, V3 a, V3 b, V3 c) {
    const uint32_t base = static_cast<uint32_t>(m.vertices.size());
    m.vertices.push_back(a);
    m.vertices.push_back(b);
    m.vertices.push_back(c);
    m.triangles.push_back({base, base + 1, base + 2});
}

// make_icosphere, mesh.cpp:163-207: golden-ratio icosahedron, edge-midpoint
// subdivision projected to the unit sphere, then scaled about the centre.
TriMesh icosphere(V3 center, double radius, int subdiv) {
    const double g = (1.0 + std::sqrt(5.0)) / 2.0;
    std::vector<V3> v = {{-1, g, 0}, {1, g, 0},  {-1, -g, 0}, {1, -g, 0}, {0, -1, g},  {0, 1, g},
                         {0, -1, -g}, {0, 1, -g}, {g, 0, -1},  {g, 0, 1},  {-g, 0, -1}, {-g, 0, 1}};
    std::vector<std::array<uint32_t, 3>> f = {
        {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11}, {1, 5, 9},  {5, 11, 4},
        {11, 10, 2}, {10, 7, 6}, {7, 1, 8},  {3, 9, 4},  {3, 4, 2},   {3, 2, 6},  {3, 6, 8},
        {3, 8, 9},  {4, 9, 5},  {2, 4, 11}, {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
    auto unit = [](V3 p) {
        const double n = norm(p);
        return V3{p.x / n, p.y / n, p.z / n};
    };
    for (auto& p : v) p = unit(p);
    for (int s = 0; s < subdiv; ++s) {
        std::map<std::pair<uint32_t, uint32_t>, uint32_t> cache;
        auto midpoint = [&](uint32_t a, uint32_t b) -> uint32_t {
            const auto key = std::make_pair(std::min(a, b), std::max(a, b));
            auto it = cache.find(key);
            if (it != cache.end()) return it->second;
            v.push_back(unit((v[a] + v[b]) * 0.5));
            const uint32_t id = static_cast<uint32_t>(v.size() - 1);
            cache.emplace(key, id);
            return id;
        };
        std::vector<std::array<uint32_t, 3>> nf;
        nf.reserve(f.size() * 4);
        for (const auto& t : f) {
            const uint32_t ab = midpoint(t[0], t[1]), bc = midpoint(t[1], t[2]), ca = midpoint(t[2], t[0]);
            nf.push_back({t[0], ab, ca});
            nf.push_back({t[1], bc, ab});
            nf.push_back({t[2], ca, bc});
            nf.push_back({ab, bc, ca});
        }
        f.swap(nf);
    }
    TriMesh m;
    for (const auto& p : v) m.vertices.push_back(center + p * radius);
    m.triangles = std::move(f);
    return m;
}

// make_box, mesh.cpp:150-161.
TriMesh box(V3 lo, V3 hi) {
    TriMesh m;
    V3 c[8];
    for (int i = 0; i < 8; ++i) c[i] = {(i & 1) ? hi.x : lo.x, (i & 2) ? hi.y : lo.y, (i & 4) ? hi.z : lo.z};
    static const int quads[6][4] = {{0, 2, 3, 1}, {4, 5, 7, 6}, {0, 1, 5, 4},
                                    {2, 6, 7, 3}, {0, 4, 6, 2}, {1, 3, 7, 5}};
    for (const auto& q : quads) {
        add_tri(m, c[q[0]], c[q[1]], c[q[2]]);
        add_tri(m, c[q[0]], c[q[2]], c[q[3]]);
    }
    return m;
}

// make_fin_comb, mesh.cpp:209-231: base plate + double-sided fins normal to y.
TriMesh fin_comb(V3 o, int fins, double len, double height, double spacing) {
    TriMesh m;
    const double depth = (fins - 1) * spacing;
    const V3 p1 = o + V3{len, 0, 0}, p2 = o + V3{len, depth, 0}, p3 = o + V3{0, depth, 0};
    add_tri(m, o, p1, p2);
    add_tri(m, o, p2, p3);
    for (int k = 0; k < fins; ++k) {
        const double y = o.y + k * spacing;
        const V3 a{o.x, y, o.z}, b{o.x + len, y, o.z}, c{o.x + len, y, o.z + height}, d{o.x, y, o.z + height};
        add_tri(m, a, b, c);
        add_tri(m, a, c, d);
    }
    return m;
}

// make_quad, mesh.cpp:143-148.
TriMesh quad(double size, double z) {
    TriMesh m;
    add_tri(m, {0, 0, z}, {size, 0, z}, {size, size, z});
    add_tri(m, {0, 0, z}, {size, size, z}, {0, size, z});
    return m;
}

// mt19937_64 bits -> [0,1) (ib.cpp:33).
inline double unit_draw(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// Area-weighted point on the surface (ib.cpp:81-105 semantics).
struct AreaTable {
    std::vector<std::array<V3, 3>> tris;
    std::vector<double> cum;
    double total = 0;
    size_t degenerate = 0;

    explicit AreaTable(const TriMesh& m) {
        for (const auto& t : m.triangles) {
            const V3 a = m.vertices[t[0]], b = m.vertices[t[1]], c = m.vertices[t[2]];
            const double ar = tri_area(a, b, c);
            if (ar <= 1e-14) {
                ++degenerate;
                continue;
            }
            total += ar;
            tris.push_back({a, b, c});
            cum.push_back(total);
        }
    }
    V3 draw(std::mt19937_64& rng) const {
        const double r = unit_draw(rng) * total;
        const size_t t = std::min<size_t>(std::lower_bound(cum.begin(), cum.end(), r) - cum.begin(),
                                          tris.size() - 1);
        double u = unit_draw(rng), v = unit_draw(rng);
        if (u + v > 1.0) {
            u = 1.0 - u;
            v = 1.0 - v;
        }
        const auto& T = tris[t];
        return T[0] + (T[1] - T[0]) * u + (T[2] - T[0]) * v;
    }
};

// Uniform bucket grid with cell edge = radius: every point closer than the
// radius lies in one of the 27 buckets around the query.
class Buckets {
public:
    explicit Buckets(double h) : h_(h) {}
    static int64_t pack(int64_t i, int64_t j, int64_t k) {
        const int64_t o = int64_t(1) << 20;
        return (i + o) | ((j + o) << 21) | ((k + o) << 42);
    }
    int64_t cell(double v) const { return static_cast<int64_t>(std::floor(v / h_)); }
    void add(V3 p, uint32_t id) { map_[pack(cell(p.x), cell(p.y), cell(p.z))].push_back(id); }
    template <class F>
    void visit(V3 p, F&& f) const {
        const int64_t i = cell(p.x), j = cell(p.y), k = cell(p.z);
        for (int64_t dk = -1; dk <= 1; ++dk)
            for (int64_t dj = -1; dj <= 1; ++dj)
                for (int64_t di = -1; di <= 1; ++di) {
                    auto it = map_.find(pack(i + di, j + dj, k + dk));
                    if (it == map_.end()) continue;
                    for (uint32_t id : it->second) f(id);
                }
    }

private:
    double h_;
    std::unordered_map<int64_t, std::vector<uint32_t>> map_;
};

inline double dist2(V3 a, V3 b) { return dot(a - b, a - b); }

void fill_report(const std::vector<V3>& pts, SamplingReport* rep) {
    rep->n_samples = pts.size();
    std::map<std::array<int, 3>, size_t> cells;
    for (const auto& p : pts)
        ++cells[{int(std::floor(p.x)), int(std::floor(p.y)), int(std::floor(p.z))}];
    rep->occupied_cells = cells.size();
    if (cells.empty()) return;
    double mn = 1e300, mx = 0, sum = 0;
    size_t band = 0;
    for (const auto& kv : cells) {
        const double d = double(kv.second);
        mn = std::min(mn, d);
        mx = std::max(mx, d);
        sum += d;
        if (kv.second >= 10 && kv.second <= 100) ++band;
    }
    rep->density_min = mn;
    rep->density_max = mx;
    rep->density_mean = sum / cells.size();
    rep->in_band_fraction = double(band) / cells.size();
}

}  // namespace

TriMesh build_mesh(const lbmg_mesh& m) {
    switch (m.type) {
        case LBMG_MESH_SPHERE: return icosphere(v3(m.center), m.radius, m.subdivisions);
        case LBMG_MESH_BOX: return box(v3(m.lo), v3(m.hi));
        case LBMG_MESH_FIN_COMB:
            return fin_comb(v3(m.origin), m.fins, m.fin_length, m.fin_height, m.fin_spacing);
        case LBMG_MESH_QUAD: return quad(m.size, m.plane_z);
    }
    throw ConfigError("mesh: unknown type");
}

// sample_surface, ib.cpp:156-229 (dart throwing / greedy elimination).
SampleSet sample_surface(const TriMesh& mesh, double radius, uint64_t seed, int method,
                         SamplingReport* report) {
    if (!(radius > 0.0)) throw ConfigError("sampling: radius must be > 0");
    AreaTable surf(mesh);
    if (surf.tris.empty()) throw ConfigError("sampling: mesh has no non-degenerate triangles");
    std::mt19937_64 rng(seed);
    const double r2 = radius * radius;
    const double estimate = 0.7 * surf.total / (M_PI * r2 / 4.0);
    std::vector<V3> pts;
    size_t attempts = 0;
    if (method == LBMG_SAMPLING_DART) {
        Buckets grid(radius);
        const size_t budget = std::max<size_t>(static_cast<size_t>(60.0 * estimate), 20000);
        size_t streak = 0;
        while (attempts < budget && streak < 8000) {
            ++attempts;
            const V3 p = surf.draw(rng);
            bool ok = true;
            grid.visit(p, [&](uint32_t id) {
                if (ok && dist2(pts[id], p) < r2) ok = false;
            });
            if (!ok) {
                ++streak;
                continue;
            }
            grid.add(p, static_cast<uint32_t>(pts.size()));
            pts.push_back(p);
            streak = 0;
        }
    } else {
        const size_t m = std::max<size_t>(static_cast<size_t>(3.0 * estimate), 64);
        std::vector<V3> cand(m);
        for (auto& p : cand) p = surf.draw(rng);
        attempts = m;
        Buckets grid(radius);
        for (size_t i = 0; i < m; ++i) grid.add(cand[i], static_cast<uint32_t>(i));
        std::vector<std::vector<uint32_t>> nb(m);
        for (size_t i = 0; i < m; ++i)
            grid.visit(cand[i], [&](uint32_t j) {
                if (j != i && dist2(cand[i], cand[j]) < r2) nb[i].push_back(j);
            });
        std::vector<char> alive(m, 1);
        std::vector<size_t> cnt(m);
        for (size_t i = 0; i < m; ++i) cnt[i] = nb[i].size();
        for (;;) {
            size_t worst = m, wc = 0;
            for (size_t i = 0; i < m; ++i)
                if (alive[i] && cnt[i] > wc) {
                    worst = i;
                    wc = cnt[i];
                }
            if (worst == m) break;
            alive[worst] = 0;
            for (uint32_t j : nb[worst])
                if (alive[j] && cnt[j] > 0) --cnt[j];
        }
        for (size_t i = 0; i < m; ++i)
            if (alive[i]) pts.push_back(cand[i]);
    }
    SampleSet set;
    set.positions = pts;
    set.reference_positions = pts;
    set.source_id.resize(pts.size());
    std::iota(set.source_id.begin(), set.source_id.end(), 0u);
    set.poisson_radius = radius;
    set.bbox_lo = {1e300, 1e300, 1e300};
    set.bbox_hi = {-1e300, -1e300, -1e300};
    for (const auto& p : pts)
        for (int a = 0; a < 3; ++a) {
            set.bbox_lo[a] = std::min(set.bbox_lo[a], p[a]);
            set.bbox_hi[a] = std::max(set.bbox_hi[a], p[a]);
        }
    if (report) {
        report->degenerate = surf.degenerate;
        report->attempts = attempts;
        fill_report(pts, report);
    }
    return set;
}

// morton3, ib.cpp:13-25: x in the least-significant bit of each triple.
uint64_t morton3(uint32_t x, uint32_t y, uint32_t z) {
    auto dilate = [](uint64_t v) {
        v &= 0x1fffffull;
        v = (v | (v << 32)) & 0x001f00000000ffffull;
        v = (v | (v << 16)) & 0x001f0000ff0000ffull;
        v = (v | (v << 8)) & 0x100f00f00f00f00full;
        v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
        v = (v | (v << 2)) & 0x1249249249249249ull;
        return v;
    };
    return dilate(x) | (dilate(y) << 1) | (dilate(z) << 2);
}

// reorder_samples, ib.cpp:231-292: key = (block id x-fastest over the floored
// bbox in blocks of ell cells, Morton code of the cell inside its block,
// source id).
std::vector<uint32_t> reorder_permutation(const std::vector<V3>& pos,
                                          const std::vector<uint32_t>& src, int ell) {
    if (ell < 1) throw ConfigError("reorder_samples: block edge must be >= 1");
    const size_t n = pos.size();
    std::vector<uint32_t> perm(n);
    if (n == 0) return perm;
    V3 lo{1e300, 1e300, 1e300}, hi{-1e300, -1e300, -1e300};
    for (const auto& p : pos)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], p[a]);
            hi[a] = std::max(hi[a], p[a]);
        }
    int base[3], nb[3];
    for (int a = 0; a < 3; ++a) {
        base[a] = static_cast<int>(std::floor(lo[a]));
        nb[a] = (static_cast<int>(std::floor(hi[a])) - base[a]) / ell + 1;
    }
    struct Key {
        uint64_t block, code;
        uint32_t src, idx;
    };
    std::vector<Key> keys(n);
    for (size_t s = 0; s < n; ++s) {
        int b[3], l[3];
        for (int a = 0; a < 3; ++a) {
            const int c = static_cast<int>(std::floor(pos[s][a])) - base[a];
            b[a] = c / ell;
            l[a] = c - b[a] * ell;
        }
        keys[s].block = uint64_t(b[0]) + uint64_t(nb[0]) * (uint64_t(b[1]) + uint64_t(nb[1]) * uint64_t(b[2]));
        keys[s].code = morton3(uint32_t(l[0]), uint32_t(l[1]), uint32_t(l[2]));
        keys[s].src = src[s];
        keys[s].idx = uint32_t(s);
    }
    std::sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
        if (a.block != b.block) return a.block < b.block;
        if (a.code != b.code) return a.code < b.code;
        return a.src < b.src;
    });
    for (size_t s = 0; s < n; ++s) perm[s] = keys[s].idx;
    return perm;
}

void reorder_samples(SampleSet& set, int ell) {
    const auto perm = reorder_permutation(set.positions, set.source_id, ell);
    set.block_edge = ell;
    if (set.size() == 0) return;
    SampleSet out = set;
    for (size_t s = 0; s < set.size(); ++s) {
        out.positions[s] = set.positions[perm[s]];
        out.reference_positions[s] = set.reference_positions[perm[s]];
        out.source_id[s] = set.source_id[perm[s]];
    }
    out.bbox_lo = {1e300, 1e300, 1e300};
    out.bbox_hi = {-1e300, -1e300, -1e300};
    for (const auto& p : out.positions)
        for (int a = 0; a < 3; ++a) {
            out.bbox_lo[a] = std::min(out.bbox_lo[a], p[a]);
            out.bbox_hi[a] = std::max(out.bbox_hi[a], p[a]);
        }
    set = std::move(out);
}

// split_domain, decomp.cpp:5-18: sizes differ by at most one, larger first.
std::vector<std::array<int, 2>> split_domain(int nz, int m) {
    if (m < 1 || m > nz)
        throw ConfigError("decomp: region count must satisfy 1 <= m <= nz (got m=" + std::to_string(m) +
                          ", nz=" + std::to_string(nz) + ")");
    std::vector<std::array<int, 2>> s(m);
    const int q = nz / m, r = nz % m;
    int z = 0;
    for (int k = 0; k < m; ++k) {
        const int len = q + (k < r ? 1 : 0);
        s[k] = {z, z + len};
        z += len;
    }
    return s;
}

// Moment rows sorted by degree, ties by (qz, qy, qx) (collision.cpp:18-42).
const ModelTables& model_tables() {
    static const ModelTables t = [] {
        ModelTables m;
        std::array<int, 27> mus;
        std::iota(mus.begin(), mus.end(), 0);
        auto deg = [](int mu) { return mu % 3 + (mu / 3) % 3 + mu / 9; };
        std::stable_sort(mus.begin(), mus.end(), [&](int a, int b) {
            if (deg(a) != deg(b)) return deg(a) < deg(b);
            if (a / 9 != b / 9) return a / 9 < b / 9;
            if ((a / 3) % 3 != (b / 3) % 3) return (a / 3) % 3 < (b / 3) % 3;
            return a % 3 < b % 3;
        });
        for (int r = 0; r < 27; ++r) {
            m.row_to_mu[r] = mus[r];
            m.mu_to_row[mus[r]] = r;
            m.degree[r] = deg(mus[r]);
        }
        return m;
    }();
    return t;
}

// CollisionModel::{bgk,raw_mrt,central_mrt} + SceneConfig::make_model
// (collision.cpp:109-146, scene.cpp:28-45).
std::array<double, 27> make_rates(const lbmg_scene_config& c) {
    if (!(c.viscosity > 0.0)) throw ConfigError("collision: viscosity must be > 0");
    const double omega = 1.0 / (3.0 * c.viscosity + 0.5);
    std::array<double, 27> r{};
    const auto& T = model_tables();
    for (int row = 0; row < 27; ++row) {
        if (c.kind == LBMG_BGK) r[row] = omega;
        else r[row] = T.degree[row] < 2 ? 1.0 : (T.degree[row] == 2 ? omega : c.high_order_rate);
    }
    if (c.has_explicit_rates)
        for (int row = 0; row < 27; ++row) r[row] = c.rates[row];
    for (int row = 0; row < 27; ++row) {
        if (T.degree[row] < 2) continue;
        if (!(r[row] > 0.0 && r[row] < 2.0))
            throw ConfigError("collision: relaxation rate out of (0,2) at moment row " + std::to_string(row));
    }
    return r;
}

// Scene-level validation mirroring the reference's parser/constructor checks
// (scene.cpp:132-331, boundary.cpp:7-15).
void validate_config(const lbmg_scene_config& c) {
    if (c.nx < 2 || c.ny < 2 || c.nz < 2) throw ConfigError("config: $.grid: extents must be >= 2");
    if (c.kind < LBMG_BGK || c.kind > LBMG_CENTRAL_MRT) throw ConfigError("config: $.collision.kind invalid");
    if (c.policy < 0 || c.policy > 1) throw ConfigError("config: $.collision.policy invalid");
    if (!(c.policy_eps0 > 0)) throw ConfigError("config: $.collision.policy_eps0: must be > 0");
    for (int a = 0; a < 3; ++a) {
        const bool lo = c.faces[2 * a].condition == LBMG_PERIODIC;
        const bool hi = c.faces[2 * a + 1].condition == LBMG_PERIODIC;
        if (lo != hi)
            throw ConfigError("boundary: periodic faces must come in opposing pairs (axis " + std::to_string(a) + ")");
    }
    for (int f = 0; f < 6; ++f)
        if (c.faces[f].condition < 0 || c.faces[f].condition > 3) throw ConfigError("config: $.faces: bad condition");
    if (c.init_density <= 0) throw ConfigError("config: $.initial.density: must be > 0");
    if (c.regions < 1 || c.regions > c.nz) throw ConfigError("config: $.regions: must be <= grid.nz");
    if (c.block_edge < 1) throw ConfigError("config: $.layout.block_edge: must be >= 1");
    if (c.alpha < 1) throw ConfigError("layout: alpha and beta must be >= 1");
    for (int s = 0; s < c.n_solids; ++s)
        if (!(c.solids[s].poisson_radius > 0))
            throw ConfigError("config: $.solids[" + std::to_string(s) + "].poisson_radius: must be > 0");
    make_rates(c);
}

// Rigid motion row of step t (ib.cpp:456-475): centre(t), Rodrigues R(t)
// with the reference's expressions (glibc cos/sin), v, omega.
void motion_table_row(const V3& linear_velocity, const V3& angular_velocity, const V3& center0, long t,
                      double* row) {
    const double td = double(t);
    const V3 center = center0 + linear_velocity * td;
    const double wn = std::sqrt(dot(angular_velocity, angular_velocity));
    double R[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    if (wn > 0.0) {
        const V3 ax = angular_velocity * (1.0 / wn);
        const double th = wn * td, ct = std::cos(th), st = std::sin(th), vt = 1.0 - ct;
        R[0][0] = ct + ax.x * ax.x * vt;
        R[0][1] = ax.x * ax.y * vt - ax.z * st;
        R[0][2] = ax.x * ax.z * vt + ax.y * st;
        R[1][0] = ax.y * ax.x * vt + ax.z * st;
        R[1][1] = ct + ax.y * ax.y * vt;
        R[1][2] = ax.y * ax.z * vt - ax.x * st;
        R[2][0] = ax.z * ax.x * vt - ax.y * st;
        R[2][1] = ax.z * ax.y * vt + ax.x * st;
        R[2][2] = ct + ax.z * ax.z * vt;
    }
    row[0] = center.x;
    row[1] = center.y;
    row[2] = center.z;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) row[3 + 3 * a + b] = R[a][b];
    for (int a = 0; a < 3; ++a) {
        row[12 + a] = linear_velocity[a];
        row[15 + a] = angular_velocity[a];
    }
}

}  // namespace lbmg
