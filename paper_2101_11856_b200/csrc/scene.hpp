// Host-side scene setup (grid/solid setup half of the drop-in boundary):
// procedural meshes, seeded Poisson-disk surface sampling, block/Morton sample
// ordering, z-slab split and the collision-model tables.  Re-implemented from
// the reference's documented semantics; integer outputs (sample order,
// source ids, slabs) are bit-exact with the reference (tests/test_setup.py).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbmg.h"

namespace lbmg {

struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};

struct V3 {
    double x = 0, y = 0, z = 0;
    double operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
    double& operator[](int a) { return a == 0 ? x : (a == 1 ? y : z); }
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V3 v3(const double* p) { return {p[0], p[1], p[2]}; }

struct TriMesh {
    std::vector<V3> vertices;
    std::vector<std::array<uint32_t, 3>> triangles;
};

TriMesh build_mesh(const lbmg_mesh& m);

struct SamplingReport {
    size_t n_samples = 0, degenerate = 0, attempts = 0, occupied_cells = 0;
    double density_min = 0, density_mean = 0, density_max = 0, in_band_fraction = 0;
};

struct SampleSet {
    std::vector<V3> positions;
    std::vector<V3> reference_positions;
    std::vector<uint32_t> source_id;
    int block_edge = 1;
    V3 bbox_lo, bbox_hi;
    double poisson_radius = 0;
    size_t size() const { return positions.size(); }
};

SampleSet sample_surface(const TriMesh& mesh, double radius, uint64_t seed, int method,
                         SamplingReport* report);

uint64_t morton3(uint32_t x, uint32_t y, uint32_t z);
// Storage permutation perm[new] = old (reorder_samples, ib.cpp:231-292).
std::vector<uint32_t> reorder_permutation(const std::vector<V3>& pos,
                                          const std::vector<uint32_t>& src, int ell);
void reorder_samples(SampleSet& set, int ell);

std::vector<std::array<int, 2>> split_domain(int nz, int m);

// Collision model (collision.hpp:33-49): canonical row order tables + rates.
struct ModelTables {
    std::array<int, 27> row_to_mu{};
    std::array<int, 27> mu_to_row{};
    std::array<int, 27> degree{};  // per row
};
const ModelTables& model_tables();
// SceneConfig::make_model incl. validation; returns rates in row order.
std::array<double, 27> make_rates(const lbmg_scene_config& cfg);
void validate_config(const lbmg_scene_config& cfg);

struct SolidInstance {
    lbmg_solid_config cfg;
    SampleSet samples;
    bool moving = false;
    V3 linear_velocity, angular_velocity, center;  // RigidMotion
    SamplingReport report;
};

// Rigid motion row of step t (ib.cpp:456-475): centre(t)[3], R(t)[9], v[3],
// omega[3] (kMotionRow doubles), computed with the reference's expressions.
void motion_table_row(const V3& linear_velocity, const V3& angular_velocity, const V3& center0, long t,
                      double* row);

}  // namespace lbmg

struct lbmg_scene {
    lbmg_scene_config cfg;  // solids pointer re-targeted to solid_cfgs
    std::vector<lbmg_solid_config> solid_cfgs;
    std::vector<lbmg::SolidInstance> solids;
    std::vector<lbmg_emitter> emitters;  // SceneConfig::emitters (scene.hpp:60)
};
