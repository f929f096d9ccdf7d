// Unit-level calls as the reference's own tests make them, on the B200 engine:
// step() on an explicit state (solver.hpp:82-83), the IB free functions
// (ib.hpp:96-128) over a sample set, and Runner(scene, regions, devices).
#include <cmath>
#include <cstdio>

#include "lbm_b200.hpp"

int main() {
    try {
        // step(SimState&): one step from a loaded state equals one advance step
        lbm::SceneConfig cfg;
        cfg.dims = {24, 16, 16};
        cfg.viscosity = 0.02;
        cfg.boundary.faces[5] = {lbm::FaceCondition::VelocityInlet, {0.05, 0.0, 0.0}};
        lbm::Scene scene = lbm::build_scene(cfg);
        lbm::Runner a(scene), b(scene);
        a.advance(7);
        const lbm::FieldStore f7 = a.gather_f();
        a.advance(1);
        b.load_state(f7, lbm::FieldStore{}, 7);
        const lbm::StepStatus st = lbm::step(b);
        const lbm::FieldStore fa = a.gather_f(), fb = b.gather_f();
        double df = 0.0;
        for (std::size_t k = 0; k < fa.size(); ++k) df = std::fmax(df, std::fabs(fa.data()[k] - fb.data()[k]));
        std::printf("step ok=%d t=%ld max_df=%.3e\n", int(st.ok), b.step_count(), df);

        // IB free functions over a uniform field: interpolation is exact, the
        // spread conserves the total force, the reaction is its negative
        const lbm::GridDims dims{16, 16, 16};
        lbm::SolidSampleSet set;
        for (int k = 0; k < 64; ++k) {
            const double th = 0.1 * k, ph = 0.37 * k;
            set.reference_positions.push_back({3.0 * std::sin(th) * std::cos(ph), 3.0 * std::sin(th) * std::sin(ph),
                                               3.0 * std::cos(th)});
        }
        const lbm::RigidMotion motion{{0.0, 0.0, 0.0}, {0.0, 0.0, 0.01}, {8.0, 8.0, 8.0}};
        lbm::update_rigid_motion(set, motion, 5, dims);
        lbm::FieldStore u(dims.n_nodes(), 3), rho(dims.n_nodes(), 1), g(dims.n_nodes(), 3);
        for (std::size_t k = 0; k < dims.n_nodes(); ++k) {
            u.data()[3 * k] = 0.1;
            rho.data()[k] = 1.0;
        }
        const lbm::SlabContext whole{dims};
        lbm::interpolate_velocity(set, u, whole);
        lbm::penalty_forces(set, rho, whole);
        lbm::spread_forces(set, g, whole);
        double fsum = 0.0, gsum = 0.0, uerr = 0.0;
        for (std::size_t s = 0; s < set.size(); ++s) {
            fsum += set.penalty_force[s].x;
            uerr = std::fmax(uerr, std::fabs(set.sampled_velocity[s].x - 0.1));
        }
        for (std::size_t k = 0; k < dims.n_nodes(); ++k) gsum += g.data()[3 * k];
        const lbm::ReactionTotals tot = lbm::reaction_totals(set, motion.center, 0, dims.nz);
        std::printf("ib samples=%zu uerr=%.3e spread_err=%.3e reaction_err=%.3e\n", set.size(), uerr,
                    std::fabs(fsum - gsum), std::fabs(tot.force.x + fsum));

        // Runner(scene, regions, devices): two slabs (on device 0 twice when
        // only one GPU is present) equal the single-slab run
        lbm::Runner one(scene, 2, 0u), two(scene, 2, std::vector<int>{0, 0});
        one.advance(10);
        two.advance(10);
        const lbm::FieldStore r1 = one.gather_rho(), r2 = two.gather_rho();
        double dr = 0.0;
        for (std::size_t k = 0; k < r1.size(); ++k) dr = std::fmax(dr, std::fabs(r1.data()[k] - r2.data()[k]));
        std::printf("devices regions=%d dev1=%d max_drho=%.3e\n", two.region_count(), two.region_device(1), dr);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
