// A reference-style `run_scene` slice (driver.cpp:22-82) on the B200 engine:
// tune (autotune.hpp search on a clone), apply, advance in chunks with
// asynchronous rho* snapshots written as LBF1 dumps (io.hpp dump_field).
//   g++ -std=c++17 -Iinclude examples/tune_and_snapshot.cpp -Lpaper_2101_11856_b200/_build -llbmg
//       -Wl,-rpath,$PWD/paper_2101_11856_b200/_build -o tune_and_snapshot
#include <cstdio>
#include <string>

#include "lbm_b200.hpp"

int main(int argc, char** argv) {
    const std::string out = argc > 1 ? argv[1] : "/tmp";
    lbm::SceneConfig cfg;
    cfg.dims = {32, 24, 24};
    cfg.viscosity = 0.02;
    cfg.kind = lbm::CollisionKind::CentralMomentMRT;
    cfg.high_order_rate = 1.5;
    cfg.policy = lbm::RatePolicy::RelaxTowardOne;
    cfg.boundary.faces[5] = {lbm::FaceCondition::VelocityInlet, {0.05, 0.0, 0.0}};
    try {
        lbm::Scene scene = lbm::build_scene(cfg);
        lbm::Runner runner(scene);
        lbm::TuneSpec spec;
        spec.alphas = {256, 4096, std::size_t(1) << 20};
        spec.variants = {{0, 0}, {1, 0}};
        spec.n_steps = 3;
        spec.warmup = 1;
        const lbm::TuneOutcome best = lbm::search(runner, spec);
        runner.set_variant(best.variant[0], best.variant[1]);
        runner.set_layout(best.ell, best.alpha);
        std::printf("tuned rows=%zu variant=%d,%d alpha=%zu step_count=%ld\n", best.rows.size(), best.variant[0],
                    best.variant[1], best.alpha, runner.step_count());
        lbm::FieldStore rho, u;
        for (int chunk = 0; chunk < 3; ++chunk) {
            runner.advance(10);
            if (chunk > 0) {  // previous snapshot drained while this chunk ran
                const long t = runner.snapshot_wait(rho, u);
                lbm::dump_field(rho, runner.dims(), out + "/rho_" + std::to_string(t) + ".lbf");
            }
            runner.snapshot_begin();
        }
        const long t = runner.snapshot_wait(rho, u);
        lbm::dump_field(rho, runner.dims(), out + "/rho_" + std::to_string(t) + ".lbf");
        std::printf("last_snapshot=%ld steps=%ld\n", t, runner.step_count());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
