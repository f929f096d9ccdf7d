// A reference-style client: the 64^3 lid-driven cavity (BASELINE configs[0])
// written against the reference API names, built on the B200 engine.
//   g++ -std=c++17 -Iinclude examples/cavity.cpp -Lpaper_2101_11856_b200/_build -llbmg
//       -Wl,-rpath,$PWD/paper_2101_11856_b200/_build -o cavity
#include <cstdio>

#include "lbm_b200.hpp"

int main(int argc, char** argv) {
    lbm::SceneConfig cfg;
    cfg.dims = {64, 64, 64};
    cfg.viscosity = 0.02;
    cfg.kind = lbm::CollisionKind::CentralMomentMRT;
    cfg.high_order_rate = 1.5;
    cfg.policy = lbm::RatePolicy::RelaxTowardOne;
    cfg.boundary.faces[5] = {lbm::FaceCondition::VelocityInlet, {0.05, 0.0, 0.0}};
    const long steps = argc > 1 ? std::atol(argv[1]) : 100;
    try {
        lbm::Scene scene = lbm::build_scene(cfg);
        lbm::Runner runner(scene);
        lbm::StepStatus st = runner.advance(steps);
        lbm::FieldStore rho = runner.gather_rho();
        double mass = 0.0;
        for (std::size_t k = 0; k < rho.n_nodes(); ++k) mass += rho.get(k, 0);
        std::printf("steps=%ld ok=%d mass=%.10f\n", runner.step_count(), int(st.ok), mass);
    } catch (const lbm::ConfigError& e) {
        std::fprintf(stderr, "config: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
