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
    // smoke tracers under the lid (tracer.hpp), emitted and advected on the device
    cfg.emitters.push_back({{8.0, 8.0, 48.0}, {56.0, 56.0, 60.0}, 10});
    const long steps = argc > 1 ? std::atol(argv[1]) : 100;
    try {
        lbm::Scene scene = lbm::build_scene(cfg);
        lbm::Runner runner(scene);
        lbm::StepStatus st = runner.advance(steps);
        lbm::FieldStore rho = runner.gather_rho();
        double mass = 0.0;
        for (std::size_t k = 0; k < rho.n_nodes(); ++k) mass += rho.get(k, 0);
        const lbm::TracerCloud cloud = runner.tracers();
        double smoke = 0.0;
        for (double v : runner.tracer_density()) smoke += v;
        std::printf("steps=%ld ok=%d mass=%.10f tracers=%zu smoke=%.6f\n", runner.step_count(), int(st.ok), mass,
                    cloud.size(), smoke);
    } catch (const lbm::ConfigError& e) {
        std::fprintf(stderr, "config: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
