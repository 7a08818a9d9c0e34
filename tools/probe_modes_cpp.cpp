// Diagnostics: host/device time split of the C++ drop-in run_batch per run mode on the
// acceptance criterion 6 workload (1000 clones, N = 200, 0.35 period, Sun + planets).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pswarm.hpp"

using namespace pswarm;

int main() {
    PropagationConfig config;
    config.n_nodes = 200;
    config.tolerance = 1e-12;
    config.force = make_reference_force_model();
    const auto states = make_clone_batch(make_reference_state(), 1000, 1e-5);
    const double period = osculating_period(states[0], mu_sun_km3s2);
    const auto segments = plan_segments(states[0], 0.0, 0.35 * period, mu_sun_km3s2, SegmentPolicy::single, 200);
    for (int rep = 0; rep < 6; ++rep)
        for (RunMode mode : {RunMode::independent, RunMode::augmented_sequential}) {
            const auto t0 = std::chrono::steady_clock::now();
            const auto o = run_batch(states, config, segments, mode, 1);
            const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            std::fprintf(stderr, "%-22s wall %.3f ms (run_batch %.3f ms)\n", to_string(mode).c_str(), 1e3 * t,
                         1e3 * o.wall_time_s);
        }
    return 0;
}
