// The step-seam binding end to end, as a reference user would call it: the
// reference builds a problem (wb::riemann4, src/problems.cpp) and runs
// Engine::init; one copy is stepped by the reference's own Engine::run on the
// host cores, the other by run_fcsg on the B200; the states must agree to
// round-off. Both classifier variants. TEST INFRASTRUCTURE.
//   dropin_engine_check <fcnn weight file> [steps]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>

#include "fcs/workbench.hpp"
#include "run_fcsg.hpp"

using namespace fcs;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s weights.bin [steps]\n", argv[0]);
        return 2;
    }
    const long steps = argc > 2 ? std::atol(argv[2]) : 5;
    int fails = 0;
    for (int variant = 0; variant < 2; ++variant) {
        auto make = [&] { return wb::riemann4(2, 2, 37, 9, 1e9); };
        run::EngineConfig cfg;
        cfg.cfl = 0.5;
        cfg.T = 1e9;
        cfg.workers = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        cfg.max_steps = steps;
        cfg.classifier.variant = variant == 0 ? visc::ClassifierConfig::Variant::ann
                                              : visc::ClassifierConfig::Variant::fallback;
        cfg.classifier.weight_path = argv[1];
        auto pa = make();
        run::Engine ref(pa.dec, pa.bcs, pa.ic, cfg);
        ref.init();
        const auto ra = ref.run();
        auto pb = make();
        run::Engine dut(pb.dec, pb.bcs, pb.ic, cfg);
        dut.init();
        const auto rb = run::run_fcsg(dut, cfg, steps);
        double worst = 0.0;
        for (size_t k = 0; k < ref.subs().size(); ++k)
            for (int c = 0; c < 4; ++c) {
                const auto& a = dut.subs()[k].e[c].v;
                const auto& b = ref.subs()[k].e[c].v;
                double dn = 0.0, bn = 0.0;
                for (size_t p = 0; p < a.size(); ++p) {
                    dn += (a[p] - b[p]) * (a[p] - b[p]);
                    bn += b[p] * b[p];
                }
                worst = std::max(worst, std::sqrt(dn / std::max(bn, 1e-300)));
            }
        const bool ok = ra.steps == rb.steps && std::fabs(ra.t - rb.t) <= 1e-12 * std::fabs(ra.t) && worst <= 1e-10;
        std::printf("%s classifier: %ld steps, t %.15g (reference %.15g), worst per-field rel L2 %.3e, "
                    "B200 %.3f ms/step vs reference %.3f ms/step (%d threads): %s\n",
                    variant == 0 ? "ann" : "fallback", rb.steps, rb.t, ra.t, worst, 1e3 * rb.seconds_per_step,
                    1e3 * ra.seconds_per_step, cfg.workers, ok ? "ok" : "MISMATCH");
        fails += ok ? 0 : 1;
    }
    return fails;
}
