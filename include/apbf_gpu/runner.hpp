// apbf_gpu/runner.hpp -- C++ drop-in of the reference harness's GPU backend
// (SURVEY.md §8f row 1): runScenario (/root/reference/proj/src/runner.cpp:
// 60-98) and runBench (src/bench.cpp:58-91) with the frames stepped on the
// B200 by apbf::gpu::Solver, the state resident on the device between frames.
// Same RunOptions, RunReport, metrics.csv (written by the reference's own
// writeMetricsCsv), frame_XXXXXX.ppm level images (rendered on the device:
// only the image is downloaded) and particles_XXXXXX.csv snapshots, so the
// reference CLI can offer `apbf run --backend gpu` and `apbf compare` reads
// the result.  Include next to the reference's src/ headers; link the
// reference's src/*.cpp and paper_1608_04721_b200/libapbf_gpu.so.
#pragma once

#include <cstdio>
#include <filesystem>
#include <string>
#include <utility>
#include <vector>

#include "apbf_gpu/solver.hpp"
#include "bench.hpp"
#include "metrics.hpp"
#include "runner.hpp"
#include "scenario.hpp"

namespace apbf::gpu {

namespace detail {

inline std::string g17(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

// The config echo that heads metrics.csv (runner.cpp:20-45), in its order.
inline std::vector<std::pair<std::string, std::string>> runEcho(const ScenarioSpec& s,
                                                                const RunOptions& opt, int frames,
                                                                int particles) {
    const SolverConfig<double>& c = s.solver;
    auto flag = [](bool b) { return std::string(b ? "1" : "0"); };
    return {{"scenario", s.name},
            {"scale", g17(s.scale)},
            {"particles", std::to_string(particles)},
            {"frames", std::to_string(frames)},
            {"seed", std::to_string(opt.seed)},
            {"mode", modeName(c.mode)},
            {"lod_model", lodModelName(s.lod.model)},
            {"iterations", std::to_string(c.range.nMin) + ".." + std::to_string(c.range.nMax)},
            {"deterministic", flag(opt.deterministic)},
            {"dt_frame", g17(c.dtFrame)},
            {"substeps", std::to_string(c.substeps)},
            {"rest_density", g17(c.restDensity)},
            {"smoothing_length", g17(c.h)},
            {"epsilon", g17(c.epsilon)},
            {"particle_radius", g17(c.effectiveParticleRadius())},
            {"stab_iterations", std::to_string(c.stabIterations)},
            {"stab_threshold", std::to_string(c.effectiveStabThreshold())},
            {"velocity_cap", g17(c.effectiveVelocityCap())},
            {"inactive_lambda_zero", flag(c.inactiveLambdaZero)},
            {"jitter", g17(s.jitter)}};
}

inline std::filesystem::path dumpPath(const std::filesystem::path& dir, const char* stem, int frame,
                                      const char* ext) {
    char b[64];
    std::snprintf(b, sizeof b, "%s_%06d.%s", stem, frame, ext);
    return dir / b;
}

}  // namespace detail

/// runScenario on the B200: spawn (makeState, double), simulate in float32 on
/// the device, and optionally persist metrics.csv plus frame dumps.
inline RunReport runScenario(const ScenarioSpec& spec, const RunOptions& opt, int device = 0) {
    ScenarioSpec s = spec;
    if (opt.range) {
        s.solver.range = *opt.range;
        s.lod.range = *opt.range;
    }
    if (opt.lodModel) s.lod.model = *opt.lodModel;
    s.solver.mode = opt.mode;
    s.solver.deterministic = opt.deterministic;
    const int frames = opt.frames > 0 ? opt.frames : s.frames;

    ParticleSet<double> state = makeState(s, opt.seed);
    Solver<double> solver(s.solver, s.scene, device);

    RunReport report;
    report.hash = scenarioHash(s, opt.seed);
    report.zeroTime = opt.deterministic;
    report.echo = detail::runEcho(s, opt, frames, state.count());
    report.frames.reserve(static_cast<size_t>(frames));

    const bool persist = !opt.outDir.empty();
    if (persist) std::filesystem::create_directories(opt.outDir);

    solver.setState(state);
    for (int f = 0; f < frames; ++f) {
        report.frames.push_back(solver.stepFrameResident(s.camera, s.lod, f));
        if (persist && opt.dumpImagesEvery > 0 && f % opt.dumpImagesEvery == 0) {
            writePpm(solver.renderLevelImage(s.camera, s.solver.effectiveParticleRadius(), s.solver.range),
                     detail::dumpPath(opt.outDir, "frame", f, "ppm"));
        }
        if (persist && opt.dumpParticlesEvery > 0 && f % opt.dumpParticlesEvery == 0) {
            solver.getState(state);
            writeParticleSnapshot(detail::dumpPath(opt.outDir, "particles", f, "csv"), state);
        }
    }
    if (persist) writeMetricsCsv(opt.outDir / "metrics.csv", report);
    return report;
}

/// runBench with the GPU runScenario: repetitions interleaved across modes,
/// per mode the median over repetitions of each run's median frame time.
inline std::vector<BenchResult> runBench(const ScenarioSpec& spec, const std::vector<BenchMode>& modes,
                                         int reps, int frames, std::uint64_t seed, int device = 0) {
    if (reps < 1) throw std::invalid_argument("bench repetitions must be at least 1");
    std::vector<BenchResult> results(modes.size());
    std::vector<std::vector<double>> medians(modes.size());
    for (int rep = 0; rep < reps; ++rep) {
        for (std::size_t k = 0; k < modes.size(); ++k) {
            RunOptions opt;
            opt.mode = modes[k].mode;
            opt.lodModel = modes[k].lodModel;
            if (modes[k].mode == SolverMode::Pbf)
                opt.range = IterationRange(modes[k].pbfIterations, modes[k].pbfIterations);
            opt.frames = frames;
            opt.seed = seed;
            const RunReport r = runScenario(spec, opt, device);
            medians[k].push_back(r.medianFrameMs());
            results[k].token = modes[k].token;
            results[k].iterations = r.totalIterations();
            results[k].frames = static_cast<int>(r.frames.size());
        }
    }
    for (std::size_t k = 0; k < modes.size(); ++k) {
        results[k].medianFrameMs = medianOf(std::move(medians[k]));
        results[k].particles = spec.particleCount();
    }
    return results;
}

}  // namespace apbf::gpu
