// runner_demo.cpp -- TEST INFRASTRUCTURE: the harness drop-in
// (include/apbf_gpu/runner.hpp) next to the reference's own runScenario.
// Checks, on the GPU, the reference harness test expectations
// (tests/test_harness.cpp: "runScenario writes metrics and frame dumps",
// "honors mode and range overrides", "bench totals are exact") for
// apbf::gpu::runScenario / runBench, and that the reference's compareRuns
// accepts the GPU metrics.csv against the reference's Solver<double> run of
// the same scenario (identical config header, same hash).  Prints
// "RUNNER OK" and exits 0 when everything holds.
// Built by oracle/Makefile into oracle/_ref/ (needs /root/reference to build).
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <string>

#include "apbf_gpu/runner.hpp"

using namespace apbf;
namespace fs = std::filesystem;

static int failures = 0;
#define EXPECT(c)                                                             \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);        \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

static std::vector<std::string> headerLines(const fs::path& p) {
    std::ifstream is(p);
    std::vector<std::string> out;
    for (std::string l; std::getline(is, l);)
        if (!l.empty() && l[0] == '#') out.push_back(l);
    return out;
}

int main(int argc, char** argv) {
    const fs::path dir = fs::temp_directory_path() / "apbf_runner_demo";
    fs::remove_all(dir);
    const double scale = argc > 1 ? std::atof(argv[1]) : 8000.0 / 216000.0;
    const int frames = argc > 2 ? std::atoi(argv[2]) : 10;

    // 1. dumps and metrics (test_harness.cpp:515-561) on the GPU backend
    {
        const ScenarioSpec spec = buildScenario("dam_break", 0.001);
        RunOptions opt;
        opt.frames = 2;
        opt.seed = 11;
        opt.deterministic = true;
        opt.outDir = dir / "dumps";
        opt.dumpImagesEvery = 1;
        opt.dumpParticlesEvery = 1;
        const RunReport r = gpu::runScenario(spec, opt);
        EXPECT(r.frames.size() == 2);
        EXPECT(r.hash == scenarioHash(spec, 11));
        EXPECT(r.zeroTime);
        for (const char* f : {"metrics.csv", "frame_000000.ppm", "frame_000001.ppm", "particles_000000.csv",
                              "particles_000001.csv"})
            EXPECT(fs::exists(opt.outDir / f));
        const MetricsFile m = readMetricsCsv(opt.outDir / "metrics.csv");
        EXPECT(m.hash && *m.hash == r.hash);
        EXPECT(m.rows.size() == 2 && m.rows[1].timeMs == 0.0);
    }
    // 2. mode and range overrides: uniform budget totals are exact
    {
        const ScenarioSpec spec = buildScenario("dam_break", 0.001);
        RunOptions opt;
        opt.mode = SolverMode::Pbf;
        opt.range = IterationRange(2, 2);
        opt.frames = 1;
        opt.deterministic = true;
        const RunReport r = gpu::runScenario(spec, opt);
        EXPECT(r.frames[0].totalIterations == 2LL * 216 * spec.solver.substeps);
    }
    // 3. bench totals (test_harness.cpp:586-611)
    {
        const ScenarioSpec spec = buildScenario("dam_break", 0.001);
        const auto res = gpu::runBench(spec, parseBenchModes("pbf:6,pbf:3,apbf:dtc"), 1, 2, 1);
        const long long n = 216, S = spec.solver.substeps;
        EXPECT(res[0].iterations == 6 * n * 2 * S);
        EXPECT(res[1].iterations == 3 * n * 2 * S);
        EXPECT(res[2].iterations >= 3 * n * 2 * S && res[2].iterations < 6 * n * 2 * S);
        std::printf("%s", formatBenchReport(res).c_str());
    }
    // 4. GPU run vs the reference's Solver<double> run: same header, compare passes
    {
        const ScenarioSpec spec = buildScenario("dam_break", scale);
        RunOptions opt;
        opt.frames = frames;
        opt.seed = 1;
        opt.deterministic = true;
        opt.outDir = dir / "gpu";
        gpu::runScenario(spec, opt);
        opt.outDir = dir / "ref";
        runScenario(spec, opt);
        EXPECT(headerLines(dir / "gpu" / "metrics.csv") == headerLines(dir / "ref" / "metrics.csv"));
        const CompareResult c =
            compareRuns(readMetricsCsv(dir / "ref" / "metrics.csv"), readMetricsCsv(dir / "gpu" / "metrics.csv"), 4.0);
        std::printf("compare: frames = %d, max |avg density delta| = %.6f pct pts, pass = %d\n", c.frames,
                    c.maxDelta, int(c.pass));
        EXPECT(c.pass && c.frames == frames);
    }
    fs::remove_all(dir);
    if (failures) return 1;
    std::printf("RUNNER OK\n");
    return 0;
}
