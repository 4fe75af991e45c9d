// e2e_cpp.cpp -- the end-to-end cost of the binding a reference maintainer
// would add (include/apbf_gpu/solver.hpp): the reference's
// own scenario loader and ParticleSet<Scalar> (src/scenario.cpp), stepped by
// apbf::gpu::Solver<Scalar>::stepFrame -- i.e. what runScenario
// (runner.cpp:71-84) does per frame after the one-line swap.  Timed with
// std::chrono around each stepFrame call (host conversion, page-locked
// staging, upload, frame, overlapped download, conversion back), after
// warm-up frames.  Prints one JSON line.
//
// Usage: e2e_cpp <scenario file> <frames> <warmup> [f32|f64]
// Built by tools/Makefile into tools/_bin/ (needs /root/reference to build;
// the binary runs anywhere libapbf_gpu.so loads).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "apbf_gpu/solver.hpp"
#include "scenario.hpp"

using namespace apbf;

template <class T>
static ParticleSet<T> castState(const ParticleSet<double>& d) {
    ParticleSet<T> o;
    const int n = d.count();
    o.x.resize(3, n);
    o.xStar.resize(3, n);
    o.v.resize(3, n);
    o.mass.resize(n);
    o.invMass.resize(n);
    o.lambda.resize(n);
    o.level.resize(n);
    for (int i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            o.x(a, i) = T(d.x(a, i));
            o.xStar(a, i) = T(d.xStar(a, i));
            o.v(a, i) = T(d.v(a, i));
        }
        o.mass[i] = T(d.mass[i]);
        o.invMass[i] = T(d.invMass[i]);
        o.lambda[i] = T(d.lambda[i]);
        o.level[i] = d.level[i];
    }
    return o;
}

template <class T>
static SolverConfig<T> castCfg(const SolverConfig<double>& c) {
    SolverConfig<T> o;
    o.dtFrame = T(c.dtFrame);
    o.substeps = c.substeps;
    o.range = c.range;
    o.restDensity = T(c.restDensity);
    o.h = T(c.h);
    o.epsilon = T(c.epsilon);
    o.gravity = Vec3<T>(T(c.gravity[0]), T(c.gravity[1]), T(c.gravity[2]));
    o.stabIterations = c.stabIterations;
    o.stabThreshold = c.stabThreshold;
    o.particleRadius = T(c.particleRadius);
    o.mode = c.mode;
    o.velocityCap = T(c.velocityCap);
    o.inactiveLambdaZero = c.inactiveLambdaZero;
    o.deterministic = c.deterministic;
    o.recordResiduals = c.recordResiduals;
    return o;
}

template <class T>
static SdfScene<T> castScene(const SdfScene<double>& s) {
    SdfScene<T> o;
    o.gradientStep = T(s.gradientStep);
    for (const auto& prim : s.primitives) {
        std::visit(
            [&](const auto& g) {
                using P = std::decay_t<decltype(g)>;
                if constexpr (std::is_same_v<P, Box<double>>)
                    o.primitives.emplace_back(Box<T>(Vec3<T>(T(g.center[0]), T(g.center[1]), T(g.center[2])),
                                                     Vec3<T>(T(g.halfExtents[0]), T(g.halfExtents[1]),
                                                             T(g.halfExtents[2])),
                                                     g.interior));
                else if constexpr (std::is_same_v<P, Cone<double>>)
                    o.primitives.emplace_back(Cone<T>(Vec3<T>(T(g.baseCenter[0]), T(g.baseCenter[1]),
                                                              T(g.baseCenter[2])),
                                                      T(g.baseRadius), T(g.height)));
                else
                    throw std::runtime_error("e2e_cpp: scenario primitive kind not handled");
            },
            prim);
    }
    return o;
}

template <class T>
static Camera<T> castCam(const Camera<double>& c) {
    Camera<T> o;
    o.eye = Vec3<T>(T(c.eye[0]), T(c.eye[1]), T(c.eye[2]));
    o.lookAt = Vec3<T>(T(c.lookAt[0]), T(c.lookAt[1]), T(c.lookAt[2]));
    o.up = Vec3<T>(T(c.up[0]), T(c.up[1]), T(c.up[2]));
    o.verticalFov = T(c.verticalFov);
    o.width = c.width;
    o.height = c.height;
    o.nearClip = T(c.nearClip);
    return o;
}

template <class T>
static LodModelConfig<T> castLod(const LodModelConfig<double>& l) {
    LodModelConfig<T> o;
    o.model = l.model;
    o.dMin = T(l.dMin);
    o.dMax = T(l.dMax);
    o.range = l.range;
    o.autoRange = l.autoRange;
    return o;
}

template <class T>
static int run(const ScenarioSpec& spec, int frames, int warmup, const char* prec) {
    ParticleSet<T> st = castState<T>(makeState(spec, 1));
    const Camera<T> cam = castCam<T>(spec.camera);
    const LodModelConfig<T> lod = castLod<T>(spec.lod);
    gpu::Solver<T> solver(castCfg<T>(spec.solver), castScene<T>(spec.scene));
    for (int f = 0; f < warmup; ++f) solver.stepFrame(st, cam, lod, f);
    std::vector<double> ms;
    long long its = 0;
    for (int f = 0; f < frames; ++f) {
        const auto t0 = std::chrono::steady_clock::now();
        its += solver.stepFrame(st, cam, lod, warmup + f).totalIterations;
        const auto t1 = std::chrono::steady_clock::now();
        ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    double total = 0;
    for (double v : ms) total += v;
    std::vector<double> sorted = ms;
    std::sort(sorted.begin(), sorted.end());
    std::printf(
        "{\"binding\": \"apbf::gpu::Solver<%s>::stepFrame (include/apbf_gpu/solver.hpp)\", \"scenario\": \"%s\", "
        "\"particles\": %d, \"frames\": %d, \"warmup\": %d, \"ms_per_step\": %.4f, \"median_ms\": %.4f, "
        "\"particle_iterations_per_s\": %.6e}\n",
        prec, spec.name.c_str(), st.count(), frames, warmup, total / frames, sorted[sorted.size() / 2],
        double(its) / (total / 1e3));
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: e2e_cpp <scenario file> <frames> <warmup> [f32|f64]\n");
        return 2;
    }
    const ScenarioSpec spec = loadScenarioFile(argv[1], 1.0);
    const int frames = std::max(1, std::atoi(argv[2]));
    const int warmup = std::max(0, std::atoi(argv[3]));
    const std::string prec = argc > 4 ? argv[4] : "f64";
    try {
        if (prec == "f32") return run<float>(spec, frames, warmup, "float");
        return run<double>(spec, frames, warmup, "double");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "e2e_cpp: %s\n", e.what());
        return 1;
    }
}
