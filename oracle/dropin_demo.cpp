// dropin_demo.cpp -- TEST INFRASTRUCTURE: the reference harness types driving
// apbf::gpu::Solver (include/apbf_gpu/solver.hpp) next to the reference's
// own apbf::Solver<float>; exits 0 when every frame is bit-identical.
// Built by oracle/Makefile into oracle/_ref/ (needs /root/reference to build,
// runs anywhere the GPU library loads).
#include <cstdio>
#include <cstring>
#include <limits>

#include "apbf_gpu/solver.hpp"
#include "scenario.hpp"

using namespace apbf;

template <class T>
static ParticleSet<T> cast(const ParticleSet<double>& d) {
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
        o.invMass[i] = T(1) / o.mass[i];
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
    o.deterministic = true;
    return o;
}

template <class T>
static SdfScene<T> castScene(const SdfScene<double>& s) {
    SdfScene<T> o;
    o.gradientStep = T(s.gradientStep);
    for (const auto& p : s.primitives) {
        std::visit([&](const auto& g) {
            using G = std::decay_t<decltype(g)>;
            if constexpr (std::is_same_v<G, Box<double>>)
                o.primitives.emplace_back(Box<T>(Vec3<T>(T(g.center[0]), T(g.center[1]), T(g.center[2])),
                                                 Vec3<T>(T(g.halfExtents[0]), T(g.halfExtents[1]), T(g.halfExtents[2])),
                                                 g.interior));
            else if constexpr (std::is_same_v<G, Cone<double>>)
                o.primitives.emplace_back(Cone<T>(Vec3<T>(T(g.baseCenter[0]), T(g.baseCenter[1]), T(g.baseCenter[2])),
                                                  T(g.baseRadius), T(g.height)));
        }, p);
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

int main(int argc, char** argv) {
    const char* name = argc > 1 ? argv[1] : "multi_dam_break";
    const double scale = argc > 2 ? std::atof(argv[2]) : 0.05;
    const int frames = argc > 3 ? std::atoi(argv[3]) : 4;
    const ScenarioSpec spec = buildScenario(name, scale);
    const ParticleSet<double> s0 = makeState(spec, 1);
    ParticleSet<float> a = cast<float>(s0), b = cast<float>(s0);
    const SolverConfig<float> cfg = castCfg<float>(spec.solver);
    const SdfScene<float> scene = castScene<float>(spec.scene);
    LodModelConfig<float> lod;
    lod.model = spec.lod.model;
    lod.range = spec.lod.range;
    lod.autoRange = spec.lod.autoRange;
    const Camera<float> cam = castCam<float>(spec.camera);
    apbf::Solver<float> ref(cfg, scene);
    apbf::gpu::Solver<float> gpu(cfg, scene);   // with an observer: the resident path
    apbf::gpu::Solver<float> host(cfg, scene);  // stepFrame via apbf_gpu_step_frame_host
    ParticleSet<float> c = cast<float>(s0);
    int iters = 0;
    gpu.iterationObserver = [&](int, int, const ParticleSet<float>&) { ++iters; };
    auto same_as = [&](const ParticleSet<float>& p, const ParticleSet<float>& q) {
        return p.count() == q.count() &&
               std::memcmp(p.x.data(), q.x.data(), sizeof(float) * 3 * p.count()) == 0 &&
               std::memcmp(p.xStar.data(), q.xStar.data(), sizeof(float) * 3 * p.count()) == 0 &&
               std::memcmp(p.v.data(), q.v.data(), sizeof(float) * 3 * p.count()) == 0 &&
               std::memcmp(p.mass.data(), q.mass.data(), sizeof(float) * p.count()) == 0 &&
               std::memcmp(p.invMass.data(), q.invMass.data(), sizeof(float) * p.count()) == 0 &&
               std::memcmp(p.lambda.data(), q.lambda.data(), sizeof(float) * p.count()) == 0 &&
               std::memcmp(p.level.data(), q.level.data(), sizeof(int) * p.count()) == 0;
    };
    for (int f = 0; f < frames; ++f) {
        const FrameStats sr = ref.stepFrame(a, cam, lod, f);
        const FrameStats sg = gpu.stepFrame(b, cam, lod, f);
        const FrameStats sh = host.stepFrame(c, cam, lod, f);
        const bool same = same_as(a, b) && same_as(a, c) && sr.totalIterations == sg.totalIterations &&
                          sr.contacts == sg.contacts && sr.totalIterations == sh.totalIterations &&
                          sr.contacts == sh.contacts;
        std::printf("frame %d: %d particles, totalIterations ref %lld gpu %lld host-path %lld, %s\n", f,
                    a.count(), sr.totalIterations, sg.totalIterations, sh.totalIterations,
                    same ? "bit-identical" : "DIFFERENT");
        if (!same) return 1;
    }
    // a failing host-path frame leaves the caller's ParticleSet untouched
    {
        ParticleSet<float> bad = c;
        bad.v(1, 7) = std::numeric_limits<float>::quiet_NaN();
        const ParticleSet<float> before = bad;
        try {
            host.stepFrame(bad, cam, lod, frames);
            std::printf("expected NumericalError from the host path\n");
            return 1;
        } catch (const NumericalError& e) {
            std::printf("host path NumericalError pass=%s particle=%d\n", e.pass().c_str(), e.particle());
        }
        bool untouched = bad.count() == before.count();
        for (int i = 0; untouched && i < bad.count(); ++i)
            for (int q = 0; q < 3; ++q)
                untouched = untouched && (bad.x(q, i) == before.x(q, i)) &&
                            (bad.xStar(q, i) == before.xStar(q, i)) &&
                            (std::memcmp(&bad.v.data()[3 * i + q], &before.v.data()[3 * i + q], sizeof(float)) == 0);
        if (!untouched) {
            std::printf("host path: failing frame modified the caller's state\n");
            return 1;
        }
    }
    std::printf("iteration observer calls: %d\n", iters);
    // error path: a NaN must surface as apbf::NumericalError("predict", 2)
    ParticleSet<float> bad = cast<float>(s0);
    bad.x(1, 2) = std::numeric_limits<float>::quiet_NaN();
    try {
        gpu.stepFrameWithLevels(bad, 0);
        std::printf("expected NumericalError\n");
        return 1;
    } catch (const NumericalError& e) {
        std::printf("NumericalError pass=%s particle=%d: %s\n", e.pass().c_str(), e.particle(), e.what());
        if (e.pass() != "predict" || e.particle() != 2) return 1;
    }
    std::printf("DROPIN OK\n");
    return 0;
}
