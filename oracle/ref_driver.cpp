// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference code
// (/root/reference/proj/include/apbf/*.hpp + src/scenario.cpp), compiled
// against the Eigen-subset shim in oracle/eigen_min by oracle/Makefile into
// oracle/_ref/libapbf_ref.so.  Used (a) in this container to pin the C
// restatement (apbf_oracle.c) and to generate tests/golden/, (b) on the GPU
// box as bench.py's CPU baseline (`--impl reference`), Solver<double> with
// OpenMP over all host cores exactly as the reference ships.
//
// Precision: `prec` 4 = Solver<float>, 8 = Solver<double>.  Array arguments
// are double on the ABI and cast to Scalar inside, so both precisions see the
// same (Scalar)value conversion the float GPU path sees.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "apbf/solver.hpp"
#include "bench.hpp"
#include "metrics.hpp"
#include "runner.hpp"
#include "scenario.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

struct ref_config {
    double dt_frame;
    int32_t substeps, n_min, n_max;
    double rest_density, h, epsilon, gravity[3];
    int32_t stab_iterations, stab_threshold;
    double particle_radius;
    int32_t mode;
    double velocity_cap;
    int32_t inactive_lambda_zero, deterministic, record_residuals;
};
struct ref_prim {
    int32_t kind, interior;
    double p[3], q[3], a, b;
};
struct ref_camera {
    double eye[3], look_at[3], up[3], vertical_fov;
    int32_t width, height;
    double near_clip;
};
struct ref_lod {
    int32_t model;
    double d_min, d_max;
    int32_t n_min, n_max, auto_range;
};
struct ref_stats {
    int32_t frame, n_residuals;
    double wall_ms, avg_density_pct, min_density_pct, max_density_pct;
    int64_t total_iterations, contacts;
    double residuals[256];
};
struct ref_error {
    int32_t code, particle;
    char pass[32];
    char message[224];
};

}  // extern "C"

namespace {

using namespace apbf;

void fill_error(ref_error* e, int code, const std::string& pass, int particle, const char* what) {
    if (!e) return;
    e->code = code;
    e->particle = particle;
    std::snprintf(e->pass, sizeof e->pass, "%s", pass.c_str());
    std::snprintf(e->message, sizeof e->message, "%s", what);
}

template <class F>
int32_t guarded(ref_error* e, F&& f) {
    if (e) std::memset(e, 0, sizeof *e);
    try {
        f();
        return 0;
    } catch (const NumericalError& x) {
        fill_error(e, 3, x.pass(), x.particle(), x.what());
        return 3;
    } catch (const std::invalid_argument& x) {
        fill_error(e, 1, "", -1, x.what());
        return 1;
    } catch (const std::out_of_range& x) {
        fill_error(e, 5, "", -1, x.what());
        return 5;
    } catch (const std::runtime_error& x) {
        fill_error(e, 2, "", -1, x.what());
        return 2;
    } catch (const std::exception& x) {
        fill_error(e, 2, "", -1, x.what());
        return 2;
    }
}

template <class S>
SolverConfig<S> to_cfg(const ref_config& c) {
    SolverConfig<S> o;
    o.dtFrame = S(c.dt_frame);
    o.substeps = c.substeps;
    o.range = IterationRange(c.n_min, c.n_max);
    o.restDensity = S(c.rest_density);
    o.h = S(c.h);
    o.epsilon = S(c.epsilon);
    o.gravity = Vec3<S>(S(c.gravity[0]), S(c.gravity[1]), S(c.gravity[2]));
    o.stabIterations = c.stab_iterations;
    o.stabThreshold = c.stab_threshold;
    o.particleRadius = S(c.particle_radius);
    o.mode = c.mode == 0 ? SolverMode::Pbf : SolverMode::Apbf;
    o.velocityCap = S(c.velocity_cap);
    o.inactiveLambdaZero = c.inactive_lambda_zero != 0;
    o.deterministic = c.deterministic != 0;
    o.recordResiduals = c.record_residuals != 0;
    return o;
}

template <class S>
Vec3<S> v3(const double* p) {
    return Vec3<S>(S(p[0]), S(p[1]), S(p[2]));
}

template <class S>
SdfScene<S> to_scene(const ref_prim* prims, int n, double step) {
    SdfScene<S> sc;
    sc.gradientStep = S(step);
    for (int k = 0; k < n; ++k) {
        const ref_prim& p = prims[k];
        switch (p.kind) {
            case 0: sc.primitives.emplace_back(HalfSpace<S>(v3<S>(p.p), S(p.a))); break;
            case 1: sc.primitives.emplace_back(Sphere<S>(v3<S>(p.p), S(p.a), p.interior != 0)); break;
            case 2: sc.primitives.emplace_back(Box<S>(v3<S>(p.p), v3<S>(p.q), p.interior != 0)); break;
            default: sc.primitives.emplace_back(Cone<S>(v3<S>(p.p), S(p.a), S(p.b))); break;
        }
    }
    return sc;
}

template <class S>
Camera<S> to_cam(const ref_camera& c) {
    Camera<S> o;
    o.eye = v3<S>(c.eye);
    o.lookAt = v3<S>(c.look_at);
    o.up = v3<S>(c.up);
    o.verticalFov = S(c.vertical_fov);
    o.width = c.width;
    o.height = c.height;
    o.nearClip = S(c.near_clip);
    return o;
}

template <class S>
LodModelConfig<S> to_lod(const ref_lod& l) {
    LodModelConfig<S> o;
    o.model = l.model == 0 ? LodModel::Dtc : LodModel::Dtvs;
    o.dMin = S(l.d_min);
    o.dMax = S(l.d_max);
    o.range = IterationRange(l.n_min, l.n_max);
    o.autoRange = l.auto_range != 0;
    return o;
}

template <class S>
Mat3X<S> to_mat3(int n, const double* p) {
    Mat3X<S> m(3, n);
    for (int i = 0; i < 3 * n; ++i) m.data()[i] = S(p[i]);
    return m;
}

template <class S>
void from_mat3(const Mat3X<S>& m, double* p) {
    if (!p) return;
    for (Eigen::Index i = 0; i < m.size(); ++i) p[i] = double(m.data()[i]);
}

void fill_stats(const FrameStats& st, ref_stats* out) {
    out->frame = st.frame;
    out->wall_ms = st.wallMs;
    out->avg_density_pct = st.avgDensityPct;
    out->min_density_pct = st.minDensityPct;
    out->max_density_pct = st.maxDensityPct;
    out->total_iterations = st.totalIterations;
    out->contacts = st.contacts;
    out->n_residuals = int32_t(st.residuals.size());
    for (size_t k = 0; k < st.residuals.size() && k < 256; ++k) out->residuals[k] = st.residuals[k];
}

struct Handle {
    int prec;
    std::unique_ptr<Solver<float>> sf;
    std::unique_ptr<Solver<double>> sd;
    ParticleSet<float> pf;
    ParticleSet<double> pd;
};

template <class S>
ParticleSet<S> make_set(int n, const double* x, const double* xs, const double* v, const double* m,
                        const double* w, const double* lam, const int32_t* lvl) {
    ParticleSet<S> p;
    p.x = to_mat3<S>(n, x);
    p.xStar = to_mat3<S>(n, xs);
    p.v = to_mat3<S>(n, v);
    p.mass.resize(n);
    p.invMass.resize(n);
    p.lambda.resize(n);
    p.level.resize(n);
    for (int i = 0; i < n; ++i) {
        p.mass[i] = S(m[i]);
        p.invMass[i] = S(w[i]);
        p.lambda[i] = S(lam[i]);
        p.level[i] = lvl[i];
    }
    return p;
}

template <class S>
void read_set(const ParticleSet<S>& p, double* x, double* xs, double* v, double* m, double* w,
              double* lam, int32_t* lvl) {
    from_mat3(p.x, x);
    from_mat3(p.xStar, xs);
    from_mat3(p.v, v);
    for (int i = 0; i < p.count(); ++i) {
        if (m) m[i] = double(p.mass[i]);
        if (w) w[i] = double(p.invMass[i]);
        if (lam) lam[i] = double(p.lambda[i]);
        if (lvl) lvl[i] = p.level[i];
    }
}

}  // namespace

extern "C" {

int32_t ref_omp_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void* ref_solver_create(int32_t prec, const ref_config* cfg, const ref_prim* prims, int32_t n_prims,
                        double grad_step, ref_error* err) {
    Handle* h = nullptr;
    guarded(err, [&] {
        auto hh = std::make_unique<Handle>();
        hh->prec = prec;
        if (prec == 4)
            hh->sf = std::make_unique<Solver<float>>(to_cfg<float>(*cfg),
                                                     to_scene<float>(prims, n_prims, grad_step));
        else
            hh->sd = std::make_unique<Solver<double>>(to_cfg<double>(*cfg),
                                                      to_scene<double>(prims, n_prims, grad_step));
        h = hh.release();
    });
    return h;
}

void ref_solver_destroy(void* h) { delete static_cast<Handle*>(h); }

int32_t ref_set_state(void* hv, int32_t n, const double* x, const double* xs, const double* v,
                      const double* m, const double* w, const double* lam, const int32_t* lvl) {
    Handle* h = static_cast<Handle*>(hv);
    if (h->prec == 4) h->pf = make_set<float>(n, x, xs, v, m, w, lam, lvl);
    else h->pd = make_set<double>(n, x, xs, v, m, w, lam, lvl);
    return 0;
}

int32_t ref_get_state(void* hv, double* x, double* xs, double* v, double* m, double* w, double* lam,
                      int32_t* lvl) {
    Handle* h = static_cast<Handle*>(hv);
    if (h->prec == 4) read_set(h->pf, x, xs, v, m, w, lam, lvl);
    else read_set(h->pd, x, xs, v, m, w, lam, lvl);
    return 0;
}

int32_t ref_step_frame(void* hv, const ref_camera* cam, const ref_lod* lod, int32_t frame,
                       ref_stats* out, ref_error* err) {
    Handle* h = static_cast<Handle*>(hv);
    return guarded(err, [&] {
        if (h->prec == 4) fill_stats(h->sf->stepFrame(h->pf, to_cam<float>(*cam), to_lod<float>(*lod), frame), out);
        else fill_stats(h->sd->stepFrame(h->pd, to_cam<double>(*cam), to_lod<double>(*lod), frame), out);
    });
}

int32_t ref_step_frame_with_levels(void* hv, int32_t frame, ref_stats* out, ref_error* err) {
    Handle* h = static_cast<Handle*>(hv);
    return guarded(err, [&] {
        if (h->prec == 4) fill_stats(h->sf->stepFrameWithLevels(h->pf, frame), out);
        else fill_stats(h->sd->stepFrameWithLevels(h->pd, frame), out);
    });
}

// --- component functions (float or double) ---

int32_t ref_grid_build(int32_t prec, int32_t n, const double* pos, double h, double pad, int32_t* perm,
                       double* origin, int32_t* dims, int32_t* cell_start, int64_t cap,
                       int64_t* cells, ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            UniformGrid<S> g;
            g.build(to_mat3<S>(n, pos), S(h), S(pad));
            for (size_t k = 0; k < g.permutation().size(); ++k) perm[k] = g.permutation()[k];
            for (int a = 0; a < 3; ++a) {
                origin[a] = double(g.origin()[a]);
                dims[a] = g.dims()[a];
            }
            *cells = g.cellCount();
            if (cell_start && cap >= g.cellCount() + 1) {
                // cellStart is private; rebuild it from particlesInCell.
                int64_t acc = 0;
                cell_start[0] = 0;
                for (int64_t c = 0; c < g.cellCount(); ++c) {
                    const int cz = int(c / (int64_t(g.dims()[0]) * g.dims()[1]));
                    const int cy = int((c / g.dims()[0]) % g.dims()[1]);
                    const int cx = int(c % g.dims()[0]);
                    acc += g.particlesInCell(Eigen::Vector3i(cx, cy, cz));
                    cell_start[c + 1] = int32_t(acc);
                }
            }
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

int32_t ref_neighbor_lists(int32_t prec, int32_t n, const double* pos, double h, double pad,
                           int32_t* offsets, int32_t* indices, int64_t cap, int64_t* total,
                           ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            UniformGrid<S> g;
            g.build(to_mat3<S>(n, pos), S(h), S(pad));
            const NeighborLists nl = g.buildNeighborLists();
            *total = int64_t(nl.indices.size());
            if (offsets)
                for (size_t k = 0; k < nl.offsets.size(); ++k) offsets[k] = nl.offsets[k];
            if (indices && cap >= *total)
                for (size_t k = 0; k < nl.indices.size(); ++k) indices[k] = nl.indices[k];
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

int32_t ref_all_densities(int32_t prec, int32_t n, const double* pos, const double* m, double h,
                          double* rho, ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            VecX<S> mm(n);
            for (int i = 0; i < n; ++i) mm[i] = S(m[i]);
            const VecX<S> r = allDensities(to_mat3<S>(n, pos), mm, S(h));
            for (int i = 0; i < n; ++i) rho[i] = double(r[i]);
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

int32_t ref_lod_levels(int32_t prec, int32_t n, const double* pos, const ref_camera* cam, const ref_lod* lod,
                double radius, int32_t* levels, ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            const LodModelConfig<S> lc = to_lod<S>(*lod);
            const VecXi l = lc.model == LodModel::Dtc
                                ? lodDtc(to_mat3<S>(n, pos), to_cam<S>(*cam), lc)
                                : lodDtvs(to_mat3<S>(n, pos), to_cam<S>(*cam), lc, S(radius));
            for (int i = 0; i < n; ++i) levels[i] = l[i];
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

int32_t ref_splat(int32_t prec, int32_t n, const double* pos, double radius, const ref_camera* cam,
                  double* depth, ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            const DepthBuffer<S> b = splat(to_mat3<S>(n, pos), S(radius), to_cam<S>(*cam));
            for (size_t k = 0; k < b.depth.size(); ++k) depth[k] = double(b.depth[k]);
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

int32_t ref_scene_distance(int32_t prec, const ref_prim* prims, int32_t n_prims, double step,
                           const double* p, double* phi, double* grad, ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            const SdfScene<S> sc = to_scene<S>(prims, n_prims, step);
            const SdfSample<S> s = sceneDistance(sc, v3<S>(p));
            *phi = double(s.phi);
            for (int a = 0; a < 3; ++a) grad[a] = double(s.gradient[a]);
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

double ref_density_kernel_r2(int32_t prec, double r2, double h) {
    return prec == 4 ? double(densityKernelR2<float>(float(r2), float(h)))
                     : densityKernelR2<double>(r2, h);
}

void ref_gradient_kernel(int32_t prec, const double* r, double h, double* out) {
    if (prec == 4) {
        const Vec3<float> g = gradientKernel(v3<float>(r), float(h));
        for (int a = 0; a < 3; ++a) out[a] = g[a];
    } else {
        const Vec3<double> g = gradientKernel(v3<double>(r), h);
        for (int a = 0; a < 3; ++a) out[a] = g[a];
    }
}

// --- scenario library (src/scenario.cpp), double as shipped ---

struct ref_scenario {
    int32_t n_particles;
    int32_t n_prims;
    double mass;
    ref_config cfg;
    ref_prim prims[8];
    double grad_step;
    ref_camera cam;
    ref_lod lod;
    int32_t frames;
    uint64_t hash;
};

int32_t ref_build_scenario(const char* name, double scale, uint64_t seed, ref_scenario* out,
                           double* positions /* 3n or NULL */, ref_error* err) {
    return guarded(err, [&] {
        const ScenarioSpec spec = buildScenario(name, scale);
        out->n_particles = spec.particleCount();
        const SolverConfig<double>& s = spec.solver;
        out->cfg = ref_config{s.dtFrame, s.substeps, s.range.nMin, s.range.nMax, s.restDensity, s.h,
                              s.epsilon, {s.gravity[0], s.gravity[1], s.gravity[2]},
                              s.stabIterations, s.stabThreshold, s.particleRadius,
                              s.mode == SolverMode::Pbf ? 0 : 1, s.velocityCap,
                              s.inactiveLambdaZero ? 1 : 0, s.deterministic ? 1 : 0,
                              s.recordResiduals ? 1 : 0};
        out->n_prims = int32_t(spec.scene.primitives.size());
        for (int k = 0; k < out->n_prims && k < 8; ++k) {
            ref_prim& p = out->prims[k];
            std::memset(&p, 0, sizeof p);
            std::visit(
                [&](const auto& g) {
                    using T = std::decay_t<decltype(g)>;
                    if constexpr (std::is_same_v<T, HalfSpace<double>>) {
                        p.kind = 0;
                        for (int a = 0; a < 3; ++a) p.p[a] = g.normal[a];
                        p.a = g.offset;
                    } else if constexpr (std::is_same_v<T, Sphere<double>>) {
                        p.kind = 1;
                        for (int a = 0; a < 3; ++a) p.p[a] = g.center[a];
                        p.a = g.radius;
                        p.interior = g.interior;
                    } else if constexpr (std::is_same_v<T, Box<double>>) {
                        p.kind = 2;
                        for (int a = 0; a < 3; ++a) {
                            p.p[a] = g.center[a];
                            p.q[a] = g.halfExtents[a];
                        }
                        p.interior = g.interior;
                    } else {
                        p.kind = 3;
                        for (int a = 0; a < 3; ++a) p.p[a] = g.baseCenter[a];
                        p.a = g.baseRadius;
                        p.b = g.height;
                    }
                },
                spec.scene.primitives[size_t(k)]);
        }
        out->grad_step = spec.scene.gradientStep;
        const Camera<double>& c = spec.camera;
        out->cam = ref_camera{{c.eye[0], c.eye[1], c.eye[2]}, {c.lookAt[0], c.lookAt[1], c.lookAt[2]},
                              {c.up[0], c.up[1], c.up[2]}, c.verticalFov, c.width, c.height, c.nearClip};
        out->lod = ref_lod{spec.lod.model == LodModel::Dtc ? 0 : 1, spec.lod.dMin, spec.lod.dMax,
                           spec.lod.range.nMin, spec.lod.range.nMax, spec.lod.autoRange ? 1 : 0};
        out->frames = spec.frames;
        out->hash = scenarioHash(spec, seed);
        const ParticleSet<double> st = makeState(spec, seed);
        out->mass = st.mass.size() > 0 ? st.mass[0] : 0.0;
        if (positions) from_mat3(st.x, positions);
    });
}

// renderLevelImage<S> (depth_splat.hpp:314-350) -> width*height*3 bytes.
int32_t ref_render_level_image(int32_t prec, int32_t n, const double* pos, const int32_t* levels,
                               double radius, const ref_camera* cam, int32_t nmin, int32_t nmax,
                               uint8_t* rgb, ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            VecXi lv(n);
            for (int i = 0; i < n; ++i) lv[i] = levels[i];
            const ImageRgb img = renderLevelImage(to_mat3<S>(n, pos), lv, S(radius), to_cam<S>(*cam),
                                                  IterationRange(nmin, nmax));
            std::memcpy(rgb, img.rgb.data(), img.rgb.size());
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

// writeParticleSnapshot<S> (particle_state.hpp:148-167) of n particles.
int32_t ref_write_particle_snapshot(int32_t prec, int32_t n, const double* pos, const int32_t* levels,
                                    const char* path, ref_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using S = decltype(tag);
            ParticleSet<S> st(to_mat3<S>(n, pos), S(1), 1);
            for (int i = 0; i < n; ++i) st.level[i] = levels[i];
            writeParticleSnapshot(std::filesystem::path(path), st);
        };
        if (prec == 4) run(float{});
        else run(double{});
    });
}

// runScenario (runner.cpp:60-98) -- the reference's own harness, Solver<double>.
// lod: -1 keep the scenario's, 0 dtc, 1 dtvs; nmin 0 = keep the range.
int32_t ref_run_scenario(const char* name, double scale, int32_t mode, int32_t lod, int32_t nmin,
                         int32_t nmax, int32_t frames, uint64_t seed, int32_t deterministic,
                         const char* out_dir, int32_t images_every, int32_t particles_every,
                         ref_error* err) {
    return guarded(err, [&] {
        const ScenarioSpec spec = buildScenario(name, scale);
        RunOptions opt;
        opt.mode = mode == 0 ? SolverMode::Pbf : SolverMode::Apbf;
        if (lod >= 0) opt.lodModel = lod == 0 ? LodModel::Dtc : LodModel::Dtvs;
        if (nmin > 0) opt.range = IterationRange(nmin, nmax);
        opt.frames = frames;
        opt.seed = seed;
        opt.deterministic = deterministic != 0;
        opt.outDir = out_dir ? out_dir : "";
        opt.dumpImagesEvery = images_every;
        opt.dumpParticlesEvery = particles_every;
        (void)runScenario(spec, opt);
    });
}

// formatBenchReport (bench.cpp:93-123) of caller-made results.
int32_t ref_format_bench_report(int32_t k, const char* const* tokens, const double* median_ms,
                                const int64_t* iterations, const int32_t* frames,
                                const int32_t* particles, char* out, int32_t cap, ref_error* err) {
    return guarded(err, [&] {
        std::vector<BenchResult> rs(static_cast<size_t>(k));
        for (int i = 0; i < k; ++i) {
            rs[size_t(i)].token = tokens[i];
            rs[size_t(i)].medianFrameMs = median_ms[i];
            rs[size_t(i)].iterations = iterations[i];
            rs[size_t(i)].frames = frames[i];
            rs[size_t(i)].particles = particles[i];
        }
        const std::string s = formatBenchReport(rs);
        std::snprintf(out, size_t(cap), "%s", s.c_str());
    });
}

// parseBenchMode (bench.cpp:9-42): 0 ok (mode, iterations, lod -1/0/1), or
// the invalid_argument message in err.
int32_t ref_parse_bench_mode(const char* token, int32_t* mode, int32_t* iters, int32_t* lod,
                             ref_error* err) {
    return guarded(err, [&] {
        const BenchMode m = parseBenchMode(token);
        *mode = m.mode == SolverMode::Pbf ? 0 : 1;
        *iters = m.pbfIterations;
        *lod = m.lodModel ? (*m.lodModel == LodModel::Dtc ? 0 : 1) : -1;
    });
}

uint64_t ref_splitmix64_first(uint64_t seed) {
    SplitMix64 r(seed);
    return r.next();
}

}  // extern "C"
