// apbf_gpu/solver.hpp -- C++ drop-in for apbf::Solver<Scalar>
// (/root/reference/proj/include/apbf/solver.hpp:208-392) over the C-ABI in
// apbf_gpu.h.  Include it next to the reference headers and replace
//     apbf::Solver<double> solver(cfg, scene);          // runner.cpp:72
// by
//     apbf::gpu::Solver<double> solver(cfg, scene);
// Same constructor, config()/scene(), iterationObserver, stepFrame and
// stepFrameWithLevels; the caller's ParticleSet<Scalar> is uploaded, stepped
// on the B200 in float32 and written back (reordered into the last
// substep's cell order exactly like the reference).  Exceptions:
// std::invalid_argument, std::runtime_error, apbf::NumericalError(pass,
// particle), std::out_of_range -- as thrown by the reference.
// Link with paper_1608_04721_b200/libapbf_gpu.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "apbf/depth_splat.hpp"
#include "apbf/solver.hpp"
#include "apbf_gpu.h"

namespace apbf::gpu {

inline void throwIfError(int32_t rc, const apbf_error& e) {
    switch (rc) {
        case APBF_OK: return;
        case APBF_ERR_INVALID_ARGUMENT: throw std::invalid_argument(e.message);
        case APBF_ERR_NUMERICAL: {
            // NumericalError prefixes its own text; pass back the detail part.
            std::string m = e.message;
            const auto k = m.find(": ");
            throw NumericalError(e.pass, e.particle, k == std::string::npos ? m : m.substr(k + 2));
        }
        case APBF_ERR_OUT_OF_RANGE: throw std::out_of_range(e.message);
        default: throw std::runtime_error(e.message);
    }
}

template <class Scalar>
class Solver {
public:
    Solver(SolverConfig<Scalar> cfg, SdfScene<Scalar> scene, int device = 0)
        : cfg_(std::move(cfg)), scene_(std::move(scene)) {
        cfg_.validate();  // the reference validates in double/float first
        apbf_solver_config c{};
        c.dt_frame = float(cfg_.dtFrame);
        c.substeps = cfg_.substeps;
        c.n_min = cfg_.range.nMin;
        c.n_max = cfg_.range.nMax;
        c.rest_density = float(cfg_.restDensity);
        c.h = float(cfg_.h);
        c.epsilon = float(cfg_.epsilon);
        for (int a = 0; a < 3; ++a) c.gravity[a] = float(cfg_.gravity[a]);
        c.stab_iterations = cfg_.stabIterations;
        c.stab_threshold = cfg_.stabThreshold;
        c.particle_radius = float(cfg_.particleRadius);
        c.mode = cfg_.mode == SolverMode::Pbf ? APBF_MODE_PBF : APBF_MODE_APBF;
        c.velocity_cap = float(cfg_.velocityCap);
        c.inactive_lambda_zero = cfg_.inactiveLambdaZero;
        c.deterministic = cfg_.deterministic;
        c.record_residuals = cfg_.recordResiduals;
        std::vector<apbf_sdf_primitive> prims;
        for (const auto& prim : scene_.primitives) {
            apbf_sdf_primitive p{};
            std::visit(
                [&](const auto& g) {
                    using T = std::decay_t<decltype(g)>;
                    if constexpr (std::is_same_v<T, HalfSpace<Scalar>>) {
                        p.kind = APBF_SDF_HALF_SPACE;
                        for (int a = 0; a < 3; ++a) p.p[a] = float(g.normal[a]);
                        p.a = float(g.offset);
                    } else if constexpr (std::is_same_v<T, Sphere<Scalar>>) {
                        p.kind = APBF_SDF_SPHERE;
                        for (int a = 0; a < 3; ++a) p.p[a] = float(g.center[a]);
                        p.a = float(g.radius);
                        p.interior = g.interior;
                    } else if constexpr (std::is_same_v<T, Box<Scalar>>) {
                        p.kind = APBF_SDF_BOX;
                        for (int a = 0; a < 3; ++a) {
                            p.p[a] = float(g.center[a]);
                            p.q[a] = float(g.halfExtents[a]);
                        }
                        p.interior = g.interior;
                    } else {
                        p.kind = APBF_SDF_CONE;
                        for (int a = 0; a < 3; ++a) p.p[a] = float(g.baseCenter[a]);
                        p.a = float(g.baseRadius);
                        p.b = float(g.height);
                    }
                },
                prim);
            prims.push_back(p);
        }
        apbf_error e{};
        const int32_t rc = apbf_gpu_solver_create(&c, prims.data(), int32_t(prims.size()),
                                                  float(scene_.gradientStep), device, &h_, &e);
        throwIfError(rc, e);
    }
    Solver(const Solver&) = delete;
    Solver& operator=(const Solver&) = delete;
    ~Solver() { apbf_gpu_solver_destroy(h_); }

    const SolverConfig<Scalar>& config() const { return cfg_; }
    const SdfScene<Scalar>& scene() const { return scene_; }

    // The fast build of the lambda / delta-p pair arithmetic (apbf_gpu_set_fast_math):
    // outside the bitwise contract, within the tier-B tolerance of Solver<double>.
    void setFastMath(bool on) { apbf_gpu_set_fast_math(h_, on ? 1 : 0); }

    // Called after every iteration's position application with the substep
    // index, the 1-based iteration and the current state (solver.hpp:222-224).
    std::function<void(int, int, const ParticleSet<Scalar>&)> iterationObserver;

    // stepFrame(ParticleSet&) through apbf_gpu_step_frame_host, the
    // reference-facing call bench.py's e2e measures: only the frame's inputs
    // (x, v, mass, invMass) go up, from page-locked float staging; the whole
    // reordered state comes back with the download overlapping the frame's
    // end.  A failing frame leaves the caller's ParticleSet untouched.  With
    // an iterationObserver the frame runs through the resident path (the
    // observer needs the state downloaded mid-frame).
    FrameStats stepFrame(ParticleSet<Scalar>& state, const Camera<Scalar>& cam,
                         const LodModelConfig<Scalar>& lodCfg, int frameIndex) {
        const apbf_camera c = toC(cam);
        const apbf_lod_config l = toC(lodCfg);
        if (iterationObserver) {
            upload(state);
            return run(state, [&](apbf_frame_stats* st, apbf_error* e) {
                return apbf_gpu_step_frame(h_, &c, &l, frameIndex, st, e);
            });
        }
        const int n = state.count();
        Pinned& b = pinned(n);
        const Scalar* x = state.x.data();
        const Scalar* v = state.v.data();
#pragma omp parallel for schedule(static)
        for (long long k = 0; k < 3LL * n; ++k) {  // Mat3X is column-major: xyz per particle
            b.x[k] = float(x[k]);
            b.v[k] = float(v[k]);
        }
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) {
            b.m[i] = float(state.mass[i]);
            b.w[i] = float(state.invMass[i]);
            b.xs[3LL * i] = b.xs[3LL * i + 1] = b.xs[3LL * i + 2] = 0.0f;  // not read by stepFrame
            b.l[i] = 0.0f;
            b.lv[i] = cfg_.range.nMax;
        }
        std::vector<double> res(size_t(cfg_.substeps) * size_t(cfg_.range.nMax) + 1);
        apbf_frame_stats st{};
        st.residuals = res.data();
        st.residuals_capacity = int32_t(res.size());
        apbf_error e{};
        throwIfError(apbf_gpu_step_frame_host(h_, n, b.x, b.xs, b.v, b.m, b.w, b.l, b.lv, &c, &l, frameIndex,
                                              &st, &e),
                     e);
        Scalar* ox = state.x.data();
        Scalar* oxs = state.xStar.data();
        Scalar* ov = state.v.data();
#pragma omp parallel for schedule(static)
        for (long long k = 0; k < 3LL * n; ++k) {
            ox[k] = Scalar(b.x[k]);
            oxs[k] = Scalar(b.xs[k]);
            ov[k] = Scalar(b.v[k]);
        }
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) {
            state.mass[i] = Scalar(b.m[i]);
            state.invMass[i] = Scalar(b.w[i]);
            state.lambda[i] = Scalar(b.l[i]);
            state.level[i] = b.lv[i];
        }
        return toStats(st, res);
    }

    // ---- device-resident use (the harness drop-in, apbf_gpu/runner.hpp) ----
    // setState uploads once; stepFrameResident steps the resident state with
    // stepFrame's semantics; getState downloads it (storage order).
    void setState(const ParticleSet<Scalar>& state) { upload(state); }
    void getState(ParticleSet<Scalar>& state) { download(state); }
    FrameStats stepFrameResident(const Camera<Scalar>& cam, const LodModelConfig<Scalar>& lodCfg,
                                 int frameIndex) {
        const apbf_camera c = toC(cam);
        const apbf_lod_config l = toC(lodCfg);
        std::vector<double> res(size_t(cfg_.substeps) * size_t(cfg_.range.nMax) + 1);
        apbf_frame_stats st{};
        st.residuals = res.data();
        st.residuals_capacity = int32_t(res.size());
        apbf_error e{};
        throwIfError(apbf_gpu_step_frame(h_, &c, &l, frameIndex, &st, &e), e);
        return toStats(st, res);
    }
    // renderLevelImage (depth_splat.hpp:314-350) of the resident state, on
    // the device (float32 positions, like the solver's).
    ImageRgb renderLevelImage(const Camera<Scalar>& cam, Scalar r, const IterationRange& range) {
        const apbf_camera c = toC(cam);
        ImageRgb img(cam.width, cam.height);
        apbf_error e{};
        throwIfError(apbf_gpu_render_levels(h_, &c, float(r), range.nMin, range.nMax, img.rgb.data(), &e), e);
        return img;
    }

    FrameStats stepFrameWithLevels(ParticleSet<Scalar>& state, int frameIndex) {
        for (int i = 0; i < state.count(); ++i) {
            if (!cfg_.range.contains(state.level[i])) {
                throw std::invalid_argument("particle level outside configured iteration range");
            }
        }
        upload(state);
        return run(state, [&](apbf_frame_stats* st, apbf_error* e) {
            return apbf_gpu_step_frame_with_levels(h_, frameIndex, st, e);
        });
    }

private:
    static apbf_camera toC(const Camera<Scalar>& cam) {
        apbf_camera c{};
        for (int a = 0; a < 3; ++a) {
            c.eye[a] = float(cam.eye[a]);
            c.look_at[a] = float(cam.lookAt[a]);
            c.up[a] = float(cam.up[a]);
        }
        c.vertical_fov = float(cam.verticalFov);
        c.width = cam.width;
        c.height = cam.height;
        c.near_clip = float(cam.nearClip);
        return c;
    }
    static apbf_lod_config toC(const LodModelConfig<Scalar>& lodCfg) {
        apbf_lod_config l{};
        l.model = lodCfg.model == LodModel::Dtc ? APBF_LOD_DTC : APBF_LOD_DTVS;
        l.d_min = float(lodCfg.dMin);
        l.d_max = float(lodCfg.dMax);
        l.n_min = lodCfg.range.nMin;
        l.n_max = lodCfg.range.nMax;
        l.auto_range = lodCfg.autoRange;
        return l;
    }
    static FrameStats toStats(const apbf_frame_stats& st, const std::vector<double>& res) {
        FrameStats out;
        out.frame = st.frame;
        out.wallMs = st.wall_ms;
        out.avgDensityPct = st.avg_density_pct;
        out.minDensityPct = st.min_density_pct;
        out.maxDensityPct = st.max_density_pct;
        out.totalIterations = st.total_iterations;
        out.contacts = st.contacts;
        out.residuals.assign(res.begin(),
                             res.begin() + std::min<int32_t>(st.n_residuals, int32_t(res.size())));
        return out;
    }

    static void trampoline(void* user, int32_t substep, int32_t iter) {
        auto* self = static_cast<Solver*>(user);
        self->download(*self->observed_);
        self->iterationObserver(substep, iter, *self->observed_);
    }

    template <class F>
    FrameStats run(ParticleSet<Scalar>& state, F&& step) {
        observed_ = &state;
        apbf_gpu_set_iteration_observer(h_, iterationObserver ? &Solver::trampoline : nullptr, this);
        std::vector<double> res(size_t(cfg_.substeps) * size_t(cfg_.range.nMax) + 1);
        apbf_frame_stats st{};
        st.residuals = res.data();
        st.residuals_capacity = int32_t(res.size());
        apbf_error e{};
        const int32_t rc = step(&st, &e);
        download(state);
        throwIfError(rc, e);
        return toStats(st, res);
    }

    void upload(const ParticleSet<Scalar>& s) {
        const int n = s.count();
        auto cvt3 = [&](const Mat3X<Scalar>& m, std::vector<float>& o) {
            o.resize(size_t(3) * n);
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < 3; ++a) o[size_t(3) * i + a] = float(m(a, i));
        };
        auto cvt1 = [&](const VecX<Scalar>& v, std::vector<float>& o) {
            o.resize(size_t(n));
            for (int i = 0; i < n; ++i) o[size_t(i)] = float(v[i]);
        };
        cvt3(s.x, x_);
        cvt3(s.xStar, xs_);
        cvt3(s.v, v_);
        cvt1(s.mass, m_);
        cvt1(s.invMass, w_);
        cvt1(s.lambda, l_);
        lv_.resize(size_t(n));
        for (int i = 0; i < n; ++i) lv_[size_t(i)] = s.level[i];
        apbf_error e{};
        throwIfError(apbf_gpu_set_state(h_, n, x_.data(), xs_.data(), v_.data(), m_.data(), w_.data(),
                                        l_.data(), lv_.data(), &e),
                     e);
    }

    void download(ParticleSet<Scalar>& s) {
        const int n = apbf_gpu_particle_count(h_);
        x_.resize(size_t(3) * n);
        xs_.resize(size_t(3) * n);
        v_.resize(size_t(3) * n);
        m_.resize(size_t(n));
        w_.resize(size_t(n));
        l_.resize(size_t(n));
        lv_.resize(size_t(n));
        apbf_error e{};
        throwIfError(apbf_gpu_get_state(h_, x_.data(), xs_.data(), v_.data(), m_.data(), w_.data(),
                                        l_.data(), lv_.data(), &e),
                     e);
        s.x.resize(3, n);
        s.xStar.resize(3, n);
        s.v.resize(3, n);
        s.mass.resize(n);
        s.invMass.resize(n);
        s.lambda.resize(n);
        s.level.resize(n);
        for (int i = 0; i < n; ++i) {
            for (int a = 0; a < 3; ++a) {
                s.x(a, i) = Scalar(x_[size_t(3) * i + a]);
                s.xStar(a, i) = Scalar(xs_[size_t(3) * i + a]);
                s.v(a, i) = Scalar(v_[size_t(3) * i + a]);
            }
            s.mass[i] = Scalar(m_[size_t(i)]);
            s.invMass[i] = Scalar(w_[size_t(i)]);
            s.lambda[i] = Scalar(l_[size_t(i)]);
            s.level[i] = lv_[size_t(i)];
        }
    }

    // page-locked float staging of stepFrame (apbf_gpu_host_alloc)
    struct Pinned {
        int cap = -1;
        float *x = nullptr, *xs = nullptr, *v = nullptr, *m = nullptr, *w = nullptr, *l = nullptr;
        int32_t* lv = nullptr;
        void release() {
            for (void* p : {(void*)x, (void*)xs, (void*)v, (void*)m, (void*)w, (void*)l, (void*)lv})
                apbf_gpu_host_free(p);
            x = xs = v = m = w = l = nullptr;
            lv = nullptr;
            cap = -1;
        }
        ~Pinned() { release(); }
    };
    Pinned pin_;
    Pinned& pinned(int n) {
        if (pin_.cap < n) {
            pin_.release();
            const size_t c = size_t(std::max(n, 1));
            auto a = [](size_t bytes) {
                void* p = apbf_gpu_host_alloc(bytes);
                if (!p) throw std::runtime_error("page-locked host allocation failed");
                return p;
            };
            pin_.x = static_cast<float*>(a(12 * c));
            pin_.xs = static_cast<float*>(a(12 * c));
            pin_.v = static_cast<float*>(a(12 * c));
            pin_.m = static_cast<float*>(a(4 * c));
            pin_.w = static_cast<float*>(a(4 * c));
            pin_.l = static_cast<float*>(a(4 * c));
            pin_.lv = static_cast<int32_t*>(a(4 * c));
            pin_.cap = n;
        }
        return pin_;
    }

    SolverConfig<Scalar> cfg_;
    SdfScene<Scalar> scene_;
    apbf_gpu_solver* h_ = nullptr;
    ParticleSet<Scalar>* observed_ = nullptr;
    std::vector<float> x_, xs_, v_, m_, w_, l_;
    std::vector<int32_t> lv_;
};

}  // namespace apbf::gpu
