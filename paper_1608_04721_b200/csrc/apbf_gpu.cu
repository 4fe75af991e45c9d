// apbf_gpu.cu -- host side of the B200 APBF step behind the C-ABI in
// include/apbf_gpu.h.  One solver handle = one device, one stream, device-
// resident ParticleSet.  See DESIGN.md for the pipeline and data layout.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>
#include <array>

#include "apbf_post.cuh"
#include "apbf_dist.cuh"
#include "apbf_transport.h"

// CTA size of the passes that fold an AABB into the control block (predict,
// aabb): one block-reduced atomic per coordinate bound per CTA, so large
// CTAs (predict 28 -> 18 us, aabb 18 -> 11 us per 1M-particle launch, ncu)
static constexpr int kAabbBlock = 1024;

#include <memory>
#include <functional>

#include <nvtx3/nvToolsExt.h>

// NVTX ranges around the host-side phases (frames, slab substeps), for
// Nsight Systems timelines.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#include <thread>

using namespace apbf_gpu;

namespace {

// ------------------------------------------------------------- errors

struct ApiError {
    int code;
    std::string pass;
    int particle;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw ApiError{code, "", -1, msg}; }

[[noreturn]] void numerical(const std::string& pass, int particle, const std::string& detail) {
    throw ApiError{APBF_ERR_NUMERICAL, pass, particle,
                   "numerical abort in pass '" + pass + "' at particle " + std::to_string(particle) +
                       ": " + detail};
}

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess)                                                                \
            throw ApiError{APBF_ERR_CUDA, "", -1,                                             \
                           std::string(#x) + ": " + cudaGetErrorString(e_) + " at " +         \
                               __FILE__ + ":" + std::to_string(__LINE__)};                    \
    } while (0)

#define LAUNCH_CHECK() CK(cudaGetLastError())

// Counts every kernel this library launches (bench.py reports it).
static unsigned long long g_launches = 0;
#define KL(...)          \
    do {                 \
        __VA_ARGS__;     \
        ++g_launches;    \
    } while (0)

// A kernel launched with programmatic stream serialization (it starts with
// pdl_wait(), apbf_device.cuh): its launch may overlap the predecessor's tail
// in the stream (also inside a captured graph, as a programmatic edge).  Only
// kernels whose first statement is pdl_wait() may be launched this way.
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(block);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, k, static_cast<KArgs>(args)...));
    ++g_launches;
}

int32_t to_err(const ApiError& e, apbf_error* out) {
    if (out) {
        out->code = e.code;
        out->particle = e.particle;
        std::snprintf(out->pass, sizeof out->pass, "%s", e.pass.c_str());
        std::snprintf(out->message, sizeof out->message, "%s", e.msg.c_str());
    }
    return e.code;
}

template <class F>
int32_t guarded(apbf_error* err, F&& f) {
    if (err) std::memset(err, 0, sizeof *err);
    try {
        f();
        return APBF_OK;
    } catch (const ApiError& e) {
        return to_err(e, err);
    } catch (const std::bad_alloc&) {
        return to_err(ApiError{APBF_ERR_RUNTIME, "", -1, "host allocation failed"}, err);
    } catch (const std::exception& e) {
        return to_err(ApiError{APBF_ERR_RUNTIME, "", -1, e.what()}, err);
    }
}

inline int blocks(long long n, int t) { return (int)std::max<long long>(1, (n + t - 1) / t); }

// ------------------------------------------------------------- buffers

// Bumped by every device (re)allocation: a captured frame graph holds raw
// pointers, so it is re-recorded only when this changes.
static unsigned long long g_alloc_gen = 0;
// Set while a slab-frame segment is being recorded into a CUDA graph: a
// device allocation there would synchronise the capturing thread (the slab
// path preallocates every buffer its segments use, set_state_local).
static thread_local bool g_segment_capture = false;

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void ensure(size_t m) {
        if (m <= n && p) return;
        if (g_segment_capture)
            throw ApiError{APBF_ERR_RUNTIME, "", -1, "internal: device allocation during slab graph capture"};
        release();
        const size_t bytes = sizeof(T) * std::max<size_t>(m, 1) + kBufSlack;
        CK(cudaMalloc(&p, bytes));
        // zeroed once: the scans' read-ahead past a run or list end (tail
        // slack, kListPad rows) then reads defined, unused values
        // (compute-sanitizer --tool initcheck stays clean)
        CK(cudaMemsetAsync(p, 0, bytes, 0));
        CK(cudaStreamSynchronize(0));
        n = std::max<size_t>(m, 1);
        ++g_alloc_gen;
    }
};

struct SetBufs {
    DBuf<float4> X, V, XS;
    DBuf<float> W, L;
    DBuf<int> LV;
    void ensure(size_t n) {
        X.ensure(n);
        V.ensure(n);
        XS.ensure(n);
        W.ensure(n);
        L.ensure(n);
        LV.ensure(n);
    }
    StateSet view() { return StateSet{X.p, V.p, XS.p, W.p, L.p, LV.p}; }
};

// Device scratch shared by the solver and the component entry points.
struct Workspace {
    int device = 0;
    cudaStream_t stream = nullptr;
    DBuf<Ctl> ctl;
    Ctl* h_ctl = nullptr;  // pinned mirror
    DBuf<int> cellCount;   // kMaxCells + 1 (cellStart after the scan)
    DBuf<int> partial;
    DBuf<int> key, slot, bucket, perm;
    DBuf<int> heavy;  // cells with > kRankDirect members (k_heavy_sort)
    DBuf<Scene> scene;
    DBuf<RadixSel> rs;
    DBuf<int> depth;
    DBuf<float4> rays;  // per-pixel ray direction + |d|^2 (k_splat_prep)
    DBuf<float> raysa;  // per-pixel sqrt(|d|^2)
    DBuf<float> dist;
    DBuf<unsigned> keys;
    DBuf<float4> tmp4;
    DBuf<unsigned long long> owner;  // renderLevelImage: (depth bits, index) per pixel
    DBuf<unsigned char> rgb;
    DBuf<int> tmpi;

    explicit Workspace(int dev) : device(dev) {
        CK(cudaSetDevice(dev));
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        ctl.ensure(1);
        CK(cudaMallocHost(&h_ctl, sizeof(Ctl)));
        partial.ensure(kScanGrid);
        scene.ensure(1);
        rs.ensure(1);
    }
    ~Workspace() {
        if (h_ctl) cudaFreeHost(h_ctl);
        if (stream) cudaStreamDestroy(stream);
    }
    void ensure_particles(size_t n) {
        key.ensure(n);
        slot.ensure(n);
        bucket.ensure(n);
        perm.ensure(n);
        heavy.ensure(n / (kRankDirect + 1) + 1);
    }
    void ensure_cells() { cellCount.ensure((size_t)kMaxCells + 1); }

    // UniformGrid::build on float4 positions P (AABB already in grid g):
    // params, histogram, scan, stable counting sort -> perm, cellStart.
    // ownLo/ownHi (slab mode, device pointers): contacts of the owned layers
    // only; params = false when the caller already ran k_grid_params for g.
    void run_grid(int g, const float4* P, int n, float h, float pad, bool contacts, float radius,
                  const int* ownLo = nullptr, const int* ownHi = nullptr, bool params = true,
                  SelfMap self = SelfMap{}) {
        ensure_cells();
        ensure_particles(n);
        if (params) launch_pdl(k_grid_params, (unsigned)(1), 1, 0, stream, ctl.p, g, h, pad);
        launch_pdl(k_zero_cells, (unsigned)(4 * 148), 256, 0, stream, ctl.p, g, cellCount.p);
        launch_pdl(k_cell_keys, (unsigned)(blocks(n, 256)), 256, 0, stream, n, P, ctl.p, g, h, cellCount.p, key.p, slot.p,
                                                        scene.p, radius, contacts ? 1 : 0, ownLo, ownHi, self);
        launch_pdl(k_scan_reduce, (unsigned)(kScanGrid), kScanBlock, 0, stream, ctl.p, g, cellCount.p, partial.p);
        launch_pdl(k_scan_partials, (unsigned)(1), kScanBlock, 0, stream, ctl.p, partial.p, kScanGrid);
        launch_pdl(k_scan_apply, (unsigned)(kScanGrid), kScanBlock, 0, stream, ctl.p, g, cellCount.p, partial.p);
        launch_pdl(k_bucket_fill, (unsigned)(blocks(n, 256)), 256, 0, stream, n, ctl.p, key.p, slot.p, cellCount.p,
                                                          bucket.p);
        launch_pdl(k_stable_rank, (unsigned)(blocks(n, 256)), 256, 0, stream, n, ctl.p, key.p, slot.p, cellCount.p, bucket.p,
                                                          perm.p, heavy.p);
        launch_pdl(k_heavy_sort, (unsigned)(148), kHeavyThreads, 0, stream, n, ctl.p, heavy.p, cellCount.p, bucket.p, perm.p);
        LAUNCH_CHECK();
    }

    void read_ctl() {
        CK(cudaMemcpyAsync(h_ctl, ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
    }
};

// ------------------------------------------------------- host helpers

bool finite3h(const float* p) { return std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2]); }

// SdfScene from the C-ABI primitives, with the reference constructors'
// validation and the half-space normalisation in float (sdf.hpp:23-73).
Scene make_scene(const apbf_sdf_primitive* prims, int n, float step) {
    if (n < 0) fail(APBF_ERR_INVALID_ARGUMENT, "negative primitive count");
    if (n > kMaxPrims) fail(APBF_ERR_INVALID_ARGUMENT, "too many SDF primitives for the GPU scene");
    Scene sc;
    std::memset(&sc, 0, sizeof sc);
    sc.n = n;
    sc.step = step;
    for (int k = 0; k < n; ++k) {
        apbf_sdf_primitive p = prims[k];
        switch (p.kind) {
            case APBF_SDF_HALF_SPACE: {
                const float len = std::sqrt(sqn3(p.p[0], p.p[1], p.p[2]));
                if (!(len > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "half-space normal must be nonzero");
                p.p[0] /= len;
                p.p[1] /= len;
                p.p[2] /= len;
                break;
            }
            case APBF_SDF_SPHERE:
                if (!(p.a > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "sphere radius must be positive");
                break;
            case APBF_SDF_BOX:
                if (!(min_std(p.q[0], min_std(p.q[1], p.q[2])) > 0.0f))
                    fail(APBF_ERR_INVALID_ARGUMENT, "box half extents must be positive");
                break;
            case APBF_SDF_CONE:
                if (!(p.a > 0.0f) || !(p.b > 0.0f))
                    fail(APBF_ERR_INVALID_ARGUMENT, "cone radius and height must be positive");
                break;
            default:
                fail(APBF_ERR_INVALID_ARGUMENT, "unknown primitive kind");
        }
        sc.prim[k] = p;
    }
    return sc;
}

// CameraFrame (depth_splat.hpp:29-71) on the host, in float.
CamFrame make_frame(const apbf_camera& cam) {
    if (cam.width <= 0 || cam.height <= 0)
        fail(APBF_ERR_INVALID_ARGUMENT, "camera resolution must be positive in both axes");
    float d[3] = {cam.look_at[0] - cam.eye[0], cam.look_at[1] - cam.eye[1], cam.look_at[2] - cam.eye[2]};
    if (!(sqn3(d[0], d[1], d[2]) > 0.0f))
        fail(APBF_ERR_INVALID_ARGUMENT, "camera look-at must differ from eye");
    if (!(cam.vertical_fov > 0.0f) || !(cam.vertical_fov < kPi))
        fail(APBF_ERR_INVALID_ARGUMENT, "vertical fov must lie in (0, pi)");
    if (!(cam.near_clip > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "near clip must be positive");
    CamFrame f;
    const float z = sqn3(d[0], d[1], d[2]);
    if (z > 0.0f) {
        const float s = std::sqrt(z);
        d[0] /= s;
        d[1] /= s;
        d[2] /= s;
    }
    for (int a = 0; a < 3; ++a) {
        f.eye[a] = cam.eye[a];
        f.forward[a] = d[a];
    }
    const float* u = cam.up;
    f.right[0] = f.forward[1] * u[2] - f.forward[2] * u[1];
    f.right[1] = f.forward[2] * u[0] - f.forward[0] * u[2];
    f.right[2] = f.forward[0] * u[1] - f.forward[1] * u[0];
    const float len = std::sqrt(sqn3(f.right[0], f.right[1], f.right[2]));
    if (!(len > 1e-12f)) fail(APBF_ERR_INVALID_ARGUMENT, "camera up is parallel to the view direction");
    for (int a = 0; a < 3; ++a) f.right[a] /= len;
    f.trueUp[0] = f.right[1] * f.forward[2] - f.right[2] * f.forward[1];
    f.trueUp[1] = f.right[2] * f.forward[0] - f.right[0] * f.forward[2];
    f.trueUp[2] = f.right[0] * f.forward[1] - f.right[1] * f.forward[0];
    f.tanY = std::tan(cam.vertical_fov / 2.0f);
    f.tanX = f.tanY * (float)cam.width / (float)cam.height;
    f.width = cam.width;
    f.height = cam.height;
    f.nearClip = cam.near_clip;
    return f;
}

void validate_lod(const apbf_lod_config& l) {
    if (!l.auto_range && !(l.d_min < l.d_max))
        fail(APBF_ERR_INVALID_ARGUMENT, "lod distance range requires d_min < d_max");
}

// LOD on device for positions X (float4): levels into LV.
// lodDtc (lod.hpp:83-104) / lodDtvs (lod.hpp:109-156).
void run_lod(Workspace& ws, const float4* X, int n, const apbf_camera& cam, const apbf_lod_config& lod,
             float radius, int* LV, cudaStream_t on = nullptr) {
    cudaStream_t st = on ? on : ws.stream;
    ws.dist.ensure(n);
    ws.keys.ensure(n);
    const bool dtvs = lod.model == APBF_LOD_DTVS;
    if (dtvs) {
        const CamFrame f = make_frame(cam);
        const size_t px = (size_t)cam.width * cam.height;
        ws.depth.ensure(px);
        ws.rays.ensure(px);
        ws.raysa.ensure(px);
        launch_pdl(k_splat_prep, (unsigned)(blocks((long long)px, 256)), 256, 0, st, f, ws.depth.p, ws.rays.p, ws.raysa.p);
        launch_pdl(k_splat, (unsigned)(blocks(n, 256)), 256, 0, st, n, X, radius, f, ws.depth.p, ws.rays.p, ws.raysa.p);
        // each LOD pass counts its own visible sample (several per frame with cameras)
        CK(cudaMemsetAsync(&ws.ctl.p->sample_count, 0, sizeof(int), st));
        launch_pdl(k_dtvs_gap, (unsigned)(blocks(n, 256)), 256, 0, st, n, X, radius, f, ws.depth.p, ws.dist.p, ws.keys.p,
                                                   ws.ctl.p);
    } else {
        launch_pdl(k_dtc_dist, (unsigned)(blocks(n, 256)), 256, 0, st, n, X, cam.eye[0], cam.eye[1], cam.eye[2], ws.dist.p,
                                                   ws.keys.p);
    }
    if (lod.auto_range) {
        launch_pdl(k_rs_init, (unsigned)(1), 1024, 0, st, ws.rs.p, ws.ctl.p, n, dtvs ? 1 : 0);
        const int hb = std::min(blocks(n, 256), 16 * 148);  // ~2 keys per thread: no load chain
        for (int pass = 0; pass < 3; ++pass) {
            launch_pdl(k_rs_hist, (unsigned)(hb), 256, 0, st, n, ws.keys.p, ws.rs.p, pass);
            launch_pdl(k_rs_select, (unsigned)(1), 1024, 0, st, ws.rs.p, pass);
        }
    }
    launch_pdl(k_lod_params, (unsigned)(1), 1, 0, st, ws.rs.p, ws.ctl.p, lod.auto_range, lod.d_min, lod.d_max, dtvs ? 1 : 0);
    launch_pdl(k_lod_map, (unsigned)(blocks(n, 256)), 256, 0, st, n, ws.ctl.p, ws.dist.p, ws.keys.p, dtvs ? 1 : 0, lod.n_min,
                                              lod.n_max, LV);
    LAUNCH_CHECK();
}

std::vector<Workspace*>& global_workspaces() {
    static std::vector<Workspace*> w;
    return w;
}

Workspace& component_ws() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto& v = global_workspaces();
    if ((int)v.size() <= dev) v.resize(dev + 1, nullptr);
    if (!v[dev]) v[dev] = new Workspace(dev);
    return *v[dev];
}

// renderLevelImage (depth_splat.hpp:314-350) of n device positions/levels
// into the caller's width*height*3 bytes.
void render_levels(Workspace& ws, int n, const float4* X, const int* LV, float radius, const apbf_camera& cam,
                   int nMin, int nMax, unsigned char* rgb_out) {
    if (!(radius > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "splat radius must be positive");
    const CamFrame f = make_frame(cam);
    const int px = cam.width * cam.height;
    ws.owner.ensure((size_t)px);
    ws.rgb.ensure((size_t)px * 3);
    cudaStream_t st = ws.stream;
    CK(cudaMemsetAsync(ws.owner.p, 0xff, sizeof(unsigned long long) * px, st));
    if (n > 0) KL(k_render_splat<<<blocks(n, 256), 256, 0, st>>>(n, X, radius, f, ws.owner.p));
    KL(k_render_color<<<blocks(px, 256), 256, 0, st>>>(px, ws.owner.p, LV, nMin, nMax, ws.rgb.p));
    LAUNCH_CHECK();
    CK(cudaMemcpyAsync(rgb_out, ws.rgb.p, (size_t)px * 3, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

void upload_pos4(Workspace& ws, int n, const float* pos, const float* mass = nullptr) {
    std::vector<float4> h((size_t)n);
    for (int i = 0; i < n; ++i)
        h[i] = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], mass ? mass[i] : 0.f);
    ws.tmp4.ensure(n);
    CK(cudaMemcpyAsync(ws.tmp4.p, h.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, ws.stream));
}

}  // namespace

// ============================================================== solver

struct apbf_gpu_solver {
    apbf_solver_config cfg;
    Scene scene;
    Workspace ws;
    int n = 0;
    // Three state sets.  A single-rank frame never writes the set it starts
    // from (predict of the first substep writes into the third set, whose
    // buffers the second substep's reorder fills only afterwards), so a
    // list-overflow retry restarts from it without a backup copy; successive
    // frames rotate through the sets (one cached graph per start set).  The
    // slab path keeps a rank's state in set[0] or set[1], receives records into
    // the other, sorts into set[3] and keeps its retry copy in set[2].
    SetBufs set[4];  // set[3]: slab mode's sorted local set
    int cur = 0;
    DBuf<float4> PB;
    DBuf<float4> PL;  // (x*, lambda) published by the lambda pass for the delta-p gathers
    DBuf<int> order, nbrCount, nbr, tileCount, levelCount, activeCount, bucketStart;
    DBuf<long long> groupBase;
    DBuf<int> lvTmp;             // multi-camera frames: one camera's levels before the blend
    DBuf<float4> sortedPM;
    DBuf<float> stage;  // compact host<->device staging (13 words per particle)
    DBuf<double> resid;
    long long nbrCap = 0;
    int numTiles = 0;
    bool levels_valid = true;
    bool metrics = true;
    bool phase_timing = false;
    float phase_ms[5] = {0, 0, 0, 0, 0};
    cudaEvent_t ev[8];
    cudaEvent_t ev_lam = nullptr;  // the frame's last lambda pass is done (lambda final)
    apbf_iteration_observer observer = nullptr;
    void* observer_user = nullptr;
    // observer view of the in-flight state
    bool in_iteration = false;
    const float4* obs_xs = nullptr;
    // derived config (solver.hpp:44-51), float as in SolverConfig<float>
    float dt = 0, radius = 0, cap = 0;
    int S = 0;
    unsigned long long last_list_entries = 0, last_list_alloc = 0;
    // per-launch CUDA-event timing of the lambda and delta-p kernels
    bool kernel_timing = false;
    std::vector<std::array<cudaEvent_t, 3>> kt_ev;
    size_t kt_used = 0;
    double kt_lambda_ms = 0, kt_deltap_ms = 0;
    long long kt_launches = 0, kt_items = 0;

    // Switching re-records the frame graph (the events are graph nodes);
    // re-enabling while on only resets the accumulators (apbf_gpu_set_kernel_timing).
    void enable_kernel_timing(bool on) {
        if (on == kernel_timing) return;
        drop_graph();
        eager_seen = false;
        kernel_timing = on;
        const size_t need = (size_t)cfg.substeps * cfg.n_max;
        while (on && kt_ev.size() < need) {
            std::array<cudaEvent_t, 3> e;
            for (auto& x : e) CK(cudaEventCreate(&x));
            kt_ev.push_back(e);
        }
    }
    void collect_kernel_timing(unsigned long long items) {
        for (size_t k = 0; k < kt_used; ++k) {
            float a = 0, b = 0;
            CK(cudaEventElapsedTime(&a, kt_ev[k][0], kt_ev[k][1]));
            CK(cudaEventElapsedTime(&b, kt_ev[k][1], kt_ev[k][2]));
            kt_lambda_ms += a;
            kt_deltap_ms += b;
        }
        kt_launches += (long long)kt_used;
        kt_items += (long long)items;
        kt_used = 0;
    }

    apbf_gpu_solver(const apbf_solver_config& c, const Scene& sc, int dev) : cfg(c), scene(sc), ws(dev) {
        dt = cfg.dt_frame / (float)cfg.substeps;
        radius = cfg.particle_radius > 0.0f ? cfg.particle_radius : cfg.h / 4.0f;
        cap = cfg.velocity_cap > 0.0f ? cfg.velocity_cap : cfg.h / dt;
        S = cfg.stab_threshold > 0 ? cfg.stab_threshold : cfg.n_max;
        for (auto& e : ev) CK(cudaEventCreate(&e));
        CK(cudaEventCreateWithFlags(&ev_lam, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&lod_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_lod_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_lod_join, cudaEventDisableTiming));
        const unsigned evf = std::getenv("APBF_E2E_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
        CK(cudaEventCreateWithFlags(&ev_x, evf));
        CK(cudaEventCreateWithFlags(&ev_inputs, evf));
        CK(cudaEventCreateWithFlags(&ev_vm, evf));
        if (const char* v = std::getenv("APBF_GRAPHS")) use_graphs = std::atoi(v) != 0;
        configure_carveouts();
        CK(cudaMemcpy(ws.scene.p, &scene, sizeof(Scene), cudaMemcpyHostToDevice));
        levelCount.ensure(cfg.n_max + 2);
        activeCount.ensure(cfg.n_max + 2);
        bucketStart.ensure(cfg.n_max + 2);
        resid.ensure((size_t)cfg.substeps * cfg.n_max);

    }
    ~apbf_gpu_solver() {
        drop_graph();
        for (auto& e : ev) cudaEventDestroy(e);
        if (ev_lam) cudaEventDestroy(ev_lam);
        if (ev_x) cudaEventDestroy(ev_x);
        if (ev_vm) cudaEventDestroy(ev_vm);
        if (ev_inputs) cudaEventDestroy(ev_inputs);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (comm_stream) cudaStreamDestroy(comm_stream);
        if (lod_stream) cudaStreamDestroy(lod_stream);
        if (ev_lod_fork) cudaEventDestroy(ev_lod_fork);
        if (ev_lod_join) cudaEventDestroy(ev_lod_join);
        if (ev_halo_ready) cudaEventDestroy(ev_halo_ready);
        if (ev_halo_done) cudaEventDestroy(ev_halo_done);
        if (ev_cls) cudaEventDestroy(ev_cls);
        if (hostCls) cudaFreeHost(hostCls);
    }

    void allocate(int nn) {
        const unsigned long long gen0 = g_alloc_gen;
        allocate_buffers(nn);
        if (g_alloc_gen != gen0) {  // new device pointers: the frame graph is stale
            drop_graph();
            eager_seen = false;
        }
    }
    void allocate_buffers(int nn) {
        n = nn;
        const size_t m = (size_t)std::max(nn, 1);
        set[0].ensure(m);
        set[1].ensure(m);
        set[2].ensure(m);
        PB.ensure(m);
        PL.ensure(m);
        if (post_pass()) {
            postOm.ensure(m);
            postV.ensure(m);
        }
        order.ensure(m);
        const size_t groups = (m + 31) / 32 + 1;
        nbrCount.ensure(groups * 32);
        groupBase.ensure(groups);
        list_groups = (long long)groups;
        const long long need = packed_lists ? (long long)m * 48 + 4096 : list_groups * list_stride * 32;
        if (nbrCap < need) {
            nbrCap = need;
            alloc_lists();
        }
        numTiles = (int)((m + kTileSize - 1) / kTileSize);
        tileCount.ensure((size_t)(cfg.n_max + 1) * numTiles);
        sortedPM.ensure(m);
        stage.ensure(13 * m);
        ws.ensure_particles(m);
        ws.ensure_cells();
    }

    void copy_set(SetBufs& dst, SetBufs& src) {
        const size_t m = (size_t)n;
        cudaStream_t st = ws.stream;
        CK(cudaMemcpyAsync(dst.X.p, src.X.p, sizeof(float4) * m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.V.p, src.V.p, sizeof(float4) * m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.XS.p, src.XS.p, sizeof(float4) * m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.W.p, src.W.p, sizeof(float) * m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.L.p, src.L.p, sizeof(float) * m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(dst.LV.p, src.LV.p, sizeof(int) * m, cudaMemcpyDeviceToDevice, st));
    }

    SolverConsts consts() const {
        SolverConsts sc;
        sc.kc = make_kernel_consts(cfg.h);
        sc.invRho0 = 1.0f / cfg.rest_density;
        sc.rho0 = cfg.rest_density;
        sc.eps = cfg.epsilon;
        sc.radius = radius;
        sc.invRho0sq = sc.invRho0 * sc.invRho0;
        // preconditions of k_lambda's cheap division-range test
        volatile float sh = sc.kc.spiky * sc.kc.h;
        volatile float shh = sh * sc.kc.h;
        sc.fastDiv = (cfg.h > 0.0f && cfg.h <= 0x1p60f && sc.kc.spiky < 0.0f && -shh < 0x1p61f) ? 1 : 0;
        sc.w0 = w0;
        return sc;
    }

    // every particle has the same inverse mass w0 (bitwise; checked at upload,
    // frames only permute it); single-GPU only -- a slab rank cannot see its ghosts'
    // what the uploaded inverse masses allow k_lambda to assume (its kW): 0
    // nothing, 1 all finite, 2 all equal to the finite w0 -- checked at
    // upload, and frames only permute them
    int w_mode = 0;
    float w0 = 0.0f;
    bool w_agreed = false;  // slab mode: w_mode / w0 made global (agree_uniform_w)

    bool w_known = false;               // w_mode/w0 hold a scan of an earlier upload
    const float* pending_scan = nullptr;  // upload_split's host inverse mass, scanned in finish_frame
    bool w_mismatch = false;            // that scan disagreed with the mode the frame ran with
    void scan_inv_mass(int nn, const float* inv_mass) {
        unsigned diff = 0, nonfinite = 0;
        const unsigned* b = reinterpret_cast<const unsigned*>(inv_mass);
        for (int i = 0; i < nn; ++i) {  // branch-free so it vectorises
            diff |= b[i] ^ b[0];
            nonfinite |= (b[i] & 0x7f800000u) == 0x7f800000u;
        }
        w0 = inv_mass[0];
        w_mode = nonfinite ? 0 : (diff == 0 ? 2 : 1);
    }
    DBuf<int> wflags;

    // Slab mode: every rank uses the uniform-w lambda only if all ranks hold
    // the same single inverse mass (ghosts come from other ranks).
    void agree_uniform_w(Transport& T) {
        if (w_agreed) return;
        unsigned bits = 0;
        std::memcpy(&bits, &w0, sizeof bits);
        const bool any = n > 0;
        int h[3] = {any ? w_mode : 2, any ? (int)bits : 0x7fffffff, any ? (int)bits : (int)0x80000000};
        wflags.ensure(3);
        CK(cudaMemcpyAsync(wflags.p, h, sizeof h, cudaMemcpyHostToDevice, ws.stream));
        T.allreduce(wflags.p, 2, RType::I32, ROp::Min, ws.stream);
        T.allreduce(wflags.p + 2, 1, RType::I32, ROp::Max, ws.stream);
        CK(cudaMemcpyAsync(h, wflags.p, sizeof h, cudaMemcpyDeviceToHost, ws.stream));
        CK(cudaStreamSynchronize(ws.stream));
        w_mode = h[0] == 2 ? (h[1] == h[2] ? 2 : 1) : h[0];  // min over ranks; equal w0 for 2
        if (w_mode == 2) std::memcpy(&w0, &h[1], sizeof w0);
        w_agreed = true;
    }
    // opt-in PBF velocity post-pass (config xsph_viscosity / vorticity_epsilon)
    bool post_pass() const { return cfg.xsph_viscosity != 0.0f || cfg.vorticity_epsilon != 0.0f; }
    DBuf<float4> postOm, postV;
    // rows per lane of every warp slab (k_build_lists_direct); grows on
    // overflow, never shrinks
    int list_stride = 64;
    long long list_groups = 0;
    // lists longer than this make the uniform stride too wasteful: fall back
    // to k_build_lists (per-warp slabs from an atomic allocator)
    static constexpr int kMaxListStride = 128;
    bool packed_lists = false;
    int ownB_ = 0, ownE_ = 0x7fffffff;  // owned slot range (slab mode); everything otherwise
    int n_iter = 0;                     // particles the solver passes cover (n, or owned+ghosts)

    // CTA sizes of the two solver passes (measured: lambda runs best in
    // 128-thread CTAs, delta-p in 256) and the neighbour gathers in flight
    // per batch.
    static constexpr int kLambdaThreads = 128, kDeltapThreads = 256, kBatch = 4;
    // apbf_gpu_set_fast_math: the contracted lambda / delta-p pair arithmetic
    // (fast_pair_coef), outside the bitwise contract
    bool fast_math = false;

    // which: 1 the lambda pass, 2 the delta-p pass, 3 both
    template <bool kZ, bool kF>
    void launch_pair_t(int it, int s, const float4* Pc, float4* Pn, const StateSet& dst,
                       const SolverConsts& sc, int tslot, int which) {
        cudaStream_t st = ws.stream;
        Ctl* ctl = ws.ctl.p;
        constexpr int B = kLambdaThreads, K = kBatch, D = kDeltapThreads;
        const int sb = blocks(n_iter, B), sd = blocks(n_iter, D);
        // inverse-mass specialisations (w_mode, checked at upload)
        auto lam = [&](auto kern) {
            launch_pdl(kern, sb, B, 0, st, n_iter, it, ctl, (const int*)activeCount.p, (const int*)order.p, Pc,
                       (const float*)dst.W, dst.L, (const int*)nbr.p, (const int*)nbrCount.p,
                       (const long long*)groupBase.p, sc, s, ownB_, ownE_, PL.p);
        };
        // inverse-mass specialisations (w_mode, checked at upload)
        if (!(which & 1)) {
        } else if (w_mode == 2)
            lam(k_lambda<B, K, kZ, 2, kF>);
        else if (w_mode == 1)
            lam(k_lambda<B, K, kZ, 1, kF>);
        else
            lam(k_lambda<B, K, kZ, 0, kF>);
        if (tslot >= 0) rec(kt_ev[tslot][1]);
        if (which & 2)
            launch_pdl(k_deltap_apply<kZ, D, K, kF>, sd, D, 0, st, n_iter, it, ctl, (const int*)activeCount.p,
                       (const int*)order.p, Pc, Pn, (const float*)dst.W, (const float*)dst.L,
                       (const int*)dst.LV, (const int*)nbr.p, (const int*)nbrCount.p,
                       (const long long*)groupBase.p, (const Scene*)ws.scene.p, sc, s, ownB_, ownE_,
                       (const float4*)PL.p);
    }

    // The list build and the residual pass.
    void launch_build_lists(int nn, const StateSet& dst) {
        cudaStream_t st = ws.stream;
        if (packed_lists)
            KL(k_build_lists<<<blocks(nn, kListThreads), kListThreads, 0, st>>>(
                nn, ws.ctl.p, order.p, dst.XS, ws.cellCount.p, cfg.h, cfg.h * cfg.h, nbr.p, nbrCount.p,
                groupBase.p, nbrCap, activeCount.p + 1));
        else
            launch_pdl(k_build_lists_direct, (unsigned)(blocks(nn, kListThreads)), kListThreads, 0, st, nn, ws.ctl.p, order.p, dst.XS, ws.cellCount.p, cfg.h, cfg.h * cfg.h, nbr.p, nbrCount.p,
                groupBase.p, list_stride, activeCount.p + 1);
    }
    void launch_residual(int nn, int it, const float4* Pn, const SolverConsts& sc, double* out, int oB,
                         int oE) {
        KL(k_residual<<<blocks(nn, 256), 256, 0, ws.stream>>>(nn, it, ws.ctl.p, activeCount.p, order.p, Pn,
                                                              nbr.p, nbrCount.p, groupBase.p, sc, out, oB, oE));
    }

    // The gather passes want L1, not shared memory (they use none).
    template <bool kF>
    static void carveouts_f() {
        const int a = cudaSharedmemCarveoutMaxL1;
        constexpr int B = kLambdaThreads, D = kDeltapThreads, K = kBatch;
        cudaFuncSetAttribute(k_lambda<B, K, false, 0, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
        cudaFuncSetAttribute(k_lambda<B, K, false, 1, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
        cudaFuncSetAttribute(k_lambda<B, K, false, 2, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
        cudaFuncSetAttribute(k_lambda<B, K, true, 0, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
        cudaFuncSetAttribute(k_lambda<B, K, true, 1, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
        cudaFuncSetAttribute(k_lambda<B, K, true, 2, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
        cudaFuncSetAttribute(k_deltap_apply<false, D, K, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
        cudaFuncSetAttribute(k_deltap_apply<true, D, K, kF>, cudaFuncAttributePreferredSharedMemoryCarveout, a);
    }
    void configure_carveouts() {
        carveouts_f<false>();
        carveouts_f<true>();
        // level tables in shared memory: (n_max + 1) ints per CTA, 9x that in
        // the stable level scatter -- past the 48 KB default from n_max 1365
        const int lvl = (kMaxLevels + 1) * (int)sizeof(int);
        CK(cudaFuncSetAttribute(k_level_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 9 * lvl));
        CK(cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, lvl));
        CK(cudaFuncSetAttribute(k_mask_level_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, lvl));
        cudaGetLastError();
    }

    // which: 1 the lambda pass, 2 the delta-p pass, 3 both
    void launch_solver_pair(int it, int s, const float4* Pc, float4* Pn, const StateSet& dst,
                            const SolverConsts& sc, int tslot, int which = 3) {
        const int v = (cfg.inactive_lambda_zero ? 1 : 0) | (fast_math ? 2 : 0);
        switch (v) {
            case 0: launch_pair_t<false, false>(it, s, Pc, Pn, dst, sc, tslot, which); break;
            case 1: launch_pair_t<true, false>(it, s, Pc, Pn, dst, sc, tslot, which); break;
            case 2: launch_pair_t<false, true>(it, s, Pc, Pn, dst, sc, tslot, which); break;
            default: launch_pair_t<true, true>(it, s, Pc, Pn, dst, sc, tslot, which); break;
        }
    }

    // Slab mode: a second iteration set (order, level bucketing and frozen
    // lists) for the halo-dependent particles, so that the interior's passes
    // overlap the x* halo exchange.  swap_sets() exchanges the two sets'
    // buffers; every launch helper works on the current one.
    DBuf<int> orderB, nbrCountB, nbrB, levelCountB, activeCountB, bucketStartB;
    DBuf<long long> groupBaseB;
    static void swap_buf(DBuf<int>& a, DBuf<int>& b) {
        std::swap(a.p, b.p);
        std::swap(a.n, b.n);
    }
    void swap_sets() {
        swap_buf(order, orderB);
        swap_buf(nbrCount, nbrCountB);
        swap_buf(nbr, nbrB);
        swap_buf(levelCount, levelCountB);
        swap_buf(activeCount, activeCountB);
        swap_buf(bucketStart, bucketStartB);
        std::swap(groupBase.p, groupBaseB.p);
        std::swap(groupBase.n, groupBaseB.n);
    }
    void ensure_set_b() {
        orderB.ensure(order.n);
        nbrCountB.ensure(nbrCount.n);
        nbrB.ensure(nbr.n);
        levelCountB.ensure(levelCount.n);
        activeCountB.ensure(activeCount.n);
        bucketStartB.ensure(bucketStart.n);
        groupBaseB.ensure(groupBase.n);
    }

    // (Re)allocate the order-based list store at nbrCap entries.
    void alloc_lists() {
        nbr.release();
        nbr.ensure((size_t)nbrCap);
        if (nbrB.p) {  // slab mode's second iteration set follows
            nbrB.release();
            nbrB.ensure((size_t)nbrCap);
        }
    }

    // After an overflowed list build: grow the per-lane stride, or switch to
    // per-warp slabs when a few lists are very long, or grow the packed store.
    void grow_lists(unsigned long long used, unsigned long long used_fb) {
        const int why = ws.h_ctl->list_overflow;
        if ((why & 1) && packed_lists) nbrCap = std::max<long long>(nbrCap * 2, (long long)(used * 3 / 2));
        if ((why & 1) && !packed_lists) {
            const int want = list_rows(std::max(list_stride + 16, (int)used_fb + 8));
            if (want > kMaxListStride) {
                // a few very long lists: a uniform stride would cost n x max;
                // switch to per-warp slabs from the allocating builder
                packed_lists = true;
                nbrCap = std::max<long long>(nbrCap, (long long)(used * 3 / 2));
            } else {
                list_stride = want;
            }
        }
        if (!packed_lists) nbrCap = std::max(nbrCap, list_groups * list_stride * 32);
        alloc_lists();
    }

    // Event records that also work inside stream capture (graph event nodes).
    bool capturing = false;
    void rec(cudaEvent_t e) {
        if (capturing) CK(cudaEventRecordWithFlags(e, ws.stream, cudaEventRecordExternal));
        else CK(cudaEventRecord(e, ws.stream));
    }
    void mark(int k) {
        if (phase_timing) rec(ev[k]);
    }

    // One frame on the device; returns after the control block is on the host.
    // Enqueue one frame on the solver stream (no host synchronisation unless an
    // iteration observer is installed): captured as a CUDA Graph by frame().
    void enqueue_frame(bool assign_lod, const apbf_camera* cam, const apbf_lod_config* lod) {
        cudaStream_t st = ws.stream;
        Ctl* ctl = ws.ctl.p;
        const SolverConsts sc = consts();
        const int nMax = cfg.n_max;
        rec(ev[0]);
        kt_used = 0;
        n_iter = n;
        launch_pdl(k_frame_begin, (unsigned)(1), 1, 0, st, ctl);
        // The LOD pass (APBF) reads only x and writes only the levels and its
        // own control fields; nothing before the first reorder reads levels.
        // So it forks onto lod_stream and runs beside the first substep's
        // predict and grid build (graph branches), joined before k_gather.
        // (Serial under phase timing or an observer.)
        bool lod_forked = false;
        if (assign_lod) {
            if (cfg.mode == APBF_MODE_PBF) {
                KL(k_fill_int<<<blocks(n, 256), 256, 0, st>>>(set[cur].LV.p, n, nMax));
            } else {
                apbf_lod_config lc = *lod;
                lc.n_min = cfg.n_min;
                lc.n_max = cfg.n_max;
                lod_forked = !phase_timing && !observer;
                if (lod_forked) {
                    CK(cudaEventRecord(ev_lod_fork, st));
                    CK(cudaStreamWaitEvent(lod_stream, ev_lod_fork, 0));
                    run_lod(ws, set[cur].X.p, n, *cam, lc, radius, set[cur].LV.p, lod_stream);
                    CK(cudaEventRecord(ev_lod_join, lod_stream));
                } else {
                    run_lod(ws, set[cur].X.p, n, *cam, lc, radius, set[cur].LV.p);
                }
            }
        }
        mark(1);
        const int sa = cur, sb = (cur + 1) % 3, sc3 = (cur + 2) % 3;
        for (int s = 0; s < cfg.substeps; ++s) {
            // substeps: a -> b, then b -> c, c -> b, ... (a is never written)
            const int si = s == 0 ? sa : ((s & 1) ? sb : sc3);
            const int di = s == 0 ? sb : ((s & 1) ? sc3 : sb);
            StateSet src = set[si].view(), dst = set[di].view();
            launch_pdl(k_substep_reset, (unsigned)(1), 1, 0, st, ctl);
            // substep 0 predicts into the third set's V/x* (free until the
            // next substep's reorder), keeping the start set intact
            StateSet pin = src;
            if (s == 0) {
                pin.V = set[sc3].V.p;
                pin.XS = set[sc3].XS.p;
                if (capturing) CK(cudaStreamWaitEvent(st, ev_vm, cudaEventWaitExternal));
                else CK(cudaStreamWaitEvent(st, ev_vm, 0));
            }
            launch_pdl(k_predict, (unsigned)(blocks(n, kAabbBlock)), kAabbBlock, 0, st, n, src.X, src.V, pin.V, src.XS, pin.XS, dt,
                                                      cfg.gravity[0], cfg.gravity[1], cfg.gravity[2], ctl, s);
            ws.run_grid(0, pin.XS, n, cfg.h, cfg.h, scene.n > 0, radius);
            const int smemG = (nMax + 1) * (int)sizeof(int);
            if (s == 0) {
                // a host stepFrame uploads inverse mass last (upload_split); a
                // no-op wait when nothing was uploaded that way
                if (capturing) CK(cudaStreamWaitEvent(st, ev_inputs, cudaEventWaitExternal));
                else CK(cudaStreamWaitEvent(st, ev_inputs, 0));
            }
            if (s == 0 && lod_forked) {
                // the fields now, the levels once the forked LOD pass joins
                launch_pdl(k_gather, (unsigned)(numTiles), kTileThreads, smemG, st, n, ctl, ws.perm.p, pin, dst, nMax, numTiles,
                                                               tileCount.p, 1, SelfMap{});
                CK(cudaStreamWaitEvent(st, ev_lod_join, 0));
                launch_pdl(k_gather, (unsigned)(numTiles), kTileThreads, smemG, st, n, ctl, ws.perm.p, pin, dst, nMax, numTiles,
                                                               tileCount.p, 2, SelfMap{});
            } else {
                launch_pdl(k_gather, (unsigned)(numTiles), kTileThreads, smemG, st, n, ctl, ws.perm.p, pin, dst, nMax, numTiles,
                                                               tileCount.p, 3, SelfMap{});
            }
            if (s == cfg.substeps - 1) rec(ev[7]);  // final storage order (overlapped download)
            launch_pdl(k_level_scan, (unsigned)(nMax + 1), 1024, 0, st, ctl, numTiles, tileCount.p, levelCount.p);
            launch_pdl(k_level_finish, (unsigned)(1), 32, 0, st, ctl, n, nMax, levelCount.p, activeCount.p, bucketStart.p, 1);
            launch_pdl(k_level_scatter, (unsigned)(numTiles), kTileThreads, 9 * smemG, st, n, ctl, dst.LV, nMax, numTiles,
                                                                         tileCount.p, bucketStart.p, order.p);
            launch_build_lists(n, dst);
            if (S > 1)
                launch_pdl(k_prestabilize, (unsigned)(blocks(n, 256)), 256, 0, st, n, ctl, activeCount.p, S, order.p, dst.XS,
                                                               dst.X, ws.scene.p, radius, cfg.stab_iterations,
                                                               s);
            LAUNCH_CHECK();
            mark(2);
            float4* P[2] = {dst.XS, PB.p};
            int lastIter = nMax;
            std::vector<int> hActive;
            if (observer) {
                hActive.resize(nMax + 2);
                CK(cudaMemcpyAsync(hActive.data(), activeCount.p, sizeof(int) * (nMax + 2),
                                   cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
            }
            for (int it = 1; it <= nMax; ++it) {
                if (observer) {
                    ws.read_ctl();
                    if (ws.h_ctl->abort) break;
                    if (hActive[it] == 0) {
                        lastIter = it - 1;
                        break;
                    }
                }
                const float4* Pc = P[(it - 1) & 1];
                float4* Pn = P[it & 1];
                const int tslot = kernel_timing ? (int)kt_used++ : -1;
                if (tslot >= 0) rec(kt_ev[tslot][0]);
                if (s == cfg.substeps - 1 && it == nMax && !observer) {
                    // lambda is final after the frame's last lambda pass: its
                    // download may start under the last delta-p and finalize
                    launch_solver_pair(it, s, Pc, Pn, dst, sc, tslot, 1);
                    rec(ev_lam);
                    launch_solver_pair(it, s, Pc, Pn, dst, sc, -1, 2);
                } else {
                    launch_solver_pair(it, s, Pc, Pn, dst, sc, tslot);
                }
                if (tslot >= 0) rec(kt_ev[tslot][2]);
                if (cfg.record_residuals) {
                    CK(cudaMemsetAsync(resid.p + (size_t)s * nMax + (it - 1), 0, sizeof(double), st));
                    launch_residual(n, it, Pn, sc, resid.p + (size_t)s * nMax + (it - 1), 0, 0x7fffffff);
                }
                LAUNCH_CHECK();
                if (observer) {
                    ws.read_ctl();
                    if (ws.h_ctl->abort) break;
                    in_iteration = true;
                    obs_xs = Pn;
                    const int c = cur;
                    cur = di;  // expose dst as the current set to get_state
                    observer(observer_user, s, it);
                    cur = c;
                    in_iteration = false;
                }
            }
            if (s == cfg.substeps - 1 && observer) rec(ev_lam);
            mark(3);
            float4* Pf = P[lastIter & 1];
            launch_pdl(k_finalize, (unsigned)(blocks(n, 256)), 256, 0, st, n, ctl, Pf, dst.XS, dst.X, dst.V, dt, cap,
                                                       Pf != dst.XS ? 1 : 0, s);
            if (post_pass()) {  // opt-in XSPH / vorticity confinement (apbf_post.cuh)
                const KernelConsts kc = make_kernel_consts(cfg.h);
                KL(k_post_omega<<<blocks(n, 256), 256, 0, st>>>(n, ctl, order.p, dst.X, dst.V, nbr.p,
                                                             nbrCount.p, groupBase.p, kc,
                                                             cfg.xsph_viscosity, postOm.p, postV.p));
                KL(k_post_apply<<<blocks(n, 256), 256, 0, st>>>(n, ctl, order.p, dst.X, postOm.p, postV.p,
                                                             nbr.p, nbrCount.p, groupBase.p, kc, dt,
                                                             cfg.vorticity_epsilon, cap, dst.V));
            }
            LAUNCH_CHECK();
            cur = di;
            mark(4);
        }
        rec(ev[5]);
        if (metrics) {
            // allDensities(x) over a throwaway grid (solver.hpp:271-279).
            launch_pdl(k_grid_reset, (unsigned)(1), 1, 0, st, ctl, 1);
            launch_pdl(k_aabb, (unsigned)(blocks(n, kAabbBlock)), kAabbBlock, 0, st, n, set[cur].X.p, ctl, 1);
            ws.run_grid(1, set[cur].X.p, n, cfg.h, cfg.h, false, radius);
            launch_pdl(k_gather_posmass, (unsigned)(blocks(n, 256)), 256, 0, st, n, ctl, ws.perm.p, set[cur].X.p,
                                                             set[cur].XS.p, sortedPM.p);
            launch_pdl(k_density_stats, (unsigned)(blocks(n, 256)), 256, 0, st, n, ctl, sortedPM.p, ws.cellCount.p, sc.kc);
            LAUNCH_CHECK();
        }
        rec(ev[6]);
        CK(cudaMemcpyAsync(ws.h_ctl, ws.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    }

    void run_frame(bool assign_lod, const apbf_camera* cam, const apbf_lod_config* lod) {
        enqueue_frame(assign_lod, cam, lod);
        finish_frame();
    }

    // ---- stepFrame on host arrays with the download overlapped ----
    // When host_out is set, the frame's result is packed and copied to the
    // caller's arrays on copy_stream as soon as the last substep is done
    // (event ev[5]), concurrently with the end-of-frame metrics pass.
    struct HostOut {
        float *x, *xs, *v, *mass, *inv_mass, *lambda;
        int32_t* level;
        bool queued;
    };
    // The caller's x*, lambda and level as passed in (stepFrame overwrites
    // them before reading them, so the frame never needs them): uploaded raw
    // on copy_stream while the frame runs, so that a failing frame can hand
    // the caller back exactly the arrays it passed (restore_host_inputs).
    DBuf<float> keep;
    HostOut* host_out = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_x = nullptr, ev_inputs = nullptr;  // upload_split: x unpacked / everything unpacked
    cudaEvent_t ev_vm = nullptr;                      // upload_split: v and mass unpacked

    // The inputs of a host stepFrame: x on the solver stream (the LOD pass
    // needs only x), v, mass and inverse mass on copy_stream, unpacked there
    // once x is; the frame waits for ev_vm before its first predict and for
    // ev_inputs before its first reorder.
    void upload_split(int nn, const float* x, const float* v, const float* mass, const float* inv_mass,
                      const float* x_star = nullptr, const float* lambda = nullptr,
                      const int32_t* level = nullptr) {
        n = nn;
        levels_valid = nn == 0;
        if (nn == 0) return;
        if (!copy_stream) CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
        cudaStream_t st = ws.stream;
        float* d = stage.p;
        const size_t n1 = sizeof(float) * (size_t)nn, n3 = 3 * n1;
        CK(cudaMemcpyAsync(d, x, n3, cudaMemcpyHostToDevice, st));
        KL(k_unpack_x<<<blocks(nn, 256), 256, 0, st>>>(nn, d, set[0].X.p));
        CK(cudaEventRecord(ev_x, st));
        // v and mass (predict), then inverse mass (first reorder): the frame
        // waits for each right where it first reads it
        CK(cudaMemcpyAsync(d + 6LL * nn, v, n3, cudaMemcpyHostToDevice, copy_stream));
        CK(cudaMemcpyAsync(d + 9LL * nn, mass, n1, cudaMemcpyHostToDevice, copy_stream));
        CK(cudaStreamWaitEvent(copy_stream, ev_x, 0));
        KL(k_unpack_vm<<<blocks(nn, 256), 256, 0, copy_stream>>>(nn, d, set[0].view()));
        CK(cudaEventRecord(ev_vm, copy_stream));
        CK(cudaMemcpyAsync(d + 10LL * nn, inv_mass, n1, cudaMemcpyHostToDevice, copy_stream));
        KL(k_unpack_w<<<blocks(nn, 256), 256, 0, copy_stream>>>(nn, d, set[0].view()));
        LAUNCH_CHECK();
        CK(cudaEventRecord(ev_inputs, copy_stream));
        if (x_star && lambda && level) {  // nothing waits on these (restore_host_inputs only)
            keep.ensure(5 * (size_t)nn);
            CK(cudaMemcpyAsync(keep.p, x_star, n3, cudaMemcpyHostToDevice, copy_stream));
            CK(cudaMemcpyAsync(keep.p + 3LL * nn, lambda, n1, cudaMemcpyHostToDevice, copy_stream));
            CK(cudaMemcpyAsync(keep.p + 4LL * nn, level, n1, cudaMemcpyHostToDevice, copy_stream));
        }
        w_agreed = false;
        // The inverse-mass mode picks the lambda variant, so it is part of the
        // frame graph's key.  Scanning 4 B/particle on the host would delay the
        // launch; once a mode is known the frame launches with it and the scan
        // runs while the GPU works (finish_frame), re-running the frame in the
        // rare case the mode changed.
        if (w_known) {
            pending_scan = inv_mass;
        } else {
            scan_inv_mass(nn, inv_mass);
            w_known = true;
        }
    }

    // The frame's result to the caller's arrays on `st`: the fields that are
    // final after the last substep's reorder once ev[7] has fired (during that
    // substep's iterations), the rest once ev[5] has (during the metrics pass).
    void enqueue_download(cudaStream_t st, HostOut& o) {
        const StateSet fin = set[cur].view();
        float* d = stage.p;
        const size_t n1 = sizeof(float) * (size_t)n, n3 = 3 * n1;
        CK(cudaStreamWaitEvent(st, ev[7], 0));
        KL(k_pack_static<<<blocks(n, 256), 256, 0, st>>>(n, fin, d));
        if (o.mass) CK(cudaMemcpyAsync(o.mass, d + 9LL * n, n1, cudaMemcpyDeviceToHost, st));
        if (o.inv_mass) CK(cudaMemcpyAsync(o.inv_mass, d + 10LL * n, n1, cudaMemcpyDeviceToHost, st));
        if (o.level) CK(cudaMemcpyAsync(o.level, d + 12LL * n, n1, cudaMemcpyDeviceToHost, st));
        // lambda straight from the final set once the last lambda pass is done
        CK(cudaStreamWaitEvent(st, ev_lam, 0));
        if (o.lambda) CK(cudaMemcpyAsync(o.lambda, fin.L, n1, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamWaitEvent(st, ev[5], 0));
        KL(k_pack_dynamic<<<blocks(n, 256), 256, 0, st>>>(n, fin, d));
        LAUNCH_CHECK();
        // (x* equals x after the frame, but filling the caller's x* from x
        // on the host competed with the DMA for host memory bandwidth on
        // some boxes: it stays a PCIe copy)
        if (o.x) CK(cudaMemcpyAsync(o.x, d, n3, cudaMemcpyDeviceToHost, st));
        if (o.xs) CK(cudaMemcpyAsync(o.xs, d + 3LL * n, n3, cudaMemcpyDeviceToHost, st));
        if (o.v) CK(cudaMemcpyAsync(o.v, d + 6LL * n, n3, cudaMemcpyDeviceToHost, st));
    }

    // A frame that failed after its overlapped download was queued: give the
    // caller back the arrays it passed in.  x, v, mass and inverse mass come
    // from the frame's start set (a single-rank frame never writes those
    // fields of it), x*, lambda and level from the raw copy of the inputs.
    void restore_host_inputs(int start) {
        HostOut& o = *host_out;
        cudaStream_t st = ws.stream;
        const StateSet s0 = set[start].view();
        float* d = stage.p;
        const size_t n1 = sizeof(float) * (size_t)n, n3 = 3 * n1;
        CK(cudaStreamSynchronize(copy_stream));
        KL(k_pack_static<<<blocks(n, 256), 256, 0, st>>>(n, s0, d));
        KL(k_pack_dynamic<<<blocks(n, 256), 256, 0, st>>>(n, s0, d));
        LAUNCH_CHECK();
        CK(cudaMemcpyAsync(o.x, d, n3, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(o.v, d + 6LL * n, n3, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(o.mass, d + 9LL * n, n1, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(o.inv_mass, d + 10LL * n, n1, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(o.xs, keep.p, n3, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(o.lambda, keep.p + 3LL * n, n1, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(o.level, keep.p + 4LL * n, n1, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        o.queued = false;
    }

    // Wait for the enqueued frame (and its overlapped download, if any).
    void finish_frame() {
        if (pending_scan) {
            // while the GPU runs the frame, and before the download into the
            // same host arrays is enqueued
            const int used = w_mode;
            const float used_w0 = w0;
            scan_inv_mass(n, pending_scan);
            pending_scan = nullptr;
            w_mismatch = w_mode != used || (w_mode == 2 && std::memcmp(&w0, &used_w0, sizeof w0) != 0);
        }
        if (host_out && n > 0 && !w_mismatch) {  // a mismatched frame is re-run, then downloaded
            if (!copy_stream) CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
            enqueue_download(copy_stream, *host_out);
            host_out->queued = true;
        }
        CK(cudaStreamSynchronize(ws.stream));
        if (host_out && n > 0) CK(cudaStreamSynchronize(copy_stream));
    }

    // ---- CUDA Graph of the whole frame (LOD + substeps + metrics) ----
    struct GraphKey {
        int start, assign_lod, metrics, ktime, ptime, n, flags, stride;
        unsigned w0bits;
        long long caps[3];
        apbf_camera cam;
        apbf_lod_config lod;
    };
    bool use_graphs = true;  // APBF_GRAPHS=0 disables
    bool eager_seen = false;  // seen[] holds keys of frames run eagerly since the last reset
    struct FrameGraph {
        GraphKey key;
        cudaGraphExec_t exec;
        size_t kt_used;
        unsigned long long kernels;  // kernel nodes of the frame graph
    };
    std::vector<FrameGraph> graphs;  // one per start set (frames rotate through three)
    std::vector<GraphKey> seen;
    static constexpr size_t kMaxGraphs = 3;

    GraphKey make_key(bool assign_lod, const apbf_camera* cam, const apbf_lod_config* lod) const {
        GraphKey k;
        std::memset(&k, 0, sizeof k);
        k.start = cur;
        k.assign_lod = assign_lod;
        k.metrics = metrics;
        k.ktime = kernel_timing;
        k.ptime = phase_timing;
        k.n = n;
        k.flags = (w_mode << 20) | (packed_lists ? 0x400000 : 0) | (fast_math ? 1 : 0);
        k.caps[0] = nbrCap;
        k.stride = list_stride;
        if (w_mode == 2) std::memcpy(&k.w0bits, &w0, sizeof w0);
        if (assign_lod && cam) k.cam = *cam;
        if (assign_lod && lod) k.lod = *lod;
        return k;
    }
    void drop_graph() {
        for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
        graphs.clear();
    }
    // The set a frame starting from set a ends in (enqueue_frame's rotation).
    int final_set(int a) const { return (a + ((cfg.substeps & 1) ? 1 : 2)) % 3; }

    // One frame: replay a captured graph when one matches the frame's key;
    // when the same configuration ran before (from any start set), capture the
    // graphs of all three start sets (frames rotate through them) and launch
    // this frame's; run eagerly otherwise (first frame, observer, changing
    // configuration).
    FrameGraph capture_graph(const GraphKey& key, bool assign_lod, const apbf_camera* cam,
                             const apbf_lod_config* lod) {
        cudaStream_t st = ws.stream;
        const int c0 = cur;
        cur = key.start;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        const unsigned long long l0 = g_launches;
        capturing = true;
        try {
            enqueue_frame(assign_lod, cam, lod);
            capturing = false;
        } catch (...) {
            capturing = false;
            cur = c0;
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        CK(cudaStreamEndCapture(st, &g));
        FrameGraph fg{key, nullptr, kt_used, g_launches - l0};  // captured, not run: counted per replay
        g_launches = l0;
        cur = c0;
        const cudaError_t e = cudaGraphInstantiate(&fg.exec, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        return fg;
    }
    void launch_frame(bool assign_lod, const apbf_camera* cam, const apbf_lod_config* lod) {
        const GraphKey key = make_key(assign_lod, cam, lod);
        const bool graphable = use_graphs && !observer;
        cudaStream_t st = ws.stream;
        auto same = [&](const GraphKey& k) { return std::memcmp(&k, &key, sizeof key) == 0; };
        auto same_config = [&](GraphKey k) {
            k.start = key.start;
            return same(k);
        };
        if (!eager_seen) seen.clear();
        const FrameGraph* hit = nullptr;
        if (graphable) {
            for (auto& g : graphs)
                if (same(g.key)) hit = &g;
            if (!hit && std::any_of(seen.begin(), seen.end(), same_config)) {
                drop_graph();
                for (int k = 0; k < 3; ++k) {
                    GraphKey kk = key;
                    kk.start = (key.start + k) % 3;
                    graphs.push_back(capture_graph(kk, assign_lod, cam, lod));
                }
                hit = &graphs.front();
            }
        }
        if (hit) {
            CK(cudaGraphLaunch(hit->exec, st));
            g_launches += hit->kernels;
            cur = final_set(key.start);
            kt_used = hit->kt_used;
            finish_frame();
            return;
        }
        run_frame(assign_lod, cam, lod);
        if (seen.size() >= kMaxGraphs) seen.erase(seen.begin());
        seen.push_back(key);
        eager_seen = true;
    }

    void frame(bool assign_lod, const apbf_camera* cam, const apbf_lod_config* lod, int frame_index,
               apbf_frame_stats* out) {
        NvtxRange range(transport ? "apbf slab frame" : "apbf frame");
        CK(cudaSetDevice(ws.device));
        if (transport) {
            if (post_pass()) fail(APBF_ERR_INVALID_ARGUMENT, "the velocity post-pass runs on one rank");
            frame_dist(assign_lod, cam, lod, frame_index, out);
            return;
        }
        if (assign_lod && cfg.mode == APBF_MODE_APBF) {
            apbf_lod_config lc = *lod;
            validate_lod(lc);
            if (n > 0 && lc.model == APBF_LOD_DTVS) {
                if (!(radius > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "splat radius must be positive");
                (void)make_frame(*cam);  // camera validation (depth_splat.hpp:29-42, 59-63)
            }
        }
        apbf_frame_stats st;
        std::memset(&st, 0, sizeof st);
        st.frame = frame_index;
        if (n == 0) {
            if (out) {
                double* r = out->residuals;
                int rc = out->residuals_capacity;
                *out = st;
                out->residuals = r;
                out->residuals_capacity = rc;
            }
            return;
        }
        const int start_set = cur;
        for (int attempt = 0;; ++attempt) {
            if (attempt == 0) launch_frame(assign_lod, cam, lod);
            else run_frame(assign_lod, cam, lod);
            if (w_mismatch) {
                // ran with the previous upload's inverse-mass mode: run again
                // from the (unwritten) start set
                w_mismatch = false;
                cur = start_set;
                --attempt;
                continue;
            }
            if (!ws.h_ctl->list_overflow) break;
            // Neighbour storage too small: double the capacity and run the
            // frame again from the start set (levels included: a retry's LOD
            // recomputes the same ones from the same x).
            if (attempt > 6) fail(APBF_ERR_RUNTIME, "neighbor list overflow");
            cur = start_set;
            grow_lists(ws.h_ctl->list_alloc, ws.h_ctl->list_alloc_fb);
            drop_graph();
            eager_seen = false;
        }
        const Ctl& c = *ws.h_ctl;
        if (kernel_timing) collect_kernel_timing(c.total_iterations);
        last_list_entries = c.list_entries;
        last_list_alloc = c.list_alloc;
        if (c.abort || c.runtime_error) {
            // A failed frame leaves the state it started from (the reference
            // throws mid-frame; here the caller gets the frame-start state,
            // with the frame's LOD levels on the device as assignLevels
            // wrote them, solver.hpp:247-258), and a host stepFrame's arrays
            // exactly as they were passed in.
            cur = start_set;
            if (host_out && host_out->queued) restore_host_inputs(start_set);
        }
        if (c.runtime_error) fail(APBF_ERR_RUNTIME, "grid cell count exceeds limit; domain blew up");
        static const char* names[kNumPassSlots] = {"predict", "prestabilize", "lambda",
                                                   "apply",   "finalize",     "finalize"};
        static const char* details[kNumPassSlots] = {
            "non-finite predicted position", "non-finite predicted position", "non-finite lambda",
            "non-finite predicted position", "non-finite velocity",           "non-finite position"};
        // The earliest failing pass: they abort the frame, so only one pass
        // (finalize: velocity before position) can hold a record.
        for (int s = 0; s < kNumPassSlots; ++s)
            if (c.bad[s] != 0x7fffffff) numerical(names[s], c.bad[s], details[s]);
        if (c.abort) fail(APBF_ERR_RUNTIME, "frame aborted without a recorded cause");
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[0], ev[5]));
        st.wall_ms = ms;
        st.total_iterations = (int64_t)c.total_iterations;
        st.contacts = (int64_t)c.contacts;
        if (metrics) {
            const double scale = 100.0 / (double)cfg.rest_density;
            st.avg_density_pct = c.rho_sum / n * scale;
            st.min_density_pct = (double)ord2f(c.rho_min_ord) * scale;
            st.max_density_pct = (double)ord2f(c.rho_max_ord) * scale;
        }
        if (cfg.record_residuals) {
            std::vector<double> r((size_t)cfg.substeps * cfg.n_max);
            CK(cudaMemcpy(r.data(), resid.p, sizeof(double) * r.size(), cudaMemcpyDeviceToHost));
            // executed iterations per substep = max level present; the
            // totalIterations sum cannot tell us, so recompute from levels
            // (levels are frame-constant).
            std::vector<int> lv((size_t)n);
            CK(cudaMemcpy(lv.data(), set[cur].LV.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
            int maxl = 0;
            for (int v : lv) maxl = std::max(maxl, v);
            int k = 0;
            for (int s = 0; s < cfg.substeps; ++s)
                for (int it = 1; it <= maxl; ++it, ++k) {
                    if (out && out->residuals && k < out->residuals_capacity)
                        out->residuals[k] = r[(size_t)s * cfg.n_max + (it - 1)] / n;
                }
            st.n_residuals = k;
        }
        if (phase_timing) {
            float t[5] = {0, 0, 0, 0, 0};
            cudaEventElapsedTime(&t[0], ev[0], ev[1]);
            cudaEventElapsedTime(&t[4], ev[5], ev[6]);
            phase_ms[0] = t[0];
            phase_ms[4] = t[4];
            // per-phase split of the last substep scaled to all substeps
            float a = 0, b = 0, d = 0;
            cudaEventElapsedTime(&a, ev[1], ev[2]);
            cudaEventElapsedTime(&b, ev[2], ev[3]);
            cudaEventElapsedTime(&d, ev[3], ev[4]);
            phase_ms[1] = a;
            phase_ms[2] = b;
            phase_ms[3] = d;
        }
        if (out) {
            double* r = out->residuals;
            int rc = out->residuals_capacity;
            *out = st;
            out->residuals = r;
            out->residuals_capacity = rc;
        }
    }

    // ================================================ z-slab decomposition
    // (kernels in apbf_dist.cuh).  Active when `transport` is
    // set: this handle is rank g of G and holds only its owned particles.

    Transport* transport = nullptr;
    long long n_global_ = 0;  // slab mode: particles over all ranks (set_state_local)
    long long send_capacity = 0;  // slab mode: exchange send buffers (set_state_local)
    std::unique_ptr<Transport> transport_owned;
    long long n_capacity = 0;
    DBuf<int> layerHist, zRange, bounds, destTile, destCountD, destStartD, sendIdx, LVo, ownedFlag,
        ownedSorted, minmax;
    DBuf<unsigned> destMask;
    DBuf<Rec> sendRec, recvRec;
    DBuf<float4> sendPM, recvPM;
    // owned counts before / after each substep: the global index of an error
    // (prefix over lower ranks) is computed from them only if a frame fails
    std::vector<long long> localPre, localPost, prefixPre, prefixPost;
    DBuf<long long> countsX;

    void exchange_prefixes(Transport& T) {
        const int G = T.size(), g = T.rank(), S2 = 2 * cfg.substeps;
        std::vector<long long> rows((size_t)G * S2, 0);
        for (int s = 0; s < cfg.substeps; ++s) {
            rows[(size_t)g * S2 + s] = localPre[s];
            rows[(size_t)g * S2 + cfg.substeps + s] = localPost[s];
        }
        countsX.ensure(rows.size());
        CK(cudaMemcpyAsync(countsX.p, rows.data(), sizeof(long long) * rows.size(), cudaMemcpyHostToDevice,
                           ws.stream));
        T.allreduce(countsX.p, rows.size(), RType::I64, ROp::Sum, ws.stream);
        CK(cudaMemcpyAsync(rows.data(), countsX.p, sizeof(long long) * rows.size(), cudaMemcpyDeviceToHost,
                           ws.stream));
        CK(cudaStreamSynchronize(ws.stream));
        prefixPre.assign(cfg.substeps, 0);
        prefixPost.assign(cfg.substeps, 0);
        for (int s = 0; s < cfg.substeps; ++s)
            for (int q = 0; q < g; ++q) {
                prefixPre[s] += rows[(size_t)q * S2 + s];
                prefixPost[s] += rows[(size_t)q * S2 + cfg.substeps + s];
            }
    }
    // Upload this rank's slice (the rank's contiguous part of the global
    // storage order) with buffers sized for the global particle count.
    void set_state_local(int nloc, long long ntotal, const float* x, const float* xs, const float* v,
                         const float* mass, const float* inv_mass, const float* lambda,
                         const int32_t* level) {
        // Capacities that no input can exceed, so that no rank ever has to
        // fail on its own between collectives:
        // * a rank receives every particle at most once: local (owned +
        //   ghost) counts <= n_global;
        // * a substep sends each particle to at most 3 ranks (its owner and
        //   the two neighbours whose 2-layer halo it may sit in; slabs are
        //   >= 2 layers thick), the metrics exchange to at most G.
        const int G = transport ? transport->size() : 1;
        const long long nt = std::max<long long>(ntotal, 1);
        n_capacity = nt + 4096;
        n_global_ = ntotal;
        send_capacity = (long long)std::max(3, G) * nt + 4096;
        allocate((int)n_capacity);
        destMask.ensure(n_capacity);
        sendIdx.ensure(send_capacity);
        LVo.ensure(n_capacity);
        ownedFlag.ensure(n_capacity);
        ownedSorted.ensure(n_capacity);
        sendRec.ensure(3 * nt + 4096);
        recvRec.ensure(n_capacity);
        sendPM.ensure(send_capacity);
        recvPM.ensure(n_capacity);
        zRange.ensure(2 * kMaxRanks);
        bounds.ensure(8);
        destCountD.ensure(kMaxRanks);
        destStartD.ensure(kMaxRanks);
        minmax.ensure(2);
        // every buffer the slab segments use, at its worst case: a recorded
        // segment must not allocate (g_segment_capture)
        const long long tilesMax = (n_capacity + kTileSize - 1) / kTileSize;
        destTile.ensure((size_t)std::max(G, 1) * (size_t)std::max<long long>(tilesMax, 1));
        set[3].ensure((size_t)n_capacity);
        ws.ensure_cells();
        ws.ensure_particles((size_t)n_capacity);
        if (G > 1) ensure_set_b();
        layerHist.ensure(layer_cap);
        gridRed.ensure(8);
        clsBuf.ensure((size_t)2 * kMaxRanks * kCls);
        spanLo.ensure(kMaxRanks);
        spanHi.ensure(kMaxRanks);
        if (!hostCls) CK(cudaMallocHost(&hostCls, sizeof(int) * 2 * kMaxRanks * kCls));
        if (!ev_cls) CK(cudaEventCreateWithFlags(&ev_cls, cudaEventDisableTiming));
        cur = 0;
        upload_state(nloc, x, xs, v, mass, inv_mass, lambda, level);
    }

    // Caller arrays go straight to the device staging area (DMA from the
    // caller's memory: full PCIe rate when it is pinned), then one kernel
    // unpacks them into the float4 SoA layout.  x_star, lambda and level may
    // be NULL: stepFrame overwrites them before reading them (predict, the
    // first iteration -- every level is >= nMin >= 1 -- and the LOD pass),
    // so a caller that only steps frames need not upload them.  Without
    // levels, stepFrameWithLevels reports them out of range.
    void upload_state(int nn, const float* x, const float* xs, const float* v, const float* mass,
                      const float* inv_mass, const float* lambda, const int32_t* level, bool sync = true) {
        n = nn;
        levels_valid = level != nullptr || nn == 0;
        if (nn == 0) return;
        if (level) {  // branch-free so it vectorises (1M levels in ~0.1 ms)
            const int lo = cfg.n_min, hi = cfg.n_max;
            int bad = 0;
            for (int i = 0; i < nn; ++i) bad |= (level[i] < lo) | (level[i] > hi);
            levels_valid = bad == 0;
        }
        cudaStream_t st = ws.stream;
        float* d = stage.p;
        const size_t n1 = sizeof(float) * (size_t)nn, n3 = 3 * n1;
        CK(cudaMemcpyAsync(d, x, n3, cudaMemcpyHostToDevice, st));
        if (xs) CK(cudaMemcpyAsync(d + 3LL * nn, xs, n3, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d + 6LL * nn, v, n3, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d + 9LL * nn, mass, n1, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d + 10LL * nn, inv_mass, n1, cudaMemcpyHostToDevice, st));
        if (lambda) CK(cudaMemcpyAsync(d + 11LL * nn, lambda, n1, cudaMemcpyHostToDevice, st));
        if (level) CK(cudaMemcpyAsync(d + 12LL * nn, level, n1, cudaMemcpyHostToDevice, st));
        w_agreed = false;  // slab ranks agree on w_mode at their next frame
        scan_inv_mass(nn, inv_mass);  // on the host while the copies run
        w_known = true;
        pending_scan = nullptr;
        const int have = (xs ? 1 : 0) | (lambda ? 2 : 0) | (level ? 4 : 0);
        KL(k_unpack_state<<<blocks(nn, 256), 256, 0, st>>>(nn, d, set[0].view(), have));
        LAUNCH_CHECK();
        if (sync) CK(cudaStreamSynchronize(st));  // the caller may reuse its arrays on return
    }

    bool any_abort(Transport& T) {
        T.allreduce(&ws.ctl.p->abort, 1, RType::I32, ROp::Max, ws.stream);
        int a = 0;
        CK(cudaMemcpyAsync(&a, &ws.ctl.p->abort, sizeof(int), cudaMemcpyDeviceToHost, ws.stream));
        CK(cudaStreamSynchronize(ws.stream));
        return a != 0;
    }

    void run_lod_dist(Transport& T, const float4* X, int nn, long long nAll, const apbf_camera& cam,
                      const apbf_lod_config& lod, int* LV) {
        cudaStream_t st = ws.stream;
        ws.dist.ensure(std::max(nn, 1));
        ws.keys.ensure(std::max(nn, 1));
        const bool dtvs = lod.model == APBF_LOD_DTVS;
        const size_t px = (size_t)cam.width * cam.height;
        if (dtvs) {
            ws.depth.ensure(px);
            ws.rays.ensure(px);
            ws.raysa.ensure(px);
        }
        seg_begin(segLod);  // (buffers sized above: the recording allocates nothing)
        if (dtvs) {
            const CamFrame f = make_frame(cam);
            launch_pdl(k_splat_prep, (unsigned)(blocks((long long)px, 256)), 256, 0, st, f, ws.depth.p, ws.rays.p, ws.raysa.p);
            launch_pdl(k_splat, (unsigned)(blocks(nn, 256)), 256, 0, st, nn, X, radius, f, ws.depth.p, ws.rays.p, ws.raysa.p);
            T.allreduce(ws.depth.p, px, RType::I32, ROp::Min, st);  // positive float bits: int order
            launch_pdl(k_dtvs_gap, (unsigned)(blocks(nn, 256)), 256, 0, st, nn, X, radius, f, ws.depth.p, ws.dist.p,
                                                         ws.keys.p, ws.ctl.p);
            T.allreduce(&ws.ctl.p->sample_count, 1, RType::I32, ROp::Sum, st);
        } else {
            launch_pdl(k_dtc_dist, (unsigned)(blocks(nn, 256)), 256, 0, st, nn, X, cam.eye[0], cam.eye[1], cam.eye[2],
                                                         ws.dist.p, ws.keys.p);
        }
        if (lod.auto_range) {
            launch_pdl(k_rs_init, (unsigned)(1), 1024, 0, st, ws.rs.p, ws.ctl.p, (int)nAll, dtvs ? 1 : 0);
            const int hb = std::min(blocks(nn, 256), 16 * 148);
            for (int pass = 0; pass < 3; ++pass) {
                launch_pdl(k_rs_hist, (unsigned)(hb), 256, 0, st, nn, ws.keys.p, ws.rs.p, pass);
                T.allreduce(&ws.rs.p->hist[0][0], 4 * 2048, RType::U32, ROp::Sum, st);
                launch_pdl(k_rs_select, (unsigned)(1), 1024, 0, st, ws.rs.p, pass);
            }
        }
        launch_pdl(k_lod_params, (unsigned)(1), 1, 0, st, ws.rs.p, ws.ctl.p, lod.auto_range, lod.d_min, lod.d_max, dtvs ? 1 : 0);
        launch_pdl(k_lod_map, (unsigned)(blocks(nn, 256)), 256, 0, st, nn, ws.ctl.p, ws.dist.p, ws.keys.p, dtvs ? 1 : 0,
                                                     lod.n_min, lod.n_max, LV);
        LAUNCH_CHECK();
        seg_end(segLod);
    }

    cudaStream_t comm_stream = nullptr;  // slab mode: the x* halo exchange (overlapped)
    cudaStream_t lod_stream = nullptr;   // the frame's LOD pass, beside the first predict + grid
    cudaEvent_t ev_lod_fork = nullptr, ev_lod_join = nullptr;
    cudaEvent_t ev_halo_ready = nullptr, ev_halo_done = nullptr;

    // APBF_SLAB_TRACE=1: host enqueue time vs device time of the slab frame's
    // phases on stderr (where the decomposition's overhead goes).
    struct TracePt {
        const char* what;
        std::chrono::steady_clock::time_point host;
        cudaEvent_t ev;
    };
    std::vector<TracePt> trace_;
    bool slab_trace = std::getenv("APBF_SLAB_TRACE") != nullptr;
    void tmark(const char* what) {
        if (!slab_trace || capturing) return;
        TracePt t{what, std::chrono::steady_clock::now(), nullptr};
        CK(cudaEventCreate(&t.ev));
        CK(cudaEventRecord(t.ev, ws.stream));
        trace_.push_back(t);
    }
    void tflush() {
        if (!slab_trace || trace_.empty()) return;
        CK(cudaEventSynchronize(trace_.back().ev));
        for (size_t k = 1; k < trace_.size(); ++k) {
            float d = 0.f;
            cudaEventElapsedTime(&d, trace_[k - 1].ev, trace_[k].ev);
            const double hms = std::chrono::duration<double, std::milli>(trace_[k].host - trace_[k - 1].host).count();
            std::fprintf(stderr, "[slab] %-22s host %.3f ms  device %.3f ms\n", trace_[k].what, hms, d);
        }
        for (auto& t : trace_) cudaEventDestroy(t.ev);
        trace_.clear();
    }

    // Device capacity of the global layer histogram (grown on need_layers).
    int layer_cap = 4096;
    DBuf<int> spanLo, spanHi;  // metrics: per-rank metrics-grid layer spans
    DBuf<int> clsBuf;            // per-destination record classes: [sent G*kCls | received G*kCls]
    int* clsSend = nullptr;
    int* clsRecv = nullptr;
    DBuf<int> gridRed;           // [~abort, lo(3), ~hi(3)]: the grid's one MIN all-reduce
    int* hostCls = nullptr;      // pinned [send G*kCls | recv G*kCls] (an async read: the
                                 // host keeps enqueueing while it lands)

    // The per-destination totals and classes of an exchange: sent on the
    // stream ahead of the records (kCls ints per peer), then ONE host
    // synchronisation reads what this rank sends and receives together with
    // the (already all-reduced) abort flags.  Returns false on abort.
    // Slab-frame segments recorded into CUDA graphs (transports whose
    // collectives only enqueue stream work: NCCL).  Each substep re-records
    // its segment with that substep's sizes and updates the instantiated
    // graph in place (cudaGraphExecUpdate; a fresh instantiate when the
    // topology changed), then launches it: one launch instead of ~20 short
    // eager ones.  The loopback transport synchronises on the host inside its
    // collectives, so it runs the same code eagerly.  APBF_SLAB_GRAPHS=0 (or
    // APBF_GRAPHS=0, or APBF_SLAB_TRACE) records nothing.
    // A segment whose recordings keep changing topology (every update fails
    // and re-instantiates while the GPU waits) goes back to eager launches
    // after kSegMaxFails consecutive failures.
    static constexpr int kSegMaxFails = 8;
    struct SegGraph {
        cudaGraphExec_t exec = nullptr;
        bool active = false;  // this occurrence is being recorded
        bool off = false;     // recording abandoned (kSegMaxFails)
        int fails = 0;        // consecutive failed in-place updates
        SegGraph() = default;
        SegGraph(const SegGraph&) = delete;
        SegGraph& operator=(const SegGraph&) = delete;
        ~SegGraph() {
            if (exec) cudaGraphExecDestroy(exec);
        }
    };
    SegGraph segLod, segPre, segPost, segIter, segMetPre, segMetPost;
    bool seg_on = false;
    bool slab_graphs = [] {
        const char* e = std::getenv("APBF_SLAB_GRAPHS");
        return !(e && e[0] == '0');
    }();
    void seg_begin(SegGraph& sg) {
        sg.active = seg_on && !sg.off;
        if (!sg.active) return;
        CK(cudaStreamBeginCapture(ws.stream, cudaStreamCaptureModeThreadLocal));
        capturing = true;
        g_segment_capture = true;
    }
    void seg_end(SegGraph& sg) {
        if (!sg.active) return;
        sg.active = false;
        capturing = false;
        g_segment_capture = false;
        cudaGraph_t g = nullptr;
        CK(cudaStreamEndCapture(ws.stream, &g));
        if (sg.exec) {
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(sg.exec, g, &info) != cudaSuccess) {
                (void)cudaGetLastError();
                cudaGraphExecDestroy(sg.exec);
                sg.exec = nullptr;
                if (++sg.fails >= kSegMaxFails) sg.off = true;  // (this occurrence still runs)
            } else {
                sg.fails = 0;
            }
        }
        cudaError_t e = cudaSuccess;
        if (!sg.exec) e = cudaGraphInstantiate(&sg.exec, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        CK(cudaGraphLaunch(sg.exec, ws.stream));
    }
    // An exception while recording: leave capture mode, drop the recording.
    void seg_cancel() {
        for (SegGraph* sg : {&segLod, &segPre, &segPost, &segIter, &segMetPre, &segMetPost}) sg->active = false;
        if (!g_segment_capture) return;
        capturing = false;
        g_segment_capture = false;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(ws.stream, &g);
        if (g) cudaGraphDestroy(g);
        (void)cudaGetLastError();
    }

    // Split in two: exchange_classes_begin enqueues the exchange and the
    // reads and records ev_cls; the caller then enqueues the device-sized
    // work that does not need the host (the destination expansion and the
    // record pack) so that the GPU keeps running while the host waits in
    // exchange_classes_end.
    cudaEvent_t ev_cls = nullptr;
    void exchange_classes_begin(Transport& T, int ncls) {
        const int G = T.size(), g = T.rank();
        cudaStream_t st = ws.stream;
        std::vector<const void*> sp(G);
        std::vector<void*> rp(G);
        std::vector<size_t> sb(G), rb(G);
        for (int q = 0; q < G; ++q) {
            sp[q] = clsSend + (size_t)q * kCls;
            rp[q] = clsRecv + (size_t)q * kCls;
            sb[q] = rb[q] = sizeof(int) * ncls;
        }
        CK(cudaMemcpyAsync(clsRecv + (size_t)g * kCls, clsSend + (size_t)g * kCls, sizeof(int) * ncls,
                           cudaMemcpyDeviceToDevice, st));
        T.alltoallv(sp.data(), sb.data(), rp.data(), rb.data(), st);
        CK(cudaMemcpyAsync(hostCls, clsSend, sizeof(int) * 2 * G * kCls, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ws.h_ctl, ws.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        rec(ev_cls);  // (an external event node while a segment is recorded)
    }
    bool exchange_classes_end() {
        CK(cudaEventSynchronize(ev_cls));
        return !ws.h_ctl->abort;
    }
    // The stable expansion of destMask[0, n) by destination into sendIdx,
    // per-destination counts and starts on the device.
    void expand_dest(int G) {
        cudaStream_t st = ws.stream;
        const int tiles = std::max(1, (n + kTileSize - 1) / kTileSize);
        destTile.ensure((size_t)G * tiles);
        KL(k_mask_tile_counts<<<tiles, kTileThreads, 0, st>>>(n, destMask.p, G, tiles, destTile.p));
        KL(k_mask_scan<<<G, 1024, 0, st>>>(tiles, destTile.p, destCountD.p));
        KL(k_dest_starts<<<1, 32, 0, st>>>(destCountD.p, G, destStartD.p));
        KL(k_mask_scatter<<<tiles, kTileThreads, 0, st>>>(n, destMask.p, G, tiles, destTile.p, destStartD.p,
                                                        sendIdx.p));
    }

    // One slab frame.  Per substep the host synchronises ONCE (after the
    // class exchange): every size the rest of the substep needs -- records
    // in and out, the local count, the owned range, the layer-1 ghost range
    // and the two halo send ranges -- follows from the class counts.  The
    // grid, the partition and the destination masks stay on the device; a
    // failure anywhere aborts through the device flags, which are all-reduced
    // before that synchronisation, so every rank leaves the collective
    // sequence at the same point.
    void run_frame_dist(Transport& T, long long nAll, bool assign_lod, const apbf_camera* cam,
                        const apbf_lod_config* lod) {
        seg_on = use_graphs && slab_graphs && T.capturable() && !slab_trace;
        try {
            run_frame_dist_body(T, nAll, assign_lod, cam, lod);
        } catch (...) {
            seg_cancel();
            throw;
        }
    }
    void run_frame_dist_body(Transport& T, long long nAll, bool assign_lod, const apbf_camera* cam,
                             const apbf_lod_config* lod) {
        const int G = T.size(), g = T.rank();
        cudaStream_t st = ws.stream;
        Ctl* ctl = ws.ctl.p;
        const SolverConsts sc = consts();
        const int nMax = cfg.n_max;
        localPre.assign(cfg.substeps, 0);
        localPost.assign(cfg.substeps, 0);
        layerHist.ensure(layer_cap);
        gridRed.ensure(8);
        clsBuf.ensure((size_t)2 * kMaxRanks * kCls);
        clsSend = clsBuf.p;
        clsRecv = clsBuf.p + (size_t)G * kCls;
        CK(cudaEventRecord(ev[0], st));
        tmark("start");
        launch_pdl(k_frame_begin, (unsigned)(1), 1, 0, st, ctl);
        if (assign_lod) {
            if (cfg.mode == APBF_MODE_PBF) {
                KL(k_fill_int<<<blocks(n, 256), 256, 0, st>>>(set[cur].LV.p, n, nMax));
            } else {
                apbf_lod_config lc = *lod;
                lc.n_min = cfg.n_min;
                lc.n_max = cfg.n_max;
                run_lod_dist(T, set[cur].X.p, n, nAll, *cam, lc, set[cur].LV.p);
            }
        }
        tmark("lod");
        for (int s = 0; s < cfg.substeps; ++s) {
            NvtxRange range("apbf slab substep");
            localPre[s] = n;
            // src: this rank's state (old, then new after the finalize); rec:
            // the unsorted local set the records land in; dst: the sorted set
            StateSet src = set[cur].view(), rec = set[cur ^ 1].view(), dst = set[3].view();
            seg_begin(segPre);  // segment 1: everything up to the host synchronisation
            launch_pdl(k_substep_reset, (unsigned)(1), 1, 0, st, ctl);
            launch_pdl(k_predict, (unsigned)(blocks(n, kAabbBlock)), kAabbBlock, 0, st, n, src.X, src.V, src.V, src.XS, src.XS, dt,
                                                      cfg.gravity[0], cfg.gravity[1], cfg.gravity[2], ctl, s);
            // global grid: AABB all-reduce (ordered ints), identical params
            // everywhere; the abort flag travels alongside
            KL(k_grid_reduce_pack<<<1, 1, 0, st>>>(ctl, 0, gridRed.p));
            T.allreduce(gridRed.p, 7, RType::I32, ROp::Min, st);
            // (unpack + grid parameters, and the layer histogram and class
            // counters cleared, in one launch)
            KL(k_grid_unpack_params<<<1, 256, 0, st>>>(ctl, 0, gridRed.p, cfg.h, cfg.h, layerHist.p, layer_cap,
                                                      clsSend, G * kCls));
            // slabs: equal-work split (sum of 1 + level per layer) of the
            // global histogram, computed on the device
            KL(k_layer_hist<<<std::max(1, std::min(blocks(n, 256 * kHistItems), 148 * 8)), 256, 0, st>>>(n, src.XS, src.LV, ctl, 0, cfg.h, layerHist.p,
                                                          layer_cap));
            T.allreduce(layerHist.p, layer_cap, RType::I32, ROp::Sum, st);
            KL(k_slab_partition<<<1, 256, sizeof(int) * std::min(layer_cap, kPartSmem), st>>>(
                layerHist.p, ctl, G, 2, zRange.p, layer_cap));
            // migration + halo in one all-to-all, previous global order kept
            KL(k_dest_mask<<<std::max(1, std::min(blocks(n, 256), 148 * 4)), 256, 0, st>>>(n, src.XS, ctl, 0, cfg.h, zRange.p, zRange.p + G,
                                                         G, 2, destMask.p, clsSend));
            tmark("pre-exchange");
            exchange_classes_begin(T, kCls);
            // device-sized, ahead of the host synchronisation: expansion by
            // destination and the records for the other ranks (this rank's
            // own segment stays in the old state: SelfMap)
            expand_dest(G);
            if (G > 1)
                KL(k_pack_recs<<<std::min(blocks(n, 256), 148 * 8), 256, 0, st>>>(sendIdx.p, src, sendRec.p,
                                                                                 destCountD.p, destStartD.p, G, g));
            seg_end(segPre);
            if (!exchange_classes_end()) break;  // the substep's one host synchronisation
            tmark("class sync");
            // sizes: what goes where, and this rank's layout after the sort
            const int* sendC = hostCls;
            const int* recvC = hostCls + (size_t)G * kCls;
            std::vector<long long> sendCnt(G), sendStart(G), recvCnt(G), roff(G);
            long long nsend = 0, nLocal = 0;
            long long lowG0 = 0, lowG1 = 0, own2lo = 0, hiG0 = 0, hiG1 = 0, ownHi2 = 0;
            for (int q = 0; q < G; ++q) {
                sendCnt[q] = sendC[q * kCls];
                sendStart[q] = nsend;
                nsend += sendCnt[q];
                recvCnt[q] = recvC[q * kCls];
                roff[q] = nLocal;
                nLocal += recvCnt[q];
                const int* c = recvC + q * kCls;
                lowG0 += c[1];   // layer lo-2
                lowG1 += c[2];   // layer lo-1
                own2lo += c[3] + c[4];  // layers lo, lo+1
                ownHi2 += c[5] + c[6];  // layers hi-2, hi-1
                hiG0 += c[7];    // layer hi
                hiG1 += c[8];    // layer hi+1
            }
            // cannot happen (set_state_local sizes for the worst case); an
            // internal error, not an input condition
            if (nLocal > n_capacity || nsend > 3 * std::max<long long>(n_global_, 1) + 4096)
                fail(APBF_ERR_RUNTIME, "internal: slab exchange larger than its worst-case capacity");
            const int ownB = (int)(lowG0 + lowG1), l1B = (int)lowG0;
            const int ownE = (int)(nLocal - hiG0 - hiG1), l1E = (int)(nLocal - hiG1);
            const int lowEnd = (int)(ownB + own2lo), highB = (int)(ownE - ownHi2);
            seg_begin(segPost);  // segment 2: records, local sort, bucketing, lists
            std::vector<const void*> sp(G);
            std::vector<void*> rp(G);
            std::vector<size_t> sb(G), rb(G);
            for (int q = 0; q < G; ++q) {
                sp[q] = sendRec.p + sendStart[q];
                sb[q] = sizeof(Rec) * sendCnt[q];
                rp[q] = recvRec.p + roff[q];
                rb[q] = sizeof(Rec) * recvCnt[q];
            }
            T.alltoallv(sp.data(), sb.data(), rp.data(), rb.data(), st);
            const int nL = (int)nLocal;
            if (nL > sendCnt[g])
                KL(k_unpack_recs<<<blocks(nL, 256), 256, 0, st>>>(nL, recvRec.p, rec, (int)roff[g],
                                                                (int)(roff[g] + sendCnt[g])));
            // the unsorted local set: rec, except its own segment [roff_g,
            // roff_g + sendCnt_g), which is read from the old state
            SelfMap self;
            self.idx = sendIdx.p + sendStart[g];
            self.off = (int)roff[g];
            self.cnt = (int)sendCnt[g];
            self.from = src;
            tmark("exchange");
            // local stable sort by global cell == global order restricted
            // (contacts of the owned layers counted on the way; grid params
            // already set for this grid above)
            ws.run_grid(0, rec.XS, nL, cfg.h, cfg.h, scene.n > 0, radius, zRange.p + g, zRange.p + G + g, false,
                        self);
            const int tilesL = std::max(1, (nL + kTileSize - 1) / kTileSize);
            const int smemG = (nMax + 1) * (int)sizeof(int);
            launch_pdl(k_gather, (unsigned)(tilesL), kTileThreads, smemG, st, nL, ctl, ws.perm.p, rec, dst, nMax, tilesL,
                                                           tileCount.p, 3, self);
            const int nOwn = ownE - ownB;
            // iteration order over owned + layer-1 ghosts (lambda is computed
            // redundantly for the latter), outer ghosts never active.  With
            // neighbours the particles split into two iteration sets: A, the
            // interior owned layers [lo+2, hi-2), whose lambda never reads a
            // ghost; B, the layer-1 ghosts and the owned layers the halo sends
            // (lo, lo+1, hi-2, hi-1).  Per iteration: lambda(A) needs no halo;
            // lambda(B) waits for the previous halo; delta-p(B) produces the
            // x* the next halo sends, which then runs on comm_stream while
            // delta-p(A) and the next lambda(A) compute.  (Same per-particle
            // lists and sums: bitwise the single-set results.)
            const int a0 = g > 0 ? lowEnd : ownB, a1 = g < G - 1 ? highB : ownE;
            const bool split = G > 1 && !cfg.record_residuals && a0 < a1;
            // (the first bucket also sums the owned levels: the rank's particle-iterations)
            auto bucket = [&](int b, int e, int xb, int xe, bool total) {
                KL(k_mask_level_tiles<<<tilesL, kTileThreads, smemG, st>>>(nL, ctl, dst.LV, b, e, xb, xe, LVo.p,
                                                                          nMax, tilesL, tileCount.p,
                                                                          total ? ownB : 0, total ? ownE : 0));
                launch_pdl(k_level_scan, (unsigned)(nMax + 1), 1024, 0, st, ctl, tilesL, tileCount.p, levelCount.p);
                launch_pdl(k_level_finish, (unsigned)(1), 32, 0, st, ctl, nL, nMax, levelCount.p, activeCount.p, bucketStart.p, 0);
                launch_pdl(k_level_scatter, (unsigned)(tilesL), kTileThreads, 9 * smemG, st, nL, ctl, LVo.p, nMax, tilesL,
                                                                           tileCount.p, bucketStart.p, order.p);
                launch_build_lists(nL, dst);
            };
            if (split) {
                ensure_set_b();
                bucket(a0, a1, 0, 0, true);  // set A
                swap_sets();
                bucket(l1B, l1E, a0, a1, false);  // set B
                swap_sets();
            } else {
                bucket(l1B, l1E, 0, 0, true);
            }
            // pre-stabilization of every local copy with level < S (owners and
            // ghost copies compute the same values); errors from owned only
            if (S > 1)
                KL(k_prestabilize_slots<<<blocks(nL, 256), 256, 0, st>>>(nL, ctl, S, dst.LV, dst.XS, dst.X,
                                                                       ws.scene.p, radius, cfg.stab_iterations,
                                                                       s, ownB, ownE));
            LAUNCH_CHECK();
            seg_end(segPost);
            tmark("sort+lists");
            ownB_ = ownB;
            ownE_ = ownE;
            n_iter = nL;
            float4* P[2] = {dst.XS, PB.p};
            if (split && !comm_stream) {
                CK(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
                CK(cudaEventCreateWithFlags(&ev_halo_ready, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_halo_done, cudaEventDisableTiming));
            }
            // segment 3: the iterations (the halo forks onto comm_stream and
            // joins back inside the recording) and the finalize
            seg_begin(segIter);
            for (int it = 1; it <= nMax; ++it) {
                const float4* Pc = P[(it - 1) & 1];
                float4* Pn = P[it & 1];
                if (split) {
                    launch_solver_pair(it, s, Pc, Pn, dst, sc, -1, 1);  // lambda(A)
                    if (it > 1) CK(cudaStreamWaitEvent(st, ev_halo_done, 0));
                    swap_sets();
                    launch_solver_pair(it, s, Pc, Pn, dst, sc, -1, 3);  // lambda(B), delta-p(B)
                    swap_sets();
                    CK(cudaEventRecord(ev_halo_ready, st));
                    CK(cudaStreamWaitEvent(comm_stream, ev_halo_ready, 0));
                } else {
                    launch_solver_pair(it, s, Pc, Pn, dst, sc, -1);
                }
                if (cfg.record_residuals) {
                    CK(cudaMemsetAsync(resid.p + (size_t)s * nMax + (it - 1), 0, sizeof(double), st));
                    launch_residual(nL, it, Pn, sc, resid.p + (size_t)s * nMax + (it - 1), ownB, ownE);
                }
                // halo: owned x* of the 2 boundary layers to each neighbour
                std::vector<const void*> hs(G, nullptr);
                std::vector<void*> hr(G, nullptr);
                std::vector<size_t> hsb(G, 0), hrb(G, 0);
                if (g > 0) {
                    hs[g - 1] = Pn + ownB;
                    hsb[g - 1] = sizeof(float4) * (size_t)(lowEnd - ownB);
                    hr[g - 1] = Pn;
                    hrb[g - 1] = sizeof(float4) * (size_t)ownB;
                }
                if (g < G - 1) {
                    hs[g + 1] = Pn + highB;
                    hsb[g + 1] = sizeof(float4) * (size_t)(ownE - highB);
                    hr[g + 1] = Pn + ownE;
                    hrb[g + 1] = sizeof(float4) * (size_t)(nL - ownE);
                }
                if (split) {
                    T.alltoallv(hs.data(), hsb.data(), hr.data(), hrb.data(), comm_stream);
                    CK(cudaEventRecord(ev_halo_done, comm_stream));
                    launch_solver_pair(it, s, Pc, Pn, dst, sc, -1, 2);  // delta-p(A), overlapping the halo
                } else {
                    T.alltoallv(hs.data(), hsb.data(), hr.data(), hrb.data(), st);
                }
            }
            if (split) CK(cudaStreamWaitEvent(st, ev_halo_done, 0));  // the last halo landed
            tmark("iterations");
            ownB_ = 0;
            ownE_ = 0x7fffffff;
            float4* Pf = P[nMax & 1];
            // finalize the owned particles into the front of the other set:
            // in order, this rank's state for the next substep
            if (nOwn > 0)
                KL(k_finalize_owned<<<blocks(nOwn, 256), 256, 0, st>>>(nOwn, ownB, ctl, Pf, dst, src, dt, cap, s));
            LAUNCH_CHECK();
            seg_end(segIter);
            n = nOwn;
            localPost[s] = n;
            // (the new state is back in set[cur], which the old state was read from)
            tmark("finalize+copy");
        }
        CK(cudaEventRecord(ev[5], st));
        T.allreduce(&ctl->abort, 1, RType::I32, ROp::Max, st);
        if (metrics) run_metrics_dist(T);
        T.allreduce(&ctl->total_iterations, 1, RType::I64, ROp::Sum, st);
        T.allreduce(&ctl->contacts, 1, RType::I64, ROp::Sum, st);
        T.allreduce(&ctl->list_overflow, 1, RType::I32, ROp::Max, st);
        T.allreduce(&ctl->abort, 1, RType::I32, ROp::Max, st);
        CK(cudaEventRecord(ev[6], st));
        tmark("metrics+reduce");
        ws.read_ctl();
        tflush();
    }

    // allDensities(x) across slabs: owned particles plus every particle of
    // other ranks within one metrics-grid layer of their layer range.  The
    // ranges are all-reduced on the device; one host synchronisation (the
    // class exchange) gives the sizes.  Skipped (consistently) on abort.
    void run_metrics_dist(Transport& T) {
        const int G = T.size(), g = T.rank();
        cudaStream_t st = ws.stream;
        Ctl* ctl = ws.ctl.p;
        const StateSet cs = set[cur].view();
        spanLo.ensure(kMaxRanks);
        spanHi.ensure(kMaxRanks);
        seg_begin(segMetPre);
        launch_pdl(k_grid_reset, (unsigned)(1), 1, 0, st, ctl, 1);
        launch_pdl(k_aabb, (unsigned)(blocks(n, kAabbBlock)), kAabbBlock, 0, st, n, cs.X, ctl, 1);
        KL(k_grid_reduce_pack<<<1, 1, 0, st>>>(ctl, 1, gridRed.p));
        T.allreduce(gridRed.p, 7, RType::I32, ROp::Min, st);
        KL(k_grid_unpack_params<<<1, 256, 0, st>>>(ctl, 1, gridRed.p, cfg.h, cfg.h, clsSend, G * kCls, nullptr,
                                                  0));
        KL(k_span_init<<<1, 32, 0, st>>>(G, spanLo.p, spanHi.p));
        KL(k_layer_minmax<<<blocks(n, 256), 256, 0, st>>>(n, cs.X, ctl, 1, cfg.h, spanLo.p + g, spanHi.p + g));
        T.allreduce(spanLo.p, G, RType::I32, ROp::Min, st);
        T.allreduce(spanHi.p, G, RType::I32, ROp::Max, st);
        KL(k_metrics_ranges<<<1, 32, 0, st>>>(G, g, spanLo.p, spanHi.p));
        KL(k_dest_mask<<<std::max(1, std::min(blocks(n, 256), 148 * 4)), 256, 0, st>>>(n, cs.X, ctl, 1, cfg.h, spanLo.p, spanHi.p, G, 1,
                                                     destMask.p, clsSend));
        exchange_classes_begin(T, 1);
        expand_dest(G);
        KL(k_pack_pm<<<std::min(blocks(n, 256), 148 * 8), 256, 0, st>>>(sendIdx.p, cs.X, cs.XS, sendPM.p,
                                                                       destCountD.p, destStartD.p, clsRecv, G, g,
                                                                       recvPM.p, ownedFlag.p));
        seg_end(segMetPre);
        if (!exchange_classes_end()) return;
        const int* sendC = hostCls;
        const int* recvC = hostCls + (size_t)G * kCls;
        std::vector<long long> sendCnt(G), sendStart(G), recvCnt(G), roff(G);
        long long nsend = 0, nM = 0;
        for (int q = 0; q < G; ++q) {
            sendCnt[q] = sendC[q * kCls];
            sendStart[q] = nsend;
            nsend += sendCnt[q];
            recvCnt[q] = recvC[q * kCls];
            roff[q] = nM;
            nM += recvCnt[q];
        }
        if (nM > n_capacity || nsend > send_capacity)  // cannot happen: see set_state_local
            fail(APBF_ERR_RUNTIME, "internal: slab metrics exchange larger than its worst-case capacity");
        seg_begin(segMetPost);
        std::vector<const void*> sp(G);
        std::vector<void*> rp(G);
        std::vector<size_t> sb(G), rb(G);
        for (int q = 0; q < G; ++q) {
            sp[q] = sendPM.p + sendStart[q];
            sb[q] = sizeof(float4) * sendCnt[q];
            rp[q] = recvPM.p + roff[q];
            rb[q] = sizeof(float4) * recvCnt[q];
        }
        T.alltoallv(sp.data(), sb.data(), rp.data(), rb.data(), st);
        const int nm = (int)nM;
        ws.run_grid(1, recvPM.p, nm, cfg.h, cfg.h, false, radius, nullptr, nullptr, false);
        launch_pdl(k_gather_posmass, (unsigned)(blocks(nm, 256)), 256, 0, st, nm, ctl, ws.perm.p, recvPM.p, recvPM.p, sortedPM.p);
        KL(k_gather_int<<<blocks(nm, 256), 256, 0, st>>>(nm, ws.perm.p, ownedFlag.p, ownedSorted.p));
        KL(k_density_stats_owned<<<blocks(nm, 256), 256, 0, st>>>(nm, ctl, sortedPM.p, ownedSorted.p,
                                                                ws.cellCount.p, make_kernel_consts(cfg.h)));
        LAUNCH_CHECK();
        T.allreduce(&ctl->rho_sum, 1, RType::F64, ROp::Sum, st);
        T.allreduce(&ctl->rho_min_ord, 1, RType::I32, ROp::Min, st);
        T.allreduce(&ctl->rho_max_ord, 1, RType::I32, ROp::Max, st);
        seg_end(segMetPost);
    }

    void frame_dist(bool assign_lod, const apbf_camera* cam, const apbf_lod_config* lod, int frame_index,
                    apbf_frame_stats* out) {
        Transport& T = *transport;
        const int G = T.size(), g = T.rank();
        if (G > kMaxRanks) fail(APBF_ERR_INVALID_ARGUMENT, "too many slab ranks");
        if (observer) fail(APBF_ERR_INVALID_ARGUMENT, "iteration observer is not available with slab decomposition");
        if (cur == 2) {  // left there by single-rank frames: the slab path uses 0/1 (and 3)
            copy_set(set[0], set[2]);
            cur = 0;
        }
        const long long nAll = n_global_;  // particles are conserved: fixed at set_state
        agree_uniform_w(T);
        if (assign_lod && cfg.mode == APBF_MODE_APBF) {
            apbf_lod_config lc = *lod;
            validate_lod(lc);
            if (nAll > 0 && lc.model == APBF_LOD_DTVS) {
                if (!(radius > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "splat radius must be positive");
                (void)make_frame(*cam);
            }
        }
        apbf_frame_stats stt;
        std::memset(&stt, 0, sizeof stt);
        stt.frame = frame_index;
        if (nAll > 0) {
            const int start_set = cur;
            const int start_n = n;
            copy_set(set[2], set[start_set]);
            for (int attempt = 0;; ++attempt) {
                run_frame_dist(T, nAll, assign_lod, cam, lod);
                // the retry conditions are all-reduced (list_overflow) or global
                // (need_layers comes from the global grid): every rank retries
                const bool lists = ws.h_ctl->list_overflow != 0, layers = ws.h_ctl->need_layers > layer_cap;
                if (!lists && !layers) break;
                if (attempt > 6) fail(APBF_ERR_RUNTIME, "neighbor list overflow");
                cur = start_set;
                n = start_n;
                copy_set(set[cur], set[2]);
                if (lists) grow_lists(ws.h_ctl->list_alloc, ws.h_ctl->list_alloc_fb);
                if (layers) layer_cap = std::max(2 * layer_cap, ws.h_ctl->need_layers + 16);
            }
            const Ctl& c = *ws.h_ctl;
            if (c.abort || c.runtime_error || c.slab_error) {
                // all-or-nothing, as on one GPU: the rank's frame-start state
                // from the backup set (levels as before the frame's LOD)
                cur = start_set;
                n = start_n;
                copy_set(set[cur], set[2]);
                CK(cudaStreamSynchronize(ws.stream));
            }
            if (c.runtime_error) fail(APBF_ERR_RUNTIME, "grid cell count exceeds limit; domain blew up");
            if (c.slab_error) fail(APBF_ERR_RUNTIME, "too few grid layers for the slab decomposition");
            // global first error: (substep, iteration, pass, global index) -- only
            // when the frame aborted (the abort flag is already all-reduced)
            const long long NONE = 0x7fffffffffffffffLL;
            long long key = NONE;
            if (c.abort) exchange_prefixes(T);
            for (int sl = 0; c.abort && sl < kNumPassSlots; ++sl) {
                if (c.bad[sl] == 0x7fffffff) continue;
                const int sub = std::max(0, c.bad_substep[sl]);
                const int itr = (sl == kPassLambda || sl == kPassApply) ? std::max(0, c.bad_iter[sl])
                                : (sl >= kPassFinalizeV ? cfg.n_max + 1 : 0);
                const long long gidx = (sl == kPassPredict ? prefixPre[sub] : prefixPost[sub]) + c.bad[sl];
                const long long seq = ((long long)sub * (cfg.n_max + 2) + itr) * 8 + sl;
                const long long k = (seq << 32) | gidx;
                key = std::min(key, k);
            }
            if (c.abort) {
                long long* dkey = reinterpret_cast<long long*>(bounds.p);
                CK(cudaMemcpyAsync(dkey, &key, sizeof(key), cudaMemcpyHostToDevice, ws.stream));
                T.allreduce(dkey, 1, RType::I64, ROp::Min, ws.stream);
                CK(cudaMemcpyAsync(&key, dkey, sizeof(key), cudaMemcpyDeviceToHost, ws.stream));
                CK(cudaStreamSynchronize(ws.stream));
            }
            if (key != NONE) {
                static const char* names[kNumPassSlots] = {"predict", "prestabilize", "lambda",
                                                           "apply",   "finalize",     "finalize"};
                static const char* details[kNumPassSlots] = {
                    "non-finite predicted position", "non-finite predicted position", "non-finite lambda",
                    "non-finite predicted position", "non-finite velocity",           "non-finite position"};
                const int sl = (int)((key >> 32) & 7);
                numerical(names[sl], (int)(key & 0xffffffffLL), details[sl]);
            }
            if (c.abort) fail(APBF_ERR_RUNTIME, "frame aborted without a recorded cause");
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[0], ev[5]));
            stt.wall_ms = ms;
            stt.total_iterations = (int64_t)c.total_iterations;
            stt.contacts = (int64_t)c.contacts;
            if (metrics) {
                const double scale = 100.0 / (double)cfg.rest_density;
                stt.avg_density_pct = c.rho_sum / (double)nAll * scale;
                stt.min_density_pct = (double)ord2f(c.rho_min_ord) * scale;
                stt.max_density_pct = (double)ord2f(c.rho_max_ord) * scale;
            }
            (void)g;
        }
        if (out) {
            double* r = out->residuals;
            int rc = out->residuals_capacity;
            *out = stt;
            out->residuals = r;
            out->residuals_capacity = rc;
        }
    }
};

// =============================================================== C-ABI

extern "C" {

int32_t apbf_gpu_abi_version(void) { return APBF_GPU_ABI_VERSION; }

int32_t apbf_gpu_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

static void validate_config(const apbf_solver_config* c) {
    if (c->n_min < 1 || c->n_max < c->n_min)
        fail(APBF_ERR_INVALID_ARGUMENT, "iteration range requires 1 <= n_min <= n_max");
    if (!(c->dt_frame > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "dt_frame must be positive");
    if (c->substeps < 1) fail(APBF_ERR_INVALID_ARGUMENT, "substeps must be at least 1");
    if (!(c->rest_density > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "rest density must be positive");
    if (!(c->h > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "smoothing length must be positive");
    if (c->epsilon < 0.0f) fail(APBF_ERR_INVALID_ARGUMENT, "epsilon must be non-negative");
    if (c->stab_iterations < 0) fail(APBF_ERR_INVALID_ARGUMENT, "stab iterations must be non-negative");
    if (c->stab_threshold != 0 && (c->stab_threshold < 1 || c->stab_threshold > c->n_max))
        fail(APBF_ERR_INVALID_ARGUMENT, "stab threshold must lie in [1, n_max]");
    if (c->particle_radius < 0.0f) fail(APBF_ERR_INVALID_ARGUMENT, "particle radius must be non-negative");
    if (c->velocity_cap < 0.0f) fail(APBF_ERR_INVALID_ARGUMENT, "velocity cap must be non-negative");
    if (!finite3h(c->gravity)) fail(APBF_ERR_INVALID_ARGUMENT, "gravity must be finite");
    if (c->mode != APBF_MODE_PBF && c->mode != APBF_MODE_APBF)
        fail(APBF_ERR_INVALID_ARGUMENT, "unknown solver mode");
    if (c->n_max > kMaxLevels) fail(APBF_ERR_INVALID_ARGUMENT, "n_max above the GPU level-table limit (4096)");
}

int32_t apbf_gpu_solver_create(const apbf_solver_config* cfg, const apbf_sdf_primitive* prims,
                               int32_t n_prims, float gradient_step, int32_t device,
                               apbf_gpu_solver** out, apbf_error* err) {
    return guarded(err, [&] {
        *out = nullptr;
        validate_config(cfg);
        const Scene sc = make_scene(prims, n_prims, gradient_step);
        int count = 0;
        CK(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(APBF_ERR_INVALID_ARGUMENT, "CUDA device out of range");
        CK(cudaSetDevice(device));
        *out = new apbf_gpu_solver(*cfg, sc, device);
    });
}

void apbf_gpu_solver_destroy(apbf_gpu_solver* s) {
    if (!s) return;
    cudaSetDevice(s->ws.device);
    cudaStreamSynchronize(s->ws.stream);
    delete s;
}

int32_t apbf_gpu_set_state(apbf_gpu_solver* s, int32_t n, const float* x, const float* xs,
                           const float* v, const float* mass, const float* inv_mass,
                           const float* lambda, const int32_t* level, apbf_error* err) {
    return guarded(err, [&] {
        if (n < 0) fail(APBF_ERR_INVALID_ARGUMENT, "negative particle count");
        CK(cudaSetDevice(s->ws.device));
        if (n > 0 && (!x || !v || !mass || !inv_mass))
            fail(APBF_ERR_INVALID_ARGUMENT, "x, v, mass and inv_mass are required");
        s->allocate(n);
        s->cur = 0;
        s->upload_state(n, x, xs, v, mass, inv_mass, lambda, level);
    });
}

int32_t apbf_gpu_get_state(apbf_gpu_solver* s, float* x, float* xs, float* v, float* mass,
                           float* inv_mass, float* lambda, int32_t* level, apbf_error* err) {
    return guarded(err, [&] {
        CK(cudaSetDevice(s->ws.device));
        const int n = s->n;
        if (n == 0) return;
        cudaStream_t st = s->ws.stream;
        SetBufs& b = s->set[s->cur];
        const float4* dxs = (s->in_iteration && s->obs_xs) ? s->obs_xs : b.XS.p;
        float* d = s->stage.p;
        KL(k_pack_state<<<blocks(n, 256), 256, 0, st>>>(n, b.view(), dxs, d));
        LAUNCH_CHECK();
        const size_t n1 = sizeof(float) * (size_t)n, n3 = 3 * n1;
        if (x) CK(cudaMemcpyAsync(x, d, n3, cudaMemcpyDeviceToHost, st));
        if (xs) CK(cudaMemcpyAsync(xs, d + 3LL * n, n3, cudaMemcpyDeviceToHost, st));
        if (v) CK(cudaMemcpyAsync(v, d + 6LL * n, n3, cudaMemcpyDeviceToHost, st));
        if (mass) CK(cudaMemcpyAsync(mass, d + 9LL * n, n1, cudaMemcpyDeviceToHost, st));
        if (inv_mass) CK(cudaMemcpyAsync(inv_mass, d + 10LL * n, n1, cudaMemcpyDeviceToHost, st));
        if (lambda) CK(cudaMemcpyAsync(lambda, d + 11LL * n, n1, cudaMemcpyDeviceToHost, st));
        if (level) CK(cudaMemcpyAsync(level, d + 12LL * n, n1, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int32_t apbf_gpu_step_frame_host(apbf_gpu_solver* s, int32_t n, float* x, float* x_star, float* v, float* mass,
                                 float* inv_mass, float* lambda, int32_t* level, const apbf_camera* cam,
                                 const apbf_lod_config* lod, int32_t frame_index, apbf_frame_stats* out,
                                 apbf_error* err) {
    return guarded(err, [&] {
        if (n < 0) fail(APBF_ERR_INVALID_ARGUMENT, "negative particle count");
        if (n > 0 && (!x || !x_star || !v || !mass || !inv_mass || !lambda || !level))
            fail(APBF_ERR_INVALID_ARGUMENT, "every ParticleSet array is required");
        if (s->transport) fail(APBF_ERR_INVALID_ARGUMENT, "step_frame_host runs on one rank");
        CK(cudaSetDevice(s->ws.device));
        s->allocate(n);
        s->cur = 0;
        // what stepFrame reads, x first (the caller's arrays stay untouched
        // until this call returns, so no sync)
        // APBF_E2E_TRACE=1: print where the end-to-end frame spends its time
        static const bool trace = std::getenv("APBF_E2E_TRACE") != nullptr;
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        auto h0 = std::chrono::steady_clock::now();
        if (trace) {
            CK(cudaEventCreate(&t0));
            CK(cudaEventCreate(&t1));
            CK(cudaEventRecord(t0, s->ws.stream));
        }
        s->upload_split(n, x, v, mass, inv_mass, x_star, lambda, level);
        auto h1 = std::chrono::steady_clock::now();
        apbf_gpu_solver::HostOut o{x, x_star, v, mass, inv_mass, lambda, level, false};
        s->host_out = &o;
        try {
            s->frame(true, cam, lod, frame_index, out);
        } catch (...) {
            s->host_out = nullptr;
            if (s->pending_scan) {  // never scanned: the mode is unknown now
                s->pending_scan = nullptr;
                s->w_known = false;
            }
            throw;
        }
        s->host_out = nullptr;
        s->levels_valid = true;
        if (trace) {
            CK(cudaEventRecord(t1, s->copy_stream));
            CK(cudaEventSynchronize(t1));
            auto h2 = std::chrono::steady_clock::now();
            auto el = [&](cudaEvent_t e) {
                float ms = -1.f;
                cudaEventElapsedTime(&ms, t0, e);
                return ms;
            };
            std::fprintf(stderr,
                         "[e2e] host: upload_split %.3f ms, total %.3f ms | device from start: x %.3f, "
                         "inputs %.3f, frame start %.3f, lod %.3f, last reorder %.3f, finalize %.3f, "
                         "metrics %.3f, download done %.3f ms\n",
                         std::chrono::duration<double, std::milli>(h1 - h0).count(),
                         std::chrono::duration<double, std::milli>(h2 - h0).count(), el(s->ev_x),
                         el(s->ev_inputs), el(s->ev[0]), s->phase_timing ? el(s->ev[1]) : -1.f,
                         el(s->ev[7]), el(s->ev[5]), el(s->ev[6]), el(t1));
            cudaEventDestroy(t0);
            cudaEventDestroy(t1);
        }
    });
}

void* apbf_gpu_stream(const apbf_gpu_solver* s) { return (void*)s->ws.stream; }

void* apbf_gpu_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes ? bytes : 1) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void apbf_gpu_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int32_t apbf_gpu_particle_count(const apbf_gpu_solver* s) { return s ? s->n : 0; }

int32_t apbf_gpu_step_frame(apbf_gpu_solver* s, const apbf_camera* cam, const apbf_lod_config* lod,
                            int32_t frame_index, apbf_frame_stats* out, apbf_error* err) {
    return guarded(err, [&] {
        s->frame(true, cam, lod, frame_index, out);
        s->levels_valid = true;
    });
}

int32_t apbf_gpu_step_frame_multi(apbf_gpu_solver* s, int32_t k, const apbf_camera* cams,
                                  const apbf_lod_config* lods, int32_t frame_index, apbf_frame_stats* out,
                                  apbf_error* err) {
    return guarded(err, [&] {
        if (k < 1) fail(APBF_ERR_INVALID_ARGUMENT, "blend requires at least one level array");
        if (s->transport) fail(APBF_ERR_INVALID_ARGUMENT, "multi-camera frames run on one rank");
        CK(cudaSetDevice(s->ws.device));
        const int n = s->n;
        int* LV = s->set[s->cur].LV.p;
        cudaStream_t st = s->ws.stream;
        for (int c = 0; c < k; ++c) {  // assignLevels per camera, then blendLod
            apbf_lod_config lc = lods[c];
            lc.n_min = s->cfg.n_min;  // lc.range = cfg_.range (solver.hpp:254)
            lc.n_max = s->cfg.n_max;
            if (s->cfg.mode == APBF_MODE_APBF) {
                validate_lod(lc);
                if (n > 0 && lc.model == APBF_LOD_DTVS) {
                    if (!(s->radius > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "splat radius must be positive");
                    (void)make_frame(cams[c]);
                }
            }
            if (n == 0) continue;
            int* dst = LV;
            if (c > 0) {
                s->lvTmp.ensure((size_t)n);
                dst = s->lvTmp.p;
            }
            if (s->cfg.mode == APBF_MODE_PBF)
                KL(k_fill_int<<<blocks(n, 256), 256, 0, st>>>(dst, n, s->cfg.n_max));
            else
                run_lod(s->ws, s->set[s->cur].X.p, n, cams[c], lc, s->radius, dst);
            if (c > 0) KL(k_max_int<<<blocks(n, 256), 256, 0, st>>>(n, LV, dst));
        }
        LAUNCH_CHECK();
        s->frame(false, nullptr, nullptr, frame_index, out);
        s->levels_valid = true;
    });
}

int32_t apbf_gpu_blend_lod(int32_t k, int32_t n, const int32_t* const* levels, int32_t* out, apbf_error* err) {
    return guarded(err, [&] {
        if (k < 1) fail(APBF_ERR_INVALID_ARGUMENT, "blend requires at least one level array");
        if (n == 0) return;
        Workspace& ws = component_ws();
        ws.tmpi.ensure((size_t)n * 2);
        int* a = ws.tmpi.p;
        int* b = ws.tmpi.p + n;
        CK(cudaMemcpyAsync(a, levels[0], sizeof(int) * n, cudaMemcpyHostToDevice, ws.stream));
        for (int c = 1; c < k; ++c) {
            CK(cudaMemcpyAsync(b, levels[c], sizeof(int) * n, cudaMemcpyHostToDevice, ws.stream));
            KL(k_max_int<<<blocks(n, 256), 256, 0, ws.stream>>>(n, a, b));
        }
        LAUNCH_CHECK();
        CK(cudaMemcpyAsync(out, a, sizeof(int) * n, cudaMemcpyDeviceToHost, ws.stream));
        CK(cudaStreamSynchronize(ws.stream));
    });
}

int32_t apbf_gpu_step_frame_with_levels(apbf_gpu_solver* s, int32_t frame_index, apbf_frame_stats* out,
                                        apbf_error* err) {
    return guarded(err, [&] {
        if (!s->levels_valid)
            fail(APBF_ERR_INVALID_ARGUMENT, "particle level outside configured iteration range");
        s->frame(false, nullptr, nullptr, frame_index, out);
    });
}

int32_t apbf_gpu_set_iteration_observer(apbf_gpu_solver* s, apbf_iteration_observer cb, void* user) {
    s->observer = cb;
    s->observer_user = user;
    return APBF_OK;
}

int32_t apbf_gpu_set_fast_math(apbf_gpu_solver* s, int32_t enabled) {
    if (!s) return APBF_ERR_INVALID_ARGUMENT;
    s->fast_math = enabled != 0;
    return APBF_OK;
}

int32_t apbf_gpu_set_frame_metrics(apbf_gpu_solver* s, int32_t enabled) {
    s->metrics = enabled != 0;
    return APBF_OK;
}

int32_t apbf_gpu_set_phase_timing(apbf_gpu_solver* s, int32_t enabled) {
    s->phase_timing = enabled != 0;
    return APBF_OK;
}

int32_t apbf_gpu_last_phase_ms(const apbf_gpu_solver* s, float* out5) {
    for (int k = 0; k < 5; ++k) out5[k] = s->phase_ms[k];
    return APBF_OK;
}

int32_t apbf_gpu_set_kernel_timing(apbf_gpu_solver* s, int32_t enabled, apbf_error* err) {
    return guarded(err, [&] {
        CK(cudaSetDevice(s->ws.device));
        s->enable_kernel_timing(enabled != 0);
        s->kt_lambda_ms = s->kt_deltap_ms = 0;
        s->kt_launches = s->kt_items = 0;
    });
}

int32_t apbf_gpu_kernel_times(const apbf_gpu_solver* s, double* lambda_ms, double* deltap_ms,
                              int64_t* launches, int64_t* particle_iterations) {
    if (lambda_ms) *lambda_ms = s->kt_lambda_ms;
    if (deltap_ms) *deltap_ms = s->kt_deltap_ms;
    if (launches) *launches = s->kt_launches;
    if (particle_iterations) *particle_iterations = s->kt_items;
    return APBF_OK;
}

uint64_t apbf_gpu_launch_count(void) { return g_launches; }

int32_t apbf_gpu_last_neighbor_stats(const apbf_gpu_solver* s, int64_t* total_entries,
                                     int64_t* list_capacity) {
    if (total_entries) *total_entries = (int64_t)s->last_list_entries;
    if (list_capacity) *list_capacity = (int64_t)s->last_list_alloc;
    return APBF_OK;
}

// ----------------------------------------------------- component calls

static void check_grid_args(int n, const float* pos, float h, float pad) {
    if (!(h > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "grid cell size must be positive");
    if (pad < 0.0f) fail(APBF_ERR_INVALID_ARGUMENT, "grid padding must be non-negative");
    for (int i = 0; i < n; ++i)
        if (!finite3h(pos + 3 * i)) numerical("grid build", i, "non-finite position");
}

// Builds grid g on the uploaded tmp4 positions; returns host Ctl.
static void component_grid(Workspace& ws, int g, int n, float h, float pad) {
    cudaStream_t st = ws.stream;
    launch_pdl(k_frame_begin, (unsigned)(1), 1, 0, st, ws.ctl.p);
    launch_pdl(k_grid_reset, (unsigned)(1), 1, 0, st, ws.ctl.p, g);
    launch_pdl(k_aabb, (unsigned)(blocks(n, kAabbBlock)), kAabbBlock, 0, st, n, ws.tmp4.p, ws.ctl.p, g);
    ws.run_grid(g, ws.tmp4.p, n, h, pad, false, 0.f);
    ws.read_ctl();
    if (ws.h_ctl->runtime_error) fail(APBF_ERR_RUNTIME, "grid cell count exceeds limit; domain blew up");
}

int32_t apbf_gpu_grid_build(int32_t n, const float* positions, float h, float padding, int32_t* perm,
                            float* origin, int32_t* dims, int32_t* cell_start,
                            int64_t cell_start_capacity, int64_t* cells_out, apbf_error* err) {
    return guarded(err, [&] {
        check_grid_args(n, positions, h, padding);
        if (n == 0) {
            if (origin) origin[0] = origin[1] = origin[2] = 0.f;
            if (dims) dims[0] = dims[1] = dims[2] = 1;
            if (cells_out) *cells_out = 1;
            if (cell_start && cell_start_capacity >= 2) cell_start[0] = cell_start[1] = 0;
            return;
        }
        Workspace& ws = component_ws();
        upload_pos4(ws, n, positions);
        component_grid(ws, 0, n, h, padding);
        const GridDev& G = ws.h_ctl->grid[0];
        if (origin)
            for (int a = 0; a < 3; ++a) origin[a] = G.origin[a];
        if (dims)
            for (int a = 0; a < 3; ++a) dims[a] = G.dims[a];
        if (cells_out) *cells_out = G.cells;
        if (perm) CK(cudaMemcpy(perm, ws.perm.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
        if (cell_start) {
            if (cell_start_capacity < G.cells + 1)
                fail(APBF_ERR_INVALID_ARGUMENT, "cell_start capacity too small");
            CK(cudaMemcpy(cell_start, ws.cellCount.p, sizeof(int) * (G.cells + 1), cudaMemcpyDeviceToHost));
        }
    });
}

int32_t apbf_gpu_neighbor_lists(int32_t n, const float* positions, float h, float padding,
                                int32_t* offsets, int32_t* indices, int64_t indices_capacity,
                                int64_t* total_out, apbf_error* err) {
    return guarded(err, [&] {
        check_grid_args(n, positions, h, padding);
        if (n == 0) {
            if (offsets) offsets[0] = 0;
            if (total_out) *total_out = 0;
            return;
        }
        Workspace& ws = component_ws();
        upload_pos4(ws, n, positions);
        component_grid(ws, 0, n, h, padding);
        // sorted points (the grid's points_ copy), then the solver's own list
        // builder over the identity order (lists by slot), read back as CSR
        cudaStream_t st = ws.stream;
        const int groups = (n + 31) / 32 + 1;
        DBuf<float4> sorted;
        DBuf<int> iota, cnt, lists;
        DBuf<long long> gbase;
        sorted.ensure(n);
        iota.ensure(n);
        cnt.ensure((size_t)groups * 32);
        gbase.ensure(groups);
        launch_pdl(k_gather_posmass, (unsigned)(blocks(n, 256)), 256, 0, st, n, ws.ctl.p, ws.perm.p, ws.tmp4.p, ws.tmp4.p,
                                                         sorted.p);
        KL(k_iota<<<blocks(n, 256), 256, 0, st>>>(iota.p, n));
        long long cap = (long long)groups * 32 * 48;
        for (;;) {
            lists.release();
            lists.ensure((size_t)cap);
            launch_pdl(k_frame_begin, (unsigned)(1), 1, 0, st, ws.ctl.p);
            launch_pdl(k_list_reset, (unsigned)(1), 1, 0, st, ws.ctl.p);
            KL(k_build_lists<<<blocks(n, kListThreads), kListThreads, 0, st>>>(
                n, ws.ctl.p, iota.p, sorted.p, ws.cellCount.p, h, h * h, lists.p, cnt.p, gbase.p, cap));
            LAUNCH_CHECK();
            ws.read_ctl();
            if (!ws.h_ctl->list_overflow) break;
            cap = std::max<long long>(cap * 2, (long long)ws.h_ctl->list_alloc * 3 / 2);
        }
        const long long used = (long long)ws.h_ctl->list_alloc;
        std::vector<int> hc(n), hl((size_t)std::max<long long>(used, 1));
        std::vector<long long> hb(groups);
        CK(cudaMemcpy(hc.data(), cnt.p, sizeof(int) * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hb.data(), gbase.p, sizeof(long long) * groups, cudaMemcpyDeviceToHost));
        if (used > 0) CK(cudaMemcpy(hl.data(), lists.p, sizeof(int) * used, cudaMemcpyDeviceToHost));
        long long total = 0;
        for (int i = 0; i < n; ++i) total += hc[i];
        if (total_out) *total_out = total;
        if (offsets) {
            offsets[0] = 0;
            for (int i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + hc[i];
        }
        if (indices) {
            if (indices_capacity < total) fail(APBF_ERR_INVALID_ARGUMENT, "indices capacity too small");
            long long w = 0;
            for (int i = 0; i < n; ++i) {
                const long long b0 = hb[i >> 5] + 4 * (i & 31);  // chunked slab layout (list_at)
                for (int e = 0; e < hc[i]; ++e) indices[w++] = hl[b0 + ((long long)(e >> 2) << 7) + (e & 3)];
            }
        }
    });
}

int32_t apbf_gpu_all_densities(int32_t n, const float* positions, const float* masses, float h,
                               float* rho_out, apbf_error* err) {
    return guarded(err, [&] {
        if (n == 0) return;
        check_grid_args(n, positions, h, h);
        Workspace& ws = component_ws();
        upload_pos4(ws, n, positions, masses);
        component_grid(ws, 1, n, h, h);
        DBuf<float4> sorted;
        DBuf<float> rho;
        sorted.ensure(n);
        rho.ensure(n);
        cudaStream_t st = ws.stream;
        launch_pdl(k_gather_posmass, (unsigned)(blocks(n, 256)), 256, 0, st, n, ws.ctl.p, ws.perm.p, ws.tmp4.p, ws.tmp4.p,
                                                         sorted.p);
        KL(k_density_out<<<blocks(n, 256), 256, 0, st>>>(n, ws.ctl.p, sorted.p, ws.perm.p, ws.cellCount.p,
                                                      make_kernel_consts(h), rho.p));
        LAUNCH_CHECK();
        CK(cudaMemcpyAsync(rho_out, rho.p, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

// The vorticity estimate of the opt-in post-pass (apbf_post.cuh, eq. 15 of
// Macklin & Mueller 2013) for arbitrary positions/velocities: the same grid,
// lists and k_post_omega the solver runs, omega in input index order.
int32_t apbf_gpu_vorticity(int32_t n, const float* positions, const float* velocities, float h,
                           float* omega_out, apbf_error* err) {
    return guarded(err, [&] {
        if (n == 0) return;
        check_grid_args(n, positions, h, h);
        if (!velocities || !omega_out) fail(APBF_ERR_INVALID_ARGUMENT, "null velocities or output");
        Workspace& ws = component_ws();
        upload_pos4(ws, n, positions);
        component_grid(ws, 0, n, h, h);
        cudaStream_t st = ws.stream;
        const int groups = (n + 31) / 32 + 1;
        DBuf<float4> sorted, vin, vs, om, vx;
        DBuf<int> iota, cnt, lists;
        DBuf<long long> gbase;
        DBuf<float> stage;
        sorted.ensure(n);
        vin.ensure(n);
        vs.ensure(n);
        om.ensure(n);
        vx.ensure(n);
        iota.ensure(n);
        cnt.ensure((size_t)groups * 32);
        gbase.ensure(groups);
        stage.ensure(3 * (size_t)n);
        CK(cudaMemcpyAsync(stage.p, velocities, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, st));
        KL(k_unpack_x<<<blocks(n, 256), 256, 0, st>>>(n, stage.p, vin.p));
        launch_pdl(k_gather_posmass, (unsigned)(blocks(n, 256)), 256, 0, st, n, ws.ctl.p, ws.perm.p, ws.tmp4.p, ws.tmp4.p,
                                                         sorted.p);
        launch_pdl(k_gather_posmass, (unsigned)(blocks(n, 256)), 256, 0, st, n, ws.ctl.p, ws.perm.p, vin.p, vin.p, vs.p);
        KL(k_iota<<<blocks(n, 256), 256, 0, st>>>(iota.p, n));
        long long cap = (long long)groups * 32 * 48;
        for (;;) {
            lists.release();
            lists.ensure((size_t)cap);
            launch_pdl(k_frame_begin, (unsigned)(1), 1, 0, st, ws.ctl.p);
            launch_pdl(k_list_reset, (unsigned)(1), 1, 0, st, ws.ctl.p);
            KL(k_build_lists<<<blocks(n, kListThreads), kListThreads, 0, st>>>(
                n, ws.ctl.p, iota.p, sorted.p, ws.cellCount.p, h, h * h, lists.p, cnt.p, gbase.p, cap));
            LAUNCH_CHECK();
            ws.read_ctl();
            if (!ws.h_ctl->list_overflow) break;
            cap = std::max<long long>(cap * 2, (long long)ws.h_ctl->list_alloc * 3 / 2);
        }
        KL(k_post_omega<<<blocks(n, 256), 256, 0, st>>>(n, ws.ctl.p, iota.p, sorted.p, vs.p, lists.p, cnt.p,
                                                     gbase.p, make_kernel_consts(h), 0.0f, om.p, vx.p));
        LAUNCH_CHECK();
        std::vector<float4> ho(n);
        std::vector<int> perm(n);
        CK(cudaMemcpyAsync(ho.data(), om.p, sizeof(float4) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(perm.data(), ws.perm.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int k = 0; k < n; ++k) {
            float* o = omega_out + 3LL * perm[k];
            o[0] = ho[k].x;
            o[1] = ho[k].y;
            o[2] = ho[k].z;
        }
    });
}

static void component_lod(int n, const float* positions, const apbf_camera* cam,
                          const apbf_lod_config* lod, float radius, int32_t* levels_out) {
    validate_lod(*lod);
    if (lod->n_min < 1 || lod->n_max < lod->n_min)
        fail(APBF_ERR_INVALID_ARGUMENT, "iteration range requires 1 <= n_min <= n_max");
    if (n == 0) return;
    if (lod->model == APBF_LOD_DTVS) {
        if (!(radius > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "splat radius must be positive");
        (void)make_frame(*cam);
    }
    Workspace& ws = component_ws();
    upload_pos4(ws, n, positions);
    DBuf<int> lv;
    lv.ensure(n);
    launch_pdl(k_frame_begin, (unsigned)(1), 1, 0, ws.stream, ws.ctl.p);
    run_lod(ws, ws.tmp4.p, n, *cam, *lod, radius, lv.p);
    CK(cudaMemcpyAsync(levels_out, lv.p, sizeof(int) * n, cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaStreamSynchronize(ws.stream));
}

int32_t apbf_gpu_lod_dtc(int32_t n, const float* positions, const apbf_camera* cam,
                         const apbf_lod_config* lod, int32_t* levels_out, apbf_error* err) {
    return guarded(err, [&] {
        apbf_lod_config l = *lod;
        l.model = APBF_LOD_DTC;
        component_lod(n, positions, cam, &l, 0.f, levels_out);
    });
}

int32_t apbf_gpu_lod_dtvs(int32_t n, const float* positions, const apbf_camera* cam,
                          const apbf_lod_config* lod, float radius, int32_t* levels_out,
                          apbf_error* err) {
    return guarded(err, [&] {
        apbf_lod_config l = *lod;
        l.model = APBF_LOD_DTVS;
        component_lod(n, positions, cam, &l, radius, levels_out);
    });
}

int32_t apbf_gpu_splat(int32_t n, const float* positions, float radius, const apbf_camera* cam,
                       float* depth_out, apbf_error* err) {
    return guarded(err, [&] {
        if (!(radius > 0.0f)) fail(APBF_ERR_INVALID_ARGUMENT, "splat radius must be positive");
        const CamFrame f = make_frame(*cam);
        Workspace& ws = component_ws();
        const size_t px = (size_t)cam->width * cam->height;
        ws.depth.ensure(px);
        ws.rays.ensure(px);
        ws.raysa.ensure(px);
        launch_pdl(k_splat_prep, (unsigned)(blocks((long long)px, 256)), 256, 0, ws.stream, f, ws.depth.p, ws.rays.p, ws.raysa.p);
        if (n > 0) {
            upload_pos4(ws, n, positions);
            launch_pdl(k_splat, (unsigned)(blocks(n, 256)), 256, 0, ws.stream, n, ws.tmp4.p, radius, f, ws.depth.p, ws.rays.p,
                                                           ws.raysa.p);
        }
        LAUNCH_CHECK();
        CK(cudaMemcpyAsync(depth_out, ws.depth.p, sizeof(float) * px, cudaMemcpyDeviceToHost, ws.stream));
        CK(cudaStreamSynchronize(ws.stream));
    });
}

int32_t apbf_gpu_render_level_image(int32_t n, const float* positions, const int32_t* levels, float radius,
                                    const apbf_camera* cam, int32_t n_min, int32_t n_max, uint8_t* rgb_out,
                                    apbf_error* err) {
    return guarded(err, [&] {
        Workspace& ws = component_ws();
        if (n > 0) {
            upload_pos4(ws, n, positions);
            ws.tmpi.ensure((size_t)n);
            CK(cudaMemcpyAsync(ws.tmpi.p, levels, sizeof(int) * n, cudaMemcpyHostToDevice, ws.stream));
        }
        render_levels(ws, n, ws.tmp4.p, ws.tmpi.p, radius, *cam, n_min, n_max, rgb_out);
    });
}

int32_t apbf_gpu_render_levels(apbf_gpu_solver* s, const apbf_camera* cam, float radius, int32_t n_min,
                               int32_t n_max, uint8_t* rgb_out, apbf_error* err) {
    return guarded(err, [&] {
        if (s->transport) fail(APBF_ERR_INVALID_ARGUMENT, "render_levels needs the whole state on one rank");
        CK(cudaSetDevice(s->ws.device));
        render_levels(s->ws, s->n, s->set[s->cur].X.p, s->set[s->cur].LV.p, radius, *cam, n_min, n_max,
                      rgb_out);
    });
}

int32_t apbf_gpu_count_contacts(int32_t n, const float* positions, const apbf_sdf_primitive* prims,
                                int32_t n_prims, float gradient_step, float radius, int64_t* count_out,
                                apbf_error* err) {
    return guarded(err, [&] {
        const Scene sc = make_scene(prims, n_prims, gradient_step);
        *count_out = 0;
        if (n == 0 || sc.n == 0) return;
        Workspace& ws = component_ws();
        CK(cudaMemcpyAsync(ws.scene.p, &sc, sizeof(Scene), cudaMemcpyHostToDevice, ws.stream));
        upload_pos4(ws, n, positions);
        launch_pdl(k_frame_begin, (unsigned)(1), 1, 0, ws.stream, ws.ctl.p);
        KL(k_count_contacts<<<blocks(n, 256), 256, 0, ws.stream>>>(n, ws.tmp4.p, ws.scene.p, radius, ws.ctl.p));
        LAUNCH_CHECK();
        ws.read_ctl();
        *count_out = (int64_t)ws.h_ctl->contacts;
    });
}


// ------------------------------------------------- z-slab decomposition API

struct apbf_gpu_group {
    std::vector<std::unique_ptr<apbf_gpu_solver>> ranks;
    std::unique_ptr<LoopbackHub> hub;
    std::vector<std::unique_ptr<LoopbackTransport>> tr;
    std::vector<int> devices;
};

static int32_t group_run(apbf_gpu_group* g, apbf_error* err,
                         const std::function<void(apbf_gpu_solver&, int)>& fn) {
    const int G = (int)g->ranks.size();
    std::vector<apbf_error> errs(G);
    std::vector<int32_t> rcs(G, APBF_OK);
    g->hub->reset();
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r) {
        th.emplace_back([&, r] {
            rcs[r] = guarded(&errs[r], [&] {
                CK(cudaSetDevice(g->devices[r]));
                try {
                    fn(*g->ranks[r], r);
                } catch (...) {
                    g->hub->poison();
                    throw;
                }
            });
        });
    }
    for (auto& t : th) t.join();
    // a numerical / argument error is global (every rank reports the same);
    // otherwise the first rank that failed for its own reason
    for (int r = 0; r < G; ++r)
        if (rcs[r] != APBF_OK && std::strcmp(errs[r].message, "slab peer rank failed") != 0) {
            if (err) *err = errs[r];
            return rcs[r];
        }
    for (int r = 0; r < G; ++r)
        if (rcs[r] != APBF_OK) {
            if (err) *err = errs[r];
            return rcs[r];
        }
    return APBF_OK;
}

int32_t apbf_gpu_group_create(const apbf_solver_config* cfg, const apbf_sdf_primitive* prims,
                              int32_t n_prims, float gradient_step, int32_t nranks,
                              const int32_t* devices, apbf_gpu_group** out, apbf_error* err) {
    return guarded(err, [&] {
        *out = nullptr;
        validate_config(cfg);
        if (nranks < 1 || nranks > kMaxRanks) fail(APBF_ERR_INVALID_ARGUMENT, "slab rank count out of range");
        const Scene sc = make_scene(prims, n_prims, gradient_step);
        int count = 0;
        CK(cudaGetDeviceCount(&count));
        auto g = std::make_unique<apbf_gpu_group>();
        for (int r = 0; r < nranks; ++r) {
            const int d = devices ? devices[r] : 0;
            if (d < 0 || d >= count) fail(APBF_ERR_INVALID_ARGUMENT, "CUDA device out of range");
            g->devices.push_back(d);
        }
        for (int r = 0; r < nranks; ++r)
            for (int q = 0; q < nranks; ++q)
                if (g->devices[r] != g->devices[q]) {
                    CK(cudaSetDevice(g->devices[r]));
                    const cudaError_t e = cudaDeviceEnablePeerAccess(g->devices[q], 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                    cudaGetLastError();
                }
        g->hub = std::make_unique<LoopbackHub>(nranks, g->devices);
        for (int r = 0; r < nranks; ++r) {
            CK(cudaSetDevice(g->devices[r]));
            g->ranks.emplace_back(new apbf_gpu_solver(*cfg, sc, g->devices[r]));
            g->tr.emplace_back(new LoopbackTransport(g->hub.get(), r));
            g->ranks.back()->transport = g->tr.back().get();
        }
        *out = g.release();
    });
}

void apbf_gpu_group_destroy(apbf_gpu_group* g) { delete g; }

int32_t apbf_gpu_group_size(const apbf_gpu_group* g) { return g ? (int32_t)g->ranks.size() : 0; }

int32_t apbf_gpu_group_set_state(apbf_gpu_group* g, int32_t n, const float* x, const float* xs,
                                 const float* v, const float* mass, const float* inv_mass,
                                 const float* lambda, const int32_t* level, apbf_error* err) {
    if (n < 0) {
        guarded(err, [] { fail(APBF_ERR_INVALID_ARGUMENT, "negative particle count"); });
        return APBF_ERR_INVALID_ARGUMENT;
    }
    if (n > 0 && (!x || !v || !mass || !inv_mass)) {
        guarded(err, [] { fail(APBF_ERR_INVALID_ARGUMENT, "x, v, mass and inv_mass are required"); });
        return APBF_ERR_INVALID_ARGUMENT;
    }
    const int G = (int)g->ranks.size();
    return group_run(g, err, [&](apbf_gpu_solver& s, int r) {
        // rank r takes the contiguous storage range [n r / G, n (r+1) / G)
        const long long b = (long long)n * r / G, e = (long long)n * (r + 1) / G;
        s.set_state_local((int)(e - b), n, x + 3 * b, xs ? xs + 3 * b : nullptr, v + 3 * b, mass + b,
                          inv_mass + b, lambda ? lambda + b : nullptr, level ? level + b : nullptr);
    });
}

int32_t apbf_gpu_group_particle_counts(const apbf_gpu_group* g, int32_t* counts) {
    for (size_t r = 0; r < g->ranks.size(); ++r) counts[r] = g->ranks[r]->n;
    return APBF_OK;
}

int32_t apbf_gpu_group_get_state(apbf_gpu_group* g, float* x, float* xs, float* v, float* mass,
                                 float* inv_mass, float* lambda, int32_t* level, apbf_error* err) {
    // global storage order = owned particles of rank 0, 1, ... (the slabs are
    // increasing cell-layer ranges of the global cell order)
    long long off = 0;
    for (auto& s : g->ranks) {
        const int32_t rc = apbf_gpu_get_state(s.get(), x ? x + 3 * off : nullptr, xs ? xs + 3 * off : nullptr,
                                              v ? v + 3 * off : nullptr, mass ? mass + off : nullptr,
                                              inv_mass ? inv_mass + off : nullptr, lambda ? lambda + off : nullptr,
                                              level ? level + off : nullptr, err);
        if (rc) return rc;
        off += s->n;
    }
    return APBF_OK;
}

int32_t apbf_gpu_group_step_frame(apbf_gpu_group* g, const apbf_camera* cam, const apbf_lod_config* lod,
                                  int32_t frame_index, apbf_frame_stats* out, apbf_error* err) {
    const int G = (int)g->ranks.size();
    std::vector<apbf_frame_stats> st(G);
    std::vector<std::vector<double>> res(G);
    for (int r = 0; r < G; ++r) {
        std::memset(&st[r], 0, sizeof st[r]);
        if (out && out->residuals) {
            res[r].resize(out->residuals_capacity);
            st[r].residuals = res[r].data();
            st[r].residuals_capacity = out->residuals_capacity;
        }
    }
    const int32_t rc = group_run(g, err, [&](apbf_gpu_solver& s, int r) {
        s.frame(cam != nullptr, cam, lod, frame_index, &st[r]);
        s.levels_valid = true;
    });
    if (rc == APBF_OK && out) {
        double* rr = out->residuals;
        const int cap = out->residuals_capacity;
        *out = st[0];
        out->residuals = rr;
        out->residuals_capacity = cap;
    }
    return rc;
}

int32_t apbf_gpu_group_step_frame_with_levels(apbf_gpu_group* g, int32_t frame_index,
                                              apbf_frame_stats* out, apbf_error* err) {
    for (auto& s : g->ranks)
        if (!s->levels_valid) {
            guarded(err, [] { fail(APBF_ERR_INVALID_ARGUMENT, "particle level outside configured iteration range"); });
            return APBF_ERR_INVALID_ARGUMENT;
        }
    return apbf_gpu_group_step_frame(g, nullptr, nullptr, frame_index, out, err);
}

int32_t apbf_gpu_nccl_unique_id(uint8_t* id128, apbf_error* err) {
    return guarded(err, [&] {
        NcclApi& api = NcclApi::get();
        if (api.getUniqueId(id128) != 0) fail(APBF_ERR_CUDA, "ncclGetUniqueId failed");
    });
}

int32_t apbf_gpu_solver_attach_nccl(apbf_gpu_solver* s, int32_t rank, int32_t nranks, const uint8_t* id128,
                                    apbf_error* err) {
    return guarded(err, [&] {
        if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
            fail(APBF_ERR_INVALID_ARGUMENT, "slab rank out of range");
        CK(cudaSetDevice(s->ws.device));
        s->transport_owned.reset(new NcclTransport(rank, nranks, id128));
        s->transport = s->transport_owned.get();
    });
}

int32_t apbf_gpu_slab_set_state(apbf_gpu_solver* s, int32_t n_local, int64_t n_global, const float* x,
                                const float* xs, const float* v, const float* mass, const float* inv_mass,
                                const float* lambda, const int32_t* level, apbf_error* err) {
    return guarded(err, [&] {
        if (!s->transport) fail(APBF_ERR_INVALID_ARGUMENT, "solver is not attached to a slab transport");
        if (n_local > 0 && (!x || !v || !mass || !inv_mass))
            fail(APBF_ERR_INVALID_ARGUMENT, "x, v, mass and inv_mass are required");
        CK(cudaSetDevice(s->ws.device));
        s->set_state_local(n_local, n_global, x, xs, v, mass, inv_mass, lambda, level);
    });
}

// Pure host logic of the decomposition, exposed for tests: equal-count
// partition of a per-layer histogram into slabs of >= min_layers layers.
int32_t apbf_slab_partition(const int64_t* layer_hist, int32_t layers, int32_t nranks, int32_t min_layers,
                            int32_t* zlo, int32_t* zhi) {
    std::vector<long long> h(layer_hist, layer_hist + layers);
    std::vector<int> a(nranks), b(nranks);
    if (!slab_partition(h.data(), layers, nranks, min_layers, a.data(), b.data())) return APBF_ERR_RUNTIME;
    for (int g = 0; g < nranks; ++g) {
        zlo[g] = a[g];
        zhi[g] = b[g];
    }
    return APBF_OK;
}

}  // extern "C"
