/*
 * apbf_gpu.h -- C-ABI of the B200-native APBF simulation step.
 *
 * This is the drop-in boundary for the reference's hot path,
 * `apbf::Solver<Scalar>` (/root/reference/proj/include/apbf/solver.hpp:208-392),
 * plus the free functions that the solver is built from and that the
 * reference exposes publicly (grid, densities, LOD, splat, contacts).
 *
 * Every entry point takes plain pointers and sizes; no CUDA or torch types
 * cross the boundary.  Arrays of 3-vectors are interleaved xyz per particle,
 * i.e. exactly the memory layout of the reference's column-major
 * `Mat3X<Scalar>` (types.hpp:14-16), in float32.
 *
 * Error convention (types.hpp:25-39, solver.hpp:53-66, uniform_grid.hpp:76-78):
 * every function returns an `int32_t` status that is also written to
 * `err->code` when `err` is non-NULL:
 *   APBF_OK                     0
 *   APBF_ERR_INVALID_ARGUMENT   1  -- std::invalid_argument in the reference
 *   APBF_ERR_RUNTIME            2  -- std::runtime_error (cell-count guard, list overflow)
 *   APBF_ERR_NUMERICAL          3  -- apbf::NumericalError(pass, particle, detail)
 *   APBF_ERR_CUDA               4  -- device failure (no reference counterpart)
 *   APBF_ERR_OUT_OF_RANGE       5  -- std::out_of_range
 * For APBF_ERR_NUMERICAL `err->pass` holds the pass name ("predict",
 * "prestabilize", "lambda", "apply", "finalize", "grid build") and
 * `err->particle` the first offending storage index, as NumericalError does.
 *
 * Threading: a solver handle owns one CUDA stream on one device and is not
 * reentrant (the reference Solver owns its scratch too, solver.hpp:382-391).
 */
#ifndef APBF_GPU_H
#define APBF_GPU_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APBF_GPU_ABI_VERSION 1

#define APBF_OK 0
#define APBF_ERR_INVALID_ARGUMENT 1
#define APBF_ERR_RUNTIME 2
#define APBF_ERR_NUMERICAL 3
#define APBF_ERR_CUDA 4
#define APBF_ERR_OUT_OF_RANGE 5

typedef struct apbf_error {
    int32_t code;
    int32_t particle;   /* NumericalError::particle() (types.hpp:36) or -1 */
    char pass[32];      /* NumericalError::pass() (types.hpp:35) or "" */
    char message[224];  /* what() */
} apbf_error;

/* SolverMode (solver.hpp:24) */
enum { APBF_MODE_PBF = 0, APBF_MODE_APBF = 1 };
/* LodModel (lod.hpp:14) */
enum { APBF_LOD_DTC = 0, APBF_LOD_DTVS = 1 };
/* SdfPrimitive alternatives (sdf.hpp:18-77) */
enum { APBF_SDF_HALF_SPACE = 0, APBF_SDF_SPHERE = 1, APBF_SDF_BOX = 2, APBF_SDF_CONE = 3 };

/* SolverConfig<float> (solver.hpp:26-51); zero means "derived default" for
 * stab_threshold, particle_radius and velocity_cap exactly as there. */
typedef struct apbf_solver_config {
    float dt_frame;
    int32_t substeps;
    int32_t n_min; /* IterationRange range (particle_state.hpp:16-29) */
    int32_t n_max;
    float rest_density;
    float h;
    float epsilon;
    float gravity[3];
    int32_t stab_iterations;
    int32_t stab_threshold;
    float particle_radius;
    int32_t mode;
    float velocity_cap;
    int32_t inactive_lambda_zero;
    int32_t deterministic;    /* accepted for API parity; the GPU path is always deterministic */
    int32_t record_residuals;
    /* Opt-in PBF velocity post-pass (Macklin & Mueller 2013, eqs. 15-17), absent
     * from the reference: XSPH viscosity c and vorticity-confinement epsilon.
     * 0 (the default) = off, and frames stay bit-identical to the reference. */
    float xsph_viscosity;
    float vorticity_epsilon;
} apbf_solver_config;

/* One SDF primitive (sdf.hpp:18-74).  Constructors' validation and the
 * half-space normal normalisation (sdf.hpp:23-29) happen inside
 * apbf_gpu_solver_create, in float, as the reference constructors do. */
typedef struct apbf_sdf_primitive {
    int32_t kind;
    int32_t interior; /* Sphere/Box interior flag */
    float p[3];       /* half_space: normal; sphere, box: center; cone: base center */
    float q[3];       /* box: half extents */
    float a;          /* half_space: offset; sphere: radius; cone: base radius */
    float b;          /* cone: height */
} apbf_sdf_primitive;

/* Camera<float> (depth_splat.hpp:19-43).  The CameraFrame basis and tan()
 * are evaluated on the host side of the library (depth_splat.hpp:55-71). */
typedef struct apbf_camera {
    float eye[3];
    float look_at[3];
    float up[3];
    float vertical_fov;
    int32_t width;
    int32_t height;
    float near_clip;
} apbf_camera;

/* LodModelConfig<float> (lod.hpp:16-29) */
typedef struct apbf_lod_config {
    int32_t model;
    float d_min;
    float d_max;
    int32_t n_min;
    int32_t n_max;
    int32_t auto_range;
} apbf_lod_config;

/* FrameStats (solver.hpp:69-78).  `residuals` is caller-owned storage of
 * `residuals_capacity` doubles (may be NULL); `n_residuals` reports how many
 * were produced (substeps * executed iterations when record_residuals). */
typedef struct apbf_frame_stats {
    int32_t frame;
    int32_t n_residuals;
    double wall_ms;
    double avg_density_pct;
    double min_density_pct;
    double max_density_pct;
    int64_t total_iterations;
    int64_t contacts;
    double* residuals;
    int32_t residuals_capacity;
    int32_t reserved;
} apbf_frame_stats;

typedef struct apbf_gpu_solver apbf_gpu_solver;

/* Library / device info. */
int32_t apbf_gpu_abi_version(void);
int32_t apbf_gpu_device_count(void);

/* Solver(SolverConfig, SdfScene) (solver.hpp:211-217, validate :53-66).
 * `device` selects the CUDA device (the caller's rank-local GPU). */
int32_t apbf_gpu_solver_create(const apbf_solver_config* cfg, const apbf_sdf_primitive* prims,
                               int32_t n_prims, float gradient_step, int32_t device,
                               apbf_gpu_solver** out, apbf_error* err);
void apbf_gpu_solver_destroy(apbf_gpu_solver* s);

/* Upload / download the ParticleSet (particle_state.hpp:33-42) in storage
 * order.  3-vector arrays hold 3*n floats.  In get_state any pointer may be
 * NULL to skip that field.  In set_state x, v, mass and inv_mass are
 * required; x_star, lambda and level may be NULL (stepFrame overwrites them
 * before reading them; without levels stepFrameWithLevels rejects the state).  The solver reorders storage every substep
 * (uniform_grid.hpp:102-105), exactly as the reference leaves the caller's
 * ParticleSet in the last substep's cell order. */
int32_t apbf_gpu_set_state(apbf_gpu_solver* s, int32_t n, const float* x, const float* x_star,
                           const float* v, const float* mass, const float* inv_mass,
                           const float* lambda, const int32_t* level, apbf_error* err);
int32_t apbf_gpu_get_state(apbf_gpu_solver* s, float* x, float* x_star, float* v, float* mass,
                           float* inv_mass, float* lambda, int32_t* level, apbf_error* err);
int32_t apbf_gpu_particle_count(const apbf_gpu_solver* s);

/* The cudaStream_t (as void*) every kernel of this handle is launched on,
 * so callers can record CUDA events on the launching stream. */
void* apbf_gpu_stream(const apbf_gpu_solver* s);

/* Solver::stepFrame (solver.hpp:228-233) and stepFrameWithLevels (:236-244).
 * The state stays resident on the device between calls. */
int32_t apbf_gpu_step_frame(apbf_gpu_solver* s, const apbf_camera* cam, const apbf_lod_config* lod,
                            int32_t frame_index, apbf_frame_stats* out, apbf_error* err);
int32_t apbf_gpu_step_frame_with_levels(apbf_gpu_solver* s, int32_t frame_index,
                                        apbf_frame_stats* out, apbf_error* err);

/* stepFrame(ParticleSet& state, ...) on host arrays in one call: uploads what
 * the frame reads (x, v, mass, inv_mass), steps, and writes the whole
 * reordered state back into the same seven arrays.  Equivalent to
 * set_state + step_frame + get_state, with the download started as soon as
 * the last substep is done, overlapping the end-of-frame metrics pass. */
int32_t apbf_gpu_step_frame_host(apbf_gpu_solver* s, int32_t n, float* x, float* x_star, float* v,
                                 float* mass, float* inv_mass, float* lambda, int32_t* level,
                                 const apbf_camera* cam, const apbf_lod_config* lod, int32_t frame_index,
                                 apbf_frame_stats* out, apbf_error* err);

/* Page-locked host memory for the arrays of apbf_gpu_step_frame_host (copies
 * from/to it run at full PCIe rate and overlap the frame).  NULL on failure;
 * apbf_gpu_host_free(NULL) is a no-op. */
void* apbf_gpu_host_alloc(size_t bytes);
void apbf_gpu_host_free(void* p);

/* Multi-camera stepFrame (the paper's multi-camera remark): per camera i
 * the levels assignLevels would give (lod config i with the solver's range,
 * solver.hpp:247-258), blended with blendLod (lod.hpp:160-172, elementwise
 * max), then stepFrameWithLevels (:236-244) -- all on the device.  k >= 1.
 * Single rank only. */
int32_t apbf_gpu_step_frame_multi(apbf_gpu_solver* s, int32_t k, const apbf_camera* cams,
                                  const apbf_lod_config* lods, int32_t frame_index, apbf_frame_stats* out,
                                  apbf_error* err);

/* Solver::iterationObserver (solver.hpp:222-224, called at :344).  The
 * callback runs on the host after each iteration; it may call
 * apbf_gpu_get_state on the same handle.  NULL removes it. */
typedef void (*apbf_iteration_observer)(void* user, int32_t substep, int32_t iteration);
int32_t apbf_gpu_set_iteration_observer(apbf_gpu_solver* s, apbf_iteration_observer cb, void* user);

/* Fast build of the lambda and delta-p pair arithmetic (default off):
 * FMA contraction, |g|^2 = c^2 r^2, and 1/|r| from one rsqrt approximation
 * instead of the correctly rounded sqrt and division of the reference's
 * gradientKernel (kernels.hpp:52-65).  Outside the bitwise contract: results
 * stay within the tier-B tolerance of the reference's Solver<double> (2x its
 * own float-vs-double divergence, tests/test_gpu_fast_math.py).  Takes effect
 * at the next frame. */
int32_t apbf_gpu_set_fast_math(apbf_gpu_solver* s, int32_t enabled);

/* Frame-time switch for the end-of-frame density metrics pass
 * (solver.hpp:271-279); on by default like the reference. */
int32_t apbf_gpu_set_frame_metrics(apbf_gpu_solver* s, int32_t enabled);

/* Device time (ms) of each phase of the last frame, for profiling:
 * [0] LOD, [1] predict+grid+lists, [2] solver iterations, [3] finalize,
 * [4] metrics.  Requires apbf_gpu_set_phase_timing(s, 1). */
int32_t apbf_gpu_set_phase_timing(apbf_gpu_solver* s, int32_t enabled);
int32_t apbf_gpu_last_phase_ms(const apbf_gpu_solver* s, float* out5);

/* Per-launch CUDA-event timing of the two solver passes (lambda and
 * delta-p+apply), on the solver's own stream, accumulated over frames since
 * the last call (each call resets the sums; switching on/off re-records the
 * frame graph); particle_iterations = sum of active particles over those
 * launches (FrameStats.totalIterations).  Profiling hook, off by default. */
int32_t apbf_gpu_set_kernel_timing(apbf_gpu_solver* s, int32_t enabled, apbf_error* err);
int32_t apbf_gpu_kernel_times(const apbf_gpu_solver* s, double* lambda_ms, double* deltap_ms,
                              int64_t* launches, int64_t* particle_iterations);

/* Number of kernels this library has launched so far (process-wide; the
 * kernel nodes of every replayed frame graph included). */
uint64_t apbf_gpu_launch_count(void);

/* Sum of frozen-list lengths (incl. self) of the last substep and the
 * sliced-ELL storage it used; entries / n is the n-bar of the flop model
 * (SURVEY.md 8d). */
int32_t apbf_gpu_last_neighbor_stats(const apbf_gpu_solver* s, int64_t* total_entries,
                                     int64_t* list_capacity);

/* ---- z-slab domain decomposition ----
 * The reference has no distributed code; these entry points run the same
 * stepFrame over G ranks that own z-slabs of the substep's global grid,
 * with migration + 2-layer halos exchanged as particle records and one x*
 * halo exchange per solver iteration.  Results equal the single-GPU run bit
 * for bit.  Global storage order = rank 0's owned particles, then rank 1's,
 * ... (set_state splits the caller's arrays into contiguous ranges). */
typedef struct apbf_gpu_group apbf_gpu_group;

/* G ranks in this process (host thread per rank); devices[r] is rank r's
 * GPU (NULL: all on device 0 -- the single-GPU test mode). */
int32_t apbf_gpu_group_create(const apbf_solver_config* cfg, const apbf_sdf_primitive* prims,
                              int32_t n_prims, float gradient_step, int32_t nranks,
                              const int32_t* devices, apbf_gpu_group** out, apbf_error* err);
void apbf_gpu_group_destroy(apbf_gpu_group* g);
int32_t apbf_gpu_group_size(const apbf_gpu_group* g);
int32_t apbf_gpu_group_set_state(apbf_gpu_group* g, int32_t n, const float* x, const float* x_star,
                                 const float* v, const float* mass, const float* inv_mass,
                                 const float* lambda, const int32_t* level, apbf_error* err);
int32_t apbf_gpu_group_get_state(apbf_gpu_group* g, float* x, float* x_star, float* v, float* mass,
                                 float* inv_mass, float* lambda, int32_t* level, apbf_error* err);
int32_t apbf_gpu_group_particle_counts(const apbf_gpu_group* g, int32_t* counts);
int32_t apbf_gpu_group_step_frame(apbf_gpu_group* g, const apbf_camera* cam,
                                  const apbf_lod_config* lod, int32_t frame_index,
                                  apbf_frame_stats* out, apbf_error* err);
int32_t apbf_gpu_group_step_frame_with_levels(apbf_gpu_group* g, int32_t frame_index,
                                              apbf_frame_stats* out, apbf_error* err);

/* One process per GPU: rank r of nranks joins an NCCL communicator (unique
 * id from rank 0, broadcast by the caller), then uploads its contiguous
 * slice of the global state with apbf_gpu_slab_set_state; step_frame /
 * get_state then act on this rank's owned particles. */
int32_t apbf_gpu_nccl_unique_id(uint8_t* id128, apbf_error* err);
int32_t apbf_gpu_solver_attach_nccl(apbf_gpu_solver* s, int32_t rank, int32_t nranks,
                                    const uint8_t* id128, apbf_error* err);
int32_t apbf_gpu_slab_set_state(apbf_gpu_solver* s, int32_t n_local, int64_t n_global,
                                const float* x, const float* x_star, const float* v,
                                const float* mass, const float* inv_mass, const float* lambda,
                                const int32_t* level, apbf_error* err);

/* Host logic of the decomposition (no GPU needed): equal-count partition of
 * a per-layer particle histogram into nranks slabs of >= min_layers layers. */
int32_t apbf_slab_partition(const int64_t* layer_hist, int32_t layers, int32_t nranks,
                            int32_t min_layers, int32_t* zlo, int32_t* zhi);

/* ---- component entry points (reference free functions / classes) ---- */

/* UniformGrid<float>::build (uniform_grid.hpp:42-98).  perm: n ints;
 * origin: 3 floats; dims: 3 ints; cell_start (may be NULL) must hold
 * cells+1 ints where cells = dims product (query with cell_start = NULL
 * first).  *cells_out receives the cell count. */
int32_t apbf_gpu_grid_build(int32_t n, const float* positions, float h, float padding,
                            int32_t* perm, float* origin, int32_t* dims, int32_t* cell_start,
                            int64_t cell_start_capacity, int64_t* cells_out, apbf_error* err);

/* UniformGrid::build + buildNeighborLists (uniform_grid.hpp:179-213) in CSR:
 * offsets n+1 ints, indices up to indices_capacity ints (call with
 * indices = NULL to get *total_out).  Slots are sorted-slot indices. */
int32_t apbf_gpu_neighbor_lists(int32_t n, const float* positions, float h, float padding,
                                int32_t* offsets, int32_t* indices, int64_t indices_capacity,
                                int64_t* total_out, apbf_error* err);

/* allDensities (solver.hpp:145-162): densities in original index order. */
int32_t apbf_gpu_all_densities(int32_t n, const float* positions, const float* masses, float h,
                               float* rho_out, apbf_error* err);

/* Not in the reference: the vorticity estimate of the
 * opt-in post-pass, omega_i = sum_j (v_i - v_j) x gradW(x_i - x_j) over the
 * strict r^2 < h^2 neighbours (Macklin & Mueller 2013 eq. 15), for n
 * positions/velocities (xyz interleaved); omega_out (3n) in input order. */
int32_t apbf_gpu_vorticity(int32_t n, const float* positions, const float* velocities, float h,
                           float* omega_out, apbf_error* err);

/* lodDtc (lod.hpp:83-104) and lodDtvs (lod.hpp:109-156); the level range is
 * taken from lod->n_min/n_max. */
int32_t apbf_gpu_lod_dtc(int32_t n, const float* positions, const apbf_camera* cam,
                         const apbf_lod_config* lod, int32_t* levels_out, apbf_error* err);
int32_t apbf_gpu_lod_dtvs(int32_t n, const float* positions, const apbf_camera* cam,
                          const apbf_lod_config* lod, float radius, int32_t* levels_out,
                          apbf_error* err);

/* blendLod (lod.hpp:160-172): out = elementwise max of k >= 1 level arrays
 * of length n (levels[i] points at array i). */
int32_t apbf_gpu_blend_lod(int32_t k, int32_t n, const int32_t* const* levels, int32_t* out, apbf_error* err);

/* splat (depth_splat.hpp:201-228): width*height depths, +inf where unwritten. */
int32_t apbf_gpu_splat(int32_t n, const float* positions, float radius, const apbf_camera* cam,
                       float* depth_out, apbf_error* err);

/* renderLevelImage (depth_splat.hpp:314-350): opaque splat render, each
 * pixel coloured by the level of its nearest particle (ties: lowest index)
 * with levelColor (:296-310); rgb_out holds width*height*3 bytes, row-major,
 * black where nothing was hit -- the ImageRgb that writePpm (:251-262)
 * stores.  Runs on the device; only the image is downloaded. */
int32_t apbf_gpu_render_level_image(int32_t n, const float* positions, const int32_t* levels, float radius,
                                    const apbf_camera* cam, int32_t n_min, int32_t n_max, uint8_t* rgb_out,
                                    apbf_error* err);
/* The same for the solver's resident state (x and level, storage order);
 * runScenario's frame_XXXXXX.ppm dumps (runner.cpp:85-90). */
int32_t apbf_gpu_render_levels(apbf_gpu_solver* s, const apbf_camera* cam, float radius, int32_t n_min,
                               int32_t n_max, uint8_t* rgb_out, apbf_error* err);

/* findContacts(...).size() (sdf.hpp:226-250). */
int32_t apbf_gpu_count_contacts(int32_t n, const float* positions, const apbf_sdf_primitive* prims,
                                int32_t n_prims, float gradient_step, float radius,
                                int64_t* count_out, apbf_error* err);

#ifdef __cplusplus
}
#endif

#endif /* APBF_GPU_H */
