/*
 * apbf_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, float32) of the reference APBF simulation step
 * (/root/reference/proj/include/apbf/ headers).  It is the checker for the CUDA
 * product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_1608_04721_b200/libapbf_gpu.so) never links or calls it.
 *
 * Parity pin: the restatement is checked bit-for-bit against the reference
 * itself, compiled from /root/reference with oracle/Makefile into
 * oracle/_ref/ (Solver<float> through the Eigen-subset shim), and against the
 * golden fixtures in tests/golden/ that were generated from that build
 * (tests/golden/make_golden.py).  Known-answer values of the reference's own
 * unit tests (test_kernels.cpp, test_solver.cpp, test_lod.cpp, ...) are
 * re-asserted in tests/test_oracle.py.
 *
 * Arithmetic contract: no FMA contraction, IEEE
 * division and sqrt, fixed-size-3 float reductions in Eigen's unrolled order
 * x0 + (x1 + x2), expression trees as written in the reference.
 */
#ifndef APBF_ORACLE_H
#define APBF_ORACLE_H

#include <stdint.h>

#include "../include/apbf_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_solver orc_solver;

orc_solver* orc_solver_create(const apbf_solver_config* cfg, const apbf_sdf_primitive* prims,
                              int32_t n_prims, float gradient_step, apbf_error* err);
void orc_solver_destroy(orc_solver* s);
int32_t orc_set_state(orc_solver* s, int32_t n, const float* x, const float* x_star,
                      const float* v, const float* mass, const float* inv_mass,
                      const float* lambda, const int32_t* level, apbf_error* err);
int32_t orc_get_state(const orc_solver* s, float* x, float* x_star, float* v, float* mass,
                      float* inv_mass, float* lambda, int32_t* level);
int32_t orc_step_frame(orc_solver* s, const apbf_camera* cam, const apbf_lod_config* lod,
                       int32_t frame_index, apbf_frame_stats* out, apbf_error* err);
int32_t orc_step_frame_with_levels(orc_solver* s, int32_t frame_index, apbf_frame_stats* out,
                                   apbf_error* err);
void orc_set_iteration_observer(orc_solver* s, apbf_iteration_observer cb, void* user);
void orc_set_frame_metrics(orc_solver* s, int32_t enabled);
/* Permutation of the last grid build (sorted slot -> pre-build index). */
int32_t orc_last_permutation(const orc_solver* s, int32_t* perm);

/* kernels.hpp:38-65 */
float orc_density_kernel_r2(float r2, float h);
void orc_gradient_kernel(const float r[3], float h, float out[3]);

/* uniform_grid.hpp:42-98 (+ 179-213 via orc_neighbor_lists) */
int32_t orc_grid_build(int32_t n, const float* positions, float h, float padding, int32_t* perm,
                       float* origin, int32_t* dims, int32_t* cell_start,
                       int64_t cell_start_capacity, int64_t* cells_out, apbf_error* err);
int32_t orc_neighbor_lists(int32_t n, const float* positions, float h, float padding,
                           int32_t* offsets, int32_t* indices, int64_t indices_capacity,
                           int64_t* total_out, apbf_error* err);

/* solver.hpp:82-141 over caller CSR lists (the reference's unit tests use
 * hand-built lists, test_solver.cpp:43-48). */
float orc_compute_density(int32_t i, const int32_t* offsets, const int32_t* indices,
                          const float* masses, const float* positions, float h);
float orc_compute_lambda(int32_t i, const int32_t* offsets, const int32_t* indices,
                         const float* x_star, const float* mass, const float* inv_mass,
                         const apbf_solver_config* cfg);
void orc_compute_deltap(int32_t i, const int32_t* offsets, const int32_t* indices,
                        const float* x_star, const float* inv_mass, const float* lambda,
                        const int32_t* level, const apbf_solver_config* cfg, int32_t iteration,
                        float out[3]);

int32_t orc_all_densities(int32_t n, const float* positions, const float* masses, float h,
                          float* rho_out, apbf_error* err);
int32_t orc_lod_dtc(int32_t n, const float* positions, const apbf_camera* cam,
                    const apbf_lod_config* lod, int32_t* levels_out, apbf_error* err);
int32_t orc_lod_dtvs(int32_t n, const float* positions, const apbf_camera* cam,
                     const apbf_lod_config* lod, float radius, int32_t* levels_out,
                     apbf_error* err);
int32_t orc_splat(int32_t n, const float* positions, float radius, const apbf_camera* cam,
                  float* depth_out, apbf_error* err);
int32_t orc_count_contacts(int32_t n, const float* positions, const apbf_sdf_primitive* prims,
                           int32_t n_prims, float gradient_step, float radius, int64_t* count_out,
                           apbf_error* err);
/* sceneDistance (sdf.hpp:202-223): phi + unit gradient. */
int32_t orc_scene_distance(const apbf_sdf_primitive* prims, int32_t n_prims, float gradient_step,
                           const float p[3], float* phi, float grad[3], apbf_error* err);
int32_t orc_map_distance_to_level(float d, float d_min, float d_max, int32_t n_min, int32_t n_max);
float orc_percentile(const float* values, int32_t n, float p);

#ifdef __cplusplus
}
#endif

#endif
