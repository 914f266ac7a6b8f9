/*
 * lk_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's global-registration path
 * (/root/reference/proj/src/registration.cpp and friends), used as the parity
 * checker for the B200 product and as the reference arm's CPU baseline.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product
 * (paper_1801_01572_b200/) never links or calls it.
 *
 * Parity pinning: the reference cannot be compiled here (Eigen3, doctest,
 * CLI11 and nlohmann-json are absent), so this restatement is pinned against
 * the reference's own known-answer and property tests
 * (proj/tests/test_registration.cpp, test_grid.cpp, test_geometry.cpp,
 * test_line_process.cpp), ported to tests/test_oracle_*.py. Eigen's
 * floating-point evaluation order is restated per SURVEY.md Appendix A;
 * transform bits vs the real Eigen binary are unpinned beyond ~1e-9.
 *
 * All functions return an lk status code (same numbering as
 * include/loopkit_b200.h) and never throw across the ABI.
 */
#ifndef LK_ORACLE_H
#define LK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    OR_OK = 0,
    OR_NO_ALIGNMENT = 1,
    OR_EMPTY_CLOUD = 2,
    OR_TOO_FEW_POINTS = 3,
    OR_MISSING_DATA = 4,
    OR_MISSING_NORMALS = 5,
    OR_NO_CORRESPONDENCES = 6,
    OR_DEGENERATE = 7,
    OR_INVALID_ARGUMENT = 8,
    OR_ERROR = 99
};

/* Field-for-field the same layout as lk_reg_params (include/loopkit_b200.h),
 * which mirrors RegistrationParams (proj/include/loopkit/registration.hpp:17-32). */
typedef struct or_params {
    double leaf;
    double normal_radius;
    double feature_radius;
    int64_t hypothesis_count;
    double similarity_tau;
    double d_max;
    double min_inlier_ratio;
    double max_fitness; /* < 0 => d_max^2 / 2 (resolved_max_fitness) */
    double normal_angle_max;
    uint64_t seed;
    int32_t threads;
    int32_t device_count;
} or_params;

typedef struct or_result {
    double R[9]; /* row-major */
    double t[3];
    double inlier_ratio;
    double fitness;
    int64_t inliers;
    int64_t hypothesis_index;
    int32_t found;
    int32_t _pad;
} or_result;

typedef struct or_stats {
    int64_t sampled;
    int64_t prerejected;
    int64_t degenerate;
    int64_t evaluated;
    int64_t qualified;
    /* work counters: W_ref, o*W_ref, k*W_ref, h*W_ref */
    int64_t w_ref;
    int64_t near_occupied;
    int64_t slots_scanned;
    int64_t nn_hits;
    double prepare_seconds;
    double hypothesis_seconds;
} or_stats;

const char* or_last_error(void);

/* ---- RNG (proj/include/loopkit/rng.hpp:14-46) ---- */
uint64_t or_splitmix64(uint64_t x);
void or_rng_u64(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out);
void or_rng_bounded(uint64_t seed, uint64_t stream, uint32_t bound, int64_t n, uint32_t* out);
void or_rng_double(uint64_t seed, uint64_t stream, int64_t n, double* out);

/* ---- sampling / pre-rejection (registration.cpp:21-51) ---- */
int or_sample_quadruples(int32_t source_size, const int32_t* cache, int64_t cache_len, uint64_t seed,
                         uint64_t stream, int32_t trials, int32_t* out_src, int32_t* out_tgt);
int or_prerejected(const double* src12, const double* dst12, double tau);

/* ---- Kabsch (geometry.cpp:62-91), Jacobi SVD restated ---- */
int or_kabsch(const double* src, const double* dst, int64_t n, double* R9, double* t3, double* sigma3);
int or_svd3(const double* A9, double* U9, double* S3, double* V9);

/* ---- SearchGrid / nn (grid.cpp:26-174) ---- */
void* or_search_grid_build(const double* xyz, int64_t n, double cell, const double* center3, int* status);
void or_search_grid_free(void* g);
int or_nn_within(void* g, const double* q3, double d_max, int32_t* idx, double* dist);
int or_nn_nearest(void* g, const double* q3, int32_t* idx, double* dist);
int64_t or_radius_search(void* g, const double* q3, double radius, int32_t* out, int64_t cap);
int or_bf_nn_within(const double* xyz, int64_t n, const double* q3, double d_max, int32_t* idx, double* dist);

/* ---- EvalGrid (registration.cpp:80-148) ---- */
void* or_eval_grid_build(const double* xyz, const double* nxyz, int64_t n, double d_max, int* status);
void or_eval_grid_free(void* g);
void or_eval_grid_dims(void* g, double* origin3, double* cell, int32_t* dims3, int64_t* ncells, int64_t* npts);
void or_eval_grid_arrays(void* g, int32_t* start, int32_t* index, double* slot_pos, double* slot_nrm,
                         uint8_t* near_occupied);
/* one evaluate_against_grid call (registration.cpp:155-219); returns 1 if fully scored, 0 on early exit */
int or_evaluate_against_grid(void* g, const double* src_xyz, const double* src_n, int64_t ns, const double* R9,
                             const double* t3, double d_max, double cos_max, int64_t miss_budget, double* ratio,
                             double* fitness, int64_t* inliers, int64_t* visited);

/* ---- evaluate_hypothesis (registration.cpp:53-78) ---- */
int or_evaluate_hypothesis(const double* R9, const double* t3, const double* src_xyz, const double* src_n,
                           int64_t ns, const double* tgt_xyz, const double* tgt_n, int64_t nt, double grid_cell,
                           const or_params* p, double* ratio, double* fitness, int64_t* inliers);

/* ---- explicit candidate list: a6 (mode 0, EvalGrid, optional early exit) or a7 (mode 1,
 *      evaluate_hypothesis over a SearchGrid of cell `grid_cell`), then a8 qualification + total order */
int or_score_candidates(const double* src_xyz, const double* src_n, int64_t ns, const double* tgt_xyz,
                        const double* tgt_n, int64_t nt, const double* Rt12, int64_t C, int32_t mode,
                        int32_t early_exit, double grid_cell, const or_params* p, double* out_ratio,
                        double* out_fitness, int64_t* out_inliers, int32_t* out_scored, or_result* best,
                        int64_t* qualified);

/* ---- preprocessing (preprocess.cpp:14-59, fpfh.cpp:17-141, reference.hpp:56-76) ---- */
int or_voxel_downsample(const double* xyz, const double* nxyz, int64_t n, double leaf, double* out_xyz,
                        double* out_n, int64_t* out_count);
int or_estimate_normals(const double* xyz, int64_t n, double radius, const double* viewpoint, int32_t threads,
                        double* out);
int or_compute_fpfh(const double* xyz, const double* nxyz, int64_t n, double radius, int32_t threads, float* out);
int or_feature_nn_cache(const float* sf, int64_t ns, const float* tf, int64_t nt, int32_t threads, int32_t* out);

/* ---- RegistrationContext (registration.cpp:223-251) + run_hypotheses (:253-332) ---- */
void* or_prepare(const double* sxyz, const double* sn, int64_t ns, const double* txyz, const double* tn, int64_t nt,
                 const or_params* p, int* status);
void* or_ctx_from_prepared(const double* sxyz, const double* sn, int64_t ns, const double* txyz, const double* tn,
                           int64_t nt, const int32_t* cache, double d_max, int* status);
void or_ctx_sizes(void* ctx, int64_t* ns, int64_t* nt);
void or_ctx_get(void* ctx, double* sxyz, double* sn, double* txyz, double* tn, int32_t* cache, float* sfeat,
                float* tfeat);
void or_ctx_free(void* ctx);
/* hypotheses [begin, end) of the run; the full run is begin=0, end=hypothesis_count */
int or_run_hypotheses(void* ctx, const or_params* p, int64_t begin, int64_t end, or_result* res, or_stats* st);
/* strict total order of run_hypotheses (registration.cpp:272-276); 1 if a beats b */
int or_better(const or_result* a, const or_result* b);

/* ---- edge_info (line_process.cpp:11-33) ---- */
int or_edge_info(const double* ci, int64_t ni, const double* cj, int64_t nj, const double* Ri9, const double* ti3,
                 const double* Rj9, const double* tj3, double epsilon, double* info36, int64_t* pair_count);

/* ICP point-to-plane (no reference; the builder's frozen spec, lk_oracle.cpp
 * "ICP point-to-plane"). history (nullable): max_iter x (count, rmse, |delta|^2). */
typedef struct or_icp_result {
    int32_t iterations;
    int32_t converged;
    int64_t correspondences;
    double rmse;
    double fitness;
} or_icp_result;
int or_icp_point_to_plane(const double* sxyz, int64_t ns, const double* txyz, const double* tn, int64_t nt,
                          const double* R0, const double* t0, double max_dist, int32_t max_iter, double eps,
                          double* R9, double* t3, or_icp_result* res, double* history);

/* propose_loops' overlap hit count of one pair (fragments.cpp:67-100) */
int or_overlap_hits(const double* later, int64_t nl, const double* Rl9, const double* tl3, const double* earlier,
                    int64_t ne, const double* Re9, const double* te3, double r, int64_t* hits);

#ifdef __cplusplus
}
#endif
#endif
