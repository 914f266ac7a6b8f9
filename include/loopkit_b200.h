/*
 * loopkit_b200.h -- C ABI of the B200-native global registration path.
 *
 * Drop-in boundary for the reference registration API
 * (/root/reference/proj/include/loopkit/registration.hpp). Every entry point
 * below names the reference interface it replaces. Plain pointers and sizes
 * only: no C++ types, no exceptions, no torch types. Errors are lk_status
 * codes mirroring proj/include/loopkit/errors.hpp; the message of the last
 * failure on the calling thread is available from lk_last_error().
 *
 * Clouds are caller-owned host arrays of packed FP64 xyz triples -- exactly
 * the memory layout of the reference's std::vector<Eigen::Vector3d>, so the
 * reference's PointCloud can be passed without copying.
 *
 * There is no CPU fallback: a call that needs the GPU returns LK_CUDA_ERROR
 * when no CUDA device is usable.
 */
#ifndef LOOPKIT_B200_H
#define LOOPKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LK_ABI_VERSION 2

/* proj/include/loopkit/errors.hpp:9-74 */
typedef enum lk_status {
    LK_OK = 0,
    LK_NO_ALIGNMENT = 1,        /* std::nullopt from register_global / run_hypotheses (not an error) */
    LK_EMPTY_CLOUD = 2,         /* EmptyCloud */
    LK_TOO_FEW_POINTS = 3,      /* TooFewPoints */
    LK_MISSING_DATA = 4,        /* MissingData */
    LK_MISSING_NORMALS = 5,     /* MissingNormals */
    LK_NO_CORRESPONDENCES = 6,  /* NoCorrespondences */
    LK_DEGENERATE = 7,          /* DegenerateConfiguration */
    LK_INVALID_ARGUMENT = 8,    /* Error (bad cell length / leaf, null pointers) */
    LK_CUDA_ERROR = 9,
    LK_NCCL_ERROR = 10,
    LK_ROTATION_TOO_LARGE = 11, /* RotationTooLarge (twist_from_transform at >= pi/2) */
    LK_INTERNAL_ERROR = 99
} lk_status;

/* proj/include/loopkit/geometry.hpp:92-99 (PointCloud): positions + optional normals */
typedef struct lk_cloud {
    const double* xyz;  /* n x 3, packed */
    const double* nxyz; /* n x 3 or NULL; a zero normal marks "invalid" */
    int64_t n;
} lk_cloud;

/* proj/include/loopkit/registration.hpp:17-32 (RegistrationParams) */
typedef struct lk_reg_params {
    double leaf;             /* 0.05 */
    double normal_radius;    /* 0.1 */
    double feature_radius;   /* 0.25 */
    int64_t hypothesis_count;/* 4,000,000 */
    double similarity_tau;   /* 0.9 */
    double d_max;            /* 0.075 */
    double min_inlier_ratio; /* 0.25 */
    double max_fitness;      /* < 0 => d_max^2 / 2 (resolved_max_fitness) */
    double normal_angle_max; /* 30 deg in radians */
    uint64_t seed;           /* 0 */
    int32_t threads;         /* host threads for the host prepare stage; 0 = all */
    int32_t device;          /* CUDA device ordinal; -1 = current */
    /* Devices one call uses (the reference's params.threads across GPUs,
     * registration.cpp:280): 0 or 1 = `device` alone; G > 1 = devices
     * device .. device + G - 1 (device -1 = from 0); -1 = every visible
     * device. A G-device context is prepared once on the first device and
     * broadcast over NCCL (ncclBroadcast); run_hypotheses gives device g the
     * contiguous hypothesis range [g H / G, (g + 1) H / G) and merges the G
     * rank records with one ncclAllReduce. Results are
     * bitwise identical for every G. */
    int32_t device_count;
    int32_t _reserved;
} lk_reg_params;

/* proj/include/loopkit/registration.hpp:34-39 (RegistrationResult) + inlier count */
typedef struct lk_reg_result {
    double R[9]; /* row-major rotation, maps source into the target frame */
    double t[3];
    double inlier_ratio;
    double fitness;
    int64_t inliers;
    int64_t hypothesis_index;
    int32_t found;
    int32_t _pad;
} lk_reg_result;

/* proj/include/loopkit/registration.hpp:91-99 (HypothesisStats) + work counters */
typedef struct lk_hyp_stats {
    int64_t sampled;
    int64_t prerejected;
    int64_t degenerate;
    int64_t evaluated;
    int64_t qualified;
    int64_t w_ref;          /* point visits of the reference loop (its static miss budget) */
    int64_t evals_executed; /* point evaluations the device actually executed */
    double prepare_seconds;
    double hypothesis_seconds;
} lk_hyp_stats;

/*
 * Per-rank record exchanged by the multi-GPU merge: the rank's best qualified
 * hypothesis plus its stats counters. 24 x 8 B = 192 B; an all-reduce(sum)
 * over a zero-filled [G x record] buffer is an exact all-gather.
 */
typedef struct lk_reg_record {
    int64_t valid;
    int64_t inliers;
    double fitness;
    int64_t index;
    double R[9];
    double t[3];
    int64_t sampled, prerejected, degenerate, evaluated, qualified;
    int64_t w_ref;
    int64_t evals_executed;
    int64_t _reserved;
} lk_reg_record;

/* Explicit-candidate score (evaluate_hypothesis, registration.cpp:53-78) */
typedef struct lk_cand_score {
    double inlier_ratio;
    double fitness;
    int64_t inliers; /* -1 when the candidate exited on the miss budget (early_exit mode) */
} lk_cand_score;

typedef struct lk_reg_ctx lk_reg_ctx;   /* RegistrationContext on one device */
typedef struct lk_grid lk_grid;         /* device grid over a target cloud */

int lk_abi_version(void);
const char* lk_last_error(void);
/* number of usable CUDA devices (0 on a host without a GPU) */
int lk_device_count(void);

/* ---- RegistrationContext --------------------------------------------------
 * prepare_registration (registration.hpp:105-107, registration.cpp:223-251),
 * all on the device: voxel downsample, estimate_normals for clouds given
 * without normals, FPFH, the feature pre-match (the binary's float matcher,
 * grid.cpp:176-213) and the EvalGrid. Throws-equivalents: LK_TOO_FEW_POINTS,
 * LK_MISSING_DATA, LK_MISSING_NORMALS. Returns as soon as the checks are
 * decided: the feature match may still run on the context's stream, which
 * every later call on the context is ordered behind (lk_reg_ctx_set_stream
 * first finishes the old stream's work). */
lk_status lk_reg_prepare(const lk_cloud* src, const lk_cloud* tgt, const lk_reg_params* params, lk_reg_ctx** out);
/* A RegistrationContext from already-prepared parts (downsampled clouds with
 * normals + the feature match cache), as when the reference's caller fills
 * RegistrationContext itself. The EvalGrid is built on the device. */
lk_status lk_reg_ctx_create(const lk_cloud* src, const lk_cloud* tgt, const int32_t* cache, const lk_reg_params* params,
                            lk_reg_ctx** out);
void lk_reg_ctx_destroy(lk_reg_ctx* ctx);
/* cudaStream_t to launch on (NULL = the context's own stream) */
lk_status lk_reg_ctx_set_stream(lk_reg_ctx* ctx, void* stream);
lk_status lk_reg_ctx_sizes(const lk_reg_ctx* ctx, int64_t* n_source, int64_t* n_target);
/* Per-kernel device timing with CUDA events on the launch stream. While
 * enabled, every run records events around k_hyp_sample, k_kabsch and
 * k_score; lk_reg_ctx_kernel_times returns the accumulated milliseconds of
 * the three kernels (ms3) and the number of runs (synchronises the events). */
lk_status lk_reg_ctx_set_profiling(lk_reg_ctx* ctx, int32_t enable);
lk_status lk_reg_ctx_kernel_times(lk_reg_ctx* ctx, double* ms3, int64_t* runs, int32_t reset);
/* The same events, per phase: ms[0..5] = k_hyp_sample, k_kabsch, then the
 * scorer (k_score_units + k_score_cta) in ms[2] with ms[3..5] = 0. */
lk_status lk_reg_ctx_phase_times(lk_reg_ctx* ctx, double* ms, int32_t n_phases, int64_t* runs, int32_t reset);
/* copy the prepared context back to the host (any pointer may be NULL) */
lk_status lk_reg_ctx_download(const lk_reg_ctx* ctx, double* src_xyz, double* src_n, double* tgt_xyz, double* tgt_n,
                              int32_t* cache, float* src_features, float* tgt_features);

/* ---- run_hypotheses (registration.hpp:116-118, registration.cpp:253-332) --
 * Returns LK_OK with result->found = 1, or LK_NO_ALIGNMENT (found = 0). */
lk_status lk_reg_run_hypotheses(lk_reg_ctx* ctx, const lk_reg_params* params, lk_reg_result* result,
                                lk_hyp_stats* stats);
/* One shard [begin, end) of the hypothesis range. The rank's record is
 * written to `record` (device pointer when record_on_device != 0, e.g. the
 * rank's slot of an NCCL buffer; host pointer otherwise). Asynchronous on
 * the context stream when record_on_device != 0. */
lk_status lk_reg_run_range(lk_reg_ctx* ctx, const lk_reg_params* params, int64_t begin, int64_t end,
                           lk_reg_record* record, int32_t record_on_device);
/* Exact merge of G per-rank records under the run_hypotheses total order
 * (registration.cpp:272-276); host-only, needs no GPU. */
lk_status lk_reg_merge_records(const lk_reg_record* records, int32_t count, int64_t n_source, lk_reg_result* result,
                               lk_hyp_stats* stats);

/* ---- one process per GPU (torchrun / MPI style) ---------------------------
 * Rank 0 creates an NCCL unique id and the caller broadcasts its 128 bytes to
 * every rank by any means; each rank attaches it to its own context
 * (ncclCommInitRank; the communicator belongs to the context). From then on
 * lk_reg_run_hypotheses on that context runs the rank's contiguous share
 * [rank H / nranks, (rank + 1) H / nranks), exchanges the rank records with
 * one ncclAllReduce over NVLink and returns the merged result on every rank
 * (identical to a 1-GPU run). lk_reg_run_exchange is the same without the
 * host merge: asynchronous on the context stream, it leaves the nranks
 * records in records_dev (device, nranks x lk_reg_record). */
lk_status lk_nccl_unique_id(uint8_t id[128]);
lk_status lk_reg_ctx_attach_comm(lk_reg_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank);
lk_status lk_reg_run_exchange(lk_reg_ctx* ctx, const lk_reg_params* params, lk_reg_record* records_dev);
/* number of devices (1 for a single-device context) and this context's rank */
lk_status lk_reg_ctx_topology(const lk_reg_ctx* ctx, int32_t* n_devices, int32_t* nranks, int32_t* rank);

/* ---- register_global (registration.hpp:121-124, registration.cpp:334-343) */
lk_status lk_register_global(const lk_cloud* src, const lk_cloud* tgt, const lk_reg_params* params,
                             lk_reg_result* result, lk_hyp_stats* stats);

/* ---- build_eval_grid (registration.hpp:79, registration.cpp:80-148) -------
 * kind 0: EvalGrid (cell = d_max, origin = bbox_lo - cell, dense CSR +
 *         26-dilated occupancy); kind 1: SearchGrid semantics
 *         (proj/src/grid.cpp:32-66: cells floor((p - 0) / cell), block
 *         radius ceil(d_max / cell)) stored densely over the occupied box. */
lk_status lk_grid_build(const lk_cloud* target, int32_t kind, double cell, double d_max, int32_t device, lk_grid** out);
void lk_grid_destroy(lk_grid* grid);
lk_status lk_grid_dims(const lk_grid* grid, double* origin3, double* cell, int32_t* dims3, int64_t* ncells,
                       int64_t* npoints);
lk_status lk_grid_download(const lk_grid* grid, int32_t* start, int32_t* index, double* slot_xyz, double* slot_n,
                           uint8_t* near_occupied);

/* ---- evaluate_hypothesis over an explicit candidate list ------------------
 * registration.hpp:60-63 (per candidate), plus run_hypotheses' qualification
 * and total order for `best`. Rt = C x 12 doubles (R row-major, then t).
 * kind-1 grid: evaluate_hypothesis semantics (fitness from sqrt(d2)^2);
 * kind-0 grid: evaluate_against_grid semantics (fitness from d2), with the
 * miss-budget early exit when early_exit != 0. per_cand may be NULL. */
lk_status lk_score_candidates(lk_grid* grid, const lk_cloud* src, const double* Rt, int64_t C,
                              const lk_reg_params* params, int32_t early_exit, lk_cand_score* per_cand,
                              lk_reg_result* best, int64_t* qualified);

/* ---- edge_info (proj/src/line_process.cpp:11-33), batched -----------------
 * For pair k: cloud_i = clouds_i[k], cloud_j = clouds_j[k], poses T_i/T_j as
 * 12 doubles each (R row-major, t). info = 36 doubles per pair (row-major
 * 6x6), pair_count per pair; a pair with no correspondence reports
 * pair_count 0 (the reference throws NoCorrespondences). */
lk_status lk_edge_info_batched(const lk_cloud* clouds_i, const lk_cloud* clouds_j, const double* Ti, const double* Tj,
                               int64_t n_pairs, double epsilon, int32_t device, double* info, int64_t* pair_count);

/* ---- batched loop verification (north-star item 5, config E) -------------
 * Per pair k, with Q = clouds_i[k] (the earlier fragment, pose Ti[k]),
 * P = clouds_j[k] (the later fragment, pose Tj[k]) and the measurement
 * T[k] mapping P into Q's frame, all bit-exact against the reference:
 *   info / pair_count  edge_info(Q, P, Ti, Tj, epsilon)   line_process.cpp:11-33
 *   overlap            propose_loops' overlap of the pair  fragments.cpp:80-100
 *                      (Tj P points within overlap_radius of Ti Q)
 *   inliers / ratio / fitness
 *                      evaluate_hypothesis(T, P, Q, SearchGrid(Q, grid_cell))
 *                                                          registration.cpp:53-78
 * A pair without edge correspondences reports pair_count 0 (the reference
 * throws NoCorrespondences); clouds must be non-empty and carry normals. */
typedef struct lk_verify_params {
    double epsilon;          /* edge_info radius */
    double overlap_radius;   /* LoopParams::overlap_radius (fragments.hpp) */
    double d_max;            /* RegistrationParams::d_max */
    double grid_cell;        /* SearchGrid cell of evaluate_hypothesis's target grid; <= 0 -> d_max */
    double normal_angle_max; /* RegistrationParams::normal_angle_max (radians) */
    int32_t device;          /* -1: current device */
    /* 0 / 1: `device` alone; G > 1: the pairs split into G contiguous shares
     * on devices device .. device + G - 1 (no exchange: pairs are
     * independent); -1: every visible device */
    int32_t device_count;
} lk_verify_params;

typedef struct lk_verify_result {
    double info[36];      /* row-major 6x6 */
    int64_t pair_count;
    int64_t overlap_hits;
    double overlap;       /* overlap_hits / |P| */
    int64_t inliers;
    double inlier_ratio;  /* inliers / |P| */
    double fitness;       /* sum of distance^2 / inliers (0 without inliers) */
} lk_verify_result;

lk_status lk_verify_batch(const lk_cloud* clouds_i, const lk_cloud* clouds_j, const double* Ti, const double* Tj,
                          const double* T, int64_t n_pairs, const lk_verify_params* params, lk_verify_result* out);

/* ---- propose_loops (fragments.hpp:46-60, fragments.cpp:61-109) -----------
 * Replaces loopkit::propose_loops(std::span<const Fragment>, const PoseGraph&,
 * const LoopParams&). fragments[f] = Fragment::cloud (local frame; normals
 * ignored), poses = PoseGraph::poses (n x 12: row-major R, t), loops =
 * PoseGraph::loops as (i, j) pairs (either orientation suppresses a pair).
 * Every pair (later i, earlier j) with i >= j + 2 whose overlap -- the
 * fraction of i's posed points with a posed point of j within overlap_radius
 * (the reference SearchGrid's nn_within) -- reaches min_overlap, sorted by
 * overlap desc, then i, then j. Writes min(count, capacity) proposals and
 * the full count to n_out. Throws-equivalents: LK_EMPTY_CLOUD (an empty
 * fragment), LK_INVALID_ARGUMENT (overlap_radius <= 0). */
typedef struct lk_loop_params {
    double overlap_radius; /* LoopParams::overlap_radius (0.1) */
    double min_overlap;    /* LoopParams::min_overlap (0.2) */
    int32_t device;        /* -1 = current */
    int32_t _pad;
} lk_loop_params;
typedef struct lk_loop_proposal {
    int32_t i; /* later fragment */
    int32_t j; /* earlier fragment */
    double overlap;
} lk_loop_proposal;
lk_status lk_propose_loops(const lk_cloud* fragments, const double* poses, int32_t n, const int32_t* loops,
                           int32_t n_loops, const lk_loop_params* params, lk_loop_proposal* out, int64_t capacity,
                           int64_t* n_out);

/* ---- line-process weight of a loop edge (host; consumer of edge_info) -----
 * Transforms are 12 doubles (row-major R, then t); info is the row-major 6x6
 * of lk_verify_result / lk_edge_info_batched.
 *   lk_edge_residual  f = xi^T Lambda xi, xi = twist(rel * T_j^-1 * T_i)
 *                     line_process.cpp:35-40 (twist: geometry.cpp:28-40);
 *                     LK_ROTATION_TOO_LARGE when the residual rotation
 *                     reaches pi/2.
 *   lk_update_weight  (mu / (mu + max(f, 0)))^2 clamped to [0, 1]; 0 when
 *                     mu <= 0                         line_process.cpp:42-46
 *   lk_loop_weights   per edge: mu = mu_tau * pair_count, the residual with
 *                     the small-angle gate of loop_residual (weight 0 beyond
 *                     pi/2), the weight, and accepted = weight >= threshold
 *                     line_process.cpp:52-67, 100-103 (labels at given poses)
 * Host-only arithmetic in the reference's evaluation order (libm asin /
 * atan2 / acos); no device is used. */
lk_status lk_edge_residual(const double* Ti, const double* Tj, const double* rel, const double* info36, double* f);
double lk_update_weight(double f, double mu);
lk_status lk_loop_weights(int64_t n, const double* Ti, const double* Tj, const double* rel, const double* info36,
                          const int64_t* pair_count, double mu_tau, double threshold, double* weight,
                          int32_t* accepted);

/* ---- feature pre-match (registration.cpp:248 -> grid.cpp:176-213) ---------
 * argmin_j ||F(p_i) - F(q_j)||^2 in FP64, ties -> lowest j. */
lk_status lk_feature_nn_cache(const float* src_features, int64_t ns, const float* tgt_features, int64_t nt,
                              int32_t device, int32_t* cache);

/* ---- ICP point-to-plane refinement (north-star item 4, config D) ---------
 * No reference implementation exists (SPEC.md:332 lists ICP as a non-goal);
 * the specification is frozen in DESIGN.md "ICP" and its CPU oracle
 * (oracle/lk_oracle.cpp): correspondences are the EvalGrid NN within
 * max_correspondence_distance (registration.cpp:165-199 semantics), the
 * residual is (T p - q) . n_q with J = (T p x n_q, n_q) (the G_p convention of
 * line_process.cpp:23-28), the 6x6 system is reduced in a fixed tree order
 * and solved by LDL^T, and T is updated by the Cayley map. Refines T0 (12
 * doubles, R row-major then t); history (nullable) receives max_iterations x
 * (correspondences, rmse, |delta|^2). LK_NO_CORRESPONDENCES when the first
 * iteration finds fewer than 6 pairs; LK_MISSING_NORMALS without target
 * normals. */
typedef struct lk_icp_params {
    double max_correspondence_distance; /* > 0 (metres) */
    int32_t max_iterations;
    int32_t device;                     /* -1: current device */
    double convergence_eps;             /* stop once |delta| < eps */
} lk_icp_params;

typedef struct lk_icp_result {
    double R[9]; /* row-major */
    double t[3];
    int32_t iterations;     /* updates applied */
    int32_t converged;
    int64_t correspondences; /* of the last accumulation */
    double rmse;             /* sqrt(sum r^2 / correspondences) of the last accumulation */
    double fitness;          /* correspondences / source size */
} lk_icp_result;

lk_status lk_icp_point_to_plane(const lk_cloud* source, const lk_cloud* target, const double* T0,
                                const lk_icp_params* params, lk_icp_result* result, double* history);

/* the pieces of prepare_registration as separate device calls */
/* voxel_downsample (preprocess.hpp / preprocess.cpp:14-59) */
lk_status lk_voxel_downsample(const lk_cloud* cloud, double leaf, double* out_xyz, double* out_n, int64_t* out_count);
/* estimate_normals (preprocess.hpp / preprocess.cpp:61-96): out_normals n x 3,
 * oriented toward viewpoint (3 doubles; NULL = origin), zero where fewer than
 * 3 points lie within radius. register_global / lk_reg_prepare call it with
 * normal_radius and the origin for clouds given without normals
 * (registration.cpp:232-237). */
lk_status lk_estimate_normals(const lk_cloud* cloud, double radius, const double* viewpoint, int32_t device,
                              double* out_normals);
lk_status lk_compute_fpfh(const lk_cloud* cloud, double radius, int32_t threads, float* out);

#ifdef __cplusplus
}
#endif
#endif /* LOOPKIT_B200_H */
