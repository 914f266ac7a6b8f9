// lk_kernels.cuh -- device data layout and kernel launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lkk {

// Stream-ordered allocations from the device's default memory pool (its
// release threshold is raised when a device is selected), so building and
// dropping contexts per registration does not pay cudaMalloc / cudaFree.
template <class T>
inline cudaError_t pool_alloc(T** p, size_t bytes, cudaStream_t s) {
    return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, s);
}
inline void pool_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// LK_TRACE=2 only: a device-event mark on stream s inside a prepare phase
// (defined in lk_abi.cu; a no-op otherwise).
void trace_point(const char* what, cudaStream_t s);

// Pinned host scratch for small device->host readbacks (counts, bounding
// boxes, records), one buffer per host thread. A readback into pageable
// memory goes through the driver's staging path and queues behind in-flight
// bulk copies (the other cloud's upload); a pinned one does not.
inline void* host_scratch(size_t bytes) {
    struct Buf {
        void* p = nullptr;
        size_t cap = 0;
        ~Buf() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Buf b;
    if (bytes > b.cap) {
        if (b.p) cudaFreeHost(b.p);
        b.p = nullptr;
        b.cap = 0;
        const size_t cap = bytes < 65536 ? 65536 : bytes;
        if (cudaHostAlloc(&b.p, cap, 0) != cudaSuccess) return nullptr;
        b.cap = cap;
    }
    return b.p;
}

// Dense CSR cell grid over a target cloud.
//  kind 0 = EvalGrid   (proj/src/registration.cpp:80-148): origin = bbox_lo - cell,
//           cell = d_max, block radius 1, local cell = floor((y - origin) / cell).
//  kind 1 = SearchGrid (proj/src/grid.cpp:26-109): cells floor((y - center) / cell)
//           with center 0, stored densely over the occupied box padded by the
//           block radius r = ceil(d_max / cell); local = cell - off.
// Slots are sorted by cell, ascending original index inside a cell.
struct GridView {
    double ox, oy, oz;  // subtracted before the division (origin or center)
    double cell;
    int nx, ny, nz;
    int offx, offy, offz;
    int radius;
    int kind;
    const int32_t* start;    // ncells + 1
    const int32_t* index;    // slot -> original target index
    const double* slot_pos;  // 3 * npoints, CSR order
    const double* slot_nrm;  // 3 * npoints, CSR order (zeros when absent)
    const uint8_t* near;     // ncells: some point within the block of this cell
    // Block lists (radius-1 grids): for every cell, the points of its 3x3x3
    // block stored contiguously, so a query is one 8-byte cell load plus a
    // linear scan of 32-byte entries. count == 0 <=> not near-occupied.
    const int2* block_info;    // (offset, count) per cell; null when not built
    const double4* block_pts;  // x, y, z, original index
    const double* nrm_orig;    // 3 * npoints normals in original point order
    // FP32 image of the block lists for the guard-band fast path: local cell
    // coordinates ((x - o) / cell - off) rounded to float, original index in w.
    const float4* block_f32;
    const double* pos_orig;    // 3 * npoints positions in original point order
    // Fine lists (radius-1 grids): cells of half the size over the same box,
    // each listing the entries of its cell's block list within fine_dmax of
    // the fine box that can be the nearest neighbour somewhere in it (Voronoi
    // pruned); FP32 fine-cell coordinates ((x - o) / fcell - 2 off), original
    // index in w.
    int fnx, fny, fnz;
    double fcell;
    double fine_dmax;
    const int2* fine_info;
    const float4* fine_pts;
    // sizes (elements) of the arrays above, for L2 prefetching
    int64_t n_points, n_cells, n_fine, n_fine_entries;
    // resolution records in original point order (radius-1 grids with blocks)
    const double4* pos4_orig;  // (x, y, z, 0) FP64
    const float4* nrm32_orig;  // FP32 normals for the guarded normal gate
};

struct GridStorage {
    GridView view{};
    int64_t ncells = 0;
    int64_t npoints = 0;
    int64_t nblock = 0;
    int32_t* start = nullptr;
    int32_t* index = nullptr;
    double* slot_pos = nullptr;
    double* slot_nrm = nullptr;
    uint8_t* near = nullptr;
    int2* block_info = nullptr;
    double4* block_pts = nullptr;
    double* nrm_orig = nullptr;
    float4* block_f32 = nullptr;
    double* pos_orig = nullptr;
    int64_t nfine = 0, nfine_entries = 0;
    int2* fine_info = nullptr;
    float4* fine_pts = nullptr;
    double4* pos4_orig = nullptr;
    float4* nrm32_orig = nullptr;
    cudaStream_t stream = nullptr;  // allocation stream
    void release();
};

// Ring grid (lk_ring.cu): dense CSR of small cells for exact NN on dense
// targets, with the reference EvalGrid's frame for the window check.
struct RingGrid {
    double ox, oy, oz, cell;  // ring cells: origin = bbox_lo
    int nx, ny, nz;
    int rmax;                 // shells beyond which nothing lies within d_max
    int64_t ncells, npoints;
    float delta;              // FP32 coordinate error (cells, both sides)
    float band;               // guard on FP32 d2 (squared cells)
    float thr;                // d_max^2 in squared cells
    const int32_t* start;     // ncells + 1
    const float4* pts;        // CSR order: ring-cell coordinates, original index in w
    const double4* pos4;      // original order FP64 (x, y, z, 0)
    // Chebyshev distance (cells, capped at rmax + 2) from each cell to the
    // nearest occupied cell, or null: shells nearer than it hold no entries
    const uint8_t* dt;
    // the reference grid whose window the answer must come from: the
    // EvalGrid (origin bbox_lo - d_max, cell d_max, +-1 cells, queries outside
    // [0, en) miss; registration.cpp:82-97,165-199) or a SearchGrid (center 0,
    // cell length, +-ceil(d_max / cell) cells, unbounded; grid.cpp:26-30,78-109)
    double eox, eoy, eoz, ecell;
    int enx, eny, enz;
    int ewin;      // window half-width in reference cells
    int ebounded;  // 1: EvalGrid range check on the query cell
};
RingGrid ring_frame(const double* lo, const double* hi, double d_max, double search_cell, int64_t max_cells,
                    bool fast, double divisor = 6.0);
struct RingStorage {
    RingGrid view{};
    int32_t* start = nullptr;
    float4* pts = nullptr;
    double4* pos4 = nullptr;
    uint8_t* dt = nullptr;
    cudaStream_t stream = nullptr;
    void release();
};
cudaError_t build_ring_grid(RingStorage& rs, const double* d_pos, int64_t n, double d_max, cudaStream_t stream,
                            bool fast = true);
// Morton order of a cloud's points (d_perm: n indices), for coherent queries.
cudaError_t spatial_order(const double* d_pos, int64_t n, int32_t* d_perm, cudaStream_t stream);
// The same within each run of `block` consecutive points.
cudaError_t spatial_order_blocks(const double* d_pos, int64_t n, int64_t block, int32_t* d_perm,
                                 cudaStream_t stream);
// K ring grids in one pass over K concatenated clouds (h_offsets: K + 1 point
// offsets into d_pos). Grid k answers radius h_dmax[k] in the window of an
// EvalGrid (h_cell[k] <= 0) or of a SearchGrid with cell length h_cell[k].
// d_views (K RingGrid on the device) and the storage stay valid until release.
struct RingBatch {
    int32_t* start = nullptr;
    float4* pts = nullptr;
    double4* pos4 = nullptr;
    RingGrid* d_views = nullptr;
    cudaStream_t stream = nullptr;
    void release();
};
cudaError_t build_ring_grids(RingBatch& rb, const double* d_pos, const int64_t* h_offsets, int32_t K,
                             const double* h_dmax, const double* h_cell, cudaStream_t stream);

// Builds a grid of the given kind from device arrays pos/nrm (nrm may be null).
// Returns cudaSuccess or the first CUDA error; throws nothing.
// with_blocks = false skips the 3x3x3 block lists (neighbour grids of FPFH).
cudaError_t build_grid(GridStorage& g, int kind, const double* d_pos, const double* d_nrm, int64_t n, double cell,
                       double d_max, cudaStream_t stream, bool with_blocks = true);

// ---- hypothesis pipeline --------------------------------------------------
struct Counters {  // device-side, zeroed per run
    unsigned long long n_survivors;   // passed pre-rejection
    unsigned long long n_candidates;  // non-degenerate (= evaluated)
    unsigned long long prerejected;
    unsigned long long degenerate;
    unsigned long long qualified;
    unsigned long long w_ref;
    unsigned long long evals_executed;
    unsigned long long work_next;   // work queue head for k_score
    unsigned long long blocks_done; // last-block-done ticket
    unsigned long long n_full;      // split candidates that were fully scored
    unsigned long long fin_done;    // last-CTA ticket of the record-writing scorer
    unsigned long long work_next2;  // candidate ticket of k_score_cta (after the units)
    unsigned long long _pad[4];
};

struct BestRec {  // per-block best, then the final record
    int64_t valid;
    int64_t inliers;
    double fitness;
    int64_t index;
    int64_t slot;  // candidate slot holding R, t
};

struct RunBuffers {
    int64_t capacity = 0;        // hypotheses per launch chunk
    int64_t* surv_index = nullptr;  // survivor hypothesis index
    int32_t* surv_ids = nullptr;    // 8 per survivor: src[4], tgt[4]
    int64_t* cand_index = nullptr;  // candidate hypothesis index
    double* cand_rt = nullptr;      // 12 per candidate: R row-major, t
    Counters* counters = nullptr;
    BestRec* block_best = nullptr;
    int32_t n_blocks = 0;
    void* cand_fast = nullptr;  // per-candidate FP32 transform + guard bands (explicit lists, k_score)
    int64_t fast_capacity = 0;
    cudaStream_t stream = nullptr;  // allocation stream (set by the owner)
    void release();
    cudaError_t ensure(int64_t cap, int32_t score_blocks);
    cudaError_t ensure_fast(int64_t n);
    // candidate-CTA scoring: two scratch slots per CTA (addends + ballot words)
    double* cta_add = nullptr;
    uint32_t* cta_inl = nullptr;
    int64_t cta_slots = 0, cta_ns_pad = 0;
    cudaError_t ensure_cta(int64_t ns, int32_t n_ctas);
    // round-unit scoring: per candidate ballots, addends, sum and unit count
    uint32_t *u_miss = nullptr, *u_inl = nullptr;
    double *u_add = nullptr, *u_sum = nullptr;
    unsigned* u_done = nullptr;
    int64_t u_cap = 0, u_ns_pad = 0;
    cudaError_t ensure_units(int64_t ns, int64_t cap);
};

struct SourceView {
    const double* pos;    // 3 * ns
    const double* nrm;    // 3 * ns
    const float4* pos32;  // ns float copies (x, y, z, 0) for the fast path; null -> FP64 only
    int64_t n;
    // resolution records of the fast path (null -> FP64 arrays above):
    const double4* pos4 = nullptr;  // (x, y, z, 0) FP64, one sector per point
    const float4* nrm32 = nullptr;  // FP32 normals for the guarded normal gate
};

struct ScoreParams {
    double d2_max;
    double d_max;
    double cos_max;
    double min_ratio;
    double max_fitness;
    int64_t miss_budget;  // INT64_MAX disables the early exit
    int32_t fitness_from_distance;  // 1: sum sqrt(d2)^2 (evaluate_hypothesis), 0: sum d2
    int32_t fast;         // 1: FP32 guard-band scan with exact FP64 decisions
    float thr_cells;      // (d_max / cell)^2: d2_max in squared cell units
    float band_cells;     // guard band on d2 in squared cell units
    float eps_cells;      // guard on cell-coordinate fractions
    float pmax_cells;     // max |p| over the source, in cells
    float nmax_cells;     // max grid dimension
};

// Fills ScoreParams' fast-path fields for a grid; disables the fast path when
// the magnitudes exceed what its guard bands cover.
void configure_fast_path(ScoreParams& sp, const GridView& g, double max_abs_source);

cudaError_t make_source32(const double* d_pos, int64_t n, float4* d_out, cudaStream_t stream);
// (x, y, z, 0) FP64 records and FP32 copies of 3 * n FP64 arrays (either output may be null)
cudaError_t make_records(const double* d_pos, const double* d_nrm, int64_t n, double4* d_pos4, float4* d_nrm32,
                         cudaStream_t stream);

// Samples, pre-rejects and fits hypotheses [begin, end); scores the
// candidates; reduces the per-run best into `record` (an lk_reg_record, device).
// `events` (nullable): kPhaseEvents events on the launch stream bracketing the
// phase events: [0] k_hyp_sample [1] k_kabsch [2] [3] the scorer
// (k_score_units + k_score_cta) [4] [5] [6] (the last three coincide)
constexpr int kPhaseEvents = 7;
cudaError_t run_hypotheses_range(const SourceView& src, const double* d_tgt_pos, const int32_t* d_cache,
                                 const GridView& grid, const ScoreParams& sp, uint64_t seed, double tau, int64_t begin,
                                 int64_t end, RunBuffers& rb, void* d_record, cudaStream_t stream, int sm_count,
                                 cudaEvent_t* events = nullptr);

// ICP point-to-plane (lk_icp.cu; spec frozen in oracle/lk_oracle.cpp "ICP").
// `ring` is the target's ring grid at d_max = max_dist, d_tnrm its normals
// (3 * nt FP64, original order); d_src is 3 * n FP64.
struct IcpOutcome {
    int32_t iterations, converged, status;
    int64_t correspondences;
    double rmse, fitness;
};
cudaError_t icp_point_to_plane(const double* d_src, int64_t n, const RingStorage& ring, const double* d_tnrm,
                               double max_dist, int32_t max_iter, double eps, const double* R0, const double* t0,
                               double* R9, double* t3, IcpOutcome* out, double* d_history, cudaStream_t stream,
                               int sm_count);

// Batched loop verification (lk_verify.cu). Host arrays: clouds concatenated
// with K + 1 point offsets; T_i, T_j, T as 12 doubles per pair. `full` = 0
// computes edge_info only (normals and T unused).
struct VerifyInput {
    int32_t n_pairs;
    // per pair host pointers (3 * n doubles each); Q = cloud_i (earlier), P = cloud_j (later)
    const double* const* qpos;
    const double* const* qnrm;
    const double* const* ppos;
    const double* const* pnrm;
    const int64_t *offq, *offp;
    const double *Ti, *Tj, *T;
    double epsilon, overlap_radius, d_max, grid_cell, cos_max;
    int32_t full;
};
struct VerifyOutput {
    double info[36];
    int64_t pair_count, overlap_hits, inliers;
    double sq_sum;  // evaluate_hypothesis's sequential sum of distance^2
};
cudaError_t verify_batch(const VerifyInput& in, VerifyOutput* out, cudaStream_t stream);
// propose_loops (proj/src/fragments.cpp:61-109): hit counts of the K pairs
// (h_pairs[2k] = later i, [2k+1] = earlier j) over n fragments (h_xyz packed,
// fragment f = points [h_foff[f], h_foff[f+1]) in its local frame, pose h_T12[12 f]).
cudaError_t propose_loops(const double* h_xyz, const int64_t* h_foff, int32_t n, const double* h_T12,
                          const int32_t* h_pairs, int32_t K, double radius, int64_t* h_hits, cudaStream_t stream);

// Scores an explicit candidate list (Rt on device, C x 12) and reduces the best.
cudaError_t score_candidates(const SourceView& src, const GridView& grid, const ScoreParams& sp, const double* d_rt,
                             int64_t C, RunBuffers& rb, int64_t* d_out_inliers, double* d_out_sum,
                             void* d_record, cudaStream_t stream, int sm_count, const RingGrid* ring = nullptr);

// exclusive scan of n int32 into out[0..n] (out[n] = total), stream-ordered
cudaError_t exclusive_scan(const int32_t* d_in, int64_t n, int32_t* d_out, cudaStream_t stream);
// the same with caller-provided temporary storage (scan_temp_bytes(n)), and
// d_out[0] left to the caller when zero_first is false: no allocation, no
// memset, only the scan's two kernels go on the stream
size_t scan_temp_bytes(int64_t n);
cudaError_t exclusive_scan(const int32_t* d_in, int64_t n, int32_t* d_out, cudaStream_t stream, void* temp,
                           size_t temp_bytes, bool zero_first);

// Stream-ordered scratch for the prepare's temporaries: one device buffer per
// stream, reused by every call on that stream (its earlier users are ordered
// before on the stream, so reuse needs no wait), held by one host scope at a
// time. Replaces the cudaMallocAsync / cudaFreeAsync pairs of a call: each is
// a stream command, ~3 us of the device front end's time while the other
// cloud's upload saturates PCIe (tools/launch_under_dma.cu).
class Scratch {
  public:
    Scratch(cudaStream_t s, size_t bytes);  // locks the stream's buffer, grows it to `bytes`
    ~Scratch();
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    static size_t round(size_t bytes) { return (bytes + 255) & ~size_t(255); }
    // nullptr (and status() an error) past the reserved size
    template <class T>
    T* take(size_t count) {
        const size_t b = round((count > 0 ? count : 1) * sizeof(T));
        if (err_ != cudaSuccess || top_ + b > cap_) {
            if (err_ == cudaSuccess) err_ = cudaErrorMemoryAllocation;
            return nullptr;
        }
        T* p = reinterpret_cast<T*>(base_ + top_);
        top_ += b;
        return p;
    }
    cudaError_t status() const { return err_; }

  private:
    struct Entry;
    Entry* e_ = nullptr;
    char* base_ = nullptr;
    size_t cap_ = 0, top_ = 0;
    cudaError_t err_ = cudaSuccess;
};

// ---- device prepare_registration ---------------------
// voxel_downsample (proj/src/preprocess.cpp:14-59) on the device: returns the
// downsampled count; out_pos / out_nrm (capacity n) in first-index order.
// Status: 0 ok, 5 invalid normals (MissingNormals), 2 empty, or a CUDA error
// reported through cudaError_t. h_stats (optional, page-locked, 2 words):
// cloud_stats_async of the output, copied back on the stream (d_nrm given).
cudaError_t voxel_downsample(const double* d_pos, const double* d_nrm, int64_t n, double leaf, double* d_out_pos,
                             double* d_out_nrm, int64_t* out_count, int* status, cudaStream_t stream,
                             unsigned long long* h_stats = nullptr);
// estimate_normals (proj/src/preprocess.cpp:61-96) on the device: n x 3 normals
// oriented to `viewpoint` (3 doubles, host), zero where fewer than 3
// neighbours lie within `radius`.
cudaError_t estimate_normals(const double* d_pos, int64_t n, double radius, const double* viewpoint, double* d_out,
                             cudaStream_t stream);
// compute_fpfh (proj/src/fpfh.cpp:57-141) on the device: 33 floats per point.
cudaError_t compute_fpfh(const double* d_pos, const double* d_nrm, int64_t n, double radius, float* d_out,
                         cudaStream_t stream);

// Usable (non-zero) normal count and max |p| of a device cloud (synchronous).
// usable-normal count and max |p| into h_out2 (pinned host, 2 x u64) without
// waiting; cloud_stats_decode reads them once the stream has synchronised
cudaError_t cloud_stats_async(const double* d_pos, const double* d_nrm, int64_t n, unsigned long long* h_out2,
                              cudaStream_t stream);
void cloud_stats_decode(const unsigned long long* h2, int64_t* usable, double* max_norm);
cudaError_t cloud_stats(const double* d_pos, const double* d_nrm, int64_t n, int64_t* usable, double* max_norm,
                        cudaStream_t stream);

// Feature NN with the reference binary's float scores, ties -> lowest index
// (grid.cpp:176-213).
cudaError_t feature_nn(const float* d_sf, int64_t ns, const float* d_tf, int64_t nt, int32_t* d_out,
                       cudaStream_t stream);
// The same in two steps: fnn_prepare per cloud as soon as its features exist
// (the padded layout the match reads; for the target also |q|^2), then
// feature_nn_prepared once both are ready.
size_t fnn_padded_bytes(int64_t n);
cudaError_t fnn_prepare(const float* d_f, int64_t n, float4* d_padded, float* d_q2, cudaStream_t stream);
cudaError_t feature_nn_prepared(const float* d_sf, const float4* d_sp, int64_t ns, const float* d_tf,
                                const float4* d_tp, const float* d_q2, int64_t nt, int32_t* d_out,
                                cudaStream_t stream);

// edge_info for one pair given a kind-1 grid over posed cloud_j.
cudaError_t edge_info(const double* d_ci, int64_t ni, const double* Ti12, const GridView& grid, double eps,
                      double* d_partials, int n_partial_blocks, double* d_info, unsigned long long* d_count,
                      cudaStream_t stream);

// y = T * x for n points (device), reference evaluation order
cudaError_t transform_points(const double* d_in, int64_t n, const double* T12, double* d_out, cudaStream_t stream);

}  // namespace lkk
