/* include/netrec_b200.h — C-ABI of libnetrec_b200.so, the B200-native GCD hot path.
 *
 * The reference (netrec, arXiv 2401.01404; /root/reference/proj/include/netrec/,
 * shortened to inc/) is a header-only C++20 library whose only plug-in seam on this
 * path is the template distance callable `Dist&& d : double(NodeId, NodeId)` taken by
 * find_knn / find_best (inc/knn.hpp:150-151, inc/find_best.hpp:186-188) with
 * ModelDistance (inc/model.hpp:389-400) as the concrete plug, driven by
 * reconstruct_gcd (inc/reconstruct.hpp:148-181).  Each entry point below names the
 * reference symbol it replaces.  Plain pointers and sizes only; host buffers unless
 * a name ends in _device.
 *
 * Conventions:
 *   - every function returns 0 on success or an errno-style code:
 *       NRG_EINVAL    -> std::invalid_argument  (validation)
 *       NRG_ERANGE    -> std::out_of_range      (node ids)
 *       NRG_EOVERFLOW -> std::overflow_error    (non-finite objective)
 *       NRG_ECUDA / NRG_EIO -> std::runtime_error
 *     with a thread-local message from nrg_last_error();
 *   - warnings are counters (nrg_counters), as inc/model.hpp:270-271;
 *   - everything is synchronous on the context's CUDA stream.
 */
#ifndef NETREC_B200_H
#define NETREC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NRG_OK 0
#define NRG_EIO 5
#define NRG_EINVAL 22
#define NRG_ERANGE 34
#define NRG_EOVERFLOW 75
#define NRG_ECUDA 100

/* ModelKind (inc/model.hpp:20) */
#define NRG_ISING 0
#define NRG_GAUSSIAN 1
/* DistanceMode (inc/model.hpp:21) + device-resident test metrics standing in for the
 * generic callables of the reference tests (TableMetric test_findbest.cpp:20-37,
 * LineMetric test_knn.cpp:16-29) */
#define NRG_EXACT 0
#define NRG_GRADIENT 1
#define NRG_TABLE 2
#define NRG_LINE 3

typedef struct nrg_ctx nrg_ctx;

/* == CandidateEdge (inc/common.hpp:15-19): canonical i < j */
typedef struct {
    int32_t i, j;
    double dist;
} nrg_pair;

/* == TraceLevel (inc/find_best.hpp:19-28) */
typedef struct {
    int32_t level, k, exhaustive, knn_sweeps;
    uint64_t nodes, dedup_size;
} nrg_trace_level;

/* == IterationRecord (inc/reconstruct.hpp:22-28) */
typedef struct {
    int32_t iter, pad;
    double delta, seconds;
    uint64_t candidates;
    double objective;
} nrg_iter_record;

/* == KnnParams (inc/knn.hpp:92-104); threads is accepted and ignored (results are
 * thread-count independent, test_knn.cpp:181-194).  reverse != 0 selects the
 * reverse-list NNDescent variant (in-edges always admitted) instead of the
 * reference-exact U construction. */
typedef struct {
    double eps;
    uint64_t seed;
    int32_t max_sweeps, scan_floor, width_floor, threads;
    int32_t reverse, pad;
} nrg_knn_params;

/* == FindBestParams (inc/find_best.hpp:45-49) */
typedef struct {
    double knn_eps;
    uint64_t seed;
    int32_t threads, reverse;
} nrg_fb_params;

/* == ReconstructionConfig (inc/reconstruct.hpp:45-55) minus the std::function hook;
 * the hook is served by nrg_gcd_iteration's candidate output. */
typedef struct {
    double kappa, eps;
    int32_t max_iters, mode;
    double knn_eps;
    uint64_t seed;
    int32_t threads, reverse;
} nrg_gcd_cfg;

const char* nrg_last_error(void);
int nrg_version(void);

/* Context = PseudoLikelihood + SparseWeights + SampleMatrix + DistanceCache resident
 * on one GPU (inc/model.hpp:107-124, inc/sparse_weights.hpp:24-32).  `lambda` as
 * PseudoLikelihood(kind, lambda, ...); validation as inc/model.hpp:115-123 happens
 * when samples are uploaded. */
int nrg_create(nrg_ctx** out, int32_t n, int32_t m, int32_t kind, double lambda, int32_t device);
int nrg_destroy(nrg_ctx* ctx);

/* SampleMatrix upload (inc/sample_matrix.hpp:14-46), row-major N x M doubles.
 * Ising data must be exactly +/-1 (inc/model.hpp:118-119).  Resets the state to
 * make_empty_state (inc/model.hpp:404-416). */
int nrg_upload_samples(nrg_ctx* ctx, const double* X);
/* Ising fast path: N x M int8 spins (+1/-1). */
int nrg_upload_spins_i8(nrg_ctx* ctx, const int8_t* X);
/* Ising, bit-packed: N rows of row_bytes >= ceil(M/8) bytes, bit t (LSB first) of a row
 * set = spin t is +1 -- the row layout of nrg_write_samples_file's Ising files, and
 * 1/8 of the int8 upload.  Bits past M are ignored. */
int nrg_upload_spins_packed(nrg_ctx* ctx, const uint8_t* bits, uint64_t row_bytes);

/* make_empty_state (inc/model.hpp:404-416) on the uploaded samples: W = 0, sums 0,
 * theta 0 (Ising) / row RMS (Gaussian); clears the distance cache. */
int nrg_reset_state(nrg_ctx* ctx);

/* SparseWeights: theta (may be NULL = keep) and a list of set_edge calls applied in
 * order (inc/sparse_weights.hpp:54-85; w == 0 deletes). */
int nrg_set_theta(nrg_ctx* ctx, const double* theta);
int nrg_set_edges(nrg_ctx* ctx, uint64_t n, const int32_t* ei, const int32_t* ej, const double* w);
/* sorted_edges (inc/sparse_weights.hpp:107-117) + theta; returns the edge count in
 * *n_edges and writes min(cap, count) edges. */
int nrg_get_state(nrg_ctx* ctx, double* theta, uint64_t cap, int32_t* ei, int32_t* ej, double* w,
                  uint64_t* n_edges);
/* cached neighbour sums m_i (inc/sparse_weights.hpp:90-97), N x M row-major */
int nrg_get_sums(nrg_ctx* ctx, double* out);

/* DistanceCache::begin_generation (inc/model.hpp:40-50): drops cached pair scores;
 * the frozen-state snapshot (tanh fields / residuals, base) is rebuilt lazily. */
int nrg_begin_generation(nrg_ctx* ctx);
/* log_posterior (inc/model.hpp:133-162), fp64 */
int nrg_log_posterior(nrg_ctx* ctx, double* out);

/* distance() (inc/model.hpp:377-386) for a batch of pairs, memoized per generation.
 * mode NRG_EXACT: -(base + optimize_edge(i,j).gain); NRG_GRADIENT: -|edge_gradient|;
 * NRG_TABLE / NRG_LINE: the uploaded test metric. */
int nrg_distance(nrg_ctx* ctx, int32_t mode, uint64_t n, const int32_t* i, const int32_t* j,
                 double* dist);
/* optimize_edge (inc/model.hpp:201-217) for a batch of pairs against the CURRENT
 * state: w* (1-D maximizer), gain >= 0, warning flag.  Any of the outputs may be NULL. */
int nrg_optimize_edge(nrg_ctx* ctx, uint64_t n, const int32_t* i, const int32_t* j, double* w,
                      double* gain, uint8_t* warn);
/* edge_gradient (inc/model.hpp:175-195) */
int nrg_edge_gradient(nrg_ctx* ctx, uint64_t n, const int32_t* i, const int32_t* j, double* g);
/* optimize_theta (inc/model.hpp:222-268) for every node, without writing it back */
int nrg_optimize_theta(nrg_ctx* ctx, double* out);

/* Test metrics: TableMetric d[min*n+max] (n x n doubles), LineMetric |pos_i - pos_j|. */
int nrg_set_table(nrg_ctx* ctx, uint64_t n, const double* table);
int nrg_set_line(nrg_ctx* ctx, uint64_t n, const double* pos);

/* find_knn (inc/knn.hpp:150-306) / find_knn_exhaustive (:309-314).  ids/dists receive
 * n * (*k_out) entries, row li = out-neighbours of nodes[li] sorted by (dist, id);
 * churn receives min(churn_cap, sweeps) per-sweep ratios. */
int nrg_find_knn(nrg_ctx* ctx, int32_t mode, int32_t k, const int32_t* nodes, uint64_t n,
                 const nrg_knn_params* p, int32_t exhaustive, int32_t* ids, double* dists,
                 int32_t* k_out, int32_t* sweeps, double* churn, int32_t churn_cap,
                 int32_t* n_churn);

/* find_best (inc/find_best.hpp:186-192) / find_best_exhaustive (:196-208). */
int nrg_find_best(nrg_ctx* ctx, int32_t mode, uint64_t m, const int32_t* nodes, uint64_t n,
                  const nrg_fb_params* p, int32_t exhaustive, nrg_pair* out, uint64_t cap,
                  uint64_t* n_out, nrg_trace_level* trace, int32_t trace_cap, int32_t* n_levels,
                  int32_t* short_count);

/* detail::apply_edge_updates (inc/reconstruct.hpp:70-127) with the sequential
 * (threads <= 1) semantics, executed as dependency-ordered node-disjoint batches. */
int nrg_apply_updates(nrg_ctx* ctx, const nrg_pair* cands, uint64_t n, double* delta);
/* detail::theta_pass (inc/reconstruct.hpp:129-138) */
int nrg_theta_pass(nrg_ctx* ctx);

/* One reconstruct_gcd loop body (inc/reconstruct.hpp:162-179) for iteration `iter`
 * (1-based): begin_generation, find_best(nearbyint(kappa*N)), updates, theta pass,
 * log_posterior.  cands (optional, cap entries) receives the candidate list — the
 * candidate_hook's view (:170). */
int nrg_gcd_iteration(nrg_ctx* ctx, const nrg_gcd_cfg* cfg, int32_t iter, nrg_iter_record* rec,
                      nrg_pair* cands, uint64_t cap, uint64_t* n_cands);
/* reconstruct_gcd (inc/reconstruct.hpp:148-181) */
int nrg_reconstruct_gcd(nrg_ctx* ctx, const nrg_gcd_cfg* cfg, nrg_iter_record* recs,
                        int32_t rec_cap, int32_t* n_iters, int32_t* converged);
/* reconstruct_cd (inc/reconstruct.hpp:185-207): every iteration updates all pairs
 * i < j in row-major order (sequential semantics), then the theta pass; stops when
 * delta < eps (eps <= 0: 1e-6 N).  n(n-1)/2 < 2^31.  threads is accepted and ignored. */
int nrg_reconstruct_cd(nrg_ctx* ctx, double eps, int32_t max_iters, int32_t threads, nrg_iter_record* recs,
                       int32_t rec_cap, int32_t* n_iters, int32_t* converged);

/* counters: pairs scored (cache misses, inc/model.hpp:83-84), cache hits,
 * line-search passes and warnings (inc/model.hpp:270-271). */
int nrg_counters(nrg_ctx* ctx, uint64_t* misses, uint64_t* hits, uint64_t* evals,
                 uint64_t* warnings);
int nrg_reset_counters(nrg_ctx* ctx);

/* recall_curve (inc/find_best.hpp:211-231), host-side */
int nrg_recall_curve(uint64_t m, const nrg_pair* exact, const nrg_pair* approx, double* out);

/* Device timing of the last call's kernels, by phase (ms), for the benchmark:
 * [0] pair scoring, [1] NNDescent framework, [2] FindBest select/merge,
 * [3] updates, [4] theta pass, [5] log_posterior, [6] snapshot. */
int nrg_phase_times(nrg_ctx* ctx, double* ms, int32_t cap);

/* Device timer on the context's stream: op 0 records the start event, op 1 records
 * the stop event, synchronises and writes the elapsed milliseconds to *ms. */
int nrg_timer(nrg_ctx* ctx, int32_t op, double* ms);
/* Per-kernel statistics accumulated since the last nrg_reset_counters:
 * [0] screen (K1) device ms, [1] K1 launches, [2] pairs screened, [3] refine (K2) ms,
 * [4] K2 launches, [5] survivors refined, [6] kernel launches issued (all kernels),
 * [7] parallel rounds apply_updates spent on tie tails, [8] tensor-core all-pairs screens,
 * [9] pairs they screened, [10] distance-cache flushes (a generation outgrew 2^31 slots). */
int nrg_kernel_stats(nrg_ctx* ctx, double* out, int32_t cap);
/* Uniform sample (up to cap) of the unique pairs scored in the current generation
 * (the distance cache's keys); returns the count in *n_out. */
int nrg_sample_scored_pairs(nrg_ctx* ctx, uint64_t cap, uint64_t seed, int32_t* i, int32_t* j,
                            uint64_t* n_out);

/* Synthetic data on the device: Erdos-Renyi Ising truth
 * (mean degree, w ~ N(0, w_sigma^2), theta ~ N(0, th_sigma^2)) and graph-coloured
 * Gibbs sweeps (burn_in, thin) written as the context's samples; optionally copied
 * out as int8 (X_out, N x M). */
int nrg_generate_ising(nrg_ctx* ctx, double mean_deg, double w_sigma, double th_sigma,
                       int32_t burn_in, int32_t thin, uint64_t seed, int8_t* X_out);
/* The truth behind the last nrg_generate_* call of this context: n_edges edges (i < j)
 * with couplings w (Ising) or precision off-diagonals (Gaussian), and per node the
 * field theta (Ising) or the precision diagonal (Gaussian).  Call with cap = 0 for the
 * count; copies min(cap, n_edges) edges and, if node_out is non-null, N node values. */
int nrg_generated_truth(nrg_ctx* ctx, uint64_t cap, int32_t* ei, int32_t* ej, double* w, double* node_out,
                        uint64_t* n_edges);
/* Config 5 truth: erased configuration model, degrees P(d) ~ d^-gamma for d >= dmin
 * (capped at sqrt(N)); same Gibbs sampler and outputs as nrg_generate_ising. */
int nrg_generate_ising_powerlaw(nrg_ctx* ctx, double gamma, int32_t dmin, double w_sigma, double th_sigma,
                                int32_t burn_in, int32_t thin, uint64_t seed, int8_t* X_out);
/* Gibbs samples of a caller-supplied Ising truth (distinct edges, theta[N]). */
int nrg_generate_ising_graph(nrg_ctx* ctx, uint64_t n_edges, const int32_t* ei, const int32_t* ej,
                             const double* w, const double* theta, int32_t burn_in, int32_t thin, uint64_t seed,
                             int8_t* X_out);
/* Config 3 (Gaussian context): random degree-regular precision matrix, off-diagonals
 * U(-amp, amp), diagonal = row sum |K_ij| + 0.5; samples by graph-coloured Gibbs (the
 * stationary law of a sparse-Cholesky draw); optionally copied out (X_out, N x M). */
int nrg_generate_gaussian(nrg_ctx* ctx, int32_t degree, double amp, int32_t burn_in, int32_t thin, uint64_t seed,
                          double* X_out);
/* Gaussian samples for a caller-supplied precision matrix: off-diagonal entries kij on
 * distinct edges (ei, ej), diagonal kdiag[N] > 0 (sample_gaussian, inc/synth.hpp:95-124,
 * draws the same law by sparse Cholesky). */
int nrg_generate_gaussian_graph(nrg_ctx* ctx, uint64_t n_edges, const int32_t* ei, const int32_t* ej,
                                const double* kij, const double* kdiag, int32_t burn_in, int32_t thin, uint64_t seed,
                                double* X_out);

/* Binary sample / state files (the fast replacement for the text
 * formats of inc/io.hpp:36-115).  Samples: "NRGSMP01", u32 kind (0 Ising bit-packed,
 * 1 Gaussian f64), u32 0, u64 n, u64 m, data.  State: "NRGSTA01", u64 n, u64 n_edges,
 * theta[n] f64, n_edges x {i32 i, i32 j, f64 w}.  Host-only functions need no GPU;
 * nrg_load_* / nrg_save_* move a file into / out of a context (load_state = empty state,
 * theta, then the edges as set_edge calls). */
int nrg_write_samples_file(const char* path, int32_t n, int32_t m, int32_t kind, const double* X);
int nrg_read_samples_info(const char* path, int32_t* n, int32_t* m, int32_t* kind);
int nrg_read_samples_file(const char* path, double* X);
int nrg_load_samples_file(nrg_ctx* ctx, const char* path);
int nrg_save_samples_file(nrg_ctx* ctx, const char* path);
int nrg_write_state_file(const char* path, int32_t n, const double* theta, uint64_t n_edges, const int32_t* ei,
                         const int32_t* ej, const double* w);
int nrg_read_state_info(const char* path, int32_t* n, uint64_t* n_edges);
int nrg_read_state_file(const char* path, double* theta, int32_t* ei, int32_t* ej, double* w);
int nrg_load_state_file(nrg_ctx* ctx, const char* path);
int nrg_save_state_file(nrg_ctx* ctx, const char* path);

/* Multi-GPU: samples, sums, W and theta replicated (updates and theta
 * passes run identically on every rank); NNDescent nodes sharded by contiguous ranges;
 * the per-generation distance cache sharded by pair key, so each unique pair is scored
 * once job-wide (two all-to-alls per sweep route requests and answers); kNN rows
 * all-gathered once per sweep; churn all-reduced; base broadcast from rank 0.  Every
 * rank issues the same calls with the same inputs.
 * NCCL: rank 0 calls nrg_comm_unique_id and shares the 128-byte id; every rank then
 * calls nrg_comm_init.  world == 1 or no call = single GPU. */
int nrg_comm_unique_id(uint8_t id[128]);
int nrg_comm_init(nrg_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t world);
/* In-process loopback group (one host thread per virtual rank, contexts on one or more
 * devices of this process): the same sharded path without NCCL, for verification. */
int nrg_loopback_create(int32_t world, void** group);
int nrg_loopback_destroy(void* group);
int nrg_comm_init_loopback(nrg_ctx* ctx, void* group, int32_t rank);
/* Host transport: the sharded path's collectives carried by caller-supplied callbacks
 * on HOST buffers (MPI, gloo through torch.distributed, sockets -- a multi-node job
 * without NCCL).  The library stages device data through pinned memory around each
 * call.  Every callback is collective (all ranks call it in the same order) and returns
 * 0 on success; byte counts and offsets are per rank (arrays of `world`). */
typedef struct {
    void* user;
    int (*allgatherv)(void* user, const void* send, uint64_t send_bytes, void* recv, const uint64_t* recv_bytes);
    int (*alltoallv)(void* user, const void* send, const uint64_t* send_bytes, const uint64_t* send_off, void* recv,
                     const uint64_t* recv_bytes, const uint64_t* recv_off);
    int (*allreduce_u64)(void* user, uint64_t* v, int32_t n, int32_t is_max);
    int (*bcast_f64)(void* user, double* v, int32_t n); /* from rank 0 */
} nrg_host_transport;
int nrg_comm_init_host(nrg_ctx* ctx, const nrg_host_transport* t, int32_t rank, int32_t world);
/* Self-test of the installed communicator (collective: every rank calls it): each
 * collective the sharded path uses (all-gather, ragged all-gather, all-to-all with
 * empty pairs, u64 sum/max all-reduce up to a world x world matrix, f64 broadcast) on
 * seeded patterns, verified on every rank; NRG error 100 on a mismatch.  Without a
 * communicator (single GPU) it runs them on a one-rank NCCL communicator created for
 * the call, which checks that NCCL loads and starts on this device. */
int nrg_comm_selftest(nrg_ctx* ctx);
/* The routing plan of one key exchange of the key-sharded distance cache (host-only):
 * from the world x world request-count matrix (row = requester, column = owner; counts
 * of 8-byte keys) the alltoallv byte counts and offsets of `rank` as sender (send_*) and
 * as owner (recv_*); returns the number of keys `rank` receives in *n_recv. */
int nrg_route_plan(int32_t world, int32_t rank, const uint64_t* counts, uint64_t* send_bytes, uint64_t* send_off,
                   uint64_t* recv_bytes, uint64_t* recv_off, uint64_t* n_recv);
/* The partition functions of the sharded path (host-only, no GPU needed): the node
 * range [lo, hi) of `rank` in a level of n nodes, and the owner rank of a pair key in
 * the key-sharded distance cache. */
int nrg_shard_range(uint64_t n, int32_t rank, int32_t world, uint64_t* lo, uint64_t* hi);
int32_t nrg_key_owner(uint64_t key, int32_t world);

#ifdef __cplusplus
}
#endif
#endif
