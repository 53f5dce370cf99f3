/* mecefo_ctl.h — C-ABI of the native host control-plane streams (libmecefo_ctl.so).
 *
 * The degraded step's integer path (failure injection, token sampling) draws
 * from numpy's PCG64 in the reference. This library is a bit-exact C++
 * restatement of those streams so the control plane does not depend on numpy:
 *
 *   - SeedSequence entropy pool + generate_state (numpy bit_generator.pyx,
 *     NEP 19), as used by `np.random.PCG64(seed)`:
 *       reference cluster.py:98  `Generator(PCG64(scenario.seed))`
 *       reference data.py:95-98 `PCG64(SeedSequence((seed, 0xDA7A, i)))`
 *   - PCG64 (XSL-RR 128/64) next_uint64 / buffered next_uint32,
 *   - Generator.random()  (53-bit double)       reference cluster.py:148-150
 *   - Generator.integers(0, high) (Lemire bounded, 32- or 64-bit path)
 *                                               reference cluster.py:160-162
 *
 * Host-only (no CUDA). Every function returns 0 on success or
 * MECEFO_CTL_CONTRACT (1) on a bad argument. Streams are caller-owned
 * structs: copy one to fork the stream.
 */
#ifndef MECEFO_CTL_H
#define MECEFO_CTL_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MECEFO_CTL_OK 0
#define MECEFO_CTL_CONTRACT 1
#define MECEFO_CTL_UNRECOVERABLE 2

typedef struct {
    uint64_t state_hi, state_lo; /* 128-bit LCG state */
    uint64_t inc_hi, inc_lo;     /* 128-bit odd increment */
    int32_t has_uint32;          /* numpy's buffered upper half for next_uint32 */
    uint32_t uinteger;
} mecefo_pcg64_t;

/* np.random.PCG64(np.random.SeedSequence(entropy)) where `entropy` is a tuple of
 * n non-negative integers, each given as 64-bit words (n <= 64); n == 1 is
 * np.random.PCG64(seed). */
int mecefo_pcg64_seed(mecefo_pcg64_t* s, const uint64_t* entropy, int32_t n);

/* Raw draws (bit_generator.random_raw / next_uint32). */
int mecefo_pcg64_next_u64(mecefo_pcg64_t* s, uint64_t* out, size_t count);
int mecefo_pcg64_next_u32(mecefo_pcg64_t* s, uint32_t* out, size_t count);

/* Generator.random(size=count): doubles in [0, 1). */
int mecefo_pcg64_random(mecefo_pcg64_t* s, double* out, size_t count);

/* Generator.integers(low, high, size=count) with int64 output, high > low. */
int mecefo_pcg64_integers(mecefo_pcg64_t* s, int64_t low, int64_t high, int64_t* out, size_t count);

/* Ring-successor takeover on one ring of n members (reference cluster.py:207-218,
 * the NDB reassignment of reassign_takeover on one DP rank's stages): failed
 * members in descending order each adopt the first following member that is
 * neither failed nor already adopting. failed[j] != 0 marks member j;
 * executor[j] receives the member that runs j's work (j itself if healthy).
 * Returns MECEFO_CTL_UNRECOVERABLE when some failed member has no adopter. */
int mecefo_ring_route(int32_t n, const uint8_t* failed, int32_t* executor);

/* ---- The cluster state machine (reference cluster.py:37-271) --------------
 * ClusterState + FailureScenario: node health (0 healthy, 1 failed, 2 doubled),
 * executor map, recovery deadlines, the failure stream (PCG64(seed)),
 * step_cluster = due recoveries (sorted) -> injection -> NDB reassignment ->
 * invariants. Codes: MECEFO_CTL_CONTRACT (ContractViolation),
 * MECEFO_CTL_UNRECOVERABLE (UnrecoverableRankError), 3 (ConsistencyError). */
#define MECEFO_CTL_CONSISTENCY 3

typedef struct mecefo_cluster mecefo_cluster;

typedef struct {
    int32_t dp, pp, layers;              /* ClusterConfig (cluster.py:37-66) */
    const int32_t* stage_boundaries;     /* pp + 1 entries, or NULL: round(s * layers / pp) */
    int32_t kind;                        /* FailureScenario (cluster.py:69-89): 0 none, 1 per_iteration, 2 scheduled */
    double probability;
    int32_t recovery_iterations;
    double failure_interval_s, recovery_time_s;
    const int32_t* victims;              /* n_victims (rank, stage) pairs, or NULL = every node */
    int32_t n_victims;
    uint64_t seed;
} mecefo_cluster_config;

/* One event of cluster.py:126-133: kind 0 fail, 1 recover (details.fetched_from =
 * (from_rank, from_stage)), 2 adopt (details.stage, details.fetched_from_rank =
 * from_rank; node = the adopting node). */
typedef struct {
    double time;
    int32_t iteration, kind;
    int32_t node_rank, node_stage;
    int32_t stage;
    int32_t from_rank, from_stage;
} mecefo_cluster_event;

int mecefo_cluster_create(mecefo_cluster** out, const mecefo_cluster_config* cfg);
int mecefo_cluster_destroy(mecefo_cluster* c);
/* The state arrays (dp x pp, row-major), owned by the cluster; callers may
 * read and write them between calls (the Python wrapper views them). */
int mecefo_cluster_arrays(mecefo_cluster* c, int8_t** status, int32_t** executor);
int mecefo_cluster_rng(mecefo_cluster* c, mecefo_pcg64_t** rng);
/* next_failure_time: set if `set`, read into `get` if given. */
int mecefo_cluster_next_failure_time(mecefo_cluster* c, const double* set, double* get);
/* down_until: the (rank, stage) -> deadline map, ascending node order; *n = its size. */
int mecefo_cluster_down_until(mecefo_cluster* c, int32_t* nodes, double* until, int32_t cap, int32_t* n);
int mecefo_cluster_set_down_until(mecefo_cluster* c, int32_t rank, int32_t stage, const double* until);
/* cluster.py:136-168, 171-173, 176-187, 190-239, 253-271, 242-250. Events are
 * written to `events` (capacity cap), their count to *n. */
int mecefo_cluster_inject(mecefo_cluster* c, double sim_time, int32_t iteration, mecefo_cluster_event* events,
                          int32_t cap, int32_t* n);
int mecefo_cluster_due_recoveries(mecefo_cluster* c, double sim_time, int32_t iteration, int32_t* nodes,
                                  int32_t cap, int32_t* n);
int mecefo_cluster_recover(mecefo_cluster* c, int32_t rank, int32_t stage, double sim_time, int32_t iteration,
                           mecefo_cluster_event* events, int32_t cap, int32_t* n);
int mecefo_cluster_reassign(mecefo_cluster* c, double sim_time, int32_t iteration, mecefo_cluster_event* events,
                            int32_t cap, int32_t* n);
int mecefo_cluster_validate(const mecefo_cluster* c);
int mecefo_cluster_step(mecefo_cluster* c, double sim_time, int32_t iteration, mecefo_cluster_event* events,
                        int32_t cap, int32_t* n);

/* costmodel.py:206-238 iteration_cost on the current state: FLOPs of the
 * slowest node (worst), its first executing stage, and the total; a healthy
 * node runs costmodel block_cost MODE_STANDARD per layer, a doubled one
 * MODE_NEIGHBOR_APPROX (policy_approx) or the naive standard cost. */
int mecefo_iteration_cost(const mecefo_cluster* c, int64_t hidden, int64_t ffn, int32_t policy_approx, int64_t r,
                          int64_t tau, int64_t tokens, int64_t* worst, int32_t* worst_stage, int64_t* total);

#ifdef __cplusplus
}
#endif

#endif /* MECEFO_CTL_H */
