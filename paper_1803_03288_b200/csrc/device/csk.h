/* Internal C ABI between the host library (csrc/host) and the sm_100a
 * kernels (csrc/device). Plain pointers and sizes only; host arrays in,
 * host arrays out unless a name starts with d_ (device pointer).
 *
 * Every entry returns 0 on success or a nonzero code with a message in
 * `err` (256 bytes); CUDA failures are reported, never silently skipped.
 */
#ifndef TICTAC_CSK_H
#define TICTAC_CSK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct DeviceGraph DeviceGraph;

/* Structure only (durations travel per call, they belong to the oracle). */
DeviceGraph* csk_graph_upload(int32_t n, const int32_t* pred_off, const int32_t* pred_idx,
                              const int32_t* succ_off, const int32_t* succ_idx,
                              const int8_t* kind, const int32_t* res, int32_t n_res,
                              const int8_t* res_channel, const int32_t* res_device,
                              int32_t n_dev, char* err);
void csk_graph_free(DeviceGraph* g);

/* Exact event simulator (reference sim.cpp:61-256), one warp per run.
 * prio: B*n priorities (-1 unprioritized) in host memory, or NULL with
 * orders != NULL: orders[b*R + i] = recv column holding priority i
 * (recv columns = recv ops ascending). seeds: per-run choice_seed.
 * start/end (n each) are filled for run 0 when non-NULL; dev_end (B*n_dev)
 * gets the max event end per device when non-NULL.
 * status[b]: 0 ok, 2 stalled ("simulation stalled with no runnable op"). */
/* One run inside SURVEY A.2's regime (worker graph, one compute unit and one
 * channel, gated, noiseless, recvs prioritized, compute ops not), for its
 * event list: gate_order = recv op indices sorted by (priority, id). */
int csk_event_a2(DeviceGraph* g, const int64_t* dur, const int32_t* gate_order, int32_t R,
                 uint64_t choice_seed, int64_t* makespan, int64_t* start, int64_t* end, char* err);
int csk_event_sim(DeviceGraph* g, const int64_t* dur, int32_t B, const int32_t* prio,
                  const int32_t* orders, int32_t R, const uint64_t* seeds, int gated,
                  double noise, int64_t* makespan, int64_t* violations, int32_t* status,
                  int64_t* start, int64_t* end, int64_t* dev_end, char* err);
/* Random sweep through the exact event simulator (cases outside the closed
 * form): run b uses seed seed_lo+b for both its random schedule (per-worker
 * derived seeds when `cluster`) and its choice stream. dev_end (B*n_dev,
 * max event end per device) may be NULL. recv_worker[c] = index of recv
 * column c's device in worker_devices() order (all 0 for worker graphs).
 * Every per-run output may be NULL. With `stats` non-NULL the batch's
 * statistics are reduced on the device (csk_event_stats below) and only
 * that block is read back; worker_dev[w] = device index of worker w (for
 * the iteration time and straggler figures of clusters), U/L = the bounds
 * the E histogram is binned over (no histogram when U == L). */
typedef struct {
  int64_t min_m, max_m, sum_m, count;       /* makespan */
  int64_t imin, imax, isum;                 /* iteration time (slowest worker), clusters */
  int64_t stalled;                          /* runs that stalled */
  int64_t argmin, argmax, iargmin, iargmax; /* lowest run index reaching the extreme */
  int64_t e_hist[1000], s_hist[1000];
  double sumsq, ssum;                       /* sum m^2, sum straggler fraction */
} csk_event_stats;
int csk_event_sweep(DeviceGraph* g, const int64_t* dur, uint64_t seed_lo, int32_t B,
                    int cluster, const int32_t* recv_worker, int32_t n_workers, int gated,
                    double noise, int64_t* makespan, int64_t* violations, int32_t* status,
                    int64_t* dev_end, const int32_t* worker_dev, int64_t U, int64_t L,
                    csk_event_stats* stats, char* err);

/* Brute force: all R! lexicographic permutations of the recv columns, each
 * simulated gated with the same choice seed / noise (metrics.cpp:37-72).
 * makespans has R! entries, in lexicographic order. */
int csk_brute_force(DeviceGraph* g, const int64_t* dur, int32_t R, uint64_t choice_seed,
                    double noise, int64_t* makespans, char* err);

/* Dependency closure + properties with every recv outstanding
 * (properties.cpp:19-109). dep_bits: n * words64 uint64 (bit c = recv column
 * c); M: n; P, Mplus: R (INT64_MAX = nullopt). mode 0 literal, 1 amended. */
int csk_properties(DeviceGraph* g, const int64_t* dur, int mode, uint64_t* dep_bits,
                   int64_t* M, int64_t* P, int64_t* Mplus, char* err);

/* tic (schedule.cpp:21-42): dense ranks per recv column; *total = flag. */
int csk_tic(DeviceGraph* g, int mode, int32_t* prio, int* total, char* err);

/* tac (schedule.cpp:44-71): rank per recv column. */
int csk_tac(DeviceGraph* g, const int64_t* dur, int32_t* prio, char* err);
int csk_tac_stats(DeviceGraph* g, const int64_t* dur, int64_t* out, char* err);

/* random_schedule (schedule.cpp:73-84) for several seeds at once:
 * perms[s*R + k] = recv column at rank k for seeds[s]. */
int csk_random_orders(int32_t R, int32_t S, const uint64_t* seeds, int32_t* perms, char* err);

/* ---- closed-form batched sweep -------------------- */
typedef struct SweepPlan SweepPlan;

/* Packed statistics keys are (m << key_bits) | seed offset; every makespan
 * is <= U, so key_bits = 63 - bitlen(U), capped to 44 (>= 26 while U < 2^37). */
static inline int csk_key_bits(int64_t U) {
  int len = 0;
  while (len < 63 && (U >> len) != 0) ++len;
  const int kb = 63 - len;
  return kb > 44 ? 44 : kb;
}

/* Per-worker chain plan: R recv columns with durations d (int64), first[c]
 * = index of the first chain class containing recv c (nc = none), suffix
 * class weights pwsuf[0..nc]. send_total = total send time on the worker's
 * channel (0 for worker graphs). W workers share the layout; worker w uses
 * tables at offset w. seed derivation: worker graphs use the seed itself;
 * clusters use splitmix64(seed ^ phi*(w+1)) (cluster.cpp:112-113).
 * noise_thr != 0: gated reorder noise, a position swaps when the noise
 * stream's (output >> 11) < noise_thr (= the reference's unit() < p).
 * nch > 1 channels per worker (several parameter servers): chan [W][R] =
 * channel of each recv column, send_total [W][nch]; such plans serve
 * random sweeps only (csk_sweep_run). */
SweepPlan* csk_sweep_plan(int32_t W, int32_t R, int32_t nc, const int64_t* d,
                          const int32_t* first, const int64_t* pwsuf, int32_t nch, const int32_t* chan,
                          const int64_t* send_total, int cluster, int64_t U, int64_t L, uint64_t noise_thr,
                          char* err);
/* General worker DAGs (recv-ancestor sets not nested): per
 * worker, recv durations d and single-recv class weights wr ([W][R]), record
 * weights wj ([W][nrec]), empty-set class weights w0 ([W]); the program
 * (nrec records of 4 value indexes: three generators and the output; -1 =
 * discard output, -2 = the previous record's result (first generator
 * only), -3 = padding record; groups of four; Ls live slots;
 * csrc/host/sweep.cpp) is shared by all workers. Runs through the same
 * csk_sweep_run / _orders / _lex calls. */
SweepPlan* csk_sweep_plan_dag(int32_t W, int32_t R, const int64_t* d, const int64_t* wr, int32_t nrec,
                              const int32_t* recs, const int64_t* wj, const int64_t* w0, int32_t Ls,
                              const int64_t* send_total, int cluster, int64_t U, int64_t L,
                              uint64_t noise_thr, char* err);
void csk_sweep_plan_free(SweepPlan* p);
/* Clusters whose parameter-server ops take time: extends a cluster chain
 * plan with the send phase (sweep.cu cluster_ps_kernel). Per worker S sends
 * (op-index order) over the plan's nch channels (ch_mask [nch][ceil(S/32)]),
 * recv_sb[c] = the worker's sends before recv column c in op-index order,
 * send durations [W][S], send successors (PS op indices, CSR over w*S + s),
 * Q PS ops in op-index order (durations, predecessor counts, successors CSR)
 * on nps cores (core_mask [nps][ceil(Q/32)]), and the active resources in
 * resource order (slots: core k -> -1-k, channel ch of worker w -> w*nch+ch).
 * csk_sweep_run then simulates full makespans (makespans, per-worker
 * makespans, statistics over the makespan). */
int csk_sweep_plan_add_ps(SweepPlan* p, int32_t S, const int16_t* recv_sb, const uint32_t* ch_mask,
                          const int64_t* send_d, const int32_t* send_succ_off, const int16_t* send_succ, int32_t Q,
                          const int64_t* ps_d, const uint8_t* ps_missing, const int32_t* ps_succ_off,
                          const int16_t* ps_succ, int32_t nps, const uint32_t* core_mask, int32_t nslot,
                          const int32_t* slots, char* err);
/* Host-to-device bytes the plan's construction copied (tables, images). */
int64_t csk_sweep_plan_uploaded(const SweepPlan* p);
// The kernel a random sweep on this plan launches.
const char* csk_sweep_plan_kernel(const SweepPlan* p);
/* Stats layout documented in include/commsched.h (CS_DSTATS_*). */
int csk_stats_pack(const int64_t* d_i64, const double* d_f64, int rank, int world, int64_t* d_buf,
                   void* stream, char* err);
int csk_stats_unpack(const int64_t* d_buf, int world, int64_t* d_i64, double* d_f64, void* stream,
                     char* err);
int csk_sweep_reset(SweepPlan* p, void* stream, int64_t* d_i64, double* d_f64, char* err);
int csk_sweep_run(SweepPlan* p, uint64_t seed_lo, int64_t count, uint64_t key_base,
                  void* stream, int64_t* d_makespans, int64_t* d_worker_makespans,
                  int64_t* d_i64, double* d_f64, char* err);
/* Explicit orders on device (int32, [n][R]) instead of seeds; W must be 1. */
int csk_sweep_orders(SweepPlan* p, const int32_t* d_orders, int64_t n, void* stream,
                     int64_t* d_makespans, char* err);

/* Lexicographic permutations [first, first+count) of a worker plan's recv
 * columns through the closed form (d_out device, count entries). */
int csk_sweep_lex(SweepPlan* p, int64_t first, int64_t count, int64_t* d_out, char* err);
/* Brute force over all `perms` = R! permutations on the closed form: first
 * minimum in lexicographic order (best_m, best_k) and the ascending distinct
 * makespans (copied when *n_distinct <= cap). */
int csk_brute_force_closed(SweepPlan* p, int64_t perms, int64_t* best_m, int64_t* best_k, int64_t* distinct,
                           int64_t cap, int64_t* n_distinct, char* err);

/* Launch counter (kernels launched by this library, process-wide). */
int64_t csk_launches(void);

#ifdef __cplusplus
}
#endif
#endif
