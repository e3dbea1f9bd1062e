/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's hot path.
 *
 * This library is the parity checker for the CUDA product path. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. Nothing in paper_1803_03288_b200/ links or calls it.
 *
 * Parity is pinned: tests/test_oracle_pins.py checks every function below
 * against the reference's own known-answer tests and against
 * the reference library itself, built from /root/reference by
 * oracle/Makefile into oracle/_ref/ (goldens committed under tests/golden/).
 *
 * Graph arrays follow the reference's index model (graph.cpp:54-96): op i is
 * the i-th op in byte order of its id, adjacency lists are sorted ascending,
 * resources are sorted by (device, unit Compute<Channel, name)
 * (graph.hpp:36-40). Recv "columns" are the recv ops in ascending op index.
 */
#ifndef TICTAC_ORACLE_H
#define TICTAC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_COMPUTE = 0, ORC_RECV = 1, ORC_SEND = 2, ORC_PS_AGG = 3,
       ORC_PS_READ = 4, ORC_PS_UPDATE = 5 };

#define ORC_INF INT64_MAX /* nullopt M+ (properties.hpp:27-37) */

typedef struct {
  int32_t n;                /* ops */
  const int32_t* pred_off;  /* CSR, n+1 */
  const int32_t* pred_idx;
  const int32_t* succ_off;  /* CSR, n+1 */
  const int32_t* succ_idx;
  const int8_t* kind;       /* ORC_* */
  const int32_t* res;       /* resource index per op */
  int32_t n_res;
  const int8_t* res_channel;/* 1 if the resource unit is a channel */
  const int64_t* dur;       /* oracle duration per op (time_oracle.hpp:28) */
} orc_graph;

/* rng.hpp:14-54 */
uint64_t orc_splitmix64(uint64_t x);
typedef struct { uint64_t mt[312]; int32_t idx; } orc_mt;
void orc_mt_seed(orc_mt* m, uint64_t seed);
uint64_t orc_mt_next(orc_mt* m);
uint64_t orc_bounded(orc_mt* m, uint64_t n);
double orc_unit(orc_mt* m);

/* random_schedule (schedule.cpp:73-84): perm[k] = recv column at rank k. */
void orc_random_order(int32_t n_recv, uint64_t seed, int32_t* perm);

/* find_dependencies (properties.cpp:19-66) as bitsets: row v has words
 * [v*words, (v+1)*words), bit c set when recv column c is in dep[v]. */
int32_t orc_dep_words(const orc_graph* g);
void orc_dependencies(const orc_graph* g, uint64_t* bits);

/* update_properties (properties.cpp:68-109). outstanding[c] flags recv
 * columns. Outputs: M per op, and per recv column P and M+ (ORC_INF =
 * nullopt); entries for non-outstanding columns are left untouched.
 * mode: 0 literal, 1 amended. */
void orc_properties(const orc_graph* g, const uint8_t* outstanding, int mode,
                    int64_t* M, int64_t* P, int64_t* Mplus);

/* precedes (schedule.cpp:12-19) on (column, P, M, M+) tuples. */
int orc_precedes(int32_t a_id, int64_t a_p, int64_t a_m, int64_t a_mp,
                 int32_t b_id, int64_t b_p, int64_t b_m, int64_t b_mp);

/* tic (schedule.cpp:21-42): prio per recv column, returns total_order. */
int orc_tic(const orc_graph* g, int mode, int32_t* prio);
/* tac (schedule.cpp:44-71), literal restatement: full update_properties
 * every round. prio per recv column. */
void orc_tac(const orc_graph* g, int32_t* prio);
/* tac via SURVEY Appendix A.1 (incremental O(V+E) rounds); valid when recvs
 * are roots (every graph tac() sees). Checked against orc_tac in tests. */
void orc_tac_incremental(const orc_graph* g, int32_t* prio);
/* the same with the closure kept per row of ops sharing one dependency set
 * (large graphs: config 5's top point). */
void orc_tac_rows(const orc_graph* g, int32_t* prio);

/* simulate (sim.cpp:61-256). prio per op (-1 = unprioritized). Outputs the
 * makespan, violations, and per-op start/end. Returns 0, or 2 when the run
 * stalls (DomainError in the reference). start/end may be NULL. */
int orc_simulate(const orc_graph* g, const int32_t* prio, int gated,
                 uint64_t choice_seed, double noise, int64_t* makespan,
                 int64_t* violations, int64_t* start, int64_t* end);

#ifdef __cplusplus
}
#endif
#endif
