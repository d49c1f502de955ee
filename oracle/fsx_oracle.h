/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the reference's embedding hot path (FreeScale
 * simulator, /root/reference/proj), used ONLY as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg. Each function cites
 * the reference file:line it restates. Pinned against the reference itself
 * (oracle/_ref, tests/test_oracle_pins.py) and against the golden fixtures in
 * tests/golden/ generated from it (tests/golden/make_golden.py).
 *
 * All arithmetic is f64 / u64 exactly as in the reference; build with
 * -ffp-contract=off (oracle/Makefile).
 */
#ifndef FSX_ORACLE_H
#define FSX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror include/fsx.h */
#define FSO_OK 0
#define FSO_INVALID_ARGUMENT -1
#define FSO_DOMAIN -2
#define FSO_PROTOCOL -4

const char* fso_last_error(void);

double fso_initial_value(uint64_t seed, uint64_t row, uint32_t d);
uint64_t fso_local_rows(uint64_t total_rows, int num_shards, int shard);
/* in-place sort + unique; returns the unique count */
uint64_t fso_sorted_unique(uint64_t* v, uint64_t n);

int fso_compute_collision(const uint64_t* cur, uint64_t ncur, const uint64_t* next, uint64_t nnext,
                          uint64_t* co, uint64_t* nco, uint64_t* exc, uint64_t* nexc,
                          uint64_t* exn, uint64_t* nexn);

int fso_init_shard(uint64_t total_rows, uint32_t dim, int num_shards, int shard, uint64_t seed,
                   double* values);
int fso_lookup(const double* values, uint64_t total_rows, uint32_t dim, int num_shards, int shard,
               const uint64_t* ids, uint64_t n, double* out);
int fso_apply_gradients(double* values, uint64_t total_rows, uint32_t dim, int num_shards,
                        int shard, double lr, const uint64_t* ids, uint64_t n,
                        const double* grads, uint64_t* uniq, uint64_t* nuniq, double* rows);

int fso_route(int world, uint64_t total_rows, const uint64_t* ids, const uint64_t* lens,
              int* occ_shard, uint64_t* recv_ids, uint64_t* recv_lens, uint64_t* uniq,
              uint64_t* nuniq);

int fso_run_engine(int world, int iters, const uint64_t* ids, const uint64_t* lens,
                   uint64_t total_rows, uint32_t dim, double lr, uint64_t seed, double grad_scale,
                   double grad_shift, double* table_out, uint64_t* stats_out);

int fso_run_engine_ex(int world, int iters, const uint64_t* ids, const uint64_t* lens,
                      uint64_t total_rows, uint32_t dim, double lr, uint64_t seed, double grad_scale,
                      double grad_shift, double* table_out, uint64_t* stats_out, int store_f32);

/* + the engine's fixed chunk association (reduce_chunk) and its PRESUM
 * two-level association of collision rows (presum); see fsx_oracle.c */
int fso_run_engine_ex2(int world, int iters, const uint64_t* ids, const uint64_t* lens,
                       uint64_t total_rows, uint32_t dim, double lr, uint64_t seed, double grad_scale,
                       double grad_shift, double* table_out, uint64_t* stats_out, int store_f32,
                       uint32_t reduce_chunk, int presum);

/* pooled (bag) lookup and its backward scatter + update (see fsx_oracle.c) */
int fso_pooled_forward(const double* table, uint64_t total_rows, uint32_t dim, const uint64_t* ids,
                       const uint64_t* offs, uint64_t n_bags, int store_f32, uint32_t reduce_chunk, double* out);
int fso_pooled_backward(double* table, uint64_t total_rows, uint32_t dim, double lr, const uint64_t* ids,
                        const uint64_t* offs, uint64_t n_bags, const double* bag_grads, int store_f32,
                        uint32_t reduce_chunk);

int fso_fbs(const uint64_t* lens, const int* origin, const int* local, uint64_t m, int n,
            int* assignment, uint64_t* order, uint64_t* order_lens);
int fso_vbs(const uint64_t* lens, const int* origin, const int* local, uint64_t m, int n,
            double alpha, const int* tuned_sizes, int* sizes_out, int* assignment,
            uint64_t* order, uint64_t* order_lens);
int fso_autotune(int n, int* sizes, double* ema_local, double* ema_global, int step, double delta,
                 double decay, const double* times, int rounds);
double fso_cost(double c0, double c1, double c2, const uint64_t* lens, uint64_t n);
double fso_bruteforce(const double* w, uint64_t m, int segments);

#ifdef __cplusplus
}
#endif
#endif
