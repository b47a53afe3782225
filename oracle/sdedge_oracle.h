/*
 * sdedge_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, literal CPU oracle for the joint bandwidth / batching /
 * speculation-length solver of arXiv 2510.11331 ("Efficient LLM Inference
 * over Heterogeneous Edge Networks with Speculative Decoding").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA path (paper_2510_11331_b200/).
 *
 * Citations: P:n = PAPER.md line n.  All arithmetic is IEEE fp64, built with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 *
 * Parity status of each function: see DESIGN.md section "Oracle pins".
 * Every function is pinned (no "parity unpinned" entries).
 */
#ifndef SDEDGE_ORACLE_H
#define SDEDGE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t Jd, h1d, h2d;        /* draft model (Table I)             */
    int32_t Jv, h1v, h2v;        /* verify model                                 */
    double  c1d, c2d, c1v, c2v;  /* eq:latency_b2 coefficients (Table II)        */
    double  Bw;                  /* uplink bandwidth B_w, Hz                     */
    double  sigma2;              /* noise power, W                               */
    double  lambda;              /* bits per token; <= 0 -> 16(h1d+h1v)  */
    int64_t gamma_s;             /* SBS memory capacity Gamma_s, bytes           */
    int32_t K, O_max, gamma_min, gamma_max;
    double  downlink_s;          /* optional per-step, per-batch verify add-on   */
    int32_t bw_policy;           /* 0 optimal eq:opt_w, 1 uniform w_k = 1/K */
    int32_t batch_policy;        /* 0 Algorithm 1 (pipelined), 1 SD w/o pipeline,
                                    2 no batching, 3 static,
                                    4 max batching, 5 heuristic,
                                    6 per-batch gamma (an extension) */
    int32_t static_batch;        /* batch size of policy 3                          */
    int32_t heuristic_start;     /* policy 5: 0 sizes 2, 3, ... (reading B5); 1 from two batches,
                                    ceil(K/2), upward (reading B5')      */
} orc_params;

typedef struct {
    int32_t status;              /* 0 ok, 1 memory-infeasible, 2 bad alpha, 3 bad task */
    int32_t gamma;               /* gamma*, -1 if status != 0                    */
    int32_t M;                   /* number of batches                            */
    double  T, T_com, T_inf;
    double  min_row_gap;         /* min over gamma and rows of (2nd-best - best)/best */
    int32_t gap_gamma, gap_row;  /* where min_row_gap occurred                   */
    double  gamma_gap;           /* (2nd-best gamma T_inf - best)/best            */
    int64_t W;                   /* candidate-steps evaluated                    */
} orc_result;

/* ---- paper primitives (each pinned in tests/test_oracle_pins.py) ---- */
double  orc_expected_tokens(double alpha, int gamma);                 /* eq:ol      */
int32_t orc_decode_steps(int32_t O, double L);                        /* eq:step_n  */
int64_t orc_param_memory(int32_t J, int32_t h1, int32_t h2);          /* eq:memory_model */
int64_t orc_kv_memory_per_task(int32_t J, int32_t h1, int32_t I, int32_t O); /* eq:memory_kv */
double  orc_flops_draft(int32_t J, int32_t h1, int32_t h2, double Im, double L, int i, int n);  /* eq:flops_d */
double  orc_flops_verify(int32_t J, int32_t h1, int32_t h2, double Im, int gamma, double L, int n); /* eq:flops_v */
double  orc_runtime(double c1, double c2, double F, double b);        /* eq:latency_b2 */
double  orc_draft_time(const orc_params* P, const double* co, int b, int32_t Im, int gamma, double L, int n); /* eq:d_latency */
double  orc_verify_time(const orc_params* P, const double* co, int b, int32_t Im, int gamma, double L, int n); /* eq:v_latency */

/* eq:opt_w / t*_com. Writes w[K]; returns t*_com. */
double  orc_bandwidth(const orc_params* P, const int32_t* I, const double* p, const double* g, double* w);

/* eq:time / eq:latency_inf: literal pipeline recursion of one plan.
 * batches are given as sorted-position ends (1-based, ascending, last == K).
 * Returns T_inf (planned, uniform O_max), +inf if a batch is memory-infeasible. */
double  orc_eval_plan(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                      int gamma, int M, const int32_t* batch_end);

/* Algorithm 1 for one gamma over sorted lengths Is[0..K-1].
 * S[K] receives 1-based boundaries; returns Upsilon[K,0,0] (+inf if infeasible).
 * row_gap[K] (optional) receives per-row relative gaps (+inf if < 2 candidates).
 * force_row/force_j (optional, force_row < 1 disables) makes row force_row take
 * j = force_j (all candidates are still evaluated) -- see orc_dp_trace. */
double  orc_dp(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
               int32_t* S, double* row_gap, int64_t* W, int force_row, int force_j);

/* Near-tie branching replay (SURVEY 8(c) "T"): Algorithm 1 where row i takes
 * j = force[i-1] when that is > 0 (force may be NULL: all rows free).  Every
 * candidate of every row is evaluated as in orc_dp; row_best[K] receives each
 * row's minimum candidate value, row_taken[K] the value of the candidate taken
 * (the new Upsilon[i,0,0]).  Returns Upsilon[K,0,0] of the forced chain, +inf if
 * some row has no feasible candidate, NaN if a forced j is infeasible. */
double  orc_dp_trace(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
                     const int32_t* force, int32_t* S, double* row_gap, double* row_best,
                     double* row_taken, int64_t* W);

/* "SD w/o pipeline" evaluation of a plan: every decoding step runs draft then
 * verify of each batch sequentially, T_n = sum_m (T^d_{n,m} + T^v_{n,m}). */
double  orc_eval_plan_nopipe(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                             int gamma, int M, const int32_t* batch_end);

/* Algorithm 1 with the SD-w/o-pipeline cost (additive, exact). Same outputs as orc_dp. */
double  orc_dp_nopipe(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
                      int32_t* S, double* row_gap, int64_t* W);

/* Fixed-plan batching policies 2..5 for one gamma: writes the plan (ends), returns M
 * (0 if no memory-feasible plan exists). */
int     orc_fixed_plan(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
                       int32_t* ends);

/* Actual-output evaluation of a plan (eq:step_n, eq:latency_infer_batch
 * P:519-525, eq:latency_inf): batch m needs n_m = ceil(O_m / L) steps with O_m the
 * largest actual output length O_k of its tasks; at step n only the batches with
 * n_m >= n run, in plan order, through the eq:time recursion.
 * Is: sorted input lengths; Os: the actual output lengths in the same sorted order. */
double  orc_eval_actual(const orc_params* P, const double* co, const int32_t* Is, const int32_t* Os,
                        double alpha, int gamma, int M, const int32_t* batch_end);

/* Per-batch speculation length (an EXTENSION: the paper fixes one l,
 * P:555).  Batch m has its own gamma_m, L_m and n_m = ceil(O_max/L_m);
 * step n runs the eq:time recursion over the active batches n_m >= n (eq:latency_infer_batch,
 * P:519-525).  Returns T_inf, +inf if a batch does not fit the memory. */
double  orc_eval_plan_pbg(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                          int M, const int32_t* batch_end, const int32_t* gammas);

/* Algorithm 1 over candidates (j, gamma) (reading NB1: ties -> largest j, then smallest
 * gamma); a finished batch adds no stage time.  S[i-1] = j*, Gm[i-1] = gamma* at row i. */
double  orc_dp_pbg(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                   int32_t* S, int32_t* Gm, double* row_gap, int64_t* W);

/* Full solve of problem P for one scenario.
 * order[K], batch_end[K], w[K], tinf_gamma[gamma_max-gamma_min+1] are caller-owned;
 * batch_gamma[K] (optional) receives each batch's gamma (gamma* for every batch unless
 * batch_policy == 6; then R->gamma is the last batch's). */
void    orc_solve(const orc_params* P, const int32_t* I, const double* p, const double* g,
                  double alpha, const double* coeffs4, orc_result* R, int32_t* order,
                  int32_t* batch_end, double* w, double* tinf_gamma, int32_t* batch_gamma);

/* Exhaustive search over every contiguous partition of the sorted order and
 * every gamma (K <= 20).  Returns best T_inf; writes its plan. */
double  orc_brute_force(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                        int gamma_min, int gamma_max, int32_t* best_gamma, int32_t* best_M,
                        int32_t* best_end);

/* Batch driver: n scenarios (SoA, row-major [n][K]) on nthreads pthreads. */
void    orc_solve_batch(const orc_params* P, int64_t n, const int32_t* I, const double* p,
                        const double* g, const double* alpha, const double* coeffs,
                        int32_t* status, int32_t* gamma, int32_t* M, double* lat /*[n*3]*/,
                        int32_t* order, int32_t* batch_end, double* w, double* min_row_gap,
                        double* gamma_gap, int64_t* W, int32_t* batch_gamma, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
