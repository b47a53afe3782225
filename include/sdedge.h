/*
 * sdedge.h -- C ABI of the B200-native batched solver for the joint
 * bandwidth / batching / speculation-length problem of arXiv 2510.11331,
 * "Efficient LLM Inference over Heterogeneous Edge Networks with Speculative
 * Decoding".  Citations: P:n = PAPER.md line n.
 *
 * What one call computes, for each of n independent scenarios (problem P,
 * P:543-566):
 *   1. the closed-form optimal uplink bandwidth split w*_k and t*_com
 *      (eq:bandw1 / eq:opt_w);
 *   2. for every speculation length gamma in [gamma_min, gamma_max]
 *      (P3): L = (1-alpha^{gamma+1})/(1-alpha) (eq:ol),
 *      N = ceil(O_max / L) (eq:step_n, uniform O_max planning
 *      P:638-641), and Algorithm 1 over the tasks sorted by input
 *      length, with the candidate cost eq:t_ij1 / state update eq:tt1-tt2
 *      evaluated under the latency model eq:flops_d, eq:flops_v,
 *      eq:latency_b2, eq:d_latency, eq:v_latency, eq:time and the
 *      memory constraint eq:memory_model + eq:memory_kv;
 *   3. gamma* = the smallest gamma minimising T_inf, its batches recovered by
 *      backtracking S, and T = T_com + T_inf.
 * DESIGN.md "Readings" lists how the garbled / ambiguous passages are read
 * (bracket of eq:t_ij1, Upsilon init, S[i] at j*=1, backtrack step, ties).
 *
 * Conventions
 *   - Every array pointer in sdedge_scenarios / sdedge_schedule / out_latency
 *     is a DEVICE pointer (cudaMalloc / torch CUDA tensor) on the current
 *     device, row-major [scenario][task].  The caller owns all of them.
 *     sdedge_solve_batch_host() is the same call on HOST pointers (pinned
 *     memory recommended); it stages the copies itself.
 *   - The call is asynchronous on params->stream (NULL = legacy default
 *     stream); results are valid once that stream completes.  Workspace is
 *     stream-ordered (cudaMallocFromPoolAsync) and freed on the same stream;
 *     it comes from a library-private memory pool per device (created on
 *     first use, kept cached between calls) -- the device's default pool and
 *     the caller's allocators are not touched.
 *   - Per-scenario problems never fail the call: they set status[s] and
 *     write gamma = -1, num_batches = 0, batch_end = 0 and
 *       status 1 (memory-infeasible: some task fits in no batch, cons. (b)
 *                 P:551):  out_latency = {+inf, T_com, +inf};
 *       status 2 (alpha not in (0,1)):              {NaN, T_com, NaN};
 *       status 3 (some I_k < 1, p_k or g_k not > 0 / not finite):
 *                 {NaN, NaN, NaN}, bw_share = NaN.
 *     order[] is always the stable sort; bw_share is valid for status 0-2.
 *   - Return: 0 = enqueued; -1 = invalid argument (see sdedge_last_error());
 *     -2 = CUDA error; -3 = out of device memory.
 *   - Thread-safe and re-entrant across streams and devices (global state:
 *     the thread-local error string and the mutex-guarded per-device pool).
 */
#ifndef SDEDGE_H
#define SDEDGE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDEDGE_ABI_VERSION 3
#define SDEDGE_MAX_K 1024

typedef struct {
    int32_t layers;  /* J   (Table I)  >= 1 */
    int32_t hidden;  /* h1  >= 1                        */
    int32_t ffn;     /* h2  >= 1                        */
} sdedge_model;

typedef enum {
    SDEDGE_ALGO_ENVELOPE = 0, /* closed-form sum over the piecewise-linear Upsilon envelope
                                 (exact reformulation of eq:t_ij1, O(K^2 * segments))   */
    SDEDGE_ALGO_DENSE = 1     /* eq:t_ij1 summed step by step over n = 1..N (O(K^2 N))   */
} sdedge_algo;

#define SDEDGE_FLAG_TINY_POOL 1
/* SDEDGE_BATCH_HEURISTIC reading: equal batches of size b with b growing while the latency
 * improves; by default from b = 2 (reading B5), with this flag from two batches,
 * b = ceil(K/2) (reading B5') -- "begins with two batches, progressively
 * increases the batch size". */
#define SDEDGE_FLAG_HEURISTIC_HALF 2

/* Bandwidth policies (P:580-616 and the uniform baseline of P:936-940). */
typedef enum {
    SDEDGE_BW_OPTIMAL = 0,       /* closed-form w*_k of eq:opt_w (the proposed policy)           */
    SDEDGE_BW_UNIFORM = 1        /* w_k = 1/K, T_com = max_k T_k,com (eq:ul_latency)              */
} sdedge_bw_policy;

/* Batching policies: the proposed Algorithm 1 and the paper's baselines
 * (Sec. IV); gamma is always enumerated over
 * [gamma_min, gamma_max] (fixed speculation length "FSL" = gamma_min = gamma_max = 7). */
typedef enum {
    SDEDGE_BATCH_PROPOSED = 0,   /* Algorithm 1 with the pipelined cost              */
    SDEDGE_BATCH_NO_PIPELINE = 1,/* "SD w/o pipeline": Algorithm 1 with T_n = sum_m (T^d + T^v)  */
    SDEDGE_BATCH_NONE = 2,       /* "No batching": one task per batch, pipelined        */
    SDEDGE_BATCH_STATIC = 3,     /* fixed batch size `static_batch` in sorted order  */
    SDEDGE_BATCH_MAX = 4,        /* largest memory-feasible size for the longest input */
    SDEDGE_BATCH_HEURISTIC = 5,  /* sizes 2,3,... until the latency stops improving */
    SDEDGE_BATCH_PER_BATCH_GAMMA = 6 /* EXTENSION (not the paper's method, which fixes
                                    one l): Algorithm 1 over candidates (j, gamma) --
                                    every batch has its own gamma, L and N_gamma = ceil(O_max / L), and
                                    step n runs only the batches with N_gamma >= n (the active set of
                                    eq:latency_infer_batch).  Ties: largest j, then smallest
                                    gamma.  fp64 only, <= 32 gammas, (K+1) O_max <= 2^27.  gamma[s] is
                                    the last batch's; batch_gamma (below) has every batch's.         */
} sdedge_batch_policy;

typedef struct {
    sdedge_model draft, verify;  /* SBS draft / MBS verify models                    */
    double  c1_draft, c2_draft;  /* eq:latency_b2 coefficients of the SBS GPU, c1 > 0, c2 >= 0 */
    double  c1_verify, c2_verify;/* ... of the MBS GPU (Table II: 4.11e-13, 0.56e-3, 2.08e-14, 1.28e-2) */
    double  bandwidth_hz;        /* B_w > 0 (Table II: 20 MHz)                               */
    double  noise_w;             /* sigma^2 > 0, linear watts (-106 dBm = 2.5118864315095823e-14) */
    double  lambda_bits;         /* lambda, bits per input token; <= 0 -> 16 (h1d + h1v) */
    int64_t mem_capacity_bytes;  /* Gamma_s of the SBS (Table II "16 GB" = 16e9)             */
    int32_t K;                   /* tasks per scenario, 1..SDEDGE_MAX_K, same for all n      */
    int32_t O_max;               /* planning output length, 1..2^20 (Table II: 2048)         */
    int32_t gamma_min, gamma_max;/* 0 <= gamma_min <= gamma_max <= 64 (P:555 uses >= 1;
                                    gamma = 0 is the autoregressive reduction)               */
    int32_t precision;           /* 0 = fp64 DP arithmetic, 1 = fp32 variant                 */
    int32_t algo;                /* sdedge_algo                                              */
    int32_t flags;               /* bit set: SDEDGE_FLAG_TINY_POOL (test hook: an 8-segment first-pass
                                    envelope pool, forcing the worst-case second pass),
                                    SDEDGE_FLAG_HEURISTIC_HALF (heuristic batching reading)  */
    double  downlink_s;          /* >= 0, added to every verify stage (P:424-427 says 0)     */
    void*   stream;              /* cudaStream_t                                              */
    int32_t bandwidth_policy;    /* sdedge_bw_policy (0 = the paper's policy)                 */
    int32_t batching_policy;     /* sdedge_batch_policy (0 = the paper's policy)              */
    int32_t static_batch;        /* batch size of SDEDGE_BATCH_STATIC, >= 1                   */
    int32_t reserved;            /* must be 0                                                 */
} sdedge_params;

typedef struct {
    const int32_t* input_len;    /* [n*K] I_k (tokens)                                      */
    const double*  tx_power_w;   /* [n*K] p_k (W)                                           */
    const double*  gain;         /* [n*K] g_k (linear)                                      */
    const double*  alpha;        /* [n]   token acceptance rate                             */
    const double*  coeffs;       /* [n*4] per-scenario (c1d, c2d, c1v, c2v) or NULL -> params */
} sdedge_scenarios;

typedef struct {
    int32_t* gamma;              /* [n]   gamma* or -1                                       */
    int32_t* num_batches;        /* [n]   M                                                 */
    int32_t* batch_end;          /* [n*K] 1-based sorted position ending batch m (m < M), rest 0 */
    int32_t* order;              /* [n*K] original task index at each sorted position        */
    double*  bw_share;           /* [n*K] w*_k in ORIGINAL task order, or NULL               */
    int32_t* status;             /* [n]                                                      */
    uint64_t* work_counters;     /* optional DEVICE [5], accumulated (caller zeroes): candidates
                                    (i,j) considered, fully-evaluated candidates x predecessor-envelope
                                    segments, candidate-steps sum N (the paper's O(K^2 N) work W),
                                    DP rows, candidates fully evaluated (the rest were pruned by the
                                    exact lower bound); NULL = not counted.  Ignored by _host.      */
    int32_t* row_choice;         /* optional DEVICE [n*K] step trace (SPEC.md:422 debug export): Algorithm 1's
                                    boundary vector S at gamma*, S[i-1] = the 1-based start j* chosen at
                                    sorted row i for EVERY row (reading A4), not only the rows
                                    the backtrack visits -- so the whole DP state of the answer can be
                                    replayed (tests: near-tie branching replay, SURVEY 8(c) "T").  0 in
                                    every entry where status != 0.  NULL = not written.  Ignored by _host. */
    int32_t* batch_gamma;        /* optional DEVICE [n*K]: the speculation length of batch m (m < M), 0
                                    for m >= M -- gamma* for every batch except under
                                    SDEDGE_BATCH_PER_BATCH_GAMMA.  NULL = not written.  Ignored by _host. */
} sdedge_schedule;

/* Solve n scenarios.  out_latency: [n*3] = {T, T_com, T_inf} (seconds). */
int sdedge_solve_batch(const sdedge_scenarios* scenarios, int64_t n, const sdedge_params* params,
                       double* out_latency, sdedge_schedule* out_schedule);

/* Same, HOST pointers for every array; copies in, solves and copies out on
 * params->stream.  The caller synchronises the stream before reading. */
int sdedge_solve_batch_host(const sdedge_scenarios* scenarios, int64_t n, const sdedge_params* params,
                            double* out_latency, sdedge_schedule* out_schedule);

/* The same solve on HOST buffers with the schedule re-encoded compactly for the device->host
 * copy: the copies in both directions share the PCIe link, so fewer output bytes
 * leave more of it to the inputs.  Same values as sdedge_solve_batch_host, different layout:
 *   batch_end_mask [n * ceil(K/32)] uint32: bit (e-1) of scenario s's words is set iff a batch ends
 *                  at sorted position e (the set bits are exactly batch_end[s, 0..M-1]);
 *   order          [n * K] uint16 (K <= SDEDGE_MAX_K < 2^16): original task index per sorted position;
 *   gamma, num_batches, status [n] int32 and bw_share [n * K] fp64 (or NULL) as in sdedge_schedule.
 * Host pointers (pinned memory recommended), asynchronous on params->stream like the host entry;
 * return codes and per-scenario status as sdedge_solve_batch.  The outputs are the solve's own (Algorithm 1's
 * backtracked batches; gamma*; w*, eq:opt_w P:596-612), re-encoded only.
 * The caller owns every buffer; on failure the caller's stream still covers every copy already queued. */
typedef struct {
    int32_t*  gamma;             /* [n]                                   */
    int32_t*  num_batches;       /* [n]                                   */
    uint32_t* batch_end_mask;    /* [n * ceil(K/32)]                      */
    uint16_t* order;             /* [n * K]                               */
    double*   bw_share;          /* [n * K] or NULL                       */
    int32_t*  status;            /* [n]                                   */
} sdedge_compact_schedule;

int sdedge_solve_batch_host_compact(const sdedge_scenarios* scenarios, int64_t n, const sdedge_params* params,
                                    double* out_latency, sdedge_compact_schedule* out_schedule);

/* Actual-output evaluation of solved schedules (P:316-318,
 * eq:step_n, eq:latency_infer_batch P:519-525, eq:latency_inf).  The planner
 * assumes O_k = O_max; this call replays each scenario's plan
 * (gamma, batch_end, order from sdedge_solve_batch) with the tasks' actual
 * output lengths: batch m runs n_m = ceil(O_m / L) steps, O_m = max of its
 * tasks' O_k, and at step n only batches with n_m >= n go through eq:time
 * (or, under SDEDGE_BATCH_NO_PIPELINE, run draft then verify sequentially).
 * output_len: DEVICE [n*K] int32 >= 1 (original task order); plan: DEVICE
 * arrays gamma, num_batches, batch_end, order, status (others ignored);
 * out_t_inf: DEVICE [n] actual T_inf in seconds (NaN where status != 0,
 * some O_k < 1, or the plan is malformed: batch_end not strictly increasing in
 * 1..K with batch M-1 ending at K, an order entry outside 0..K-1, M outside
 * 1..K, gamma outside 0..64).  Uses the same params (models, coefficients, K, O_max,
 * stream) as the solve.  Asynchronous; returns 0 / -1 / -2 like the solve. */
int sdedge_evaluate_actual(const sdedge_scenarios* scenarios, const int32_t* output_len, int64_t n,
                           const sdedge_params* params, const sdedge_schedule* plan, double* out_t_inf);

/* Exhaustive search (quantifies Algorithm 1's heuristic
 * gap).  For each scenario: the exact minimum of the planned T_inf
 * (eq:time, eq:latency_inf P:505-530, uniform O_max as P:638-641) over EVERY
 * contiguous partition of the stably sorted order (the search space of
 * Algorithm 1), every gamma in [gamma_min, gamma_max] and subject to the memory
 * constraint (b) per batch.  2^(K-1) plans per gamma, so K must
 * be <= 20 (-1 otherwise).  batching_policy selects the cost: SDEDGE_BATCH_PROPOSED
 * (pipelined) or SDEDGE_BATCH_NO_PIPELINE; any other policy returns -1.  Ties keep
 * the first plan in (gamma ascending, partition mask ascending) order.
 * DEVICE pointers; async on params->stream.  out_t_inf: [n] (+inf if no plan is
 * memory-feasible, NaN for status 2/3).  out: gamma, num_batches, batch_end, order,
 * status as for sdedge_solve_batch (bw_share ignored; p_k, g_k are not read);
 * work_counters, if set, accumulates [0] plans evaluated, [1] batch-steps
 * (sum over plans of N_gamma x M).  Two launches: one CTA per (scenario, gamma)
 * item, then one warp per scenario for the min over gamma; the [n * ngamma]
 * workspace is stream-ordered.  Returns 0 / -1 / -2 / -3. */
int sdedge_brute_force(const sdedge_scenarios* scenarios, int64_t n, const sdedge_params* params,
                       double* out_t_inf, sdedge_schedule* out);

/* Multi-GPU gather: one process per GPU solves a contiguous shard of
 * the scenarios; the only exchange is the final gather of the outputs to cuda:0.
 * It is fused into the solve: rank 0 exports its output allocation once, every
 * other rank maps it and passes pointers into it (at its shard's rows) as the
 * out_latency / out_schedule arrays of sdedge_solve_batch, so the solve kernel's
 * epilogue stores each scenario's results over NVLink as it finishes -- no copy
 * after the solve.
 *   sdedge_ipc_export: dev_ptr = any address inside a cudaMalloc'd (e.g. torch)
 *     allocation on the current device; writes the allocation's 64-byte CUDA IPC
 *     handle to handle[0..63] and dev_ptr's byte offset in it to *offset.
 *   sdedge_ipc_open: maps that allocation into this process (peer access enabled
 *     lazily) and returns base + offset in *dev_ptr.  Unmap with sdedge_ipc_close
 *     (same offset).  The exporter must keep the allocation alive meanwhile.
 * Synchronous host calls; return 0, -1 (bad argument) or -2 (CUDA error). */
#define SDEDGE_IPC_HANDLE_BYTES 64
int sdedge_ipc_export(const void* dev_ptr, void* handle, uint64_t* offset);
int sdedge_ipc_open(const void* handle, uint64_t offset, void** dev_ptr);
int sdedge_ipc_close(void* dev_ptr, uint64_t offset);
/* Asynchronous device-to-device copy on `stream` (a cudaStream_t), e.g. a finished chunk of a rank's
 * outputs into cuda:0's peer-mapped arrays by the copy engines while the next chunk is solved. */
int sdedge_copy_async(void* dst, const void* src, uint64_t bytes, void* stream);

/* Per-kernel timing for measurement (bench.py's roofline): sdedge_kernel_timing(1) clears the
 * record and starts bracketing every launch the solve calls on this thread enqueue with CUDA
 * events on the launch's own stream (0 stops).  sdedge_kernel_times waits for the recorded
 * events and writes the summed milliseconds per kernel kind to ms[4] -- [0] the prep kernel of
 * the tiled path, [1] the main DP launch, [2] the worst-case-pool pass, [3] other -- and the
 * launch counts to launches[4] (optional).  At most 4096 launches are recorded. */
int sdedge_kernel_timing(int32_t enable);
int sdedge_kernel_times(double* ms, int32_t* launches);

/* Number of kernel launches the last successful call on this thread enqueued. */
int sdedge_last_launch_count(void);

/* Message for the last nonzero return on this thread ("" if none). */
const char* sdedge_last_error(void);

int sdedge_abi_version(void);

/* FP64 / FP32 pipe peak microbenchmark (the roofline denominator):
 * runs a DFMA (fp32: FFMA) chain on every SM of the current device and
 * returns achieved FMA-lane operations per second in *ops_per_s (an FMA
 * counts as one operation).  Synchronous.  Returns 0 or a negative error. */
int sdedge_pipe_peak(int32_t fp32, double* ops_per_s, double* elapsed_s);

#ifdef __cplusplus
}
#endif
#endif
