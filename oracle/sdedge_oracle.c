/*
 * sdedge_oracle.c -- TEST INFRASTRUCTURE ONLY (see sdedge_oracle.h).
 *
 * A plain, slow, literal fp64 implementation of the paper's solver:
 *   P1 closed-form bandwidth, P2 Algorithm 1 with the
 *   repairs listed in DESIGN.md ("Readings"), P3 enumeration of the
 *   speculation length.
 * Stage times are computed literally, pass by pass, from eq:flops_d /
 * eq:flops_v / eq:latency_b2 / eq:d_latency / eq:v_latency for every
 * candidate (i, j) and every decoding step n, exactly as Algorithm 1 lines
 * 12-15 prescribe.  No closed forms, no blocking, no reordering.
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -pthread (no -ffast-math).
 */
#include "sdedge_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* eq:ol: L = (1 - alpha^{1+l}) / (1 - alpha).
 * Reading A2: alpha^{1+l} by repeated multiplication, each op rounded.   */
double orc_expected_tokens(double alpha, int gamma)
{
    double A = alpha;
    for (int t = 0; t < gamma; ++t) A = A * alpha;
    return (1.0 - A) / (1.0 - alpha);
}

/* eq:step_n: n_m = ceil(O_m / L), with O_m = O_max. */
int32_t orc_decode_steps(int32_t O, double L)
{
    double q = (double)O / L;
    return (int32_t)ceil(q);
}

/* eq:memory_model: Gamma_p = J (8 h1^2 + 4 h1 h2) bytes (FP16). */
int64_t orc_param_memory(int32_t J, int32_t h1, int32_t h2)
{
    return (int64_t)J * (8 * (int64_t)h1 * h1 + 4 * (int64_t)h1 * h2);
}

/* eq:memory_kv: per task 4 J h1 (I_m + O_m) bytes. */
int64_t orc_kv_memory_per_task(int32_t J, int32_t h1, int32_t I, int32_t O)
{
    return 4 * (int64_t)J * h1 * ((int64_t)I + O);
}

/* eq:flops_d: FLOPs of the i-th draft forward pass at step n. */
double orc_flops_draft(int32_t J, int32_t h1, int32_t h2, double Im, double L, int i, int n)
{
    if (n == 1 && i == 1)
        return 4.0 * J * h1 * Im * (2.0 * h1 + Im + h2);
    double Ikv = Im + ((n - 1) * L - 1.0) + i - 1; /* I^{kv,d}_{i,n,m} */
    return 4.0 * J * h1 * (2.0 * h1 + Ikv + 1.0 + h2);
}

/* eq:flops_v: FLOPs of the verify pass at step n (l = gamma). */
double orc_flops_verify(int32_t J, int32_t h1, int32_t h2, double Im, int gamma, double L, int n)
{
    if (n == 1)
        return 4.0 * J * h1 * (Im + gamma) * (2.0 * h1 + Im + gamma + h2);
    double Ikv = Im + (n - 1) * L - 1.0; /* I^{kv,v}_{n,m} */
    return 4.0 * J * h1 * (1.0 + gamma) * (2.0 * h1 + Ikv + gamma + 1.0 + h2);
}

/* eq:latency_b2: T(b, F) = c1 F b + c2. */
double orc_runtime(double c1, double c2, double F, double b)
{
    return c1 * F * b + c2;
}

static void coeffs_of(const orc_params* P, const double* co, double* c1d, double* c2d,
                      double* c1v, double* c2v)
{
    if (co) { *c1d = co[0]; *c2d = co[1]; *c1v = co[2]; *c2v = co[3]; }
    else    { *c1d = P->c1d; *c2d = P->c2d; *c1v = P->c1v; *c2v = P->c2v; }
}

/* eq:d_latency: T^d_{n,m} = sum_{i=1}^{l} (c1d F^d_{i,n,m} b + c2d). */
double orc_draft_time(const orc_params* P, const double* co, int b, int32_t Im, int gamma,
                      double L, int n)
{
    double c1d, c2d, c1v, c2v;
    coeffs_of(P, co, &c1d, &c2d, &c1v, &c2v);
    double t = 0.0;
    for (int i = 1; i <= gamma; ++i)
        t += orc_runtime(c1d, c2d, orc_flops_draft(P->Jd, P->h1d, P->h2d, (double)Im, L, i, n), (double)b);
    return t;
}

/* eq:v_latency: T^v_{n,m} = c1v F^v_{n,m} b + c2v
 * (+ optional downlink constant, reading A12; 0 by default). */
double orc_verify_time(const orc_params* P, const double* co, int b, int32_t Im, int gamma,
                       double L, int n)
{
    double c1d, c2d, c1v, c2v;
    coeffs_of(P, co, &c1d, &c2d, &c1v, &c2v);
    return orc_runtime(c1v, c2v, orc_flops_verify(P->Jv, P->h1v, P->h2v, (double)Im, gamma, L, n),
                       (double)b) + P->downlink_s;
}

/* Memory feasibility of a batch of b tasks padded to Im (cons. (b) P:551,
 * Alg. 1 lines 10-13).  128-bit so the literal product cannot overflow. */
static int batch_fits(const orc_params* P, int b, int32_t Im)
{
    __int128 mem = (__int128)orc_param_memory(P->Jd, P->h1d, P->h2d)
                 + (__int128)b * orc_kv_memory_per_task(P->Jd, P->h1d, Im, P->O_max);
    return mem <= (__int128)P->gamma_s;
}

/* t*_com and eq:opt_w.  The printed t* has "p_k/g_k sigma^2"
 * (P:608); reading A14 uses p_k g_k / sigma^2 as in eq:ul_latency_k. */
double orc_bandwidth(const orc_params* P, const int32_t* I, const double* p, const double* g, double* w)
{
    const int K = P->K;
    const double lam = P->lambda > 0 ? P->lambda : 16.0 * (P->h1d + P->h1v);
    if (P->bw_policy == 1) {
        /* uniform scheme: w_k = 1/K; T_com = max_k T_k,com (eq:ul_latency_k, eq:ul_latency) */
        double tmax = 0.0;
        for (int k = 0; k < K; ++k) {
            double wk = 1.0 / K;
            double snr = p[k] * g[k] / P->sigma2;
            double r = wk * P->Bw * log2(1.0 + snr);
            double t = lam * I[k] / r;
            if (t > tmax) tmax = t;
            if (w) w[k] = wk;
        }
        return tmax;
    }
    double tcom = 0.0, denom = 0.0;
    for (int k = 0; k < K; ++k) {
        double snr = p[k] * g[k] / P->sigma2;
        double s = log2(1.0 + snr);
        tcom += lam * I[k] / (P->Bw * s);
        denom += I[k] / s;
    }
    if (w)
        for (int k = 0; k < K; ++k) {
            double snr = p[k] * g[k] / P->sigma2;
            double s = log2(1.0 + snr);
            w[k] = (I[k] / s) / denom;
        }
    return tcom;
}

/* eq:time, eq:latency_infer_batch, eq:latency_inf for a given
 * plan under uniform O_max planning (M_n = M). */
double orc_eval_plan(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                     int gamma, int M, const int32_t* batch_end)
{
    double L = orc_expected_tokens(alpha, gamma);
    int N = orc_decode_steps(P->O_max, L);
    for (int m = 0; m < M; ++m) {
        int start = m ? batch_end[m - 1] + 1 : 1;
        if (!batch_fits(P, batch_end[m] - start + 1, Is[batch_end[m] - 1])) return INFINITY;
    }
    double Tinf = 0.0;
    for (int n = 1; n <= N; ++n) {
        double Cd = 0.0, C = 0.0; /* C_{n,0} = 0 */
        for (int m = 0; m < M; ++m) {
            int start = m ? batch_end[m - 1] + 1 : 1;
            int b = batch_end[m] - start + 1;
            int32_t Im = Is[batch_end[m] - 1]; /* sorted: max is the last */
            Cd += orc_draft_time(P, co, b, Im, gamma, L, n);         /* C^d_{n,m} */
            double st = Cd > C ? Cd : C;                             /* max{C^d, C_{n,m-1}} */
            C = st + orc_verify_time(P, co, b, Im, gamma, L, n);     /* eq:time */
        }
        Tinf += C; /* T_n = C_{n,M} */
    }
    return Tinf;
}

double orc_eval_actual(const orc_params* P, const double* co, const int32_t* Is, const int32_t* Os,
                       double alpha, int gamma, int M, const int32_t* batch_end)
{
    double L = orc_expected_tokens(alpha, gamma);
    int* nm = (int*)malloc(sizeof(int) * (M > 0 ? M : 1));
    int N = 0;
    for (int m = 0; m < M; ++m) {
        int start = m ? batch_end[m - 1] + 1 : 1;
        int Om = 0;                                   /* O_m = max_k x_k^m O_k */
        for (int q = start; q <= batch_end[m]; ++q) if (Os[q - 1] > Om) Om = Os[q - 1];
        nm[m] = orc_decode_steps(Om, L);              /* eq:step_n */
        if (nm[m] > N) N = nm[m];                     /* N = max_m n_m */
    }
    double Tinf = 0.0;
    for (int n = 1; n <= N; ++n) {
        double Cd = 0.0, C = 0.0;
        for (int m = 0; m < M; ++m) {
            if (nm[m] < n) continue;                  /* active set M_n */
            int start = m ? batch_end[m - 1] + 1 : 1;
            int b = batch_end[m] - start + 1;
            int32_t Im = Is[batch_end[m] - 1];
            if (P->batch_policy == 1) {               /* SD w/o pipeline: sequential stages */
                C += orc_draft_time(P, co, b, Im, gamma, L, n) + orc_verify_time(P, co, b, Im, gamma, L, n);
                continue;
            }
            Cd += orc_draft_time(P, co, b, Im, gamma, L, n);
            double st = Cd > C ? Cd : C;
            C = st + orc_verify_time(P, co, b, Im, gamma, L, n);
        }
        Tinf += C;                                    /* T_n = C_{n, M_n} */
    }
    free(nm);
    return Tinf;
}

double orc_eval_plan_nopipe(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                            int gamma, int M, const int32_t* batch_end)
{
    double L = orc_expected_tokens(alpha, gamma);
    int N = orc_decode_steps(P->O_max, L);
    for (int m = 0; m < M; ++m) {
        int start = m ? batch_end[m - 1] + 1 : 1;
        if (!batch_fits(P, batch_end[m] - start + 1, Is[batch_end[m] - 1])) return INFINITY;
    }
    double Tinf = 0.0;
    for (int n = 1; n <= N; ++n) {
        double Tn = 0.0;
        for (int m = 0; m < M; ++m) {
            int start = m ? batch_end[m - 1] + 1 : 1;
            int b = batch_end[m] - start + 1;
            int32_t Im = Is[batch_end[m] - 1];
            Tn += orc_draft_time(P, co, b, Im, gamma, L, n) + orc_verify_time(P, co, b, Im, gamma, L, n);
        }
        Tinf += Tn;
    }
    return Tinf;
}

double orc_dp_nopipe(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
                     int32_t* S, double* row_gap, int64_t* W)
{
    /* Algorithm 1's loop structure with the sequential (no-overlap) step cost:
     * T_{i,j} = Upsilon[j-1,0,0] + sum_n (T^d_n + T^v_n) -- additive, so exact. */
    const int K = P->K;
    double L = orc_expected_tokens(alpha, gamma);
    int N = orc_decode_steps(P->O_max, L);
    double* V = (double*)calloc((size_t)K + 1, sizeof(double));
    double result = 0.0;
    for (int i = 1; i <= K; ++i) {
        double best = INFINITY, second = INFINITY;
        int jstar = 0;
        int32_t Im = Is[i - 1];
        for (int j = 1; j <= i; ++j) {
            int b = i - j + 1;
            if (!batch_fits(P, b, Im)) continue;
            double temp = V[j - 1];
            for (int n = 1; n <= N; ++n)
                temp += orc_draft_time(P, co, b, Im, gamma, L, n) + orc_verify_time(P, co, b, Im, gamma, L, n);
            if (W) *W += N;
            if (best >= temp) { second = best; best = temp; jstar = j; }
            else if (temp < second) second = temp;
        }
        if (jstar == 0) { result = INFINITY; if (S) S[i - 1] = 0; break; }
        V[i] = best;
        if (S) S[i - 1] = jstar;
        if (row_gap)
            row_gap[i - 1] = isinf(second) ? INFINITY : second == best ? 0.0 : (second - best) / fabs(best);
        result = best;
    }
    free(V);
    return result;
}

static int equal_plan(int K, int b, int32_t* ends)
{
    int M = 0;
    for (int e = b; e < K; e += b) ends[M++] = e;
    ends[M++] = K;
    return M;
}

int orc_fixed_plan(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
                   int32_t* ends)
{
    const int K = P->K;
    int M = 0;
    switch (P->batch_policy) {
    case 2: /* no batching: one task at a time */
        for (int k = 1; k <= K; ++k) ends[M++] = k;
        break;
    case 3: /* static batching: fixed small batch size, contiguous in sorted order */
        M = equal_plan(K, P->static_batch < K ? P->static_batch : K, ends);
        break;
    case 4: { /* max batching: largest b for which a batch of b of the arriving
                 tasks' longest input (and O_max) fits the SBS memory (reading B4) */
        int b = 0;
        while (b < K && batch_fits(P, b + 1, Is[K - 1])) ++b;
        if (b < 1) return 0;
        M = equal_plan(K, b, ends);
        break;
    }
    case 5: { /* heuristic: equal batches of size b, b growing until the
                 pipelined latency stops improving (or memory binds); reading B5 starts at
                 b = 2, reading B5' (heuristic_start = 1) at two batches,
                 b = ceil(K/2) */
        int32_t tmp[1024 + 1];
        int bbest = 1;
        double tbest = INFINITY;
        const int b0 = P->heuristic_start ? (K + 1) / 2 : (K >= 2 ? 2 : 1);
        for (int b = b0; b <= K; ++b) {
            int Mt = equal_plan(K, b, tmp);
            double t = orc_eval_plan(P, co, Is, alpha, gamma, Mt, tmp);
            if (!(t < tbest) && !isinf(tbest)) break;   /* latency starts to degrade */
            if (isinf(t)) break;                          /* memory binds */
            tbest = t;
            bbest = b;
        }
        if (isinf(tbest)) bbest = 1;                      /* even b = 2 infeasible: one at a time */
        M = equal_plan(K, bbest, ends);
        break;
    }
    default:
        return 0;
    }
    for (int m = 0; m < M; ++m) {
        int start = m ? ends[m - 1] + 1 : 1;
        if (!batch_fits(P, ends[m] - start + 1, Is[ends[m] - 1])) return 0;
    }
    return M;
}

/* Algorithm 1 with readings A1 (bracket of eq:t_ij1), A3 (K+1
 * rows, row 0 = 0, best = +inf), A4 (S[i] always set), A6 (largest j wins
 * ties: the ">=" of line 21).
 * force (optional, [K], 0 = free): row i takes j = force[i-1] instead of its
 * argmin -- every candidate is still evaluated, so row_best[i-1] receives the
 * row's minimum and row_taken[i-1] the value of the candidate taken.  This is
 * the near-tie branching replay of SURVEY 8(c) "T": a plan reached by taking,
 * at rows whose best-vs-taken gap is below a threshold, a near-best candidate
 * instead of the best (PAPER.md:738 -- the tie rule decides exact ties only).
 * A forced j that is memory-infeasible (or outside 1..i) makes the result NaN. */
double orc_dp_trace(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
                    const int32_t* force, int32_t* S, double* row_gap, double* row_best,
                    double* row_taken, int64_t* W)
{
    const int K = P->K;
    double L = orc_expected_tokens(alpha, gamma);
    int N = orc_decode_steps(P->O_max, L);
    size_t rowlen = (size_t)(N + 1) * 2;
    double* Y = (double*)calloc((size_t)(K + 1) * rowlen, sizeof(double)); /* Upsilon */
    double* Td = (double*)malloc((size_t)(N + 1) * sizeof(double));
    double* Tv = (double*)malloc((size_t)(N + 1) * sizeof(double));
#define UPS(i, n, s) Y[(size_t)(i) * rowlen + (size_t)(n) * 2 + (s)]
    double result = 0.0;
    for (int i = 1; i <= K; ++i) {
        double best = INFINITY, second = INFINITY, taken = NAN;
        int jstar = 0;
        const int jf = force ? force[i - 1] : 0;
        int32_t Im = Is[i - 1]; /* max input length of tasks j..i */
        for (int j = 1; j <= i; ++j) {
            int b = i - j + 1;
            if (!batch_fits(P, b, Im)) continue; /* Alg. 1 lines 10-13 */
            for (int n = 1; n <= N; ++n) {      /* Alg. 1 lines 14-15 */
                Tv[n] = orc_verify_time(P, co, b, Im, gamma, L, n);
                Td[n] = orc_draft_time(P, co, b, Im, gamma, L, n);
            }
            double temp = 0.0;                  /* Alg. 1 line 15, eq:t_ij1 (A1) */
            for (int n = 1; n <= N; ++n) {
                double d0 = UPS(j - 1, n, 0) + Td[n];
                double y1 = UPS(j - 1, n, 1);
                temp += (d0 > y1 ? d0 : y1) + Tv[n];
            }
            if (W) *W += N;
            if (j == jf) taken = temp;
            if (best >= temp) { second = best; best = temp; jstar = j; } /* line 21 */
            else if (temp < second) second = temp;
        }
        if (jstar == 0) { result = INFINITY; if (S) S[i - 1] = 0; break; } /* no feasible batch */
        if (jf > 0) {
            if (isnan(taken)) { result = NAN; if (S) S[i - 1] = jf; break; } /* forced j infeasible */
        } else {
            taken = best;
        }
        const int jt = jf > 0 ? jf : jstar;
        UPS(i, 0, 0) = taken;                   /* eq:rg (the taken candidate) */
        if (S) S[i - 1] = jt;
        if (row_gap) /* relative gap; an exact tie is a zero gap even at best == 0 */
            row_gap[i - 1] = isinf(second) ? INFINITY : second == best ? 0.0 : (second - best) / fabs(best);
        if (row_best) row_best[i - 1] = best;
        if (row_taken) row_taken[i - 1] = taken;
        int b = i - jt + 1;
        for (int n = 1; n <= N; ++n) {          /* eq:tt1, eq:tt2 (line 26) */
            double td = orc_draft_time(P, co, b, Im, gamma, L, n);
            double tv = orc_verify_time(P, co, b, Im, gamma, L, n);
            double d0 = UPS(jt - 1, n, 0) + td;
            double y1 = UPS(jt - 1, n, 1);
            UPS(i, n, 0) = d0;
            UPS(i, n, 1) = (d0 > y1 ? d0 : y1) + tv;
        }
        result = taken;
    }
#undef UPS
    free(Y); free(Td); free(Tv);
    return result;
}

/* Algorithm 1 as written: orc_dp_trace with every row free, or with one
 * forced row (force_row >= 1 takes j = force_j there). */
double orc_dp(const orc_params* P, const double* co, const int32_t* Is, double alpha, int gamma,
              int32_t* S, double* row_gap, int64_t* W, int force_row, int force_j)
{
    if (force_row < 1 || force_row > P->K)
        return orc_dp_trace(P, co, Is, alpha, gamma, NULL, S, row_gap, NULL, NULL, W);
    int32_t* f = (int32_t*)calloc((size_t)P->K, sizeof(int32_t));
    f[force_row - 1] = force_j;
    double t = orc_dp_trace(P, co, Is, alpha, gamma, f, S, row_gap, NULL, NULL, W);
    free(f);
    return t;
}

/* ---------------------------------------------------------------- per-batch gamma
 * an EXTENSION, not the paper's method: the paper fixes one
 * global speculation length l (cons. (f) P:555; the enumeration of P3),
 * and SPEC.md:540 lists per-batch lengths as a non-goal.  Here batch m runs gamma_m
 * draft passes per step, so it has its own L_m = eq:ol(alpha, gamma_m) and
 * n_m = ceil(O_max / L_m) (eq:step_n under uniform O_max planning), and
 * at step n only the batches with n_m >= n take part in the eq:time recursion --
 * the active set M_n of eq:latency_infer_batch, the same mechanism the
 * paper uses for batches that finish early.  Reading NB1: a row's
 * candidates are the pairs (j, gamma); ties go to the largest j, then the
 * smallest gamma. */
double orc_eval_plan_pbg(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                         int M, const int32_t* batch_end, const int32_t* gammas)
{
    double* L = (double*)malloc(sizeof(double) * (M > 0 ? M : 1));
    int* nm = (int*)malloc(sizeof(int) * (M > 0 ? M : 1));
    int N = 0;
    for (int m = 0; m < M; ++m) {
        int start = m ? batch_end[m - 1] + 1 : 1;
        if (!batch_fits(P, batch_end[m] - start + 1, Is[batch_end[m] - 1])) { free(L); free(nm); return INFINITY; }
        L[m] = orc_expected_tokens(alpha, gammas[m]);
        nm[m] = orc_decode_steps(P->O_max, L[m]);
        if (nm[m] > N) N = nm[m];
    }
    double Tinf = 0.0;
    for (int n = 1; n <= N; ++n) {
        double Cd = 0.0, C = 0.0;
        for (int m = 0; m < M; ++m) {
            if (nm[m] < n) continue;                  /* active set M_n */
            int start = m ? batch_end[m - 1] + 1 : 1;
            int b = batch_end[m] - start + 1;
            int32_t Im = Is[batch_end[m] - 1];
            Cd += orc_draft_time(P, co, b, Im, gammas[m], L[m], n);
            double st = Cd > C ? Cd : C;
            C = st + orc_verify_time(P, co, b, Im, gammas[m], L[m], n);
        }
        Tinf += C;                                    /* T_n = C_{n, M_n} */
    }
    free(L); free(nm);
    return Tinf;
}

/* Algorithm 1 (readings A1-A6) with candidates (j, gamma), gamma in
 * [gamma_min, gamma_max]: Upsilon rows run over n = 1..N_max = max_gamma N_gamma; a
 * candidate whose batch is finished at step n (n > N_gamma) adds no stage time there,
 * max{Upsilon[j-1,n,0] + 0, Upsilon[j-1,n,1]} + 0 = Upsilon[j-1,n,1] (Upsilon1 >=
 * Upsilon0 always).  S[i-1] = j*, Gm[i-1] = gamma* of the batch ending at row i. */
double orc_dp_pbg(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                  int32_t* S, int32_t* Gm, double* row_gap, int64_t* W)
{
    const int K = P->K, ng = P->gamma_max - P->gamma_min + 1;
    double* Lg = (double*)malloc(sizeof(double) * ng);
    int* Ng = (int*)malloc(sizeof(int) * ng);
    int N = 0;
    for (int q = 0; q < ng; ++q) {
        Lg[q] = orc_expected_tokens(alpha, P->gamma_min + q);
        Ng[q] = orc_decode_steps(P->O_max, Lg[q]);
        if (Ng[q] > N) N = Ng[q];
    }
    size_t rowlen = (size_t)(N + 1) * 2;
    double* Y = (double*)calloc((size_t)(K + 1) * rowlen, sizeof(double));
#define UPS(i, n, s) Y[(size_t)(i) * rowlen + (size_t)(n) * 2 + (s)]
    double result = 0.0;
    for (int i = 1; i <= K; ++i) {
        double best = INFINITY, second = INFINITY;
        int jstar = 0, qstar = -1;
        int32_t Im = Is[i - 1];
        for (int j = 1; j <= i; ++j) {
            int b = i - j + 1;
            if (!batch_fits(P, b, Im)) continue;
            for (int q = ng - 1; q >= 0; --q) {           /* gamma descending: ties -> smallest gamma */
                const int gm = P->gamma_min + q;
                double temp = 0.0;
                for (int n = 1; n <= N; ++n) {
                    double y1 = UPS(j - 1, n, 1);
                    if (n <= Ng[q]) {
                        double d0 = UPS(j - 1, n, 0) + orc_draft_time(P, co, b, Im, gm, Lg[q], n);
                        temp += (d0 > y1 ? d0 : y1) + orc_verify_time(P, co, b, Im, gm, Lg[q], n);
                    } else {
                        temp += y1;                       /* batch finished: no stage time */
                    }
                }
                if (W) *W += N;
                if (best >= temp) { second = best; best = temp; jstar = j; qstar = q; }
                else if (temp < second) second = temp;
            }
        }
        if (jstar == 0) { result = INFINITY; if (S) S[i - 1] = 0; if (Gm) Gm[i - 1] = -1; break; }
        UPS(i, 0, 0) = best;
        if (S) S[i - 1] = jstar;
        if (Gm) Gm[i - 1] = P->gamma_min + qstar;
        if (row_gap)
            row_gap[i - 1] = isinf(second) ? INFINITY : second == best ? 0.0 : (second - best) / fabs(best);
        const int b = i - jstar + 1, gm = P->gamma_min + qstar;
        for (int n = 1; n <= N; ++n) {
            double d0 = UPS(jstar - 1, n, 0), y1 = UPS(jstar - 1, n, 1);
            if (n <= Ng[qstar]) {
                d0 += orc_draft_time(P, co, b, Im, gm, Lg[qstar], n);
                y1 = (d0 > y1 ? d0 : y1) + orc_verify_time(P, co, b, Im, gm, Lg[qstar], n);
            }
            UPS(i, n, 0) = d0;
            UPS(i, n, 1) = y1;
        }
        result = best;
    }
#undef UPS
    free(Y); free(Lg); free(Ng);
    return result;
}

/* Stable ascending sort of task indices by I_k (reading A13). */
static void sort_tasks(int K, const int32_t* I, int32_t* order)
{
    for (int k = 0; k < K; ++k) order[k] = k;
    for (int a = 1; a < K; ++a) { /* insertion sort: stable */
        int32_t t = order[a];
        int c = a - 1;
        while (c >= 0 && I[order[c]] > I[t]) { order[c + 1] = order[c]; --c; }
        order[c + 1] = t;
    }
}

void orc_solve(const orc_params* P, const int32_t* I, const double* p, const double* g,
               double alpha, const double* coeffs4, orc_result* R, int32_t* order,
               int32_t* batch_end, double* w, double* tinf_gamma, int32_t* batch_gamma)
{
    const int K = P->K;
    const int ng = P->gamma_max - P->gamma_min + 1;
    memset(R, 0, sizeof(*R));
    R->gamma = -1; R->min_row_gap = INFINITY; R->gamma_gap = INFINITY;
    R->gap_gamma = -1; R->gap_row = -1;
    for (int k = 0; k < K; ++k) batch_end[k] = 0;
    if (batch_gamma) for (int k = 0; k < K; ++k) batch_gamma[k] = 0;
    sort_tasks(K, I, order);

    int bad_task = 0;
    for (int k = 0; k < K; ++k)
        if (I[k] < 1 || !(p[k] > 0) || !(g[k] > 0) || !isfinite(p[k]) || !isfinite(g[k])) bad_task = 1;
    if (bad_task) {
        R->status = 3;
        R->T = R->T_com = R->T_inf = NAN;
        for (int k = 0; k < K; ++k) w[k] = NAN;
        for (int q = 0; q < ng; ++q) tinf_gamma[q] = NAN;
        return;
    }
    R->T_com = orc_bandwidth(P, I, p, g, w);
    if (!(alpha > 0.0 && alpha < 1.0)) {
        R->status = 2;
        R->T = R->T_inf = NAN;
        for (int q = 0; q < ng; ++q) tinf_gamma[q] = NAN;
        return;
    }
    int32_t* Is = (int32_t*)malloc(sizeof(int32_t) * K);
    int32_t* S = (int32_t*)malloc(sizeof(int32_t) * K);
    int32_t* Sbest = (int32_t*)malloc(sizeof(int32_t) * K);
    double* gap = (double*)malloc(sizeof(double) * K);
    for (int k = 0; k < K; ++k) Is[k] = I[order[k]];

    double best = INFINITY, second = INFINITY;
    int gbest = -1, Mbest = 0;
    int32_t* ends = (int32_t*)malloc(sizeof(int32_t) * (K + 1));
    int32_t* ends_best = (int32_t*)malloc(sizeof(int32_t) * (K + 1));
    if (P->batch_policy == 6) {   /* per-batch gamma (NEXT-3 extension): one DP over (j, gamma) */
        int32_t* Gm = (int32_t*)malloc(sizeof(int32_t) * K);
        for (int r = 0; r < K; ++r) gap[r] = INFINITY;
        double t = orc_dp_pbg(P, coeffs4, Is, alpha, S, Gm, gap, &R->W);
        for (int q = 0; q < ng; ++q) tinf_gamma[q] = t;
        for (int r = 0; r < K; ++r)
            if (gap[r] < R->min_row_gap) { R->min_row_gap = gap[r]; R->gap_gamma = -1; R->gap_row = r + 1; }
        if (isinf(t)) {
            R->status = 1;
            R->T = R->T_inf = INFINITY;
        } else {
            int tmp[1024 + 1], i = K, M = 0;
            while (i > 0) { tmp[M++] = i; i = S[i - 1] - 1; }
            for (int m = 0; m < M; ++m) {
                batch_end[m] = tmp[M - 1 - m];
                if (batch_gamma) batch_gamma[m] = Gm[batch_end[m] - 1];
            }
            R->M = M;
            R->gamma = Gm[K - 1];          /* the last batch's length (batch_gamma has them all) */
            R->T_inf = t;
            R->T = R->T_com + t;
        }
        free(Gm);
        free(ends); free(ends_best);
        free(Is); free(S); free(Sbest); free(gap);
        return;
    }
    for (int gm = P->gamma_min; gm <= P->gamma_max; ++gm) { /* P3 */
        double t;
        int Mg = 0;
        if (P->batch_policy <= 1) {
            for (int r = 0; r < K; ++r) gap[r] = INFINITY;
            t = P->batch_policy == 0 ? orc_dp(P, coeffs4, Is, alpha, gm, S, gap, &R->W, 0, 0)
                                     : orc_dp_nopipe(P, coeffs4, Is, alpha, gm, S, gap, &R->W);
            if (!isinf(t)) {   /* backtracking (reading A5: i <- S[i] - 1) */
                int tmp[1024 + 1], i = K;
                while (i > 0) { tmp[Mg++] = i; i = S[i - 1] - 1; }
                for (int m = 0; m < Mg; ++m) ends[m] = tmp[Mg - 1 - m];
            }
        } else {
            Mg = orc_fixed_plan(P, coeffs4, Is, alpha, gm, ends);
            t = Mg > 0 ? orc_eval_plan(P, coeffs4, Is, alpha, gm, Mg, ends) : INFINITY;
            for (int r = 0; r < K; ++r) gap[r] = INFINITY;
        }
        tinf_gamma[gm - P->gamma_min] = t;
        if (isinf(t)) continue;
        for (int r = 0; r < K; ++r)
            if (gap[r] < R->min_row_gap) { R->min_row_gap = gap[r]; R->gap_gamma = gm; R->gap_row = r + 1; }
        if (t < best) { second = best; best = t; gbest = gm; Mbest = Mg; memcpy(ends_best, ends, sizeof(int32_t) * Mg); }
        else if (t < second) second = t; /* smallest gamma wins ties (reading A7) */
    }
    if (gbest < 0) {
        R->status = 1;
        R->T = R->T_inf = INFINITY;
    } else {
        R->gamma = gbest;
        R->T_inf = best;
        R->T = R->T_com + R->T_inf;
        R->gamma_gap = isinf(second) ? INFINITY : (second - best) / best;
        for (int m = 0; m < Mbest; ++m) batch_end[m] = ends_best[m];
        if (batch_gamma) for (int m = 0; m < Mbest; ++m) batch_gamma[m] = gbest;
        R->M = Mbest;
    }
    free(ends); free(ends_best);
    free(Is); free(S); free(Sbest); free(gap);
}

double orc_brute_force(const orc_params* P, const double* co, const int32_t* Is, double alpha,
                       int gamma_min, int gamma_max, int32_t* best_gamma, int32_t* best_M,
                       int32_t* best_end)
{
    const int K = P->K;
    double best = INFINITY;
    int32_t ends[32];
    *best_gamma = -1; *best_M = 0;
    if (K > 20) return NAN;
    for (int gm = gamma_min; gm <= gamma_max; ++gm) {
        for (long mask = 0; mask < (1L << (K - 1)); ++mask) {
            int M = 0;
            for (int t = 0; t < K - 1; ++t)
                if (mask & (1L << t)) ends[M++] = t + 1;
            ends[M++] = K;
            double v = orc_eval_plan(P, co, Is, alpha, gm, M, ends);
            if (v < best) {
                best = v; *best_gamma = gm; *best_M = M;
                memcpy(best_end, ends, sizeof(int32_t) * M);
            }
        }
    }
    return best;
}

/* ---------------------------------------------------------------- batch */
typedef struct {
    const orc_params* P; int64_t n; const int32_t* I; const double *p, *g, *alpha, *coeffs;
    int32_t *status, *gamma, *M; double* lat; int32_t *order, *batch_end; double* w;
    double *min_row_gap, *gamma_gap; int64_t* W; int32_t* batch_gamma; int64_t next;
} batch_ctx;

static void* batch_worker(void* arg)
{
    batch_ctx* c = (batch_ctx*)arg;
    const int K = c->P->K;
    double* tg = (double*)malloc(sizeof(double) * (c->P->gamma_max - c->P->gamma_min + 1));
    for (;;) {
        int64_t s = __atomic_fetch_add(&c->next, 1, __ATOMIC_RELAXED);
        if (s >= c->n) break;
        orc_result R;
        orc_solve(c->P, c->I + s * K, c->p + s * K, c->g + s * K, c->alpha[s],
                  c->coeffs ? c->coeffs + s * 4 : NULL, &R, c->order + s * K,
                  c->batch_end + s * K, c->w + s * K, tg, c->batch_gamma ? c->batch_gamma + s * K : NULL);
        c->status[s] = R.status; c->gamma[s] = R.gamma; c->M[s] = R.M;
        c->lat[3 * s] = R.T; c->lat[3 * s + 1] = R.T_com; c->lat[3 * s + 2] = R.T_inf;
        if (c->min_row_gap) c->min_row_gap[s] = R.min_row_gap;
        if (c->gamma_gap) c->gamma_gap[s] = R.gamma_gap;
        if (c->W) c->W[s] = R.W;
    }
    free(tg);
    return NULL;
}

void orc_solve_batch(const orc_params* P, int64_t n, const int32_t* I, const double* p,
                     const double* g, const double* alpha, const double* coeffs,
                     int32_t* status, int32_t* gamma, int32_t* M, double* lat,
                     int32_t* order, int32_t* batch_end, double* w, double* min_row_gap,
                     double* gamma_gap, int64_t* W, int32_t* batch_gamma, int nthreads)
{
    batch_ctx c = {P, n, I, p, g, alpha, coeffs, status, gamma, M, lat, order, batch_end, w,
                   min_row_gap, gamma_gap, W, batch_gamma, 0};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, &c);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}
