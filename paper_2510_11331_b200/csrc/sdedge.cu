// sdedge.cu -- sm_100a kernels and C-ABI implementation of sdedge_solve_batch
// (include/sdedge.h).  Citations: P:n = PAPER.md line n; DESIGN.md sections.
//
// One persistent CTA owns one scenario at a time (atomic work queue):
//   stage + validate  ->  stable rank sort  ->  t*_com, w* block
//   reduction (eq:opt_w)  ->  warps pull speculation lengths gamma
//   from a CTA-local queue and each runs Algorithm 1 for its
//   gamma  ->  gamma* argmin + backtrack  ->  outputs.
//
// Inside one warp's DP, row i's candidates j (lanes) read predecessor row
// p = j-1.  Upsilon is not stored as a (K+1) x N x 2 table: for n >= 2
//   Upsilon[p, n, 0] = a0[p] + s0[p] (n-1)            (affine, D2)
//   Upsilon[p, n, 1] = env_p(n-1), convex piecewise-linear, kept as segments
// which is exact up to rounding because every stage time is affine in n for
// n >= 2 (eq:flops_d, eq:flops_v with the KV lengths of P:390).
// The candidate sum of eq:t_ij1 over n = 2..N is then either
//   ALGO_ENVELOPE: esum[p] + sum_m max(P + Q m - env_p(m), 0), closed form
//                  per segment (an arithmetic series on the positive part), or
//   ALGO_DENSE:    sum_m max(P + Q m, env_p(m)) step by step (the paper's
//                  O(K^2 N) loop),
// plus the hoisted verify sum (N-1) Av + Bv (N-1)N/2 and the n = 1 term.
#include "sdedge.h"

#include <cuda.h>          // driver-API types only (entry points are fetched at run time: no -lcuda)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

// Optional per-kernel timing (sdedge_kernel_timing): while enabled, every launch of the solve is
// bracketed by CUDA events on its own stream; sdedge_kernel_times sums the durations per kernel
// kind.  Events are recycled, so a long timed region costs no allocation after the first steps.
struct KTiming {
    bool on = false;
    int used = 0;
    int kind[4096];
    cudaEvent_t ev[4096][2];
    int created = 0;
};
thread_local KTiming g_kt;

enum { KT_PREP = 0, KT_MAIN = 1, KT_BIG = 2, KT_OTHER = 3 };

inline int kt_begin(int kind, cudaStream_t st)
{
    if (!g_kt.on || g_kt.used >= 4096) return -1;
    const int q = g_kt.used++;
    if (q >= g_kt.created) {
        if (cudaEventCreate(&g_kt.ev[q][0]) != cudaSuccess || cudaEventCreate(&g_kt.ev[q][1]) != cudaSuccess) {
            --g_kt.used;
            return -1;
        }
        g_kt.created = q + 1;
    }
    g_kt.kind[q] = kind;
    cudaEventRecord(g_kt.ev[q][0], st);
    return q;
}

inline void kt_end(int q, cudaStream_t st)
{
    if (q >= 0) cudaEventRecord(g_kt.ev[q][1], st);
}

int fail(int code, const char* msg)
{
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

#ifndef SDEDGE_WARPS
#define SDEDGE_WARPS 1
#endif
constexpr int kWarps = SDEDGE_WARPS;     // warps per CTA
#ifndef SDEDGE_TILE_G
#define SDEDGE_TILE_G 1       // DPs per warp of the tiled DP (tile = 32 / G rows)
#endif
#ifndef SDEDGE_TILE_SHFL_ARGMIN
#define SDEDGE_TILE_SHFL_ARGMIN 1
#endif
#ifndef SDEDGE_LBB_FIRST
#define SDEDGE_LBB_FIRST 0    // 1: the batch-count bound also screens the first gamma of the queue (0: only the later ones)
#endif
#ifndef SDEDGE_QCHUNK
#define SDEDGE_QCHUNK 4       // scenarios taken from the work queue per atomic (persistent CTAs)
#endif
#ifndef SDEDGE_CHUNK_SKIP
#define SDEDGE_CHUNK_SKIP 1   // phase A: skip a 16-row chunk whose smallest bound exceeds every lane's threshold
#endif
#ifndef SDEDGE_POOL_SMEM
#define SDEDGE_POOL_SMEM 0    // 1: first-pass envelope pool in shared memory for draft-bound pairs (measured slower: 4.12 vs 4.33 M/s, r2k)
#endif
#ifndef SDEDGE_RS_MAX_K
#define SDEDGE_RS_MAX_K 160   // tiled DP keeps its row store in shared memory up to this K
#endif
#ifndef SDEDGE_TILE_MIN_K
#define SDEDGE_TILE_MIN_K 0   // tiled DP above this K (all K since the push-style phase B)
#endif
// G = DPs per warp: with ALGO_ENVELOPE and small K a warp runs G independent DPs
// (different gamma) side by side in G lane groups of 32/G lanes, so every
// per-row instruction (stage constants, argmin, update) serves G DPs; for
// large K one DP per warp keeps more warps resident (chosen in launch_all).
constexpr int kThreads = kWarps * 32;

// ------------------------------------------------------------ call constants
// Byte offsets of the shared-memory arrays of one CTA (computed on the host by smem_layout, so that
// the kernel forms each array address as base + constant instead of re-deriving the layout)
struct SmemOff {
    unsigned I, Is, ord, key, glb, gord, nq, dq, pI, pI2, jlo, jf, jw, tinf, red, sid, ctl, rows, rec, rbar;
};

struct Consts {
    int K, O_max, gmin, ng;
    int Jd, hd, h2d, Jv, hv, h2v;
    double c1d, c2d, c1v, c2v;           // defaults when coeffs == NULL
    double Bw, sigma2, lambda, dl;
    double isig2;                        // 1 / sigma2
    long long gamma_s, Gp, kvunit;       // Gamma_s, Gamma_p (eq:memory_model), 4 Jd hd
    int bw_policy, batch_policy, static_batch;   // SDEDGE_BW_* / SDEDGE_BATCH_* (paper baselines)
    int flags;                           // SDEDGE_FLAG_*
    int rows_in_smem;                    // DP row state in shared (1) or global (0) memory
    long long pool_cap;                  // envelope segments per warp slot
    long long rows_stride;               // bytes of one warp's global row state
    long long ybuf_stride;               // doubles of one CTA's per-batch-gamma rows, (K+1) x (3 O_max + 1)
    long long prep_stride;               // bytes of one scenario's prep record (two-kernel path)
    SmemOff so;                          // shared layout of this launch's kernel (PHASE 0/2; set per launch)
    int pool_smem;                       // first-pass envelope pool in shared memory (TILE == 2)
    long long pool_cap_smem;             // its capacity in segments
};

struct Inputs {
    const int32_t* I;
    const double* p;
    const double* g;
    const double* alpha;
    const double* coeffs;
};

struct Outputs {
    double* lat;
    int32_t* gamma;
    int32_t* M;
    int32_t* bend;
    int32_t* order;
    double* w;
    int32_t* status;
    unsigned long long* work;   // [5] or null: candidates, candidate x segments, candidate-steps, rows, full evals
    int32_t* trace;             // [n*K] or null: S vector of gamma* (row choices, the step-trace export)
    int32_t* bgam;              // [n*K] or null: gamma of each batch m < M
};

// Work actually evaluated by one lane (reduced per CTA, flushed once at exit).
// Work counters: accumulated in shared memory at the end of
// each DP (warp-reduced), not carried in registers across the gamma loop.
// Slots: candidates, candidate-segments, candidate-steps W, rows, full evaluations.
struct WorkCount {
    unsigned long long* sh;        // this thread's 5 slots in shared memory, or null (not counted)
};

// Each thread adds its own counts to its own shared slots -- no atomics, no shuffles on the
// hot path; the CTA reduces its slots once, at exit, when the caller asked for counters.
__device__ inline void work_flush(const WorkCount& wc, bool active, unsigned cand, unsigned seg, unsigned full,
                                  unsigned long long steps, unsigned rows)
{
    if (!wc.sh || !active) return;
    wc.sh[0] += cand;
    wc.sh[1] += seg;
    wc.sh[2] += steps;
    wc.sh[3] += rows;
    wc.sh[4] += full;
}

struct Work {
    short* S;                      // [grid][ng][K] boundaries j* (1-based), one block per CTA
    unsigned long long* next;      // [3] scenario queue heads (main, big, prep)
    unsigned char* prep;           // [n] prep records of C.prep_stride bytes (two-kernel path)
    unsigned int* ovf_count;       // scenarios handed to the big-pool pass
    long long* ovf_list;           // [n]
    unsigned char* rows;           // global row state (when not in smem)
    unsigned char* pool;           // envelope segment pools, one per warp slot
    double* ybuf;                  // per-batch-gamma DP rows, one block of ybuf_stride doubles per CTA
};

// DP row state of one warp (SoA of pairs, generic pointers: smem or global).
template <typename R> struct Pair;
template <> struct Pair<double> { using T = double2; };
template <> struct Pair<float> { using T = float2; };
template <typename R> using R2 = typename Pair<R>::T;

// One DP row (AoS).  80 B for fp64 (48 B for fp32): with consecutive rows on
// consecutive lanes the 16-byte loads of a warp hit distinct banks, and one
// address computation serves all five loads.
template <typename R>
struct alignas(16) RowRec {                  // 80 B (fp64) / 48 B (fp32): 16-byte multiples for TMA
    R2<R> Y;           // (Upsilon[p,1,0], Upsilon[p,1,1])
    R2<R> A;           // Upsilon[p,n,0] = A.x + A.y (n-1), n >= 2
    R2<R> E;           // (sum_{n=2}^{N} Upsilon[p,n,1], last m of the first envelope segment)
    R2<R> Ln;          // first envelope segment's line (intercept, slope in m = n-1)
    int cnt, off;      // #segments; extra segments in pool[off .. off+cnt-2]
    R key;             // Y.y + E.x = Upsilon[p,0,0] (tiled DP: the pruning bound's predecessor term)
};

template <typename R>
__host__ __device__ inline size_t rows_bytes(int K)
{
    return ((size_t)(K + 1) * sizeof(RowRec<R>) + 15) & ~(size_t)15;
}

template <typename R>
__device__ inline RowRec<R>* carve_rows(unsigned char* base, int K)
{
    return reinterpret_cast<RowRec<R>*>(base);
}

template <typename R>
struct Pool {
    int* u;    // first m of the segment
    R* a;      // intercept
    R* s;      // slope
    long long cap;
};

template <typename R>
__host__ __device__ inline size_t pool_bytes(long long cap)
{
    return (size_t)cap * (sizeof(int) + 2 * sizeof(R));
}

template <typename R>
__device__ inline Pool<R> carve_pool(unsigned char* base, long long cap)
{
    Pool<R> p;
    p.a = reinterpret_cast<R*>(base);
    p.s = p.a + cap;
    p.u = reinterpret_cast<int*>(p.s + cap);
    p.cap = cap;
    return p;
}

// ------------------------------------------------------------ small helpers
constexpr int kWarpsFwd = SDEDGE_WARPS;
// CTA-wide barrier (a warp barrier when the CTA is one warp: orders shared memory too)
__device__ inline void block_sync()
{
    if (kWarpsFwd == 1) __syncwarp();
    else __syncthreads();
}
template <typename R> __device__ inline R rmax(R a, R b) { return a > b ? a : b; }
template <typename R> __device__ inline R kinf();
template <> __device__ inline double kinf<double>() { return __longlong_as_double(0x7ff0000000000000LL); }
template <> __device__ inline float kinf<float>() { return __int_as_float(0x7f800000); }

__device__ inline double dnan() { return __longlong_as_double(0x7ff8000000000000LL); }
__device__ inline double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Warp argmin over (T, j): smallest T, then the LARGEST j (reading A6: the
// ">=" of Alg. 1 line 21).  T >= 0 or +inf, so its IEEE bit pattern orders
// like an unsigned integer: three REDUX instructions instead of a shuffle tree.
__device__ inline int warp_argmin(double t, int j, double* tmin, unsigned mask)
{
    const unsigned long long key = (unsigned long long)__double_as_longlong(t);
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_min_sync(mask, hi);
    const unsigned mlo = __reduce_min_sync(mask, hi == mhi ? lo : 0xffffffffu);
    *tmin = __hiloint2double((int)mhi, (int)mlo);
    return __reduce_max_sync(mask, (hi == mhi && lo == mlo) ? j : -1);
}

__device__ inline int warp_argmin(float t, int j, float* tmin, unsigned mask)
{
    const unsigned key = __float_as_uint(t);
    const unsigned m = __reduce_min_sync(mask, key);
    *tmin = __uint_as_float(m);
    return __reduce_max_sync(mask, key == m ? j : -1);
}

// Argmin within an aligned group of GL lanes by a butterfly of shuffles on the
// (T bits, j) key -- same order and tie rule as warp_argmin.
template <int GL>
__device__ inline int group_argmin(double t, int j, double* tmin)
{
    unsigned long long key = (unsigned long long)__double_as_longlong(t);
#pragma unroll
    for (int o = GL / 2; o > 0; o >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
        const int oj = __shfl_xor_sync(0xffffffffu, j, o);
        if (ok < key || (ok == key && oj > j)) { key = ok; j = oj; }
    }
    *tmin = __longlong_as_double((long long)key);
    return j;
}

template <int GL>
__device__ inline int group_argmin(float t, int j, float* tmin)
{
    unsigned key = __float_as_uint(t);
#pragma unroll
    for (int o = GL / 2; o > 0; o >>= 1) {
        const unsigned ok = __shfl_xor_sync(0xffffffffu, key, o);
        const int oj = __shfl_xor_sync(0xffffffffu, j, o);
        if (ok < key || (ok == key && oj > j)) { key = ok; j = oj; }
    }
    *tmin = __uint_as_float(key);
    return j;
}

// First / last integer m in [u, v] with dP + dQ m > 0, given that the sign
// changes inside [u, v] (exactly once: the function is linear).  A float
// estimate of the crossing is fixed up with exact comparisons.
template <typename R>
__device__ inline int first_pos(R dP, R dQ, int u, int v)
{
    if (fma(dQ, (R)u, dP) > (R)0) return u;
    float x = (float)(-dP) / (float)dQ;
    x = fminf(fmaxf(x, (float)u), (float)v);
    int f = min(max((int)floorf(x) + 1, u + 1), v);
    while (f > u + 1 && fma(dQ, (R)(f - 1), dP) > (R)0) --f;
    while (f < v && fma(dQ, (R)f, dP) <= (R)0) ++f;
    return f;
}

template <typename R>
__device__ inline int last_pos(R dP, R dQ, int u, int v)
{
    if (fma(dQ, (R)v, dP) > (R)0) return v;
    float x = (float)(-dP) / (float)dQ;
    x = fminf(fmaxf(x, (float)u), (float)v);
    int l = min(max((int)ceilf(x) - 1, u), v - 1);
    while (l < v - 1 && fma(dQ, (R)(l + 1), dP) > (R)0) ++l;
    while (l > u && fma(dQ, (R)l, dP) <= (R)0) --l;
    return l;
}

// sum_{m=u}^{v} max(dP + dQ m, 0): the positive part of a linear function on
// an integer range is one sub-range, summed as an arithmetic series.
template <typename R>
__device__ inline R pos_sum(R dP, R dQ, R u, R v)
{
    const R Du = fma(dQ, u, dP), Dv = fma(dQ, v, dP);
    if (Du <= (R)0 && Dv <= (R)0) return (R)0;
    if (Du > (R)0 && Dv > (R)0) return (v - u + (R)1) * (Du + Dv) * (R)0.5;
    const int ui = (int)u, vi = (int)v;
    if (Dv > (R)0) {                         // increasing: positive on [f, v]
        const int f = first_pos(dP, dQ, ui, vi);
        return (R)(vi - f + 1) * (fma(dQ, (R)f, dP) + Dv) * (R)0.5;
    }
    const int l = last_pos(dP, dQ, ui, vi);  // decreasing: positive on [u, l]
    return (R)(l - ui + 1) * (Du + fma(dQ, (R)l, dP)) * (R)0.5;
}

// Segment k >= 1 of row p (pool), as integers.
template <typename R>
struct Seg { int u, v; R a, s; };

template <typename R>
__device__ inline Seg<R> get_seg(const RowRec<R>* rw, const Pool<R>& pl, int p, int k, int c, int Mx)
{
    Seg<R> sg;
    if (k == 0) {
        const R2<R> ln = rw[p].Ln;
        sg.u = 1; sg.v = (int)rw[p].E.y; sg.a = ln.x; sg.s = ln.y;
    } else {
        const long long q = rw[p].off + k - 1;
        sg.u = pl.u[q]; sg.a = pl.a[q]; sg.s = pl.s[q];
        sg.v = (k + 1 < c) ? pl.u[q + 1] - 1 : Mx;
    }
    return sg;
}

// sum_{m=m0}^{m1} max(P + Q m, env_p(m)), one step at a time (eq:t_ij1 as
// written: the O(N) inner loop of Alg. 1 line 15).  Per segment, four steps per
// iteration with four accumulators (independent FP64 chains); the step value
// m is one shared register, the other three lines are pre-shifted by Q and s.
template <typename R>
__device__ inline R dense_sum(const RowRec<R>* rw, const Pool<R>& pl, int p, R P, R Q, int m0, int m1, int Mx)
{
    R acc0 = (R)0, acc1 = (R)0, acc2 = (R)0, acc3 = (R)0;
    if (m0 > m1) return acc0;
    const int cntp = rw[p].cnt;
    for (int k = 0; k < cntp; ++k) {
        const Seg<R> sg = get_seg(rw, pl, p, k, cntp, Mx);
        const int u = max(sg.u, m0), v = min(sg.v, m1);
        if (sg.u > m1) break;
        if (u > v) continue;
        const R P1 = P + Q, P2 = P1 + Q, P3 = P2 + Q;
        const R a1 = sg.a + sg.s, a2 = a1 + sg.s, a3 = a2 + sg.s;
        R x = (R)u;
        int m = u;
        for (; m + 3 <= v; m += 4, x += (R)4) {
            acc0 += rmax(fma(Q, x, P), fma(sg.s, x, sg.a));
            acc1 += rmax(fma(Q, x, P1), fma(sg.s, x, a1));
            acc2 += rmax(fma(Q, x, P2), fma(sg.s, x, a2));
            acc3 += rmax(fma(Q, x, P3), fma(sg.s, x, a3));
        }
        for (; m <= v; ++m, x += (R)1) acc0 += rmax(fma(Q, x, P), fma(sg.s, x, sg.a));
    }
    return (acc0 + acc1) + (acc2 + acc3);
}

// Stage-time coefficients (D1: Appendix-A closed forms of eq:d_latency /
// eq:v_latency summed over the gamma draft passes; everything per unit batch size b).
// Per (scenario, gamma): the I-independent parts.
struct DPConst {
    double kd, kv;        // c1d 4 Jd hd,  c1v 4 Jv hv
    double hd2, hv2;      // 2 hd + h2d,   2 hv + h2v
    double g, tri;        // gamma, gamma (gamma-1) / 2
    double bdc, bvc;      // draft / verify slopes in n:  kd gamma L,  kv (1+gamma) L
    double c2dg, c2vv;    // gamma c2d,  c2v + downlink
    double sumM, Mx;      // sum_{m=1}^{N-1} m,  N - 1
};

// Per sorted row i with padded length I.
struct RowCoef {
    double td1, ad;       // draft: n = 1 value, n >= 2 intercept            (x b, + c2dg)
    double tv1, av;       // verify: n = 1 value, n >= 2 intercept           (x b, + c2vv)
    double tvb, tvc;      // sum_{n>=2} T^v_n = b tvb + tvc  (closed form, hoisted)
    double vsl, vc;       // total verify time sum_{n>=1} T^v_n = b vsl + vc (the pruning bound)
};

__device__ inline RowCoef row_coef(const DPConst& D, int I)
{
    RowCoef r;
    const double Id = I;
    const double hI = D.hd2 + Id;
    if (D.g > 0.0) {
        r.td1 = D.kd * ((Id + D.g - 1.0) * hI + D.tri);      // prefill pass + (gamma-1) decode passes at n = 1
        r.ad = D.kd * (D.g * hI + D.tri);
    } else {
        r.td1 = r.ad = 0.0;                                  // gamma = 0: no draft passes
    }
    const double vI = D.hv2 + Id + D.g;
    r.tv1 = D.kv * (Id + D.g) * vI;
    r.av = D.kv * (1.0 + D.g) * vI;
    r.tvb = fma(D.bvc, D.sumM, r.av * D.Mx);
    r.tvc = D.c2vv * D.Mx;
    r.vsl = r.tv1 + r.tvb;
    r.vc = D.c2vv + r.tvc;
    return r;
}

// Candidate data of (i, j) with batch size b (as a double) for predecessor row p = j - 1.
template <typename R>
struct Cand { R d0, d1, P, Q; };

template <typename R>
__device__ inline Cand<R> cand_terms(const RowRec<R>* rw, const DPConst& D, const RowCoef& rc, int p, double bd)
{
    Cand<R> c;
    const R2<R> y = rw[p].Y, a = rw[p].A;
    c.d0 = y.x + (R)fma(bd, rc.td1, D.c2dg);             // eq:tt1 at n = 1
    c.d1 = rmax(c.d0, y.y) + (R)fma(bd, rc.tv1, D.c2vv);  // eq:tt2 at n = 1 (reading A1)
    c.P = a.x + (R)fma(bd, rc.ad, D.c2dg);               // Upsilon0 line of the candidate, n >= 2
    c.Q = a.y + (R)(bd * D.bdc);
    return c;
}

// Exact IEEE sequence shared with the oracle (reading A2):
// A = alpha^{gamma+1} by repeated multiplication, L = (1-A)/(1-alpha), N = ceil(O/L).
__device__ inline double expected_tokens(double alpha, int gamma)
{
    double A = alpha;
    for (int t = 0; t < gamma; ++t) A = __dmul_rn(A, alpha);
    return __ddiv_rn(__dsub_rn(1.0, A), __dsub_rn(1.0, alpha));
}

// The per-(scenario, gamma) stage-time constants (D1) for N = ceil(O_max / L) steps.
__device__ inline DPConst make_dpconst(const Consts& C, int gamma, double L, int N, double c1d, double c2d,
                                       double c1v, double c2v)
{
    DPConst D;
    const int Mx = N - 1;                                        // n >= 2 <-> m = n-1 in [1, Mx]
    D.g = gamma;
    D.tri = D.g * (D.g - 1.0) * 0.5;                             // sum_{i=1}^{gamma} (i-1)
    D.kd = c1d * (4.0 * C.Jd * (double)C.hd);
    D.kv = c1v * (4.0 * C.Jv * (double)C.hv);
    D.hd2 = 2.0 * C.hd + C.h2d;
    D.hv2 = 2.0 * C.hv + C.h2v;
    D.bdc = D.kd * D.g * L;
    D.bvc = D.kv * (1.0 + D.g) * L;
    D.c2dg = D.g * c2d;
    D.c2vv = c2v + C.dl;
    D.Mx = Mx;
    D.sumM = (double)Mx * (double)(Mx + 1) * 0.5;
    return D;
}

// First feasible batch start j of row i (cons. (b), Alg. 1 lines 10-13): batches of
// b <= bmax = floor(room / d) tasks fit, room = Gamma_s - Gamma_p, d = 4 Jd hd (I + O_max).
// Exact integer floor.  Below 2^52 a single-precision estimate q' of room / d (relative error
// < 2^-21) decides bmax >= i outright when q' >= 2 i + 2; otherwise q < 2^17, so floor(q') is
// within one of bmax and an exact integer fix-up (products < 2^53, no overflow) finishes it.
__device__ __noinline__ long long div_slow(long long a, long long b) { return a / b; }

__device__ inline int window_lo(long long room, long long d, int i)
{
    long long bmax = 0;
    if (room >= 0 && d > 0) {
        if (room < (1LL << 52) && d < (1LL << 52)) {
            const float qf = __fdividef((float)room, (float)d);
            if (qf >= 2.0f * (float)i + 2.0f) return 1;
            bmax = (long long)qf;
            if (bmax * d > room) --bmax;
            if ((bmax + 1) * d <= room) ++bmax;
        } else {
            bmax = div_slow(room, d);
        }
    }
    return bmax >= i ? 1 : (int)(i - bmax + 1);
}

// log2(x) for x >= 1 (x = 1 + p g / sigma^2, eq:opt_w): x = 2^e m, m in [sqrt(1/2), sqrt(2)),
// ln m = 2 atanh(f) = 2 (f + f^3/3 + ... + f^23/23), f = (m - 1) / (m + 1), |f| <= 0.1716 (the
// truncated terms < 2^-58 relative); 1/(m+1) by a single-precision seed and two Newton steps.
// A few ulp from the correctly rounded value (the tolerance on w and T_com is 1e-12 relative).
__device__ inline double log2_ge1(double x)
{
    if (!(x < 1.7976931348623157e308)) return x;               // inf, nan
    const int hi = __double2hiint(x), lo = __double2loint(x);
    int e = (hi >> 20) - 1023;
    int mh = (hi & 0x000fffff) | 0x3ff00000;
    if (mh > 0x3ff6a09e) { mh -= 0x00100000; ++e; }             // m > sqrt(2): m / 2
    const double m = __hiloint2double(mh, lo);
    const double num = m - 1.0, den = m + 1.0;                  // both exact
    double r = (double)__frcp_rn((float)den);
    r = fma(r, fma(-den, r, 1.0), r);
    r = fma(r, fma(-den, r, 1.0), r);
    const double f = num * r, f2 = f * f;
    double q = 1.0 / 23;
    q = fma(q, f2, 1.0 / 21); q = fma(q, f2, 1.0 / 19); q = fma(q, f2, 1.0 / 17);
    q = fma(q, f2, 1.0 / 15); q = fma(q, f2, 1.0 / 13); q = fma(q, f2, 1.0 / 11);
    q = fma(q, f2, 1.0 / 9);  q = fma(q, f2, 1.0 / 7);  q = fma(q, f2, 1.0 / 5);
    q = fma(q, f2, 1.0 / 3);
    const double f2x = 2.0 * f;
    const double lnm = fma(f2x * f2, q, f2x);
    return fma(lnm, 1.4426950408889634, (double)e);            // ln m / ln 2 + e
}

// Warp-register bitonic sort of 32 E 64-bit keys (element e = lane E + r in register r):
// partners at distance st >= E are in lane ^ (st / E) (shuffles), smaller distances in the
// same lane -- no shared-memory traffic and no barriers.
template <int E>
__device__ inline void warp_bitonic(unsigned long long (&x)[E], int lane)
{
    constexpr int P = 32 * E;
#pragma unroll 1
    for (int sz = 2; sz <= P; sz <<= 1) {
#pragma unroll 1
        for (int st = sz >> 1; st > 0; st >>= 1) {
            if (st >= E) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const int e = lane * E + r;
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, x[r], st / E);
                    const bool keep_min = ((e & sz) == 0) == ((e & st) == 0);   // ascending half's lower element
                    x[r] = keep_min ? (o < x[r] ? o : x[r]) : (o > x[r] ? o : x[r]);
                }
            } else {                         // st < E: pairs (r, r + st) inside the lane
#pragma unroll
                for (int sv = 1; sv < E; sv <<= 1) {   // constant register indices
                    if (st != sv) continue;
#pragma unroll
                    for (int r = 0; r < E; ++r) {
                        if (r & sv) continue;
                        const unsigned long long a = x[r], b = x[r | sv];
                        if ((a > b) == (((lane * E + r) & sz) == 0)) { x[r] = b; x[r | sv] = a; }
                    }
                }
            }
        }
    }
}

// 32-bit keys (I << 7 | e, valid when 0 <= I < 2^24 and K <= 128): half the shuffles and compares;
// the network is fully unrolled (28 stages at E = 4: distances, directions and registers are constants)
template <int E>
__device__ inline void warp_bitonic32(unsigned (&x)[E], int lane)
{
    constexpr int P = 32 * E;
#pragma unroll
    for (int sz = 2; sz <= P; sz <<= 1) {
#pragma unroll
        for (int st = sz >> 1; st > 0; st >>= 1) {
            if (st >= E) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const int e = lane * E + r;
                    const unsigned o = __shfl_xor_sync(0xffffffffu, x[r], st / E);
                    const bool keep_min = ((e & sz) == 0) == ((e & st) == 0);
                    x[r] = keep_min ? min(o, x[r]) : max(o, x[r]);
                }
            } else {
#pragma unroll
                for (int sv = 1; sv < E; sv <<= 1) {
                    if (st != sv) continue;
#pragma unroll
                    for (int r = 0; r < E; ++r) {
                        if (r & sv) continue;
                        const unsigned a = x[r], b = x[r | sv];
                        if ((a > b) == (((lane * E + r) & sz) == 0)) { x[r] = b; x[r | sv] = a; }
                    }
                }
            }
        }
    }
}

template <int E>
__device__ inline void warp_sort_tasks(const int* I, int* ord, int* Is, int K, int lane)
{
    static_assert(32 * E <= 128, "the 32-bit keys hold a 7-bit index");
    int mn = 0x7fffffff, mx = -0x7fffffff - 1;
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int e = lane * E + r;
        if (e < K) { mn = min(mn, I[e]); mx = max(mx, I[e]); }
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (mn >= 0 && mx < (1 << 24)) {
        unsigned y[E];
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int e = lane * E + r;
            y[r] = e < K ? ((unsigned)I[e] << 7) | (unsigned)e : 0xffffffffu;
        }
        warp_bitonic32<E>(y, lane);
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int e = lane * E + r;
            if (e < K) {
                const int k = (int)(y[r] & 127u);
                ord[e] = k;
                Is[e] = I[k];
            }
        }
        return;
    }
    unsigned long long x[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int e = lane * E + r;
        x[r] = e < K ? ((unsigned long long)((unsigned)I[e] ^ 0x80000000u) << 32) | (unsigned)e : ~0ULL;
    }
    warp_bitonic<E>(x, lane);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int e = lane * E + r;
        if (e < K) {
            const int k = (int)(unsigned)(x[r] & 0xffffffffULL);
            ord[e] = k;
            Is[e] = I[k];
        }
    }
}

// ------------------------------------------------------------ shared layout
struct Smem {
    int* I;        // [K] original lengths
    int* Is;       // [K] sorted lengths
    int* ord;      // [K] sorted pos -> task
    unsigned long long* key;  // [sort_len(K)] bitonic sort keys (biased I_k << 32 | k)
    double* glb;   // [ng] pre-DP lower bound of T_inf(gamma), in gamma-index order
    int* gord;     // [ng] gamma indices in the order the warps take them (most promising first)
    double* pI;    // [K/kPfx + 2] prefix sums of the sorted I (exact integers) at rows 0, kPfx, 2 kPfx, ..
    double* pI2;   // [K/kPfx + 2] ... of the sorted I^2 (the last entry: the total)
    int* nq;       // [ng] N_gamma (per-batch-gamma policy)
    DPConst* dq;   // [ng] stage-time constants per gamma
    unsigned char* rec;          // DP kernel: two prep-record buffers (current, prefetched next)
    unsigned long long* rbar;    // their mbarriers
    short* jlo;    // [K] first feasible j of row i (memory window), > i if none
    short* jf;     // [K] fixed-plan policies: start j of the batch ending at row i, 0 if none
    short* jw;     // [kWarps][K] heuristic batching: the plan under evaluation
    double* tinf;  // [ng]
    double* red;   // [5 * kWarps] per-warp partials: T_com, sum I/s, sum I, sum I^2, min single-batch T_inf
    int* ctl;      // [0] gamma queue, [2] M, [3] bad flag, [4] gamma* index
    long long* sid;
    unsigned char* rows; // [kWarps] row states when rows_in_smem
};

#ifndef SDEDGE_TILE_CH
#define SDEDGE_TILE_CH 16     // rows per TMA chunk of the tiled DP's phase A
#endif
constexpr int kTileCh = SDEDGE_TILE_CH;
#ifndef SDEDGE_DBG
#define SDEDGE_DBG 0          // 1: event counters of the tiled DP (development builds; sdedge_debug_counters)
#endif
#if SDEDGE_DBG
__device__ unsigned long long g_dbg[16];
#define DBG_ADD(i, v) atomicAdd(&g_dbg[i], (unsigned long long)(v))
#else
#define DBG_ADD(i, v) ((void)0)
#endif

// per tiled DP: tile rows, two TMA staging buffers, two mbarriers, the DP constants
template <typename R, int G>
__host__ __device__ inline size_t tile_bytes()
{
    return (size_t)(32 / G) * sizeof(RowRec<R>) +
           2 * (size_t)kTileCh * sizeof(RowRec<R>) + 2 * sizeof(unsigned long long) + sizeof(DPConst);
}

// rows past K that the shared-memory row store needs so that every tile of GL rows is in bounds
__host__ __device__ inline int rs_pad(int K, int GL)
{
    return (K + GL - 1) / GL * GL - K;
}

// prefix sums of I and I^2 are kept at rows 0, 16, 32, ... (the tile ends, GL in {8, 16, 32})
constexpr int kPfx = 8;
__host__ __device__ inline int pfx_len(int K) { return K / kPfx + 2; }

// bitonic sort length: the next power of two >= K
__host__ __device__ inline int sort_len(int K)
{
    int p = 2;
    while (p < K) p <<= 1;
    return p;
}

// Shared-memory layout of one CTA: offsets of every array and the total size.  rec > 0 is the DP
// kernel of the two-kernel path: it keeps two prep-record buffers of rec bytes (the current
// scenario's and the prefetched next one's, filled by TMA bulk copies) and points Is, jlo, pI, pI2
// and glb into them, so it has no arrays of its own for those (nor for I, ord and the sort keys).
// Arrays a kernel does not have get offset 0xffffffff.
__host__ __device__ inline size_t smem_layout(int K, int ng, int rec, SmemOff* o)
{
    size_t b = 0;
    auto at = [&](size_t bytes, size_t align) -> unsigned {
        b = (b + align - 1) & ~(align - 1);
        const unsigned off = (unsigned)b;
        b += bytes;
        return off;
    };
    const unsigned none = 0xffffffffu;
    SmemOff t;
    if (rec > 0) {
        t.rec = at((size_t)2 * rec, 16);
        t.rbar = at(2 * sizeof(unsigned long long), 8);
        t.I = t.Is = t.ord = t.key = none;
    } else {
        t.I = at((size_t)K * sizeof(int), 16);
        t.Is = at((size_t)K * sizeof(int), 4);
        t.ord = at((size_t)K * sizeof(int), 4);
        t.key = at((size_t)sort_len(K) * sizeof(unsigned long long), 16);
        t.rec = t.rbar = none;
    }
    t.glb = rec > 0 ? none : at((size_t)ng * sizeof(double), 8);
    t.gord = at((size_t)ng * sizeof(int), 4);
    t.nq = at((size_t)ng * sizeof(int), 4);
    t.dq = at((size_t)ng * sizeof(DPConst), 16);
    t.pI = rec > 0 ? none : at((size_t)pfx_len(K) * sizeof(double), 8);
    t.pI2 = rec > 0 ? none : at((size_t)pfx_len(K) * sizeof(double), 8);
    t.jlo = rec > 0 ? none : at((size_t)K * sizeof(short), 2);
    t.jf = at((size_t)K * sizeof(short), 2);
    t.jw = at((size_t)kWarps * K * sizeof(short), 2);
    t.tinf = at((size_t)ng * sizeof(double), 16);
    t.red = at(5 * kWarps * sizeof(double), 8);
    t.sid = at(2 * sizeof(long long), 8);
    t.ctl = at(8 * sizeof(int), 4);
    t.rows = at(0, 16);
    if (o) *o = t;
    return (b + 15) & ~(size_t)15;
}

template <typename R, int G>
__host__ __device__ inline size_t smem_bytes(int K, int ng, int rows_in_smem, int tile, int row_pad = 0, int rec = 0)
{
    size_t b = smem_layout(K, ng, rec, nullptr);
    if (rows_in_smem) b += (size_t)kWarps * G * rows_bytes<R>(K + row_pad);
    if (tile) b += (size_t)kWarps * G * tile_bytes<R, G>();
    return b;
}

__device__ inline Smem carve_smem(unsigned char* base, const SmemOff& o)
{
    auto p = [&](unsigned off) -> unsigned char* { return base + off; };   // (absent arrays are never used)
    Smem s;
    s.I = reinterpret_cast<int*>(p(o.I));
    s.Is = reinterpret_cast<int*>(p(o.Is));
    s.ord = reinterpret_cast<int*>(p(o.ord));
    s.key = reinterpret_cast<unsigned long long*>(p(o.key));
    s.glb = reinterpret_cast<double*>(p(o.glb));
    s.gord = reinterpret_cast<int*>(p(o.gord));
    s.nq = reinterpret_cast<int*>(p(o.nq));
    s.dq = reinterpret_cast<DPConst*>(p(o.dq));
    s.pI = reinterpret_cast<double*>(p(o.pI));
    s.pI2 = reinterpret_cast<double*>(p(o.pI2));
    s.jlo = reinterpret_cast<short*>(p(o.jlo));
    s.jf = reinterpret_cast<short*>(p(o.jf));
    s.jw = reinterpret_cast<short*>(p(o.jw));
    s.tinf = reinterpret_cast<double*>(p(o.tinf));
    s.red = reinterpret_cast<double*>(p(o.red));
    s.sid = reinterpret_cast<long long*>(p(o.sid));
    s.ctl = reinterpret_cast<int*>(p(o.ctl));
    s.rows = p(o.rows);
    s.rec = p(o.rec);
    s.rbar = reinterpret_cast<unsigned long long*>(p(o.rbar));
    return s;
}

// ------------------------------------------------------------ prep records (two-kernel hot path)
// The tiled hot path runs as two kernels: PHASE 1 (prep: staging, sort, windows, bandwidth, w*,
// prefix sums, per-gamma bounds; writes order, w*, T_com and every output of an invalid
// scenario) and PHASE 2 (the DPs and the backtrack).  Each kernel's code is small enough for the
// instruction caches, and every warp of an SM runs the same phase.  Per scenario the prep record
// carries what PHASE 2 needs:
struct PrepView {
    int* Is;       // [K] sorted lengths
    short* jlo;    // [K] first feasible j per row
    double* pI;    // [pfx_len(K)] prefix sums of I (at every kPfx-th row, then the total)
    double* pI2;   // [pfx_len(K)] ... of I^2
    double* glb;   // [ng] lower bound of T_inf(gamma)
    double* L;     // [ng] expected tokens per step (eq:ol)
    int* N;        // [ng] decoding steps (eq:step_n)
    double* misc;  // [2] seed of the best T_inf (min single-batch latency), T_com
    int* flags;    // [1] bit 0 bad task, bit 1 bad alpha, bit 2 monotone coefficients
};

__host__ __device__ inline size_t prep_stride(int K, int ng)
{
    size_t b = 0;
    b += ((size_t)K * 4 + 7) & ~(size_t)7;
    b += ((size_t)K * 2 + 7) & ~(size_t)7;
    b += 2 * (size_t)pfx_len(K) * 8;
    b += (size_t)ng * 16;
    b += ((size_t)ng * 4 + 7) & ~(size_t)7;
    b += 16 + 8;
    return (b + 15) & ~(size_t)15;
}

__device__ inline PrepView prep_view(unsigned char* base, int K, int ng)
{
    PrepView v;
    size_t b = 0;
    v.Is = reinterpret_cast<int*>(base + b); b += ((size_t)K * 4 + 7) & ~(size_t)7;
    v.jlo = reinterpret_cast<short*>(base + b); b += ((size_t)K * 2 + 7) & ~(size_t)7;
    v.pI = reinterpret_cast<double*>(base + b); b += (size_t)pfx_len(K) * 8;
    v.pI2 = reinterpret_cast<double*>(base + b); b += (size_t)pfx_len(K) * 8;
    v.glb = reinterpret_cast<double*>(base + b); b += (size_t)ng * 8;
    v.L = reinterpret_cast<double*>(base + b); b += (size_t)ng * 8;
    v.N = reinterpret_cast<int*>(base + b); b += ((size_t)ng * 4 + 7) & ~(size_t)7;
    v.misc = reinterpret_cast<double*>(base + b); b += 16;
    v.flags = reinterpret_cast<int*>(base + b);
    return v;
}

// ------------------------------------------------------------ envelope update
// Row i's Upsilon1 for n >= 2 (eq:tt2):  env_i(m) = max(P + Q m, env_p(m)) + Av + Bv m.
// The set where the new line beats the convex env_p is one interval [mlo, mhi].
// Executed by the single lane that owns j*; returns true on pool overflow.
template <typename R>
__device__ bool env_update(RowRec<R>* rw, const Pool<R>& pl, int p, int i, R P, R Q, R Av, R Bv,
                           int Mx, long long& top)
{
    const int cntp = rw[p].cnt;
    const long long base = top;
    rw[i].off = (int)base;
    if (cntp == 0) { rw[i].cnt = 0; return false; }            // N = 1: no n >= 2 steps
    if (cntp == 1) {                                           // fast path: one old line on [1, Mx]
        const R2<R> ln = rw[p].Ln;
        const R ea = ln.x, es = ln.y;
        const R dP = P - ea, dQ = Q - es;
        const R Du = dP + dQ, Dv = fma(dQ, (R)Mx, dP);
        if (!(Du > (R)0) && !(Dv > (R)0)) {                    // old line everywhere
            rw[i].Ln = R2<R>{ea + Av, es + Bv}; rw[i].E.y = (R)Mx; rw[i].cnt = 1;
            return false;
        }
        if (Du > (R)0 && Dv > (R)0) {                          // new line everywhere
            rw[i].Ln = R2<R>{P + Av, Q + Bv}; rw[i].E.y = (R)Mx; rw[i].cnt = 1;
            return false;
        }
        if (base >= pl.cap) return true;
        if (Dv > (R)0) {                                       // old on [1, f-1], new on [f, Mx]
            const int f = first_pos(dP, dQ, 1, Mx);
            rw[i].Ln = R2<R>{ea + Av, es + Bv}; rw[i].E.y = (R)(f - 1);
            pl.u[base] = f; pl.a[base] = P + Av; pl.s[base] = Q + Bv;
        } else {                                               // new on [1, l], old on [l+1, Mx]
            const int l = last_pos(dP, dQ, 1, Mx);
            rw[i].Ln = R2<R>{P + Av, Q + Bv}; rw[i].E.y = (R)l;
            pl.u[base] = l + 1; pl.a[base] = ea + Av; pl.s[base] = es + Bv;
        }
        rw[i].cnt = 2;
        top = base + 1;
        return false;
    }
    int mlo = 0, mhi = -1;
    for (int k = 0; k < cntp && mlo == 0; ++k) {
        const Seg<R> sg = get_seg(rw, pl, p, k, cntp, Mx);
        const R dP = P - sg.a, dQ = Q - sg.s;
        if (fma(dQ, (R)sg.u, dP) > (R)0 || fma(dQ, (R)sg.v, dP) > (R)0) mlo = first_pos(dP, dQ, sg.u, sg.v);
    }
    if (mlo > 0)
        for (int k = cntp - 1; k >= 0; --k) {
            const Seg<R> sg = get_seg(rw, pl, p, k, cntp, Mx);
            const R dP = P - sg.a, dQ = Q - sg.s;
            if (fma(dQ, (R)sg.u, dP) > (R)0 || fma(dQ, (R)sg.v, dP) > (R)0) {
                mhi = last_pos(dP, dQ, sg.u, sg.v);
                break;
            }
        }
    int nseg = 0;
    bool ovf = false;
    rw[i].E.y = (R)Mx;
    auto emit = [&](int u, R a, R s) {
        a += Av;
        s += Bv;
        if (nseg == 0) { rw[i].Ln = R2<R>{a, s}; }
        else {
            if (nseg == 1) rw[i].E.y = (R)(u - 1);
            const long long q = base + nseg - 1;
            if (q >= pl.cap) ovf = true;
            else { pl.u[q] = u; pl.a[q] = a; pl.s[q] = s; }
        }
        ++nseg;
    };
    bool line_done = false;
    for (int k = 0; k < cntp; ++k) {
        const Seg<R> sg = get_seg(rw, pl, p, k, cntp, Mx);
        if (mlo > 0 && sg.v >= mlo && sg.u <= mhi) {
            if (sg.u < mlo) emit(sg.u, sg.a, sg.s);            // left remainder
            if (!line_done) { emit(mlo, P, Q); line_done = true; }
            if (sg.v > mhi) emit(mhi + 1, sg.a, sg.s);         // right remainder
        } else {
            emit(sg.u, sg.a, sg.s);
        }
    }
    rw[i].cnt = nseg;
    top = base + (nseg > 1 ? nseg - 1 : 0);
    return ovf;
}

// sum over the integer sub-range of [u, v] where dP + dQ m > 0, when the sign
// changes inside [u, v] (Du = value at u, Dv = value at v).  Rare path.
template <typename R>
__device__ __noinline__ R crossing_sum(R dP, R dQ, int u, int v, R Du, R Dv)
{
    if (Dv > (R)0) {                         // increasing: positive on [f, v]
        const int f = first_pos(dP, dQ, u, v);
        return (R)(v - f + 1) * (fma(dQ, (R)f, dP) + Dv) * (R)0.5;
    }
    const int l = last_pos(dP, dQ, u, v);    // decreasing: positive on [u, l]
    return (R)(l - u + 1) * (Du + fma(dQ, (R)l, dP)) * (R)0.5;
}

// Segments k >= 1 of a multi-segment envelope (rare path).
template <typename R>
__device__ __noinline__ R extra_segments(const RowRec<R>* rw, const Pool<R>& pl, int p, int cntp, R P, R Q, int Mx)
{
    R pos = (R)0;
    for (int k = 1; k < cntp; ++k) {
        const Seg<R> sg = get_seg(rw, pl, p, k, cntp, Mx);
        pos += pos_sum(P - sg.a, Q - sg.s, (R)sg.u, (R)sg.v);
    }
    return pos;
}

// T_{i,j} of one candidate by the envelope closed form (ALGO_ENVELOPE), for
// N >= 2 (the envelope is non-empty).  Branch-light: the first segment's
// positive part is a select, crossings and further segments are rare calls.
template <typename R>
__device__ inline R env_cand(const RowRec<R>* rw, const Pool<R>& pl, const DPConst& D, const RowCoef& rc, int p,
                             double bd, int Mx, R& rest, int& nseg)
{
    const RowRec<R>* q = rw + p;
    const R2<R> y = q->Y, a = q->A, e = q->E, ln = q->Ln;
    const int cntp = q->cnt;
    const R Td1 = (R)fma(bd, rc.td1, D.c2dg), Tv1 = (R)fma(bd, rc.tv1, D.c2vv);
    const R P = a.x + (R)fma(bd, rc.ad, D.c2dg), Q = a.y + (R)(bd * D.bdc);
    const R base = e.x + (R)fma(bd, rc.tvb, rc.tvc);     // sum_{n>=2} (Upsilon1[p,n] + T^v_n)
    const R d1 = rmax(y.x + Td1, y.y) + Tv1;             // eq:t_ij1 at n = 1
    // first segment [1, e.y] with line ln: sum of max(P + Q m - ln(m), 0)
    const R dP = P - ln.x, dQ = Q - ln.y;
    const R Du = dP + dQ, Dv = fma(dQ, e.y, dP);
    const bool pu = Du > (R)0, pv = Dv > (R)0;
    R pos = (pu && pv) ? (Du + Dv) * e.y * (R)0.5 : (R)0;
    if (pu != pv && cntp > 0) pos = crossing_sum(dP, dQ, 1, (int)e.y, Du, Dv);
    if (cntp > 1) pos += extra_segments(rw, pl, p, cntp, P, Q, Mx);
    nseg = cntp;
    rest = base + pos;
    return d1 + rest;
}

// ------------------------------------------------------------ the DP of one gamma
// Returns T_inf (= Upsilon[K,0,0]) or +inf if some row has no feasible batch;
// sets *overflow if the segment pool ran out.  S[i-1] = j* (1-based).
template <typename R, int ALGO, int G>
__device__ double dp_gamma(const Consts& C, const Smem& sm, RowRec<R>* rw, Pool<R> pl, int gamma,
                           double alpha, double c1d, double c2d, double c1v, double c2v,
                           short* S, bool* overflow, WorkCount& wc, long long* top_s, bool active,
                           const short* jf)
{
    constexpr int GL = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane % GL;                                    // lane within the DP's group
    const unsigned gmask = G == 1 ? 0xffffffffu : (((1u << GL) - 1u) << (lane - gl));
    const int K = C.K;
    const double L = expected_tokens(alpha, gamma);
    const int N = (int)ceil(__ddiv_rn((double)C.O_max, L));   // eq:step_n
    const int Mx = N - 1;                                        // n >= 2 <-> m = n-1 in [1, Mx]
    const DPConst D = make_dpconst(C, gamma, L, N, c1d, c2d, c1v, c2v);
    unsigned n_cand = 0, n_seg = 0;

    if (gl == 0) {                                               // row 0 == 0 (reading A3)
        rw[0].Y = R2<R>{(R)0, (R)0};
        rw[0].A = R2<R>{(R)0, (R)0};
        rw[0].E = R2<R>{(R)0, (R)Mx};
        rw[0].Ln = R2<R>{(R)0, (R)0};
        rw[0].off = 0;
        rw[0].cnt = Mx >= 1 ? 1 : 0;
        *top_s = 0;                                              // pool bump pointer (owner lanes only)
    }
    __syncwarp();

    double T_last = 0.0;
    int rows_done = 0;
    bool ovf_any = false;
    const bool nopipe = C.batch_policy == SDEDGE_BATCH_NO_PIPELINE;
    for (int i = 1; i <= K; ++i) {
        int jlo = sm.jlo[i - 1];             // memory window (Alg. 1 lines 10-13)
        int jhi = i;
        if (jf) {                            // fixed plan: only the batch ending at i (if any)
            const int jfi = jf[i - 1];
            if (jfi == 0) {                  // not a batch end: no choice at this row (trace 0)
                if (S && gl == 0) S[i - 1] = 0;
                continue;
            }
            if (jfi < jlo) { T_last = dinf(); break; }
            jlo = jhi = jfi;
        }
        if (jlo > jhi) { T_last = dinf(); break; }
        const RowCoef rc = row_coef(D, sm.Is[i - 1]);
        if (nopipe) {
            // "SD w/o pipeline": T_n = sum_m (T^d + T^v), so T_{i,j} =
            // Upsilon[j-1,0,0] + sum_n (T^d_n + T^v_n)(b, I_i), closed form in b.
            const double slope = rc.td1 + rc.tv1 + D.Mx * (rc.ad + rc.av) + D.sumM * (D.bdc + D.bvc);
            const double fixed = (D.c2dg + D.c2vv) * (D.Mx + 1.0);
            R bT = kinf<R>();
            int bj = -1;
            double bd = (double)(i - jlo - gl + 1);
            for (int j = jlo + gl; j <= jhi; j += GL, bd -= GL) {
                const R T = rw[j - 1].E.x + (R)fma(bd, slope, fixed);
                n_cand += 1;
                if (T <= bT) { bT = T; bj = j; }
            }
            R tmin;
            const int jj = warp_argmin(bT, bj, &tmin, gmask);
            if (jj < 0) { T_last = dinf(); break; }
            if (bj == jj) {
                if (S) S[i - 1] = (short)jj;
                rw[i].E = R2<R>{tmin, (R)0};
            }
            __syncwarp(gmask);
            ++rows_done;
            T_last = (double)tmin;
            continue;
        }

        R bT = kinf<R>();
        int bj = -1;
        R brest = (R)0;
        const int nc = jhi - jlo + 1;
        if (ALGO == SDEDGE_ALGO_ENVELOPE) {
            // one lane per candidate, two candidates (j, j+GL) in flight per lane;
            // ascending j per lane, so '<=' keeps the largest j
            double bd = (double)(i - jlo - gl + 1);
            for (int j = jlo + gl; j <= jhi; j += 2 * GL, bd -= 2.0 * GL) {
                const bool two = j + GL <= jhi;
                R r0, r1;
                int c0, c1;
                const R T0 = env_cand(rw, pl, D, rc, j - 1, bd, Mx, r0, c0);
                R T1 = env_cand(rw, pl, D, rc, two ? j + GL - 1 : j - 1, two ? bd - GL : bd, Mx, r1, c1);
                if (!two) { T1 = kinf<R>(); c1 = 0; }
                n_cand += 1 + two;
                n_seg += (unsigned)(c0 + c1);
                if (T0 <= bT) { bT = T0; bj = j; brest = r0; }   // '>=' of Alg. 1 line 21
                if (T1 <= bT) { bT = T1; bj = j + GL; brest = r1; }
            }
        } else if (nc >= 17) {
            // DENSE: one lane per candidate, ascending j per lane
            double bd = (double)(i - jlo - lane + 1);
            for (int j = jlo + lane; j <= jhi; j += 32, bd -= 32.0) {
                const int p = j - 1;
                const Cand<R> c = cand_terms(rw, D, rc, p, bd);
                const R acc = dense_sum(rw, pl, p, c.P, c.Q, 1, Mx, Mx);
                n_cand += 1;
                n_seg += (unsigned)rw[p].cnt;
                const R rest = acc + (R)fma(bd, rc.tvb, rc.tvc);   // + sum_{n>=2} T^v_n
                const R T = c.d1 + rest;
                if (T <= bT) { bT = T; bj = j; brest = rest; }   // '>=' of Alg. 1 line 21
            }
        } else {
            // DENSE with few candidates: gsz lanes share one candidate's n-range
            int gsz = 1;
            while (gsz * 2 * nc <= 32) gsz *= 2;
            const int ci = lane / gsz, sub = lane % gsz;
            R rest = (R)0;
            int j = -1;
            Cand<R> c;
            const double bd = (double)(i - jlo - ci + 1);
            if (ci < nc) {
                j = jlo + ci;
                const int p = j - 1;
                c = cand_terms(rw, D, rc, p, bd);
                const int chunk = (Mx + gsz - 1) / gsz;
                const int m0 = 1 + sub * chunk, m1 = min(Mx, m0 + chunk - 1);
                rest = dense_sum(rw, pl, p, c.P, c.Q, m0, m1, Mx);
            }
            for (int o = gsz >> 1; o > 0; o >>= 1) rest += __shfl_xor_sync(0xffffffffu, rest, o);
            if (ci < nc && sub == 0) {
                n_cand += 1;
                n_seg += (unsigned)rw[j - 1].cnt;
                rest = rest + (R)fma(bd, rc.tvb, rc.tvc);
                bT = c.d1 + rest;
                bj = j;
                brest = rest;
            }
        }
        R tmin;
#if SDEDGE_TILE_SHFL_ARGMIN
        const int jj = G > 1 ? group_argmin<GL>(bT, bj, &tmin) : warp_argmin(bT, bj, &tmin, gmask);
#else
        const int jj = warp_argmin(bT, bj, &tmin, gmask);
#endif
        // Every lane prepares row i as if its own best candidate won (SIMD, so this
        // overlaps the REDUX latency instead of serialising behind it); the owner of
        // j* then only stores.  eq:rg, eq:tt1, eq:tt2 (reading A4: S[i] always set).
        const int pb = bj > 0 ? bj - 1 : 0;
        const double bdb = (double)(i - pb);
        const Cand<R> cb = cand_terms(rw, D, rc, pb, bdb);
        const R Avb = (R)fma(bdb, rc.av, D.c2vv), Bvb = (R)(bdb * D.bvc);
        const int cntb = rw[pb].cnt;
        const R2<R> lnb = rw[pb].Ln;
        const R dPb = cb.P - lnb.x, dQb = cb.Q - lnb.y;
        const bool pub = dPb + dQb > (R)0, pvb = fma(dQb, (R)Mx, dPb) > (R)0;
        if (jj < 0) { T_last = dinf(); break; }                // no finite candidate
        if (bj == jj) {                                        // the owner (exactly one lane per group)
            if (S) S[i - 1] = (short)jj;
            RowRec<R>* o = rw + i;
            o->Y = R2<R>{cb.d0, cb.d1};
            o->A = R2<R>{cb.P, cb.Q};
            if (cntb == 1 && pub == pvb) {
                // one old line and the new line does not cross it inside [1, Mx]
                o->Ln = pub ? R2<R>{cb.P + Avb, cb.Q + Bvb} : R2<R>{lnb.x + Avb, lnb.y + Bvb};
                o->E = R2<R>{brest, (R)Mx};
                o->cnt = 1;
                o->off = 0;
            } else {
                long long top = *top_s;
                o->E.x = brest;
                if (env_update(rw, pl, pb, i, cb.P, cb.Q, Avb, Bvb, Mx, top)) {
                    ovf_any = true;
                    o->cnt = min(o->cnt, 1);                   // keep later reads in bounds
                }
                *top_s = top;
            }
        }
        __syncwarp(gmask);
        ++rows_done;
        T_last = (double)tmin;
    }
    if (__ballot_sync(0xffffffffu, ovf_any) & gmask) { *overflow = true; T_last = dinf(); }
    work_flush(wc, active, n_cand, n_seg, n_cand, (unsigned long long)n_cand * (unsigned long long)N,
               gl == 0 ? (unsigned)rows_done : 0u);
    return T_last;
}

// ------------------------------------------------------------ per-batch gamma
// An EXTENSION (the paper fixes one l: P:555): Algorithm 1 over candidates (j, gamma),
// each batch with its own L, N_gamma; at step n only the batches with N_gamma >= n run
// (eq:latency_infer_batch's active set), so a finished batch passes the state through:
// max{Upsilon0 + 0, Upsilon1} + 0 = Upsilon1.  Dense, one warp, fp64: the Upsilon rows (n = 1..Nmax,
// Nmax = max N_gamma) live in a global workspace (row p: Y0[Nmax] then Y1[Nmax]); lanes take steps n,
// every (j, gamma) candidate is a lane sum + butterfly.  Ties: largest j, then smallest gamma (NB1).
#ifndef SDEDGE_PBG_WS_GIB
#define SDEDGE_PBG_WS_GIB 8   // per-batch-gamma row workspace of all CTAs (bounds the grid; one CTA's rows <= 2 GiB)
#endif
constexpr long long kPbgWorkspace = (long long)SDEDGE_PBG_WS_GIB << 30;

// Per-(row, gamma) stage constants of the per-batch-gamma DP (hoisted out of the candidate loop)
struct PbgCoef {
    double td1, tv1, ad, av, bdc, bvc;   // n = 1 values, n >= 2 intercepts (per unit b, + c2dg / c2vv), slopes in n
    double c2dg, c2vv;
    int N;
};

// Row p of the per-batch-gamma DP in the CTA's workspace: Upsilon0[n], Upsilon1[n] (n = 1..Nmax) and the
// suffix sums U[k] = sum_{n > k} Upsilon1[n] (k = 0..Nmax): a batch with n_m = N_q < Nmax contributes no
// stage time after step N_q, so its candidate's steps n > N_q add Upsilon1 of the predecessor unchanged
// (reading NB1) -- one lookup instead of Nmax - N_q terms.
__device__ inline void pbg_suffix(double* y1, double* U, int Nmax)
{
    const int lane = threadIdx.x & 31;
    double carry = 0.0;
    if (lane == 0) U[Nmax] = 0.0;
    for (int b0 = ((Nmax - 1) / 32) * 32; b0 >= 0; b0 -= 32) {
        const int k = b0 + lane;
        double v = k < Nmax ? y1[k] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {              // inclusive suffix scan within the block
            const double t = __shfl_down_sync(0xffffffffu, v, o);
            if (lane + o < 32) v += t;
        }
        if (k < Nmax) U[k] = v + carry;
        carry += __shfl_sync(0xffffffffu, v, 0);
    }
    __syncwarp();
}

__device__ double dp_pbg(const Consts& C, const Smem& sm, double* Y, int Nmax, short* S, short* Gm, WorkCount& wc)
{
    const int lane = threadIdx.x & 31, K = C.K, ng = C.ng;
    const size_t rs = 3 * (size_t)Nmax + 1;
    __shared__ PbgCoef s_pc[32];
    for (int n = lane; n < Nmax; n += 32) { Y[n] = 0.0; Y[Nmax + n] = 0.0; }   // row 0 == 0 (reading A3)
    for (int n = lane; n <= Nmax; n += 32) Y[2 * Nmax + n] = 0.0;
    __syncwarp();
    unsigned n_cand = 0, rows = 0;
    unsigned long long n_steps = 0;
    double T_last = 0.0;
    for (int i = 1; i <= K; ++i) {
        const int jlo = sm.jlo[i - 1];
        if (jlo > i) { T_last = dinf(); break; }
        const int I = sm.Is[i - 1];
        for (int q = lane; q < ng; q += 32) {          // this row's constants, one gamma per lane
            const DPConst& D = sm.dq[q];
            const RowCoef rc = row_coef(D, I);
            s_pc[q] = PbgCoef{rc.td1, rc.tv1, rc.ad, rc.av, D.bdc, D.bvc, D.c2dg, D.c2vv, sm.nq[q]};
        }
        __syncwarp();
        double best = dinf();
        int bj = -1, bq = -1;
        for (int j = jlo; j <= i; ++j) {
            const double b = (double)(i - j + 1);
            const double* y0p = Y + (size_t)(j - 1) * rs;
            const double* y1p = y0p + Nmax;
            const double* up = y0p + 2 * Nmax;
            for (int q = 0; q < ng; ++q) {
                const PbgCoef& pc = s_pc[q];
                const int Nq = pc.N;
                const double td1 = fma(b, pc.td1, pc.c2dg), tv1 = fma(b, pc.tv1, pc.c2vv);
                const double ad = fma(b, pc.ad, pc.c2dg), av = fma(b, pc.av, pc.c2vv);
                const double sd = b * pc.bdc, sv = b * pc.bvc;
                double acc = 0.0;
                for (int n = 1 + lane; n <= Nq; n += 32) {
                    const double x = (double)(n - 1);
                    const double td = n == 1 ? td1 : fma(sd, x, ad), tv = n == 1 ? tv1 : fma(sv, x, av);
                    acc += rmax(y0p[n - 1] + td, y1p[n - 1]) + tv;      // eq:t_ij1 (reading A1)
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                acc += up[Nq];                                           // steps after the batch finished
                if (acc < best || (acc == best && j > bj)) { best = acc; bj = j; bq = q; }   // NB1
            }
            n_cand += (unsigned)ng;
            n_steps += (unsigned long long)ng * (unsigned long long)Nmax;
        }
        if (bj < 0) { T_last = dinf(); break; }
        {   // eq:tt1 / eq:tt2 with (j*, gamma*)
            const PbgCoef& pc = s_pc[bq];
            const int Nq = pc.N;
            const double b = (double)(i - bj + 1);
            const double td1 = fma(b, pc.td1, pc.c2dg), tv1 = fma(b, pc.tv1, pc.c2vv);
            const double ad = fma(b, pc.ad, pc.c2dg), av = fma(b, pc.av, pc.c2vv);
            const double sd = b * pc.bdc, sv = b * pc.bvc;
            const double* y0p = Y + (size_t)(bj - 1) * rs;
            double* o0 = Y + (size_t)i * rs;
            for (int n = 1 + lane; n <= Nmax; n += 32) {
                double y0 = y0p[n - 1], y1 = y0p[Nmax + n - 1];
                if (n <= Nq) {
                    const double x = (double)(n - 1);
                    y0 += n == 1 ? td1 : fma(sd, x, ad);
                    y1 = rmax(y0, y1) + (n == 1 ? tv1 : fma(sv, x, av));
                }
                o0[n - 1] = y0;
                o0[Nmax + n - 1] = y1;
            }
            __syncwarp();
            pbg_suffix(o0 + Nmax, o0 + 2 * Nmax, Nmax);
        }
        if (lane == 0) {
            S[i - 1] = (short)bj;
            Gm[i - 1] = (short)(C.gmin + bq);
        }
        __syncwarp();
        ++rows;
        T_last = best;
    }
    work_flush(wc, true, n_cand, 0u, n_cand, n_steps, lane == 0 ? rows : 0u);
    return T_last;
}

// Lower bound of T_inf(gamma) from the verify stage's serial work with the batch count, plus the first
// batch's draft work: in every step the verify stage cannot start before the first batch's
// draft is done, so T_n >= T^d_{n,1} + sum_m T^v_{n,m}; summed over n the verify part is sum_m (b_m vsl(I_m)
// + vc).  Hence T_inf >= min over the batch count M of: M = 1, K vsl(I_K) + vc + K dsl(I_K) + dc (the exact
// single-batch latency); M = 2, the best memory-feasible split s (batches padded to their last task) with
// s vsl(I_s) + (K-s) vsl(I_K) + 2 vc + s dsl(I_s) + dc; M >= 3, sum_k vsl(I_k) + 3 vc + dsl(I_1) + dc.
// vsl, dsl are quadratics in I per unit batch size (Appendix A); dc = gamma c2d N.  Warp-collective (lanes
// take split points); evaluated only for a gamma that survived the O(1) bounds, right before its DP.
__device__ double lb_batches(const Smem& sm, const DPConst& D, int K)
{
    const int lane = threadIdx.x & 31;
    const double c = D.hv2 + D.g;
    const double qb = D.kv * (2.0 * D.g + D.hv2) + D.Mx * D.kv * (1.0 + D.g);
    const double qc = D.kv * D.g * c + D.Mx * D.kv * (1.0 + D.g) * c + D.bvc * D.sumM;
    const double vc = D.c2vv * (D.Mx + 1.0);
    // draft slope per unit batch: td1 + Mx ad + sumM bdc (row_coef), 0 at gamma = 0
    const bool gd = D.g > 0.0;
    const double da = gd ? D.kd : 0.0;
    const double db = gd ? D.kd * (D.g - 1.0 + D.hd2 + D.Mx * D.g) : 0.0;
    const double dcq = gd ? D.kd * ((D.g - 1.0) * D.hd2 + D.tri + D.Mx * (D.g * D.hd2 + D.tri)) + D.sumM * D.bdc : 0.0;
    const double dc = D.c2dg * (D.Mx + 1.0);
    const int pt = K / kPfx + 1;
    const double S1 = sm.pI[pt], S2 = sm.pI2[pt], Kd = (double)K;
    const double own = D.kv * S2 + qb * S1 + Kd * qc;                 // sum_k vsl(I_k)
    const double I1 = (double)sm.Is[0], IK = (double)sm.Is[K - 1];
    const double vK = fma(fma(D.kv, IK, qb), IK, qc);
    const double dK = fma(fma(da, IK, db), IK, dcq);
    double lb = own + 3.0 * vc + fma(fma(da, I1, db), I1, dcq) + dc;  // M >= 3
    const double l1 = Kd * (vK + dK) + vc + dc;                       // M = 1
    if (sm.jlo[K - 1] == 1 && l1 < lb) lb = l1;
    const int jK = sm.jlo[K - 1];                                     // batch sp+1..K fits iff jK <= sp+1
    // M = 2, split after row sp: four independent split points per lane per iteration (ILP)
    const double inf = dinf();
    double b2[4] = {inf, inf, inf, inf};
    for (int sp0 = max(jK - 1, 1) + lane; sp0 < K; sp0 += 128) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int sp = sp0 + 32 * u;
            if (sp < K && sm.jlo[sp - 1] == 1) {                      // batch 1..sp must fit
                const double Isp = (double)sm.Is[sp - 1];
                const double v1 = fma(fma(D.kv, Isp, qb), Isp, qc) + fma(fma(da, Isp, db), Isp, dcq);
                const double v = fma((double)sp, v1, (double)(K - sp) * vK);
                b2[u] = v < b2[u] ? v : b2[u];
            }
        }
    }
    double m2 = b2[0] < b2[1] ? b2[0] : b2[1];
    const double m3 = b2[2] < b2[3] ? b2[2] : b2[3];
    m2 = m3 < m2 ? m3 : m2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, m2, o);
        m2 = ov < m2 ? ov : m2;
    }
    const double lb2 = m2 + 2.0 * vc + dc;
    return lb2 < lb ? lb2 : lb;
}

// ------------------------------------------------------------ TMA bulk copies (sm_90+/sm_100a)
__device__ inline unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ inline void mbar_init(unsigned long long* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ inline void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// one-shot: arrive with an expected transaction count, then a 1-D bulk copy
// global -> shared that completes the transaction on the same mbarrier
__device__ inline void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar)
{
    // the buffer was last read through the generic proxy (ordered by __syncwarp)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// The same chunk of rows for all G DPs of the warp, issued by one lane: DP g's
// staging buffer b is at st0 + g tstride + b kTileCh sizeof(RowRec), its
// mbarriers right after the two buffers, its row store at rw0 + g rwstride.  All
// operands are warp-uniform, so the copies need no per-lane serialisation.
template <typename R, int G>
__device__ inline void bulk_load_groups(unsigned st0, unsigned tstride, const unsigned char* rw0, long long rwstride,
                                        int a, unsigned bytes, int b)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const unsigned st = st0 + (unsigned)g * tstride;
        const unsigned bar = st + 2u * kTileCh * (unsigned)sizeof(RowRec<R>) + 8u * (unsigned)b;
        const unsigned dst = st + (unsigned)b * kTileCh * (unsigned)sizeof(RowRec<R>);
        const unsigned char* src = rw0 + g * rwstride + (long long)a * (long long)sizeof(RowRec<R>);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
    }
}

__device__ inline void mbar_wait(unsigned long long* bar, unsigned phase)
{
    unsigned done = 0;
    for (long long spin = 0; !done; ++spin) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
        if (spin > (1LL << 28)) __trap();   // a lost transaction must fail the launch, not hang the GPU
    }
}

// generic-proxy global stores -> visible to later async-proxy (TMA) reads
__device__ inline void fence_proxy_async_global()
{
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------ tiled DP (large K)
// Exact pruning: T_{i,j} = Upsilon[p,0,0] + sum_n T^v_n(b) + [max(y0 + T^d_1 - y1, 0)
// + positive part of the envelope sum] >= LB = (y1[p] + es[p]) + (b vsl + vc).  A candidate whose LB
// exceeds the row's running best by more than any rounding (relative 1e-13, fp32 1e-6) can neither win nor tie,
// so its full evaluation is skipped; the decisions are the same as without pruning.
#ifndef SDEDGE_PRUNE
#define SDEDGE_PRUNE 1
#endif
#ifndef SDEDGE_PASS1_FAST
#define SDEDGE_PASS1_FAST 1  // phase-A bound test as one FMA + compare per predecessor
#endif
#ifndef SDEDGE_SCEN_SMEM
#define SDEDGE_SCEN_SMEM 1    // re-read alpha and the coefficients from shared memory at each DP call
#endif
#ifndef SDEDGE_GAMMA_ABORT
#define SDEDGE_GAMMA_ABORT 1  // stop a gamma's DP once its partial optimum exceeds the best finished gamma
#endif
#ifndef SDEDGE_LB2
#define SDEDGE_LB2 1          // pass 2: the Jensen bound on the envelope sum before a full evaluation
#endif
#ifndef SDEDGE_TMA_LANE0
#define SDEDGE_TMA_LANE0 0    // 1: lane 0 issues the chunk copies of all G DPs (uniform operands)
#endif
#ifndef SDEDGE_SPEC
#define SDEDGE_SPEC 2      // phase B: rows built at once from their phase-A winners (2: only the steps that matter run)
#endif
#ifndef SDEDGE_PREFETCH
#define SDEDGE_PREFETCH 0  // L1 prefetch of the phase-A winner's record before phase B
#endif
#ifndef SDEDGE_GUESS
#define SDEDGE_GUESS 1     // warm start: bit 0 same batch start, bit 1 same batch size as row i0-1
#endif
// thr = bT (1 + 1e-13), kept next to the running best bT.
template <typename R>
__device__ inline R prune_lb(const RowRec<R>* q, const RowCoef& rc, double bd)
{
    return q->key + (R)fma(bd, rc.vsl, rc.vc);
}
template <typename R>
__device__ inline bool prunable(const RowRec<R>* q, const RowCoef& rc, double bd, R thr)
{
#if SDEDGE_PRUNE
    return prune_lb(q, rc, bd) > thr;
#else
    return false;
#endif
}
// (fp32: the margin must exceed a few float roundings; 1 + 1e-13 would round to 1)
// Second bound, for the pass-2 survivors (before the full evaluation): the
// envelope sum is sum_m max(P + Q m - env_p(m), 0) >= max(Mx P + sumM Q - E.x, 0)
// (Jensen on the positive part; sum_m env_p(m) = E.x), so T >= LB + that.  The
// difference of two large sums is taken with a slack of 1e-12 (fp32 1e-5) of
// their size, far above its rounding, so this too never prunes a winner or tie.
template <typename R>
__device__ inline bool prunable2(const RowRec<R>* q, const RowCoef& rc, const DPConst& D, double bd, R lb, R thr)
{
#if SDEDGE_PRUNE && SDEDGE_LB2
    const R P = q->A.x + (R)fma(bd, rc.ad, D.c2dg), Q = q->A.y + (R)(bd * D.bdc);
    const R ex = q->E.x;
    const R X = fma((R)D.Mx, P, fma((R)D.sumM, Q, -ex));
    const R dl = (sizeof(R) == 8 ? (R)1e-12 : (R)1e-5) * (ex + ex + fabs(X));
    return lb + rmax(X - dl, (R)0) > thr;
#else
    return false;
#endif
}

template <typename R> __device__ inline R prune_thr(R bT) { return bT * (sizeof(R) == 8 ? (R)(1.0 + 1e-13) : (R)(1.0 + 1e-6)); }

// Record-pointer versions of the segment walk, candidate and update (the
// predecessor may live in global memory or in the shared tile buffer).
template <typename R>
__device__ inline Seg<R> get_seg_rec(const RowRec<R>* q, const Pool<R>& pl, int k, int c, int Mx)
{
    Seg<R> sg;
    if (k == 0) {
        sg.u = 1; sg.v = (int)q->E.y; sg.a = q->Ln.x; sg.s = q->Ln.y;
    } else {
        const long long o = q->off + k - 1;
        sg.u = pl.u[o]; sg.a = pl.a[o]; sg.s = pl.s[o];
        sg.v = (k + 1 < c) ? pl.u[o + 1] - 1 : Mx;
    }
    return sg;
}

// Segments k >= 1 of an envelope whose extra segments start at pool[off].
template <typename R>
__device__ __noinline__ R extra_segments_off(const Pool<R>& pl, int off, int cntp, R P, R Q, int Mx)
{
    R pos = (R)0;
    for (int k = 1; k < cntp; ++k) {
        const long long o = off + k - 1;
        const int u = pl.u[o], v = (k + 1 < cntp) ? pl.u[o + 1] - 1 : Mx;
        pos += pos_sum(P - pl.a[o], Q - pl.s[o], (R)u, (R)v);
    }
    return pos;
}

// The rare parts of a candidate's envelope sum, behind one branch: a crossing
// inside the first segment and/or further segments.
template <typename R>
__device__ __noinline__ R rare_pos(const Pool<R>& pl, int cntp, int off, R lv, R P, R Q, R dP, R dQ, R Du,
                                   R Dv, bool cross, R pos, int Mx)
{
    if (cross && cntp > 0) pos = crossing_sum(dP, dQ, 1, (int)lv, Du, Dv);
    if (cntp > 1) pos += extra_segments_off(pl, off, cntp, P, Q, Mx);
    return pos;
}

// T_{i,j} for predecessor record q (see env_cand).
template <typename R>
__device__ inline R env_cand_rec(const RowRec<R>* q, const Pool<R>& pl, const DPConst& D, const RowCoef& rc,
                                 double bd, int Mx, R& rest, int& nseg)
{
    const R2<R> y = q->Y, a = q->A, e = q->E, ln = q->Ln;
    const int cntp = q->cnt, off = q->off;
    const R Td1 = (R)fma(bd, rc.td1, D.c2dg), Tv1 = (R)fma(bd, rc.tv1, D.c2vv);
    const R P = a.x + (R)fma(bd, rc.ad, D.c2dg), Q = a.y + (R)(bd * D.bdc);
    const R base = e.x + (R)fma(bd, rc.tvb, rc.tvc);
    const R d1 = rmax(y.x + Td1, y.y) + Tv1;
    const R dP = P - ln.x, dQ = Q - ln.y;
    const R Du = dP + dQ, Dv = fma(dQ, e.y, dP);
    const bool pu = Du > (R)0, pv = Dv > (R)0;
    R pos = (pu && pv) ? (Du + Dv) * e.y * (R)0.5 : (R)0;
    if ((pu != pv) | (cntp > 1)) pos = rare_pos(pl, cntp, off, e.y, P, Q, dP, dQ, Du, Dv, pu != pv, pos, Mx);
    nseg = cntp;
    rest = base + pos;
    return d1 + rest;
}

// General merge of the new line into env_q (rare path, out of line so that its
// registers do not count against the DP loop); see env_update.
template <typename R>
__device__ __noinline__ bool row_merge_rec(const RowRec<R>* q, RowRec<R>* o, const Pool<R>& pl, R P, R Q, R Av,
                                           R Bv, R rest, int Mx, long long& top)
{
    const int cntp = q->cnt;
    int mlo = 0, mhi = -1;
    for (int k = 0; k < cntp && mlo == 0; ++k) {
        const Seg<R> sg = get_seg_rec(q, pl, k, cntp, Mx);
        const R sP = P - sg.a, sQ = Q - sg.s;
        if (fma(sQ, (R)sg.u, sP) > (R)0 || fma(sQ, (R)sg.v, sP) > (R)0) mlo = first_pos(sP, sQ, sg.u, sg.v);
    }
    if (mlo > 0)
        for (int k = cntp - 1; k >= 0; --k) {
            const Seg<R> sg = get_seg_rec(q, pl, k, cntp, Mx);
            const R sP = P - sg.a, sQ = Q - sg.s;
            if (fma(sQ, (R)sg.u, sP) > (R)0 || fma(sQ, (R)sg.v, sP) > (R)0) {
                mhi = last_pos(sP, sQ, sg.u, sg.v);
                break;
            }
        }
    const long long base = top;
    int nseg = 0;
    bool ovf = false;
    R lv = (R)Mx;
    R2<R> first{(R)0, (R)0};
    auto emit = [&](int u, R ea, R es) {
        ea += Av;
        es += Bv;
        if (nseg == 0) first = R2<R>{ea, es};
        else {
            if (nseg == 1) lv = (R)(u - 1);
            const long long w = base + nseg - 1;
            if (w >= pl.cap) ovf = true;
            else { pl.u[w] = u; pl.a[w] = ea; pl.s[w] = es; }
        }
        ++nseg;
    };
    bool line_done = false;
    for (int k = 0; k < cntp; ++k) {
        const Seg<R> sg = get_seg_rec(q, pl, k, cntp, Mx);
        if (mlo > 0 && sg.v >= mlo && sg.u <= mhi) {
            if (sg.u < mlo) emit(sg.u, sg.a, sg.s);
            if (!line_done) { emit(mlo, P, Q); line_done = true; }
            if (sg.v > mhi) emit(mhi + 1, sg.a, sg.s);
        } else {
            emit(sg.u, sg.a, sg.s);
        }
    }
    o->Ln = first;
    o->E = R2<R>{rest, lv};
    o->cnt = ovf ? 1 : nseg;                 // on overflow keep later reads in bounds
    top = base + (nseg > 1 ? nseg - 1 : 0);
    return ovf;
}

// Row i from predecessor record q and the winning candidate (eq:tt1, eq:tt2),
// stored to the shared tile slot o_s and the global row store o_g; the pool
// pointer lives in shared memory (only the rare merge path moves it).
// Returns 1 on pool overflow, 2 if `spec` and the row needs the merge path
// (nothing stored: the pool is allocated in row order, serially), else 0.
template <typename R>
__device__ int row_update_rec(const RowRec<R>* q, RowRec<R>* o_s, RowRec<R>* o_g, const Pool<R>& pl,
                              const DPConst& D, const RowCoef& rc, double bd, R rest, int Mx, long long* top_s,
                              bool spec = false)
{
    const R2<R> y = q->Y, a = q->A, ln = q->Ln;
    const int cntp = q->cnt;
    const R d0 = y.x + (R)fma(bd, rc.td1, D.c2dg);
    const R d1 = rmax(d0, y.y) + (R)fma(bd, rc.tv1, D.c2vv);
    const R P = a.x + (R)fma(bd, rc.ad, D.c2dg), Q = a.y + (R)(bd * D.bdc);
    const R Av = (R)fma(bd, rc.av, D.c2vv), Bv = (R)(bd * D.bvc);
    const R2<R> Y{d0, d1}, A{P, Q};
    const R dP = P - ln.x, dQ = Q - ln.y;
    const bool pu = dP + dQ > (R)0, pv = fma(dQ, (R)Mx, dP) > (R)0;
    if (cntp == 0 || (cntp == 1 && pu == pv)) {   // N = 1, or no crossing: one line, old or new
        const R2<R> Ln = cntp == 0 ? R2<R>{(R)0, (R)0}
                                   : (pu ? R2<R>{P + Av, Q + Bv} : R2<R>{ln.x + Av, ln.y + Bv});
        const R2<R> E{rest, cntp == 0 ? (R)0 : (R)Mx};
        const R key = d1 + rest;
        o_s->Y = Y; o_s->A = A; o_s->E = E; o_s->Ln = Ln; o_s->cnt = cntp; o_s->off = 0; o_s->key = key;
        if (o_g != o_s) { o_g->Y = Y; o_g->A = A; o_g->E = E; o_g->Ln = Ln; o_g->cnt = cntp; o_g->off = 0; o_g->key = key; }
        return 0;
    }
    if (spec) return 2;
    long long top = *top_s;
    o_s->Y = Y;
    o_s->A = A;
    o_s->off = (int)top;
    const bool ovf = row_merge_rec(q, o_s, pl, P, Q, Av, Bv, rest, Mx, top);
    o_s->key = d1 + rest;
    *top_s = top;
    if (o_g != o_s) *o_g = *o_s;
    return ovf ? 1 : 0;
}

// Algorithm 1 in tiles of GL rows; lane r of a group owns row i0+r throughout.
// Phase A: every lane scans the finished predecessors p < i0, the whole group
// reading the same record (a broadcast from the TMA-staged chunk) -- no per-row
// warp work.  Phase B: rows in order; lane r finalizes row i0+r from its own
// running best (no reduction), writes it to the shared tile and the global
// store, and the later rows of the tile evaluate their candidate with that row
// as predecessor.  Every lane sees its row's candidates in ascending j, so the
// '<=' update keeps the largest j: the same candidates, comparisons and tie
// rule as dp_gamma.
// RS: the row store itself lives in shared memory (small K): phase A reads the finished rows in
// place and the tile's rows are rows i0.. of the store -- no TMA staging, no global row traffic.
template <typename R, int G, bool RS>
__device__ double dp_gamma_tiled(const Consts& C, const Smem& sm, RowRec<R>* rw, Pool<R> pl, RowRec<R>* tb_buf,
                                 RowRec<R>* stage, unsigned long long* bars, unsigned& bar_phase,
                                 unsigned st0, unsigned tstride, const unsigned char* rw0, long long rwstride,
                                 int gi, short* S, bool* overflow, WorkCount& wc, long long* top_s, bool active,
                                 const double* best_s, double lbv, bool mono)
{
    constexpr int GL = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane % GL;
    const unsigned gmask = G == 1 ? 0xffffffffu : (((1u << GL) - 1u) << (lane - gl));
    const int K = C.K;
    // the per-(scenario, gamma) constants (L, N = ceil(O_max / L) by eq:ol / eq:step_n, and the
    // Appendix-A stage-time coefficients) were computed once per scenario by solve_kernel's
    // prologue; they stay in shared memory (all twelve in registers would spill the phase-A loop)
    const int N = sm.nq[gi];
    const int Mx = N - 1;
    const DPConst& D = sm.dq[gi];
    unsigned n_cand = 0, n_seg = 0, n_full = 0;
    if (gl == 0) {                           // row 0 == 0 (reading A3); empty segment pool
        *top_s = 0;
        rw[0].Y = R2<R>{(R)0, (R)0};
        rw[0].A = R2<R>{(R)0, (R)0};
        rw[0].E = R2<R>{(R)0, (R)Mx};
        rw[0].Ln = R2<R>{(R)0, (R)0};
        rw[0].off = 0;
        rw[0].cnt = Mx >= 1 ? 1 : 0;
        rw[0].key = (R)0;
        if (!RS) fence_proxy_async_global();
    }
    __syncwarp();
    int rows_done = 0;
    bool ovf_any = false, infeasible = false, aborted = !active;
#if SDEDGE_GAMMA_ABORT
    if (best_s) {
        // Before any row: T_inf >= the verify server's total work, sum_m sum_n T^v_n =
        // sum_m (b_m vsl(I_m) + vc) >= sum_k vsl(I_k) + vc, since vsl grows with I and
        // each task pays at least its own length's slope.  A gamma whose
        // bound already exceeds the best finished T_inf never starts.
        // (lbv is computed per scenario in O(1) from sum I and sum I^2: solve_kernel's prologue)
        const double mg = sizeof(R) == 8 ? 1e-11 : 1e-4;       // covers the rounding of either DP
        aborted |= lbv * (1.0 - mg) > *best_s * (1.0 + mg);
        if (__all_sync(0xffffffffu, aborted)) {
            work_flush(wc, active, 0u, 0u, 0u, 0ull, 0u);
            return dinf();
        }
    }
#endif
    R t_row = (R)0;                          // Upsilon[i,0,0] of the last row this lane finalized
    int jprev = 0;                           // j* of row i0-1 (the previous tile's last row)
    for (int i0 = 1; i0 <= K && !infeasible; i0 += GL) {
        RowRec<R>* const tb = RS ? rw + i0 : tb_buf;   // the tile's GL rows
        const int i = i0 + gl;               // this lane's row
        const bool own = i <= K;
        const int jlo_i = own ? sm.jlo[i - 1] : K + 2;
        RowCoef rc{};
        if (own) rc = row_coef(D, sm.Is[i - 1]);
        // ---- phase A: predecessors p < i0 (final rows, global store)
        R bT = kinf<R>(), thr = kinf<R>();
        int bj = -1;
        R brest = (R)0;
        const int pA = __reduce_min_sync(0xffffffffu, jlo_i) - 1;   // jlo is gamma-independent
        const int p0 = max(pA, 0);
        const int pst = own ? jlo_i - 1 : K + 1;                    // this lane's first predecessor
        // Predecessor rows p0 .. i0-1 stream through two shared staging buffers by
        // TMA bulk copies (cp.async.bulk + mbarrier): chunk c+1 is in flight while
        // chunk c is consumed with broadcast shared loads.
        static_assert(sizeof(RowRec<R>) % 16 == 0, "TMA bulk copies need 16-byte multiples");
        static_assert(kTileCh <= 32, "chunk masks are 32-bit");
        const int nrows = i0 - p0;
        const int nch = (nrows + kTileCh - 1) / kTileCh;
        if (!RS && nch > 0) {
            const int e = min(p0 + kTileCh, i0);
#if SDEDGE_TMA_LANE0
            if (lane == 0) bulk_load_groups<R, G>(st0, tstride, rw0, rwstride, p0, (unsigned)((e - p0) * sizeof(RowRec<R>)), 0);
#else
            if (gl == 0) bulk_load(stage, rw + p0, (unsigned)((e - p0) * sizeof(RowRec<R>)), bars);
#endif
        }
        // Warm start: before the scan, evaluate the candidate(s)
        // suggested by the previous row's winner -- the same batch start and/or the
        // same batch size -- so that the threshold is tight from the first
        // predecessor on.  Ties are then broken explicitly (largest j wins).
        int pg1 = -1, pg2 = -1;
#if SDEDGE_GUESS
        if (jprev > 0 && own && pst <= i0 - 1) {   // only if the window reaches before the tile
            const int jlo_c = max(jlo_i, 1);
            if (SDEDGE_GUESS & 1) pg1 = min(max(jprev, jlo_c), i0) - 1;                  // same start
            if (SDEDGE_GUESS & 2) pg2 = min(max(i - i0 + jprev + 1, jlo_c), i0) - 1;     // same size
            if (pg2 == pg1) pg2 = -1;
#pragma unroll 1
            for (int t = 0; t < 2; ++t) {
                const int pg = t ? pg2 : pg1;
                if (pg < 0) continue;
                R r0;
                int c0;
                const double bd = (double)(i - pg);
                const R T0 = env_cand_rec(rw + pg, pl, D, rc, bd, Mx, r0, c0);
                n_full += 1;
                n_seg += (unsigned)c0;
                if (T0 < bT || (T0 == bT && pg + 1 > bj)) { bT = T0; thr = prune_thr(bT); bj = pg + 1; brest = r0; }
            }
        }
#endif
        for (int c = 0; c < nch; ++c) {
            if (!RS && c + 1 < nch) {
                const int a1 = p0 + (c + 1) * kTileCh, e1 = min(a1 + kTileCh, i0);
#if SDEDGE_TMA_LANE0
                if (lane == 0)
                    bulk_load_groups<R, G>(st0, tstride, rw0, rwstride, a1, (unsigned)((e1 - a1) * sizeof(RowRec<R>)),
                                           (c + 1) & 1);
#else
                if (gl == 0)
                    bulk_load(stage + ((c + 1) & 1) * kTileCh, rw + a1, (unsigned)((e1 - a1) * sizeof(RowRec<R>)),
                              bars + ((c + 1) & 1));
#endif
            }
            if (!RS) {
                mbar_wait(bars + (c & 1), (bar_phase >> (c & 1)) & 1u);
                bar_phase ^= 1u << (c & 1);
            }
            const int a = p0 + c * kTileCh, e = min(a + kTileCh, i0);
            const RowRec<R>* buf = RS ? rw + a : stage + (c & 1) * kTileCh;
            const double bda = (double)(i - a);
            // this lane's candidates in the chunk: predecessors max(a, pst) .. e-1
            const int lo = max(pst - a, 0), hi = e - a;
            n_cand += (unsigned)max(hi - lo, 0);
#if SDEDGE_PRUNE
            // whole-chunk skip: with coefficients >= 0 the row values Upsilon[p,0,0] = key
            // are non-decreasing in p (5.2d), so every predecessor of the chunk has key >= key[a] and
            // batch size >= i - (e-1): LB1 >= key[a] + (i-e+1) vsl + vc.  A chunk whose bound exceeds
            // every lane's threshold (key[a] shaded by 1e-13, fp32 1e-6, against rounding) is skipped
            if (SDEDGE_CHUNK_SKIP && mono) {
                const R ka = buf[0].key * (sizeof(R) == 8 ? (R)(1.0 - 1e-13) : (R)(1.0 - 1e-6));
                const R lbc = ka + (R)fma(bda - (double)(e - a - 1), rc.vsl, rc.vc);
                if (__all_sync(0xffffffffu, !own || lbc > thr)) {
                    if (!RS) __syncwarp();
                    continue;
                }
            }
#endif
            // pass 1 (independent, unrolled): the bound of every predecessor of the
            // chunk against the threshold at the chunk's start -- a superset of the
            // survivors, since the threshold only falls
            unsigned m = 0;
#if SDEDGE_PRUNE && SDEDGE_PASS1_FAST
            // key + (bda - k) vsl + vc > thr  <=>  key > u + k vsl with u = thr - (bda vsl + vc):
            // two operations per predecessor.  Rounding here is a few ulp of T, far inside the
            // 1e-13 (fp32: 1e-6) margin of thr, so a pruned candidate still cannot win or tie.
            const R u = thr - (R)fma(bda, rc.vsl, rc.vc), vs = (R)rc.vsl;
#pragma unroll
            for (int k = 0; k < kTileCh; ++k)
                m |= (unsigned)!(buf[k].key > fma((R)k, vs, u)) << k;
#else
#pragma unroll
            for (int k = 0; k < kTileCh; ++k)
                m |= (unsigned)!(prunable(buf + k, rc, bda - (double)k, thr)) << k;
#endif
            m &= lo >= kTileCh ? 0u : (0xffffffffu << lo);
            if (hi < kTileCh) m &= (1u << hi) - 1u;              // the last chunk of the window
            // pass 2: the survivors in ascending j, re-tested against the current
            // threshold (lanes of the warp evaluate different predecessors together)
            while (m) {
                const int k = __ffs(m) - 1;
                m &= m - 1;
                const double bd = bda - (double)k;
                const RowRec<R>* q = buf + k;
                const R lb = prune_lb(q, rc, bd);
                if (!(SDEDGE_PRUNE && lb > thr) && a + k != pg1 && a + k != pg2 &&   // guesses: done
                    !prunable2(q, rc, D, bd, lb, thr)) {
                    R r0;
                    int c0;
                    const R T0 = env_cand_rec(q, pl, D, rc, bd, Mx, r0, c0);
                    n_full += 1;
                    n_seg += (unsigned)c0;
#if SDEDGE_GUESS
                    if (T0 < bT || (T0 == bT && a + k + 1 > bj)) { bT = T0; thr = prune_thr(bT); bj = a + k + 1; brest = r0; }
#else
                    if (T0 <= bT) { bT = T0; thr = prune_thr(bT); bj = a + k + 1; brest = r0; }   // '<=': largest j
#endif
                }
            }
            if (!RS) __syncwarp();                               // buffer (c & 1) may be refilled now
        }
        __syncwarp();
        // ---- phase B: the tile's rows in order.  Lane r already holds the best
        // of every candidate of its row except those whose predecessor is in the
        // tile; each finished row i0+r is "pushed": the later rows of the tile
        // evaluate their candidate with predecessor i0+r (broadcast from the shared
        // tile).  So no reduction is needed: lane r finalizes row i0+r itself.
#if SDEDGE_PREFETCH
        // the phase-A winner's record is in the global store (L2): start pulling it
        // into L1 now, its row update comes up in step gl of the serial phase B
        if (own && bj > 0) {
            const char* g = reinterpret_cast<const char*>(rw + (bj - 1));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(g));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(g + sizeof(RowRec<R>) - 1));
        }
#endif
        // rows of the tile up to the first one whose memory window is empty (the
        // window is gamma-independent, so every group stops at the same row)
        const unsigned bad_rows = __ballot_sync(0xffffffffu, own && jlo_i > i) & ((GL == 32 ? 0u : (1u << GL)) - 1u);
        const int rend = min(bad_rows ? __ffs(bad_rows) - 1 : GL, K - i0 + 1);
        if (bad_rows && __ffs(bad_rows) - 1 < K - i0 + 1) infeasible = true;
#if SDEDGE_SPEC
        // Speculation: every lane builds its row from its phase-A winner at once (the
        // predecessor is a finished row, p < i0).  The serial steps below then only
        // test the pushed candidates; a lane rebuilds its row in its own step if one
        // of them won, or if its row needs the merge path (pool space is taken in
        // row order).  Same candidates, comparisons and tie rule as the serial form.
        bool fin = false;                    // slot gl holds the row for the current bj
        if (own && gl < rend && bj > 0) {
            const int p = bj - 1;
            fin = row_update_rec(rw + p, tb + gl, rw + i, pl, D, rc, (double)(i - p), brest, Mx, top_s, true) == 0;
            if (SDEDGE_DBG && !fin) DBG_ADD(0, 1);                  // speculation needs the merge path
        }
        if (SDEDGE_DBG && own && gl < rend && bj <= 0) DBG_ADD(1, 1);   // no phase-A winner
        __syncwarp();
#if SDEDGE_SPEC >= 2
        // In-tile candidates j = i0+r+1 (predecessor row i0+r, r < gl) are first
        // tested against the speculative rows, all at once; then only the steps r
        // that hold a surviving candidate or a row to rebuild run.  A rebuilt row's
        // candidates are re-tested by every later row (its key may have fallen).
        const int rlo = max(jlo_i - i0 - 1, 0);          // j = i0+r+1 >= jlo_i
        const bool live = own && gl < rend;
        unsigned cm = 0;
        {
            const R u = thr - (R)fma((double)(i - i0), rc.vsl, rc.vc), vs = (R)rc.vsl;
#pragma unroll
            for (int r = 0; r < GL; ++r) cm |= (unsigned)!(SDEDGE_PRUNE && tb[r].key > fma((R)r, vs, u)) << r;
            cm &= (live && rlo < gl) ? (((1u << gl) - 1u) & (0xffffffffu << rlo)) : 0u;
            if (live) n_cand += (unsigned)max(gl - rlo, 0);
        }
        unsigned todo = __reduce_or_sync(0xffffffffu, cm | ((live && !fin) ? 1u << gl : 0u));
        while (todo) {
            const int r = __ffs(todo) - 1;
            todo &= todo - 1;
            const int ii = i0 + r;
            bool rebuilt = false;
            if (gl == r && !fin) {           // eq:rg, eq:tt1, eq:tt2 with j* = bj (reading A4)
                const int p = bj - 1;
                const RowRec<R>* q = p >= i0 ? tb + (p - i0) : rw + p;
                if (SDEDGE_DBG) DBG_ADD(3, 1);                               // serial row builds
                if (SDEDGE_DBG && rw[p].cnt > 0) DBG_ADD(4, rw[p].cnt);
                if (row_update_rec(q, tb + r, rw + ii, pl, D, rc, (double)(ii - p), brest, Mx, top_s) == 1)
                    ovf_any = true;
                fin = true;
                rebuilt = true;
            }
            __syncwarp();
            const bool chg = __shfl_sync(0xffffffffu, rebuilt, (lane - gl) + r);
            if (live && gl > r && r >= rlo && (chg || ((cm >> r) & 1u))) {
                const R lb = prune_lb(tb + r, rc, (double)(i - ii));
                if (!(SDEDGE_PRUNE && lb > thr) && !prunable2(tb + r, rc, D, (double)(i - ii), lb, thr)) {
                    R rq;
                    int c0;
                    const R t = env_cand_rec(tb + r, pl, D, rc, (double)(i - ii), Mx, rq, c0);
                    n_full += 1;
                    n_seg += (unsigned)c0;
                    if (SDEDGE_DBG && t <= bT) DBG_ADD(2, 1);               // an in-tile candidate wins
                    if (t <= bT) { bT = t; thr = prune_thr(bT); bj = ii + 1; brest = rq; fin = false; }   // '<=': largest j
                }
            }
            todo |= __reduce_or_sync(0xffffffffu, (live && !fin) ? 1u << gl : 0u);   // rows that must be rebuilt
        }
        rows_done += rend;
#else
        for (int r = 0; r < rend; ++r) {
            const int ii = i0 + r;
            if (gl == r && !fin) {           // eq:rg, eq:tt1, eq:tt2 with j* = bj (reading A4)
                const int p = bj - 1;
                const RowRec<R>* q = p >= i0 ? tb + (p - i0) : rw + p;
                if (row_update_rec(q, tb + r, rw + ii, pl, D, rc, (double)(ii - p), brest, Mx, top_s) == 1)
                    ovf_any = true;
                fin = true;
            }
            __syncwarp();
            if (own && gl > r && ii + 1 >= jlo_i) {   // candidate j = ii+1 of the later rows
                n_cand += 1;
                const R lb = prune_lb(tb + r, rc, (double)(i - ii));
                if (!(SDEDGE_PRUNE && lb > thr) && !prunable2(tb + r, rc, D, (double)(i - ii), lb, thr)) {
                    R rq;
                    int c0;
                    const R t = env_cand_rec(tb + r, pl, D, rc, (double)(i - ii), Mx, rq, c0);
                    n_full += 1;
                    n_seg += (unsigned)c0;
                    if (t <= bT) { bT = t; thr = prune_thr(bT); bj = ii + 1; brest = rq; fin = false; }   // '<=': largest j
                }
            }
            ++rows_done;
        }
#endif
        if (own && gl < rend) {
            if (S) S[i - 1] = (short)bj;
            t_row = bT;
        }
#else
        for (int r = 0; r < rend; ++r) {
            const int ii = i0 + r;
            if (gl == r) {                   // eq:rg, eq:tt1, eq:tt2 with j* = bj (reading A4)
                if (S) S[ii - 1] = (short)bj;
                const int p = bj - 1;
                const RowRec<R>* q = p >= i0 ? tb + (p - i0) : rw + p;
                if (row_update_rec(q, tb + r, rw + ii, pl, D, rc, (double)(ii - p), brest, Mx, top_s) == 1)
                    ovf_any = true;
                t_row = bT;
            }
            __syncwarp();
            if (own && gl > r && ii + 1 >= jlo_i) {   // candidate j = ii+1 of the later rows
                n_cand += 1;
                if (!prunable(tb + r, rc, (double)(i - ii), thr)) {
                    R rq;
                    int c0;
                    const R t = env_cand_rec(tb + r, pl, D, rc, (double)(i - ii), Mx, rq, c0);
                    n_full += 1;
                    n_seg += (unsigned)c0;
                    if (t <= bT) { bT = t; thr = prune_thr(bT); bj = ii + 1; brest = rq; }   // '<=': largest j
                }
            }
            ++rows_done;
        }
#endif
        jprev = __shfl_sync(0xffffffffu, bj, (lane - gl) + GL - 1);
        // later tiles bulk-read this tile's rows through TMA (async proxy): every
        // lane orders the global row stores it made before the next __syncwarp
        if (!RS) fence_proxy_async_global();
        __syncwarp();
#if SDEDGE_GAMMA_ABORT
        // Exact gamma-level pruning: the optimal latency of the first i tasks is
        // non-decreasing in i (drop the last task from its batch: the batch shrinks,
        // its padded length cannot grow, every stage time can only fall), so once
        // T*(i0+GL-1) exceeds the best T_inf of an already finished gamma, this gamma
        // cannot win or tie.  Margins cover the rounding of both DPs.
        // Stronger: Upsilon[i+1,0,0] >= Upsilon[i,0,0] + vsl(I_{i+1}) -- every
        // candidate of row i+1 either extends a candidate of row i by task i+1 (its verify
        // stage grows by at least that task's own verify time, every other stage time can only
        // grow) or appends a new batch after row i's state -- so T_inf >= Upsilon[i,0,0] + the
        // remaining tasks' own verify work sum_{k>i} vsl(I_k), quadratic in I_k: O(1) from the
        // suffix sums of I and I^2.
        if (best_s && rend == GL) {
            const int il = i0 + GL - 1;                          // the tile's last row
            const R kl = __shfl_sync(0xffffffffu, t_row, (lane - gl) + GL - 1);
            const double mg = sizeof(R) == 8 ? 1e-11 : 1e-4;
            const int pt = K / kPfx + 1, pl = il / kPfx;         // il is a multiple of GL, hence of kPfx
            const double S1 = sm.pI[pt] - sm.pI[pl], S2 = sm.pI2[pt] - sm.pI2[pl], cnt = (double)(K - il);
            const double c = D.hv2 + D.g;
            const double rest = D.kv * (S2 + (D.g + c) * S1 + cnt * D.g * c) + D.kv * (1.0 + D.g) * D.Mx * (S1 + cnt * c) +
                                cnt * D.bvc * D.sumM;
            aborted |= ((double)kl + rest) * (1.0 - mg) > *best_s * (1.0 + mg);
            if (__all_sync(0xffffffffu, aborted)) break;
        }
#endif
    }
    // T_inf = Upsilon[K,0,0], held by the lane that finalized row K
    double T_last = (double)__shfl_sync(0xffffffffu, t_row, (lane - gl) + (K - 1) % GL);
    if (infeasible) T_last = dinf();
    if (aborted) T_last = dinf();            // pruned (or an idle group)
    if (__ballot_sync(0xffffffffu, ovf_any) & gmask) { *overflow = true; T_last = dinf(); }
    work_flush(wc, active, n_cand, n_seg, n_full, (unsigned long long)n_cand * (unsigned long long)N,
               gl == 0 ? (unsigned)rows_done : 0u);
    return T_last;
}

// ------------------------------------------------------------ the fused kernel
#ifndef SDEDGE_MINB
#define SDEDGE_MINB 16    // min resident CTAs per SM requested from ptxas (128-register cap)
#endif

#ifndef SDEDGE_MINB_PREP
#define SDEDGE_MINB_PREP 32   // the prep kernel (PHASE 1): 64 registers, 32 one-warp CTAs per SM
#endif
template <typename R, int ALGO, int RSMEM, int G, int TILE, int PHASE>
__global__ void __launch_bounds__(kThreads, PHASE == 1 ? SDEDGE_MINB_PREP : SDEDGE_MINB)
solve_kernel(const Consts C, const Inputs in, const Outputs out, long long n, Work ws, int BIG)
{
    static_assert(PHASE == 0 || (TILE != 0 && kWarps == 1), "the two-kernel path is the tiled, one-warp CTA");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int K = C.K, ng = C.ng;
    // PHASE 2 keeps two prep-record buffers (the current scenario's, the next one's in flight)
    Smem sm = carve_smem(smem_raw, C.so);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int GL = 32 / G;
    const int grp = lane / GL;
    const long long slot = ((long long)blockIdx.x * kWarps + warp) * G + grp;   // one DP per (warp, group)

    // RSMEM is a template parameter so that the compiler sees shared-window
    // (32-bit, LDS/STS) addresses for the row state instead of generic ones.
    // TILE == 2 (row store in shared memory): the in-tile pass reads the GL-row tile at rows
    // i0 .. i0+GL-1 of the store even past row K (masked), so the store is padded to a whole tile
    const int kPad = TILE == 2 ? rs_pad(K, GL) : 0;
    RowRec<R>* rw = carve_rows<R>(RSMEM ? sm.rows + (size_t)(warp * G + grp) * rows_bytes<R>(K + kPad)
                                     : ws.rows + (size_t)slot * C.rows_stride, K);
    // first-pass envelope pool: shared memory after the row store when C.pool_smem (TILE == 2, one DP
    // per CTA), else this slot's block of the global pool; the worst-case pass (BIG) is always global
    const bool pool_s = TILE == 2 && PHASE == 2 && C.pool_smem && !BIG;
    Pool<R> pl = pool_s ? carve_pool<R>(sm.rows + (size_t)kWarps * G * rows_bytes<R>(K + kPad), C.pool_cap_smem)
                        : carve_pool<R>(ws.pool + (size_t)slot * pool_bytes<R>(C.pool_cap), C.pool_cap);
    RowRec<R>* tb = nullptr;
    RowRec<R>* stage = nullptr;
    unsigned long long* bars = nullptr;
    DPConst* dpc = nullptr;
    if (TILE == 1 && PHASE != 1) {           // shared tile buffer of this (warp, group) DP (none in prep)
        unsigned char* t = sm.rows + (RSMEM ? (size_t)kWarps * G * rows_bytes<R>(K + kPad) : 0) +
                           (size_t)(warp * G + grp) * tile_bytes<R, G>();
        tb = reinterpret_cast<RowRec<R>*>(t);
        stage = reinterpret_cast<RowRec<R>*>(t + (size_t)GL * sizeof(RowRec<R>));
        bars = reinterpret_cast<unsigned long long*>(stage + 2 * kTileCh);
        dpc = reinterpret_cast<DPConst*>(bars + 2);
        if (lane % GL == 0) {
            mbar_init(bars, 1);
            mbar_init(bars + 1, 1);
            fence_mbar_init();
        }
        __syncwarp();
    }
    unsigned bar_phase = 0u;                  // parity of each staging mbarrier (bit b)
    // warp-uniform addresses of group 0's staging buffer and row store (TMA issue)
    const unsigned tb_stride = (unsigned)tile_bytes<R, G>();
    const int wu = kWarps == 1 ? 0 : warp;
    const unsigned st0 = TILE == 1 ? smem_u32(sm.rows + (RSMEM ? (size_t)kWarps * G * rows_bytes<R>(K + kPad) : 0) +
                                         (size_t)(wu * G) * tb_stride) + (unsigned)(GL * sizeof(RowRec<R>)) : 0u;
    const unsigned char* rw0 = ws.rows + (size_t)((long long)blockIdx.x * kWarps + wu) * G * C.rows_stride;
    const long long n_items = BIG ? (long long)*ws.ovf_count : n;
    short* Scta = ws.S + (size_t)blockIdx.x * (ng + 1) * K;   // this CTA's S vectors (+1: per-batch gammas)
    __shared__ bool s_ovf;
    __shared__ double s_best;                // best T_inf of the finished gammas of this scenario
    __shared__ unsigned long long s_work[kThreads * 5];   // per-thread work counters
    __shared__ long long s_top[kWarps * G];
    for (int q = 0; q < 5; ++q) s_work[tid * 5 + q] = 0;
    __syncthreads();
    WorkCount wc{out.work ? s_work + tid * 5 : nullptr};
    __shared__ double s_par[5];              // alpha, c1d, c2d, c1v, c2v of the current scenario

    // backtrack stack of the epilogue: the sort keys (dead after the sort) or, in the DP kernel, the
    // shared row store / tile buffers (dead after the DPs; >= 2 K bytes); K <= 1024 fits int16
    short* const bstack = PHASE == 2 ? reinterpret_cast<short*>(sm.rows) : reinterpret_cast<short*>(sm.key);
    // PHASE 2: the record of the next scenario is fetched by a TMA bulk copy while this one is solved
    int rcur = 0;
    unsigned rphase = 0u;
    // tid 0 takes queue items SDEDGE_QCHUNK at a time (one atomic round trip per SDEDGE_QCHUNK scenarios)
    __shared__ unsigned long long s_qnext, s_qend;
    if (tid == 0) { s_qnext = 0; s_qend = 0; }
    auto take_item = [&](unsigned long long* ctr) -> unsigned long long {
        if (s_qnext == s_qend) {
            s_qnext = atomicAdd(ctr, (unsigned long long)SDEDGE_QCHUNK);
            s_qend = s_qnext + SDEDGE_QCHUNK;
        }
        return s_qnext++;
    };
    auto fetch_rec = [&](int buf) {          // tid 0: take the next queue item, start its record copy
        const unsigned long long it = take_item(ws.next + BIG);
        const long long sn = (long long)it < n_items ? (BIG ? ws.ovf_list[it] : (long long)it) : -1;
        sm.sid[1] = sn;
        if (sn >= 0)
            bulk_load(sm.rec + (size_t)buf * C.prep_stride, ws.prep + (size_t)sn * C.prep_stride,
                      (unsigned)C.prep_stride, sm.rbar + buf);
    };
    if constexpr (PHASE == 2) {
        if (tid == 0) {
            mbar_init(sm.rbar, 1);
            mbar_init(sm.rbar + 1, 1);
            fence_mbar_init();
            fetch_rec(0);
        }
        __syncthreads();
    }

    for (;;) {
        if (tid == 0) {
            if constexpr (PHASE == 2) {
                sm.sid[0] = sm.sid[1];
                if (sm.sid[0] >= 0) fetch_rec(rcur ^ 1);
            } else {
                const unsigned long long it = take_item(ws.next + (PHASE == 1 ? 2 : BIG));
                sm.sid[0] = (long long)it < n_items ? (BIG ? ws.ovf_list[it] : (long long)it) : -1;
            }
            sm.ctl[0] = 0;
            s_ovf = false;
            s_best = dinf();
        }
        __syncthreads();
        const long long s = sm.sid[0];
        if (s < 0) break;

        int bad = 0;
        const bool uniform = C.bw_policy == SDEDGE_BW_UNIFORM;
        bool bad_alpha = false, mono = true;
        double Tcom = 0.0;
        if constexpr (PHASE != 2) {
        // ---- stage + validate (SoA, coalesced)
        const int32_t* Ig = in.I + s * K;
        const double* pg = in.p + s * K;
        const double* gg = in.g + s * K;
        // t*_com and w* sums (eq:opt_w); s1, s2 = sum I_k, sum I_k^2 (exact integers)
        double tc = 0.0, q = 0.0, s1 = 0.0, s2 = 0.0;
        // fast path: one warp, K <= 128, K % 4 == 0, 16-byte aligned rows -- every lane takes 4
        // consecutive tasks with one int4 and four double2 loads, validates them and computes their
        // bandwidth terms in registers, and writes w* straight from registers after the reductions
        const bool fast = kWarps == 1 && K <= 128 && (K & 3) == 0 &&
                          ((reinterpret_cast<uintptr_t>(Ig) | reinterpret_cast<uintptr_t>(pg) |
                            reinterpret_cast<uintptr_t>(gg)) & 15u) == 0;
        if (fast) {
            const int k0 = 4 * lane;
            double u[4] = {0.0, 0.0, 0.0, 0.0};
            if (k0 < K) {
                const int4 Iv = reinterpret_cast<const int4*>(Ig)[lane];
                const double2 pa = reinterpret_cast<const double2*>(pg)[2 * lane];
                const double2 pb = reinterpret_cast<const double2*>(pg)[2 * lane + 1];
                const double2 ga = reinterpret_cast<const double2*>(gg)[2 * lane];
                const double2 gb = reinterpret_cast<const double2*>(gg)[2 * lane + 1];
                const int Ik[4] = {Iv.x, Iv.y, Iv.z, Iv.w};
                const double pk[4] = {pa.x, pa.y, pb.x, pb.y}, gk[4] = {ga.x, ga.y, gb.x, gb.y};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    sm.I[k0 + r] = Ik[r];
                    if (Ik[r] < 1 || !(pk[r] > 0.0) || !(gk[r] > 0.0) || !isfinite(pk[r]) || !isfinite(gk[r])) bad = 1;
                    const double Ikd = (double)Ik[r];
                    s1 += Ikd;
                    s2 += Ikd * Ikd;
                    const double sk = log2_ge1(1.0 + pk[r] * gk[r] * C.isig2);
                    if (uniform) {
                        tc = fmax(tc, C.lambda * Ikd / ((1.0 / K) * C.Bw * sk));
                    } else {                      // t*_com = (lambda / B_w) sum_k I_k / s_k: one division per task
                        u[r] = Ikd / sk;
                        q += u[r];
                    }
                }
            }
            bad = __any_sync(0xffffffffu, bad);
            for (int o = 16; o > 0; o >>= 1) {
                const double ot = __shfl_xor_sync(0xffffffffu, tc, o);
                tc = uniform ? (ot > tc ? ot : tc) : tc + ot;
                q += __shfl_xor_sync(0xffffffffu, q, o);
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            }
            if (!uniform) tc = (C.lambda / C.Bw) * q;
            if (out.w && k0 < K) {
                const double rq = 1.0 / q;
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    out.w[s * K + k0 + r] = bad ? dnan() : uniform ? 1.0 / K : u[r] * rq;
            }
            __syncwarp();
        } else {
        #pragma unroll 1
        for (int k = tid; k < K; k += kThreads) {
            const int Ik = Ig[k];
            const double pk = pg[k], gk = gg[k];
            sm.I[k] = Ik;
            if (Ik < 1 || !(pk > 0.0) || !(gk > 0.0) || !isfinite(pk) || !isfinite(gk)) bad = 1;
        }
        bad = __syncthreads_or(bad);
        }
        // ---- stable ascending sort by I_k (reading A13): bitonic sort of the unique keys
        // (I_k biased to unsigned) << 32 | k, padded to a power of two with ~0 -- O(K log^2 K / threads)
        if (kWarps == 1 && K <= 128) {       // in registers: one warp, 4 keys per lane
            warp_sort_tasks<4>(sm.I, sm.ord, sm.Is, K, lane);
        } else {
            const int P2 = sort_len(K);
            for (int k = tid; k < P2; k += kThreads)
                sm.key[k] = k < K ? ((unsigned long long)((unsigned)sm.I[k] ^ 0x80000000u) << 32) | (unsigned)k
                                  : ~0ULL;
            block_sync();
            for (int sz = 2; sz <= P2; sz <<= 1)
                for (int st = sz >> 1; st > 0; st >>= 1) {
                    for (int t = tid; t < (P2 >> 1); t += kThreads) {
                        const int a = ((t & ~(st - 1)) << 1) | (t & (st - 1)), b = a + st;
                        const unsigned long long ka = sm.key[a], kb = sm.key[b];
                        if ((ka > kb) == ((a & sz) == 0)) { sm.key[a] = kb; sm.key[b] = ka; }
                    }
                    block_sync();
                }
            #pragma unroll 1
            for (int r = tid; r < K; r += kThreads) {
                const int k = (int)(unsigned)(sm.key[r] & 0xffffffffULL);
                sm.ord[r] = k;
                sm.Is[r] = sm.I[k];
            }
        }
        __syncthreads();
        // prefix sums of the sorted I and I^2 at rows 0, kPfx, 2 kPfx, ... and the totals (the suffix
        // verify-work bound at tile ends): one thread per kPfx-row block, then a scan
        {
            const int nb = (K + kPfx - 1) / kPfx;
            double c1 = 0.0, c2 = 0.0;
            #pragma unroll 1
            for (int bk = tid; bk < nb; bk += kThreads)
                for (int r = bk * kPfx; r < min(K, bk * kPfx + kPfx); ++r) {
                    const double x = sm.Is[r];
                    c1 += x; c2 += x * x;
                }
            if (kWarps == 1 && nb <= 32) {
                double e1 = c1, e2 = c2;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double u1 = __shfl_up_sync(0xffffffffu, e1, o), u2 = __shfl_up_sync(0xffffffffu, e2, o);
                    if (lane >= o) { e1 += u1; e2 += u2; }
                }
                if (tid == 0) { sm.pI[0] = 0.0; sm.pI2[0] = 0.0; }
                if (tid < nb) { sm.pI[tid + 1] = e1; sm.pI2[tid + 1] = e2; }       // inclusive: row (tid+1) kPfx
                if (tid == nb - 1) { sm.pI[K / kPfx + 1] = e1; sm.pI2[K / kPfx + 1] = e2; }   // the totals
            } else {
                __syncthreads();
                if (tid == 0) {
                    double e1 = 0.0, e2 = 0.0;
                    sm.pI[0] = 0.0; sm.pI2[0] = 0.0;
                    #pragma unroll 1
                    for (int r = 0; r < K; ++r) {
                        const double x = sm.Is[r];
                        e1 += x; e2 += x * x;
                        if ((r + 1) % kPfx == 0) { sm.pI[(r + 1) / kPfx] = e1; sm.pI2[(r + 1) / kPfx] = e2; }
                    }
                    sm.pI[K / kPfx + 1] = e1; sm.pI2[K / kPfx + 1] = e2;
                }
            }
        }
        __syncthreads();
        // ---- memory window per sorted row (gamma-independent): b <= floor((Gs - Gp) / (4 Jd hd (I + O)))
        #pragma unroll 1
        for (int r = tid; r < K; r += kThreads) {
            const int i = r + 1;
            sm.jlo[r] = (short)window_lo(C.gamma_s - C.Gp, C.kvunit * ((long long)sm.Is[r] + C.O_max), i);
        }
        // ---- t*_com and w* (eq:opt_w; reading A14: p_k g_k / sigma^2), or the
        // uniform baseline w_k = 1/K with T_com = max_k T_k,com (eq:ul_latency)
        if (!bad && !fast)
            #pragma unroll 1
            for (int k = tid; k < K; k += kThreads) {
                const double Ikd = (double)sm.I[k];
                s1 += Ikd;
                s2 += Ikd * Ikd;
                const double sk = log2_ge1(1.0 + pg[k] * gg[k] * C.isig2);
                if (uniform) {
                    const double r = (1.0 / K) * C.Bw * sk;
                    tc = fmax(tc, C.lambda * (double)sm.I[k] / r);
                } else {
                    tc += C.lambda * (double)sm.I[k] / (C.Bw * sk);
                    const double u = (double)sm.I[k] / sk;
                    q += u;
                    reinterpret_cast<double*>(sm.key)[k] = u;   // w*_k = u_k / sum u (the sort keys are dead)
                }
            }
        if (!fast)
        for (int o = 16; o > 0; o >>= 1) {
            const double ot = __shfl_xor_sync(0xffffffffu, tc, o);
            tc = uniform ? fmax(tc, ot) : tc + ot;
            q += __shfl_xor_sync(0xffffffffu, q, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane == 0) {
            sm.red[warp] = tc; sm.red[kWarps + warp] = q;
            sm.red[2 * kWarps + warp] = s1; sm.red[3 * kWarps + warp] = s2;
        }
        // ---- fixed-plan baselines (gamma-independent): start of the batch ending at each row
        if (!TILE && C.batch_policy >= SDEDGE_BATCH_NONE && C.batch_policy <= SDEDGE_BATCH_MAX) {
            int b = 1;
            if (C.batch_policy == SDEDGE_BATCH_STATIC) b = min(C.static_batch, K);
            if (C.batch_policy == SDEDGE_BATCH_MAX) {      // largest size for the longest input (reading B4)
                const int jl = sm.jlo[K - 1];
                b = jl > K ? 0 : K - jl + 1;
            }
            #pragma unroll 1
            for (int r = tid; r < K; r += kThreads) {
                const int e = r + 1;
                sm.jf[r] = b < 1 ? (short)(e == K ? -1 : 0)
                                 : (short)((e % b == 0 || e == K) ? ((e - 1) / b) * b + 1 : 0);
            }
        }
        if (tid == 0) {
            s_par[0] = in.alpha[s];
            s_par[1] = in.coeffs ? in.coeffs[4 * s] : C.c1d;
            s_par[2] = in.coeffs ? in.coeffs[4 * s + 1] : C.c2d;
            s_par[3] = in.coeffs ? in.coeffs[4 * s + 2] : C.c1v;
            s_par[4] = in.coeffs ? in.coeffs[4 * s + 3] : C.c2v;
        }
        __syncthreads();
        bad_alpha = !(s_par[0] > 0.0 && s_par[0] < 1.0);
        if (out.w && !fast) {                // w* (eq:opt_w): known before any DP runs
            double qsum = 0.0;
            for (int w = 0; w < kWarps; ++w) qsum += sm.red[kWarps + w];
            #pragma unroll 1
            for (int k = tid; k < K; k += kThreads)
                out.w[s * K + k] = bad ? dnan() : uniform ? 1.0 / K : reinterpret_cast<const double*>(sm.key)[k] / qsum;
        }
        // (alpha and the coefficients are re-read from shared memory at each DP call:
        // nothing scenario-wide stays live in registers across the gamma loop)
#if SDEDGE_SCEN_SMEM
#define SDEDGE_SCEN_ARGS s_par[0], s_par[1], s_par[2], s_par[3], s_par[4]
#else
        const double alpha = s_par[0], c1d = s_par[1], c2d = s_par[2], c1v = s_par[3], c2v = s_par[4];
#define SDEDGE_SCEN_ARGS alpha, c1d, c2d, c1v, c2v
#endif

        // stage times non-decreasing in b and I (non-negative coefficients): the row
        // optimum is then monotone in the row, which the gamma-level pruning needs
        mono = s_par[1] >= 0.0 && s_par[2] >= 0.0 && s_par[3] >= 0.0 && s_par[4] >= 0.0 && C.dl >= 0.0;
        // ---- per-gamma prologue, one gamma per thread:
        //  * the verify-work lower bound T_inf(gamma) >= sum_k vsl(I_k) + vc, in O(1): vsl is a
        //    quadratic in I, so the sum needs only sum I and sum I^2;
        //  * the closed-form latency of the single batch of all K tasks -- row K's j = 1 candidate,
        //    so T_inf(gamma) <= it; its minimum over gamma seeds s_best, the best
        //    finished T_inf, before any DP runs;
        //  * the order in which the warps take the gammas: ascending lower bound (the most
        //    promising first, so s_best tightens early).  The result does not depend on the order:
        //    gamma* is the smallest argmin over the stored T_inf (reading A7).
        if (!bad && !bad_alpha) {
            double S1 = 0.0, S2 = 0.0;
            for (int w = 0; w < kWarps; ++w) { S1 += sm.red[2 * kWarps + w]; S2 += sm.red[3 * kWarps + w]; }
            const double Kd = (double)K;
            const bool one_fits = sm.jlo[K - 1] == 1;     // a batch of all K tasks fits the memory
            double one_min = dinf();
            #pragma unroll 1
            for (int gi = tid; gi < ng; gi += kThreads) {
                const int gamma = C.gmin + gi;
                const double L = expected_tokens(s_par[0], gamma);
                const int N = (int)ceil(__ddiv_rn((double)C.O_max, L));
                const DPConst D = make_dpconst(C, gamma, L, N, s_par[1], s_par[2], s_par[3], s_par[4]);
                if (PHASE != 1) sm.dq[gi] = D;      // the prep kernel ships L and N; the DP kernel rebuilds D
                if (PHASE == 1) sm.tinf[gi] = L;
                sm.nq[gi] = N;
                const double c = D.hv2 + D.g;
                const double lbv = D.kv * (S2 + (D.g + c) * S1 + Kd * D.g * c) + D.kv * (1.0 + D.g) * D.Mx * (S1 + Kd * c) +
                                   Kd * D.bvc * D.sumM + D.c2vv * (D.Mx + 1.0);
                // draft side: every step's makespan is at least the draft stage's
                // serial work plus the last batch's verify time, sum_m T^d + T^v_M >= sum_k d_n(I_k)
                // + c2d gamma + v_n(I_K) + c2v (the last batch holds task K, the longest)
                double lbd = 0.0;
                if (D.g > 0.0) {
                    const double e = D.g - 1.0 + D.hd2;
                    lbd = D.kd * (S2 + e * S1 + Kd * ((D.g - 1.0) * D.hd2 + D.tri)) +
                          D.Mx * D.kd * (D.g * S1 + Kd * (D.g * D.hd2 + D.tri)) + Kd * D.sumM * D.bdc;
                }
                lbd += row_coef(D, sm.Is[K - 1]).vsl + (D.c2dg + D.c2vv) * (D.Mx + 1.0);
                sm.glb[gi] = fmax(lbv, lbd);
                if (one_fits) {
                    const RowCoef rc = row_coef(D, sm.Is[K - 1]);
                    one_min = fmin(one_min, Kd * (rc.td1 + rc.tv1 + D.Mx * (rc.ad + rc.av) + D.sumM * (D.bdc + D.bvc)) +
                                                (D.c2dg + D.c2vv) * (D.Mx + 1.0));
                }
            }
            for (int o = 16; o > 0; o >>= 1) one_min = fmin(one_min, __shfl_xor_sync(0xffffffffu, one_min, o));
            if (lane == 0) sm.red[4 * kWarps + warp] = one_min;
            __syncthreads();
            if (warp == 0) {                 // queue: the gamma of the smallest bound first, then ascending
                double v = dinf();
                int a = ng;
                #pragma unroll 1
                for (int gi = lane; gi < ng; gi += 32)
                    if (sm.glb[gi] < v) { v = sm.glb[gi]; a = gi; }
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                    const int oa = __shfl_xor_sync(0xffffffffu, a, o);
                    if (ov < v || (ov == v && oa < a)) { v = ov; a = oa; }
                }
                if (a >= ng) a = 0;                                  // all bounds NaN / inf
                #pragma unroll 1
                for (int pos = lane; pos < ng; pos += 32) sm.gord[pos] = pos == 0 ? a : (pos <= a ? pos - 1 : pos);
            }
            if (tid == 0) {
                double m = dinf();
                for (int w = 0; w < kWarps; ++w) m = fmin(m, sm.red[4 * kWarps + w]);
                s_best = m;
            }
            __syncthreads();
        }
        for (int w = 0; w < kWarps; ++w) Tcom = uniform ? fmax(Tcom, sm.red[w]) : Tcom + sm.red[w];
        if constexpr (PHASE == 1) {
            // ---- prep record of scenario s (coalesced), and the outputs that do not need the DPs
            const PrepView pv = prep_view(ws.prep + (size_t)s * C.prep_stride, K, ng);
            #pragma unroll 1
            for (int k = tid; k < K; k += kThreads) {
                out.order[s * K + k] = sm.ord[k];
                pv.Is[k] = sm.Is[k];
                pv.jlo[k] = sm.jlo[k];
            }
            #pragma unroll 1
            for (int k = tid; k < pfx_len(K); k += kThreads) { pv.pI[k] = sm.pI[k]; pv.pI2[k] = sm.pI2[k]; }
            if (!bad && !bad_alpha) {
                #pragma unroll 1
                for (int gi = tid; gi < ng; gi += kThreads) {
                    pv.glb[gi] = sm.glb[gi];
                    pv.L[gi] = sm.tinf[gi];          // L, parked there by the prologue
                    pv.N[gi] = sm.nq[gi];
                }
            }
            if (tid == 0) {
                pv.misc[0] = s_best;
                pv.misc[1] = Tcom;
                pv.flags[0] = (bad ? 1 : 0) | (bad_alpha ? 2 : 0) | (mono ? 4 : 0);
                out.lat[3 * s + 1] = bad ? dnan() : Tcom;
                if (bad || bad_alpha) {              // status 3 / 2: no DP runs (phase 2 skips it)
                    out.lat[3 * s] = dnan();
                    out.lat[3 * s + 2] = dnan();
                    out.gamma[s] = -1;
                    out.M[s] = 0;
                    out.status[s] = bad ? 3 : 2;
                }
            }
            if (bad || bad_alpha) {
                #pragma unroll 1
                for (int k = tid; k < K; k += kThreads) {
                    out.bend[s * K + k] = 0;
                    if (out.trace) out.trace[s * K + k] = 0;
                    if (out.bgam) out.bgam[s * K + k] = 0;
                }
            }
            __syncthreads();
            continue;
        }
        } else {
            // ---- PHASE 2: scenario s's prep record, already in shared memory (or arriving) -- used in place
            mbar_wait(sm.rbar + rcur, (rphase >> rcur) & 1u);
            rphase ^= 1u << rcur;
            const PrepView pv = prep_view(sm.rec + (size_t)rcur * C.prep_stride, K, ng);
            rcur ^= 1;
            sm.Is = pv.Is;
            sm.jlo = pv.jlo;
            sm.pI = pv.pI;
            sm.pI2 = pv.pI2;
            sm.glb = pv.glb;
            const int fl = pv.flags[0];
            bad = fl & 1;
            bad_alpha = (fl & 2) != 0;
            mono = (fl & 4) != 0;
            if (bad || bad_alpha) {              // every output written by phase 1
                __syncthreads();
                continue;
            }
            const double c1d = in.coeffs ? in.coeffs[4 * s] : C.c1d, c2d = in.coeffs ? in.coeffs[4 * s + 1] : C.c2d;
            const double c1v = in.coeffs ? in.coeffs[4 * s + 2] : C.c1v, c2v = in.coeffs ? in.coeffs[4 * s + 3] : C.c2v;
            #pragma unroll 1
            for (int gi = tid; gi < ng; gi += kThreads) {
                const int N = pv.N[gi];
                sm.nq[gi] = N;
                sm.dq[gi] = make_dpconst(C, C.gmin + gi, pv.L[gi], N, c1d, c2d, c1v, c2v);
            }
            if (tid == 0) {
                s_best = pv.misc[0];
                Tcom = pv.misc[1];
                sm.red[0] = Tcom;
            }
            __syncwarp();
            Tcom = sm.red[0];
            {   // queue: the gamma of the smallest bound first, then ascending
                double v = dinf();
                int a = ng;
                #pragma unroll 1
                for (int gi = lane; gi < ng; gi += 32)
                    if (sm.glb[gi] < v) { v = sm.glb[gi]; a = gi; }
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                    const int oa = __shfl_xor_sync(0xffffffffu, a, o);
                    if (ov < v || (ov == v && oa < a)) { v = ov; a = oa; }
                }
                if (a >= ng) a = 0;
                #pragma unroll 1
                for (int pos = lane; pos < ng; pos += 32) sm.gord[pos] = pos == 0 ? a : (pos <= a ? pos - 1 : pos);
            }
            __syncwarp();
        }
        if constexpr (PHASE != 1) {
        // ---- P3: each warp pulls gamma values and runs Algorithm 1
        const bool pbg = C.batch_policy == SDEDGE_BATCH_PER_BATCH_GAMMA;
        if (pbg) {
            if constexpr (sizeof(R) == 8 && G == 1 && !TILE) {   // per-batch gamma: one dense DP (warp 0)
                if (!bad && !bad_alpha && warp == 0) {
                    int Nmax = 0;
                    for (int q = lane; q < ng; q += 32) Nmax = max(Nmax, sm.nq[q]);
                    Nmax = __reduce_max_sync(0xffffffffu, Nmax);
                    const double t = dp_pbg(C, sm, ws.ybuf + (size_t)blockIdx.x * C.ybuf_stride, Nmax, Scta,
                                            Scta + (size_t)ng * K, wc);
                    if (lane == 0) sm.tinf[0] = t;
                }
            }
        } else if (!bad && !bad_alpha) {
            // exact gamma-level pruning before the first row, for the proposed
            // policy: a gamma whose lower bound exceeds the best finished (or seeded) T_inf can
            // neither win nor tie -- it is dropped from the queue without a DP call
            const bool prune = SDEDGE_GAMMA_ABORT && mono && C.batch_policy == SDEDGE_BATCH_PROPOSED;
            const double mg = sizeof(R) == 8 ? 1e-11 : 1e-4;
            // one warp and <= 32 gammas: lane p holds queue position p; the queue is a register mask
            const bool lanes_q = kWarps == 1 && ng <= 32;
            const int q_l = lanes_q && lane < ng ? sm.gord[lane] : 0;
            const double glb_l = lanes_q && lane < ng ? sm.glb[q_l] : 0.0;
            unsigned left = lanes_q ? (ng == 32 ? 0xffffffffu : ((1u << ng) - 1u)) : 0u;
            bool ran = false;                    // a DP of this scenario has finished
            for (;;) {
                // the next G unpruned gammas of the queue (most promising first)
                int mine = -1;
                if (lanes_q) {
                    const bool dead = prune && glb_l * (1.0 - mg) > s_best * (1.0 + mg);
                    const unsigned deadm = __ballot_sync(0xffffffffu, ((left >> lane) & 1u) && dead);
                    if ((deadm >> lane) & 1u) sm.tinf[q_l] = dinf();
                    left &= ~deadm;
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        int pos = left ? __ffs(left) - 1 : -1;
                        if (pos >= 0) left &= left - 1u;
                        int sel = __shfl_sync(0xffffffffu, q_l, pos >= 0 ? pos : 0);
                        // a gamma that is not the scenario's first DP must also pass the batch-count bound
                        if constexpr (G == 1 && TILE != 0)
                            while (pos >= 0 && prune && s_best < dinf() && (SDEDGE_LBB_FIRST || ran) &&
                                   lb_batches(sm, sm.dq[sel], K) * (1.0 - mg) > s_best * (1.0 + mg)) {
                                if (lane == 0) sm.tinf[sel] = dinf();
                                pos = left ? __ffs(left) - 1 : -1;
                                if (pos >= 0) left &= left - 1u;
                                sel = __shfl_sync(0xffffffffu, q_l, pos >= 0 ? pos : 0);
                            }
                        if (g == grp) mine = pos >= 0 ? sel : -1;
                    }
                } else {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    int sel = -1;
                    if (lane == 0)
                        for (;;) {
                            const int pos = atomicAdd(&sm.ctl[0], 1);
                            if (pos >= ng) break;
                            const int q = sm.gord[pos];
                            if (prune && sm.glb[q] * (1.0 - mg) > s_best * (1.0 + mg)) { sm.tinf[q] = dinf(); continue; }
                            sel = q;
                            break;
                        }
                    sel = __shfl_sync(0xffffffffu, sel, 0);
                    if (g == grp) mine = sel;
                    if (g == 0 && sel < 0) break;
                }
                }
                const int first = __shfl_sync(0xffffffffu, mine, 0);
                if (first < 0) break;
                const bool active = mine >= 0;       // an idle group repeats the first gamma without writing
                const int gi = active ? mine : first;
                bool ovf = false;
                short* Sg = active ? Scta + (size_t)gi * K : nullptr;
                const short* jf = (C.batch_policy >= SDEDGE_BATCH_NONE && C.batch_policy <= SDEDGE_BATCH_MAX)
                                      ? sm.jf : nullptr;
                double t = 0.0;
                // baselines run only in the G = 1, untiled instantiations (launch_all), so the
                // other instantiations compile just their own DP (fewer live registers)
                constexpr bool kBase = G == 1 && !TILE;
                if constexpr (TILE) {
                    t = dp_gamma_tiled<R, G, TILE == 2>(C, sm, rw, pl, tb, stage, bars, bar_phase, st0, tb_stride, rw0,
                                             C.rows_stride, gi,
                                             Sg, &ovf, wc, &s_top[warp * G + grp], active,
                                             (SDEDGE_GAMMA_ABORT && mono) ? &s_best : nullptr, sm.glb[gi], mono);
                } else if (kBase && C.batch_policy == SDEDGE_BATCH_HEURISTIC) {
                    // heuristic batching (reading B5): equal batches of size
                    // 2, 3, ... in sorted order until the pipelined latency stops improving
                    short* jw = sm.jw + (size_t)warp * K;
                    auto plan = [&](int b) {
                        #pragma unroll 1
                        for (int r = lane; r < K; r += 32) {
                            const int e = r + 1;
                            jw[r] = (short)((e % b == 0 || e == K) ? ((e - 1) / b) * b + 1 : 0);
                        }
                        __syncwarp();
                    };
                    double tb = dinf();
                    int bb = 1;
                    const int b0 = (C.flags & SDEDGE_FLAG_HEURISTIC_HALF) ? (K + 1) / 2 : (K >= 2 ? 2 : 1);
                    for (int b = b0; b <= K; ++b) {
                        plan(b);
                        const double tt = dp_gamma<R, ALGO, G>(C, sm, rw, pl, C.gmin + gi, SDEDGE_SCEN_ARGS,
                                                               nullptr, &ovf, wc, &s_top[warp * G + grp],
                                                               active, jw);
                        if (!(tt < tb) && !isinf(tb)) break;       // latency starts to degrade
                        if (isinf(tt)) break;                      // memory binds
                        tb = tt;
                        bb = b;
                    }
                    if (isinf(tb)) bb = 1;
                    plan(bb);
                    t = dp_gamma<R, ALGO, G>(C, sm, rw, pl, C.gmin + gi, SDEDGE_SCEN_ARGS, Sg, &ovf, wc,
                                             &s_top[warp * G + grp], active, jw);
                } else {
                    t = dp_gamma<R, ALGO, G>(C, sm, rw, pl, C.gmin + gi, SDEDGE_SCEN_ARGS, Sg, &ovf, wc,
                                             &s_top[warp * G + grp], active, kBase ? jf : nullptr);
                }
                if (lane % GL == 0 && active) {
                    sm.tinf[gi] = t;
                    if (ovf) s_ovf = true;
                }
                ran = true;
                {   // best finished T_inf so far (gamma-level pruning of the later DPs)
                    double tv = (lane % GL == 0 && active) ? t : dinf();
#pragma unroll
                    for (int o = GL; o < 32; o <<= 1) tv = fmin(tv, __shfl_xor_sync(0xffffffffu, tv, o));
                    if (lane == 0 && tv < s_best) s_best = tv;
                    __syncwarp();
                }
            }
        }
        __syncthreads();

        if (s_ovf && !BIG) {
            // hand the scenario to the big-pool pass (outputs written there)
            if (tid == 0) {
                const unsigned int at = atomicAdd(ws.ovf_count, 1u);
                ws.ovf_list[at] = s;
            }
            __syncthreads();
            continue;
        }


        // ---- gamma* (smallest argmin, reading A7) and backtrack (reading A5)
        double wbest = dinf();
        int wg = -1;
        if (kWarps == 1 && ng <= 32 && !pbg) {   // one warp: the argmin as a butterfly (ties -> smaller gamma)
            if (lane < ng) { wbest = sm.tinf[lane]; wg = wbest < dinf() ? lane : -1; }
            if (wg < 0) wg = 0x7fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, wbest, o);
                const int og = __shfl_xor_sync(0xffffffffu, wg, o);
                if (ob < wbest || (ob == wbest && og < wg)) { wbest = ob; wg = og; }
            }
            if (wg == 0x7fffffff) wg = -1;
        }
        if (tid == 0) {
            int st = 0, gbest = -1, M = 0;
            double best = dinf();
            if (bad) st = 3;
            else if (bad_alpha) st = 2;
            else if (s_ovf) st = 5;          // cannot happen with the worst-case pool
            else if (pbg) {
                best = sm.tinf[0];
                gbest = best < dinf() ? 0 : -1;
                if (gbest < 0) st = 1;
            } else if (kWarps == 1 && ng <= 32) {
                best = wbest;
                gbest = wg;
                if (gbest < 0) st = 1;
            } else {
                #pragma unroll 1
                for (int gi = 0; gi < ng; ++gi)
                    if (sm.tinf[gi] < best) { best = sm.tinf[gi]; gbest = gi; }
                if (gbest < 0) st = 1;
            }
            double* lat = out.lat + 3 * s;
            sm.ctl[4] = gbest;
            if (st == 0) {
                const short* S = Scta + (size_t)gbest * K;
                int i = K;
                short* stk = bstack;                                  // dead scratch: a stack
                while (i > 0) { stk[M++] = (short)i; i = S[i - 1] - 1; }
                lat[0] = Tcom + best; lat[1] = Tcom; lat[2] = best;
                out.gamma[s] = pbg ? (int)Scta[(size_t)ng * K + K - 1] : C.gmin + gbest;   // pbg: the last batch's
            } else {
                const double nan = dnan();
                lat[0] = st == 1 ? dinf() : nan;
                lat[1] = st == 3 || st == 5 ? nan : Tcom;
                lat[2] = st == 1 ? dinf() : nan;
                out.gamma[s] = -1;
            }
            out.M[s] = M;
            out.status[s] = st;
            sm.ctl[2] = M;
            sm.ctl[3] = bad;
        }
        __syncthreads();
        const int M = sm.ctl[2];
        #pragma unroll 1
        for (int k = tid; k < K; k += kThreads) {
            if (PHASE != 2) out.order[s * K + k] = sm.ord[k];
            out.bend[s * K + k] = k < M ? bstack[M - 1 - k] : 0;
        }
        if (out.bgam)                        // each batch's gamma (gamma* for all unless per-batch)
            #pragma unroll 1
            for (int k = tid; k < K; k += kThreads)
                out.bgam[s * K + k] = k >= M ? 0 : pbg ? (int32_t)Scta[(size_t)ng * K + bstack[M - 1 - k] - 1]
                                                       : C.gmin + sm.ctl[4];
        if (out.trace) {                     // S vector of gamma* (row choices; 0 unless status 0)
            const short* S = Scta + (size_t)max(sm.ctl[4], 0) * K;
            #pragma unroll 1
            for (int k = tid; k < K; k += kThreads) out.trace[s * K + k] = M > 0 ? (int32_t)S[k] : 0;
        }

        __syncthreads();
        }   // PHASE != 1
    }
    if (out.work) {
        __syncthreads();
        if (tid < 5) {
            unsigned long long v = 0;
            #pragma unroll 1
            for (int t = 0; t < kThreads; ++t) v += s_work[t * 5 + tid];
            atomicAdd(out.work + tid, v);
        }
    }
}

// ------------------------------------------------------------ actual-output evaluation
// One warp per scenario (grid-stride).  Per batch: b_m, padded I_m and the
// closed-form stage coefficients (D1) go to shared memory with
// n_m = ceil(O_m / L) (exact IEEE sequence, reading A2); lanes then take steps
// n and run the eq:time recursion over the batches still active at n.
struct ActBatch {
    double td1, ad, bd, tv1, av, bv;   // T^d_1, T^d_n = ad + bd (n-1); T^v likewise (already x b, + c2)
    int nm, pad;
};

__global__ void __launch_bounds__(128)
actual_kernel(const Consts C, const Inputs in, const int32_t* __restrict__ O, const int32_t* __restrict__ gam,
              const int32_t* __restrict__ Mv, const int32_t* __restrict__ bend, const int32_t* __restrict__ order,
              const int32_t* __restrict__ status, long long n, double* __restrict__ out)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int K = C.K, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    ActBatch* bt = reinterpret_cast<ActBatch*>(smem_raw) + (size_t)warp * K;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long s = (long long)blockIdx.x * (blockDim.x >> 5) + warp; s < n; s += nw) {
        const int M = Mv[s];
        const int g = gam[s];
        if (status[s] != 0 || M < 1 || M > K || g < 0 || g > 64) {
            if (lane == 0) out[s] = dnan();
            continue;
        }
        {   // the plan is caller data: batch ends strictly increasing in [1, K] ending at K, order a
            // permutation range -- anything else yields NaN instead of out-of-bounds reads
            int badp = 0;
            for (int m = lane; m < M; m += 32) {
                const int e = bend[s * K + m], pv = m ? bend[s * K + m - 1] : 0;
                badp |= e < 1 || e > K || e <= pv || (m == M - 1 && e != K);
            }
            for (int q = lane; q < K; q += 32) {
                const int o = order[s * K + q];
                badp |= o < 0 || o >= K;
            }
            if (__any_sync(0xffffffffu, badp)) {
                if (lane == 0) out[s] = dnan();
                continue;
            }
        }
        const double alpha = in.alpha[s];
        double c1d = C.c1d, c2d = C.c2d, c1v = C.c1v, c2v = C.c2v;
        if (in.coeffs) {
            c1d = in.coeffs[4 * s]; c2d = in.coeffs[4 * s + 1];
            c1v = in.coeffs[4 * s + 2]; c2v = in.coeffs[4 * s + 3];
        }
        const double L = expected_tokens(alpha, g);
        DPConst D;
        D.g = g;
        D.tri = D.g * (D.g - 1.0) * 0.5;
        D.kd = c1d * (4.0 * C.Jd * (double)C.hd);
        D.kv = c1v * (4.0 * C.Jv * (double)C.hv);
        D.hd2 = 2.0 * C.hd + C.h2d;
        D.hv2 = 2.0 * C.hv + C.h2v;
        D.bdc = D.kd * D.g * L;
        D.bvc = D.kv * (1.0 + D.g) * L;
        D.c2dg = D.g * c2d;
        D.c2vv = c2v + C.dl;
        D.Mx = 0.0;
        D.sumM = 0.0;
        int nmax = 0, bad = 0;
        for (int m = lane; m < M; m += 32) {
            const int e = bend[s * K + m], st = m ? bend[s * K + m - 1] + 1 : 1;
            int Om = 0;
            for (int q = st; q <= e; ++q) {
                const int o = O[s * K + order[s * K + q - 1]];
                Om = max(Om, o);
                bad |= o < 1;
            }
            const int I = in.I[s * K + order[s * K + e - 1]];
            const RowCoef rc = row_coef(D, I);
            const double b = e - st + 1;
            ActBatch a;
            a.td1 = fma(b, rc.td1, D.c2dg);
            a.ad = fma(b, rc.ad, D.c2dg);
            a.bd = b * D.bdc;
            a.tv1 = fma(b, rc.tv1, D.c2vv);
            a.av = fma(b, rc.av, D.c2vv);
            a.bv = b * D.bvc;
            a.nm = (int)ceil(__ddiv_rn((double)Om, L));   // eq:step_n
            a.pad = 0;
            bt[m] = a;
            nmax = max(nmax, a.nm);
        }
        nmax = __reduce_max_sync(0xffffffffu, nmax);
        bad = __reduce_or_sync(0xffffffffu, bad);
        __syncwarp();
        double acc = 0.0;
        for (int step = 1 + lane; step <= nmax; step += 32) {
            const double x = step - 1;
            double Cd = 0.0, Cc = 0.0;
            for (int m = 0; m < M; ++m) {
                const ActBatch a = bt[m];
                if (a.nm < step) continue;                // M_n
                const double td = step == 1 ? a.td1 : fma(a.bd, x, a.ad);
                const double tv = step == 1 ? a.tv1 : fma(a.bv, x, a.av);
                if (C.batch_policy == SDEDGE_BATCH_NO_PIPELINE) { Cc += td + tv; continue; }  // sequential
                Cd += td;                                 // C^d_{n,m}
                Cc = rmax(Cd, Cc) + tv;                   // eq:time
            }
            acc += Cc;                                    // T_n = C_{n, M_n}
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[s] = bad ? dnan() : acc;
        __syncwarp();
    }
}

// ------------------------------------------------------------ exhaustive search
// Exact optimum of the batching subproblem over every contiguous partition of
// the sorted order (the search space of Algorithm 1) and every gamma,
// to measure Algorithm 1's heuristic gap at scale.
// bf_item_kernel: one CTA per (scenario, gamma chunk) item (grid-stride); the chunk
// is one gamma when n is too small to fill one wave of CTAs (the grid then
// balances even at a few hundred scenarios), else all of them; the per-end-position stage coefficients
// (every gamma of the chunk at once) go to shared memory, each warp takes
// (gamma, partition) pairs (bit t of the mask = a batch ends at sorted position t + 1), and its lanes take decoding steps n and run the
// eq:time recursion over the batches, as in actual_kernel.  The item's minimum
// and its first minimising mask go to a workspace; bf_final_kernel (one warp per
// scenario) takes the smallest gamma among the minima.  Ties therefore keep the
// first plan in (gamma, mask) order (the oracle's exhaustive search does the same).
constexpr int kBFMaxK = 20;
constexpr int kBFWarps = 8;

constexpr int kBFMaxG = 65;     // gamma_max - gamma_min + 1 <= 65 (gamma in 0..64)

struct BFCoef { double td1, ad, tv1, av; };       // row_coef's stage terms (x b, + c2)
struct BFGam { double bdc, bvc, c2dg, c2vv; int N, pad; };

__global__ void __launch_bounds__(kBFWarps * 32, 4)
bf_item_kernel(const Consts C, const Inputs in, long long items, int gc, double* __restrict__ wsv,
               int32_t* __restrict__ wsg, unsigned* __restrict__ wsm, unsigned long long* work)
{
    __shared__ int Is[kBFMaxK], bmx[kBFMaxK];
    __shared__ BFCoef rcs[kBFMaxG * kBFMaxK];       // [gamma of the chunk][sorted end position]
    __shared__ BFGam gms[kBFMaxG];
    __shared__ double wv[kBFWarps];
    __shared__ unsigned wm[kBFWarps];
    __shared__ int wgs[kBFWarps];
    const int K = C.K, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned nmask = 1u << (K - 1), last = 1u << (K - 1);
    const bool nopipe = C.batch_policy == SDEDGE_BATCH_NO_PIPELINE;
    const int nch = (C.ng + gc - 1) / gc;                // gamma chunks per scenario
    unsigned long long plans = 0, bsteps = 0;
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const long long s = it / nch;
        const int g0 = C.gmin + (int)(it - s * nch) * gc, gn = min(gc, C.gmin + C.ng - g0);
        __syncthreads();                                 // previous item's readers are done
        int bad = 0;
        for (int k = tid; k < K; k += blockDim.x) {      // stable rank sort
            const int Ik = in.I[s * K + k];
            bad |= Ik < 1;
            int r = 0;
            for (int q = 0; q < K; ++q) {
                const int Iq = in.I[s * K + q];
                r += (Iq < Ik) || (Iq == Ik && q < k);
            }
            Is[r] = Ik;
        }
        bad = __syncthreads_or(bad);
        const double alpha = in.alpha[s];
        if (bad || !(alpha > 0.0 && alpha < 1.0)) {      // status 3 / 2: set by bf_final_kernel
            if (tid == 0) { wsv[it] = kinf<double>(); wsg[it] = -1; wsm[it] = 0xffffffffu; }
            continue;
        }
        double c1d = C.c1d, c2d = C.c2d, c1v = C.c1v, c2v = C.c2v;
        if (in.coeffs) {
            c1d = in.coeffs[4 * s]; c2d = in.coeffs[4 * s + 1];
            c1v = in.coeffs[4 * s + 2]; c2v = in.coeffs[4 * s + 3];
        }
        // stage coefficients of every gamma of the chunk at once, so warps run through
        // (gamma, mask) pairs without a barrier per gamma
        for (int q = tid; q < gn * K + K; q += blockDim.x) {
            if (q >= gn * K) {                           // memory window
                const int r = q - gn * K;
                const long long room = C.gamma_s - C.Gp;
                const long long b = room >= 0 ? room / (C.kvunit * ((long long)Is[r] + C.O_max)) : 0;
                bmx[r] = (int)(b < K ? b : K);
                continue;
            }
            const int gi = q / K, r = q - gi * K, g = g0 + gi;
            const double L = expected_tokens(alpha, g);
            DPConst D;
            D.g = g;
            D.tri = D.g * (D.g - 1.0) * 0.5;
            D.kd = c1d * (4.0 * C.Jd * (double)C.hd);
            D.kv = c1v * (4.0 * C.Jv * (double)C.hv);
            D.hd2 = 2.0 * C.hd + C.h2d;
            D.hv2 = 2.0 * C.hv + C.h2v;
            D.bdc = D.kd * D.g * L;
            D.bvc = D.kv * (1.0 + D.g) * L;
            D.c2dg = D.g * c2d;
            D.c2vv = c2v + C.dl;
            D.Mx = 0.0;
            D.sumM = 0.0;
            const RowCoef rc = row_coef(D, Is[r]);
            rcs[gi * K + r] = BFCoef{rc.td1, rc.ad, rc.tv1, rc.av};
            if (r == 0)
                gms[gi] = BFGam{D.bdc, D.bvc, D.c2dg, D.c2vv,
                                (int)ceil(__ddiv_rn((double)C.O_max, L)), 0};   // eq:step_n, O = O_max
        }
        __syncthreads();
        double best = kinf<double>();
        int bg = -1;
        unsigned bm = 0xffffffffu;
        const unsigned total = (unsigned)gn * nmask;
        for (unsigned w = warp; w < total; w += kBFWarps) {   // (gamma, mask) ascending per warp
            const int gi = (int)(w >> (K - 1));
            const unsigned mask = w & (nmask - 1);
            const unsigned ends = mask | last;
            bool ok = true;
            int M = 0;
            for (unsigned m = ends, st = 1; m; m &= m - 1) {   // constraint (b) per batch
                const int e = __ffs(m);
                ok &= (e - (int)st + 1) <= bmx[e - 1];
                st = e + 1;
                ++M;
            }
            if (!ok) continue;
            const BFGam G = gms[gi];
            const BFCoef* rg = rcs + gi * K;
            double acc = 0.0;
            if (lane == 0) {                             // step n = 1 (prefill + first drafts), peeled
                double Cd = 0.0, Cc = 0.0;
                for (unsigned m = ends, st = 1; m; m &= m - 1) {
                    const int e = __ffs(m);
                    const double b = e - (int)st + 1;
                    st = e + 1;
                    const double td = fma(b, rg[e - 1].td1, G.c2dg), tv = fma(b, rg[e - 1].tv1, G.c2vv);
                    if (nopipe) { Cc += td + tv; continue; }
                    Cd += td;
                    Cc = rmax(Cd, Cc) + tv;
                }
                acc = Cc;
            }
            for (int step = lane == 0 ? 33 : 1 + lane; step <= G.N; step += 32) {
                const double x = step - 1;
                const double xd = G.bdc * x, xv = G.bvc * x;    // slopes in n of the per-task stage times
                double Cd = 0.0, Cc = 0.0;
                for (unsigned m = ends, st = 1; m; m &= m - 1) {
                    const int e = __ffs(m);
                    const double b = e - (int)st + 1;
                    st = e + 1;
                    const BFCoef& r = rg[e - 1];         // padded to the batch's longest input
                    const double td = fma(b, r.ad + xd, G.c2dg);   // T^d_n = b (ad + bdc (n-1)) + gamma c2d
                    const double tv = fma(b, r.av + xv, G.c2vv);   // T^v_n = b (av + bvc (n-1)) + c2v
                    if (nopipe) { Cc += td + tv; continue; }
                    Cd += td;                            // C^d_{n,m}
                    Cc = rmax(Cd, Cc) + tv;              // eq:time
                }
                acc += Cc;                               // T_n = C_{n,M}
            }
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            acc = __shfl_sync(0xffffffffu, acc, 0);      // warp-uniform decision
            ++plans;
            bsteps += (unsigned long long)G.N * M;
            if (acc < best) { best = acc; bg = g0 + gi; bm = mask; }
        }
        if (lane == 0) { wv[warp] = best; wgs[warp] = bg; wm[warp] = bm; }
        __syncthreads();
        if (tid == 0) {
            double v = kinf<double>();
            int gb = -1;
            unsigned mk = 0xffffffffu;
            for (int w = 0; w < kBFWarps; ++w)          // lexicographic (T_inf, gamma, mask)
                if (wgs[w] >= 0 && (gb < 0 || wv[w] < v ||
                                    (wv[w] == v && (wgs[w] < gb || (wgs[w] == gb && wm[w] < mk))))) {
                    v = wv[w];
                    gb = wgs[w];
                    mk = wm[w];
                }
            wsv[it] = v;
            wsg[it] = gb;
            wsm[it] = mk;
        }
    }
    if (work) {
        for (int o = 16; o > 0; o >>= 1) {
            plans += __shfl_xor_sync(0xffffffffu, plans, o);
            bsteps += __shfl_xor_sync(0xffffffffu, bsteps, o);
        }
        if (lane == 0) {          // plans/bsteps are lane-uniform: count once per warp
            atomicAdd(work + 0, plans / 32);
            atomicAdd(work + 1, bsteps / 32);
        }
    }
}

__global__ void __launch_bounds__(128)
bf_final_kernel(const Consts C, const Inputs in, long long n, int nch, const double* __restrict__ wsv,
                const int32_t* __restrict__ wsg, const unsigned* __restrict__ wsm, double* __restrict__ out_t, int32_t* __restrict__ og,
                int32_t* __restrict__ oM, int32_t* __restrict__ obend, int32_t* __restrict__ oorder,
                int32_t* __restrict__ ostatus)
{
    const int K = C.K, lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long s = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < n; s += nw) {
        int rank = 0, bad = 0;
        if (lane < K) {                                  // stable rank of task `lane`
            const int Ik = in.I[s * K + lane];
            bad = Ik < 1;
            for (int q = 0; q < K; ++q) {
                const int Iq = in.I[s * K + q];
                rank += (Iq < Ik) || (Iq == Ik && q < lane);
            }
        }
        bad = __reduce_or_sync(0xffffffffu, bad);
        const double alpha = in.alpha[s];
        double v = kinf<double>();
        int g = -1;
        unsigned mk = 0;
        for (int c = 0; c < nch; ++c) {                  // smallest gamma among equal minima
            const double x = wsv[s * nch + c];
            const int gc = wsg[s * nch + c];
            if (gc >= 0 && (g < 0 || x < v)) { v = x; g = gc; mk = wsm[s * nch + c]; }
        }
        const int st = bad ? 3 : (!(alpha > 0.0 && alpha < 1.0) ? 2 : (g < 0 ? 1 : 0));
        const unsigned ends = mk | (1u << (K - 1));
        const int M = st ? 0 : __popc(ends);
        if (lane < K) {
            oorder[s * K + rank] = lane;
            int32_t be = 0;
            if (st == 0 && lane < M) {                   // position of the (lane+1)-th set bit
                unsigned m = ends;
                for (int t = 0; t < lane; ++t) m &= m - 1;
                be = __ffs(m);
            }
            obend[s * K + lane] = be;
        }
        if (lane == 0) {
            out_t[s] = st == 0 ? v : (st == 1 ? kinf<double>() : dnan());
            og[s] = st ? -1 : g;
            oM[s] = M;
            ostatus[s] = st;
        }
    }
}

// ------------------------------------------------------------ pipe-peak microbenchmark
template <typename T>
__global__ void pipe_peak_kernel(T* sink, int iters, T seed)
{
    T a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
      a6 = a0 + 6, a7 = a0 + 7;
    const T m = (T)0.999999, c = (T)1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
            a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
        }
    }
    const T r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == (T)-1) sink[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// ------------------------------------------------------------ host side
int validate(const sdedge_scenarios* s, int64_t n, const sdedge_params* p, const double* lat,
             const sdedge_schedule* o)
{
    if (!s || !p || !o) return fail(-1, "null argument");
    if (n < 0) return fail(-1, "n < 0");
    if (p->K < 1 || p->K > SDEDGE_MAX_K) return fail(-1, "K outside 1..1024");
    if (p->gamma_min < 0 || p->gamma_max < p->gamma_min || p->gamma_max > 64)
        return fail(-1, "need 0 <= gamma_min <= gamma_max <= 64");
    if (p->O_max < 1 || p->O_max > (1 << 20)) return fail(-1, "O_max outside 1..2^20");
    const sdedge_model* ms[2] = {&p->draft, &p->verify};
    for (const sdedge_model* m : ms)
        if (m->layers < 1 || m->layers > 1024 || m->hidden < 1 || m->hidden > 65536 || m->ffn < 1 ||
            m->ffn > (1 << 20))
            return fail(-1, "model dims outside J in 1..1024, h1 in 1..65536, h2 in 1..2^20");
    const double cs[4] = {p->c1_draft, p->c2_draft, p->c1_verify, p->c2_verify};
    for (double c : cs)
        if (!(c >= 0.0) || !std::isfinite(c)) return fail(-1, "runtime coefficients must be finite and >= 0");
    if (!(p->bandwidth_hz > 0) || !std::isfinite(p->bandwidth_hz)) return fail(-1, "bandwidth_hz must be > 0");
    if (!(p->noise_w > 0) || !std::isfinite(p->noise_w)) return fail(-1, "noise_w must be > 0");
    if (!std::isfinite(p->lambda_bits)) return fail(-1, "lambda_bits must be finite");
    if (p->mem_capacity_bytes < 0) return fail(-1, "mem_capacity_bytes < 0");
    if (p->precision != 0 && p->precision != 1) return fail(-1, "precision must be 0 (fp64) or 1 (fp32)");
    if (p->algo != SDEDGE_ALGO_ENVELOPE && p->algo != SDEDGE_ALGO_DENSE) return fail(-1, "unknown algo");
    if (p->flags & ~(SDEDGE_FLAG_TINY_POOL | SDEDGE_FLAG_HEURISTIC_HALF)) return fail(-1, "unknown flags");
    if (p->bandwidth_policy != SDEDGE_BW_OPTIMAL && p->bandwidth_policy != SDEDGE_BW_UNIFORM)
        return fail(-1, "unknown bandwidth_policy");
    if (p->batching_policy < SDEDGE_BATCH_PROPOSED || p->batching_policy > SDEDGE_BATCH_PER_BATCH_GAMMA)
        return fail(-1, "unknown batching_policy");
    if (p->batching_policy == SDEDGE_BATCH_PER_BATCH_GAMMA) {
        if (p->precision != 0) return fail(-1, "per-batch gamma is fp64 only");
        if (p->gamma_max - p->gamma_min + 1 > 32) return fail(-1, "per-batch gamma: at most 32 speculation lengths");
        if ((long long)(p->K + 1) * (3LL * p->O_max + 1) * 8 > (2LL << 30)) return fail(-1, "per-batch gamma: (K+1) O_max too large");
    }
    if (p->batching_policy == SDEDGE_BATCH_STATIC && p->static_batch < 1) return fail(-1, "static_batch < 1");
    if (p->reserved != 0) return fail(-1, "reserved must be 0");
    if (!(p->downlink_s >= 0) || !std::isfinite(p->downlink_s)) return fail(-1, "downlink_s must be >= 0");
    if (n > 0) {
        if (!s->input_len || !s->tx_power_w || !s->gain || !s->alpha) return fail(-1, "null scenario array");
        if (!lat || !o->gamma || !o->num_batches || !o->batch_end || !o->order || !o->status)
            return fail(-1, "null output array");
    }
    return 0;
}

#define CU(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            snprintf(g_err, sizeof(g_err), "%s: %s", #x, cudaGetErrorString(e_)); \
            return e_ == cudaErrorMemoryAllocation ? -3 : -2;                   \
        }                                                                       \
    } while (0)

// Stream-ordered workspace comes from ONE library-private memory pool per device
// (created on first use, release threshold "never", so the workspace stays cached
// between calls); the device's default pool -- and every other allocator of the
// caller's process -- is left untouched.
int lib_pool(int dev, cudaMemPool_t* out)
{
    static std::mutex mu;
    static cudaMemPool_t pools[256] = {};
    if (dev < 0 || dev >= 256) return fail(-1, "device ordinal out of range");
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pl = nullptr;
        CU(cudaMemPoolCreate(&pl, &props));
        unsigned long long thr = ~0ULL;
        CU(cudaMemPoolSetAttribute(pl, cudaMemPoolAttrReleaseThreshold, &thr));
        pools[dev] = pl;
    }
    *out = pools[dev];
    return 0;
}

// cudaMallocAsync from the library pool of the current device
int ws_alloc(void** ptr, size_t bytes, cudaStream_t st)
{
    int dev = 0;
    CU(cudaGetDevice(&dev));
    cudaMemPool_t pl = nullptr;
    if (int rc = lib_pool(dev, &pl)) return rc;
    CU(cudaMallocFromPoolAsync(ptr, bytes, pl, st));
    return 0;
}

template <typename R, int ALGO, int G, int TILE>
int launch_all(const Consts& C0, const Inputs& in, const Outputs& out, long long n, cudaStream_t st, int flags)
{
    int dev = 0, nsm = 0, max_smem = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CU(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));

    Consts C = C0;
    const size_t rb = rows_bytes<R>(C.K);
    // row state in shared memory when it keeps >= 3 CTAs (12 warps) per SM
    // row state in shared memory when it keeps >= 3 CTAs per SM (untiled), always for TILE == 2
    C.rows_in_smem = TILE == 2 ? 1 : (!TILE && smem_bytes<R, G>(C.K, C.ng, 1, 0) <= (size_t)(220 * 1024 / 3) ? 1 : 0);
    size_t sb = smem_bytes<R, G>(C.K, C.ng, C.rows_in_smem, TILE == 1, TILE == 2 ? rs_pad(C.K, 32 / G) : 0);
    // Envelope-segment pool of the first pass in shared memory (TILE == 2) when the draft stage is
    // the slower one: then envelopes have several segments and the merge / sums walk the pool on
    // every update.  The decision compares the per-token cost of a draft pass with a verify pass
    // (the params' coefficients; per-scenario coefficients do not change it -- it only places
    // memory).  A DP that outgrows this smaller pool is redone by the worst-case pass.
    const double draft_per_tok = C.c1d * C.Jd * (double)C.hd, verify_per_tok = C.c1v * C.Jv * (double)C.hv;
    C.pool_smem = (SDEDGE_POOL_SMEM && TILE == 2 && G == 1 && kWarps == 1 && !(flags & SDEDGE_FLAG_TINY_POOL) && draft_per_tok > verify_per_tok) ? 1 : 0;
    C.pool_cap_smem = ((2LL * (C.K + 1) + 32) + 7) & ~7LL;
    if (C.pool_smem) sb += (pool_bytes<R>(C.pool_cap_smem) + 15) & ~(size_t)15;
    if (sb > (size_t)max_smem) return fail(-1, "shared memory requirement exceeds the device limit");
    C.rows_stride = (long long)((rb + 255) & ~(size_t)255);

    // tiled (TILE != 0): two kernels, prep (PHASE 1) then the DPs (PHASE 2); otherwise one fused kernel
    using KFn = void (*)(const Consts, const Inputs, const Outputs, long long, Work, int);
    KFn k_main;
    if constexpr (TILE == 2) k_main = solve_kernel<R, ALGO, 1, G, 2, 2>;
    else if constexpr (TILE == 1) k_main = solve_kernel<R, ALGO, 0, G, 1, 2>;
    else k_main = C.rows_in_smem ? solve_kernel<R, ALGO, 1, G, 0, 0> : solve_kernel<R, ALGO, 0, G, 0, 0>;
    KFn k_big = k_main;
    // the prep kernel does not depend on the row store: one instantiation serves TILE 1 and 2
    KFn k_prep = TILE ? solve_kernel<R, ALGO, 0, G, 1, 1> : k_main;
    const size_t sb_prep = smem_bytes<R, G>(C.K, C.ng, 0, 0);
    C.prep_stride = TILE ? (long long)prep_stride(C.K, C.ng) : 0;
    if (TILE) sb = smem_bytes<R, G>(C.K, C.ng, C.rows_in_smem, TILE == 1, TILE == 2 ? rs_pad(C.K, 32 / G) : 0,
                                    (int)C.prep_stride) + (C.pool_smem ? (pool_bytes<R>(C.pool_cap_smem) + 15) & ~(size_t)15 : 0);
    CU(cudaFuncSetAttribute(k_main, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    CU(cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    int occ_prep = 0;
    if (TILE) {
        CU(cudaFuncSetAttribute(k_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb_prep));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_prep, k_prep, kThreads, sb_prep));
        if (occ_prep < 1) return fail(-1, "prep kernel does not fit on an SM");
    }
    if (sb > (size_t)max_smem) return fail(-1, "shared memory requirement exceeds the device limit");
    int occ = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_main, kThreads, sb));
    if (occ < 1) return fail(-1, "kernel does not fit on an SM");
    long long grid = (long long)nsm * occ;
    const bool pbg = C.batch_policy == SDEDGE_BATCH_PER_BATCH_GAMMA;
    // per-batch gamma: (K+1) Upsilon rows of 3 Nmax + 1 doubles per CTA (Nmax <= O_max); <= SDEDGE_PBG_WS_GIB in all
    C.ybuf_stride = pbg ? (long long)(C.K + 1) * (3 * (long long)C.O_max + 1) : 0;
    if (pbg) grid = std::max(1LL, std::min(grid, (kPbgWorkspace) / (8 * C.ybuf_stride)));
    if (grid > n) grid = n;

    // typical envelopes have <= a few segments per row: 4 (K+1) + 64 extra
    // segments per warp; a DP that overflows is redone by the big-pool pass
    // with the worst-case bound sum_i 2i = K(K+1) (D3).
    const long long cap_main = (flags & SDEDGE_FLAG_TINY_POOL) ? 8LL : (4LL * (C.K + 1) + 64 + 7) & ~7LL;
    const long long cap_big = ((long long)C.K * (C.K + 1) + 64 + 7) & ~7LL;
    long long grid_big = std::max(1LL, std::min(std::min((long long)nsm, std::max(n, 1LL)),
                                  (2LL << 30) / (long long)(kWarps * G * pool_bytes<R>(cap_big))));
    if (pbg) grid_big = 1;                   // no envelopes: the second pass has nothing to do
    const long long slots = grid * kWarps * G, slots_big = grid_big * kWarps * G;

    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
    const size_t o_next = take(3 * sizeof(unsigned long long) + sizeof(unsigned int));
    const size_t o_prep = take((size_t)n * C.prep_stride);
    const size_t o_S = take((size_t)std::max(grid, grid_big) * (C.ng + 1) * C.K * sizeof(short));
    const size_t o_list = take((size_t)n * sizeof(long long));
    const size_t o_rows = take(C.rows_in_smem ? 0 : (size_t)std::max(slots, slots_big) * C.rows_stride);
    const size_t o_pool = take((size_t)slots * pool_bytes<R>(cap_main));
    const size_t o_pool_big = take(pbg ? 0 : (size_t)slots_big * pool_bytes<R>(cap_big));
    const size_t o_ybuf = take((size_t)grid * C.ybuf_stride * sizeof(double));
    unsigned char* wsb = nullptr;
    if (int rc = ws_alloc(reinterpret_cast<void**>(&wsb), off, st)) return rc;
    CU(cudaMemsetAsync(wsb + o_next, 0, 3 * sizeof(unsigned long long) + sizeof(unsigned int), st));

    Work w;
    w.S = reinterpret_cast<short*>(wsb + o_S);
    w.next = reinterpret_cast<unsigned long long*>(wsb + o_next);
    w.ovf_count = reinterpret_cast<unsigned int*>(wsb + o_next + 3 * sizeof(unsigned long long));
    w.prep = wsb + o_prep;
    w.ovf_list = reinterpret_cast<long long*>(wsb + o_list);
    w.rows = wsb + o_rows;
    w.ybuf = reinterpret_cast<double*>(wsb + o_ybuf);

    int launches = 0;
    if (n > 0) {
        C.pool_cap = cap_main;
        w.pool = wsb + o_pool;
        SmemOff so_prep, so_main;
        smem_layout(C.K, C.ng, 0, &so_prep);
        smem_layout(C.K, C.ng, TILE ? (int)C.prep_stride : 0, &so_main);
        if (TILE) {
            const long long grid_prep = std::min((long long)nsm * occ_prep, n);
            const int tq = kt_begin(KT_PREP, st);
            C.so = so_prep;
            k_prep<<<(unsigned)grid_prep, kThreads, sb_prep, st>>>(C, in, out, n, w, 0);
            kt_end(tq, st);
            ++launches;
            CU(cudaGetLastError());
        }
        int tq = kt_begin(KT_MAIN, st);
        C.so = so_main;
        k_main<<<(unsigned)grid, kThreads, sb, st>>>(C, in, out, n, w, 0);
        kt_end(tq, st);
        ++launches;
        CU(cudaGetLastError());
        C.pool_cap = cap_big;
        w.pool = wsb + o_pool_big;
        tq = kt_begin(KT_BIG, st);
        k_big<<<(unsigned)grid_big, kThreads, sb, st>>>(C, in, out, n, w, 1);
        kt_end(tq, st);
        ++launches;
        CU(cudaGetLastError());
    }
    CU(cudaFreeAsync(wsb, st));
    g_launches = launches;
    return 0;
}

Consts make_consts(const sdedge_params* p)
{
    Consts C{};
    C.K = p->K; C.O_max = p->O_max; C.gmin = p->gamma_min; C.ng = p->gamma_max - p->gamma_min + 1;
    C.Jd = p->draft.layers; C.hd = p->draft.hidden; C.h2d = p->draft.ffn;
    C.Jv = p->verify.layers; C.hv = p->verify.hidden; C.h2v = p->verify.ffn;
    C.c1d = p->c1_draft; C.c2d = p->c2_draft; C.c1v = p->c1_verify; C.c2v = p->c2_verify;
    C.Bw = p->bandwidth_hz; C.sigma2 = p->noise_w; C.isig2 = 1.0 / p->noise_w;
    C.lambda = p->lambda_bits > 0 ? p->lambda_bits : 16.0 * ((double)C.hd + (double)C.hv);
    C.dl = p->downlink_s;
    C.gamma_s = p->mem_capacity_bytes;
    C.Gp = (long long)C.Jd * (8LL * C.hd * C.hd + 4LL * C.hd * C.h2d);                      // eq:memory_model
    C.kvunit = 4LL * C.Jd * C.hd;                                                            // eq:memory_kv
    C.bw_policy = p->bandwidth_policy;
    C.batch_policy = p->batching_policy;
    C.static_batch = p->static_batch;
    C.flags = p->flags;
    return C;
}

int solve_device(const sdedge_scenarios* s, int64_t n, const sdedge_params* p, double* lat,
                 sdedge_schedule* o)
{
    Consts C = make_consts(p);
    Inputs in{s->input_len, s->tx_power_w, s->gain, s->alpha, s->coeffs};
    Outputs out{lat, o->gamma, o->num_batches, o->batch_end, o->order, o->bw_share, o->status,
                reinterpret_cast<unsigned long long*>(o->work_counters), o->row_choice, o->batch_gamma};
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    // envelope, proposed policy: small K -> G DPs per warp with row state in shared
    // memory; larger K -> the tiled DP (rows in global memory, a GL-row shared tile
    // per DP) with SDEDGE_TILE_G DPs per warp.  Baselines and dense: one DP per warp.
    const int f = p->flags;
    const bool base = p->algo == SDEDGE_ALGO_DENSE || p->batching_policy != SDEDGE_BATCH_PROPOSED;
    const bool tiled = !base && p->K > SDEDGE_TILE_MIN_K;
    // tiled DP with the row store in shared memory (no TMA staging) while it stays small
    const bool rs = tiled && p->K <= SDEDGE_RS_MAX_K;
    const int G = base ? 1 : (p->K <= 48 ? 4 : 2);
    if (p->precision == 0) {
        if (p->algo == SDEDGE_ALGO_DENSE) return launch_all<double, SDEDGE_ALGO_DENSE, 1, 0>(C, in, out, n, st, f);
        if (base) return launch_all<double, SDEDGE_ALGO_ENVELOPE, 1, 0>(C, in, out, n, st, f);
        if (rs) return launch_all<double, SDEDGE_ALGO_ENVELOPE, SDEDGE_TILE_G, 2>(C, in, out, n, st, f);
        if (tiled) return launch_all<double, SDEDGE_ALGO_ENVELOPE, SDEDGE_TILE_G, 1>(C, in, out, n, st, f);
        if (G == 4) return launch_all<double, SDEDGE_ALGO_ENVELOPE, 4, 0>(C, in, out, n, st, f);
        return launch_all<double, SDEDGE_ALGO_ENVELOPE, 2, 0>(C, in, out, n, st, f);
    }
    if (p->algo == SDEDGE_ALGO_DENSE) return launch_all<float, SDEDGE_ALGO_DENSE, 1, 0>(C, in, out, n, st, f);
    if (base) return launch_all<float, SDEDGE_ALGO_ENVELOPE, 1, 0>(C, in, out, n, st, f);
    if (rs) return launch_all<float, SDEDGE_ALGO_ENVELOPE, SDEDGE_TILE_G, 2>(C, in, out, n, st, f);
    if (tiled) return launch_all<float, SDEDGE_ALGO_ENVELOPE, SDEDGE_TILE_G, 1>(C, in, out, n, st, f);
    if (G == 4) return launch_all<float, SDEDGE_ALGO_ENVELOPE, 4, 0>(C, in, out, n, st, f);
    return launch_all<float, SDEDGE_ALGO_ENVELOPE, 2, 0>(C, in, out, n, st, f);
}

// ---- the host entry point's pipeline state (sdedge_solve_batch_host)
constexpr int kHostStreams = 4;              // 0: H2D, 1-2: solves, 3: D2H
constexpr int kHostMaxChunks = 16;

struct HostPipe {
    unsigned char* d = nullptr;
    cudaStream_t ss[kHostStreams] = {};
    cudaEvent_t ev0 = nullptr, evh[kHostMaxChunks] = {}, evc[kHostMaxChunks] = {}, evj[kHostStreams] = {};

    // Join every internal stream into the caller's stream, free, destroy.  Runs on
    // success and failure alike; returns the first error it meets (0 if none).
    int finish(cudaStream_t st)
    {
        int rc = 0;
        auto keep = [&](cudaError_t e, const char* what) {
            if (e != cudaSuccess && rc == 0) {
                snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
                rc = e == cudaErrorMemoryAllocation ? -3 : -2;
            }
        };
        for (int q = 0; q < kHostStreams; ++q) {
            if (!ss[q]) continue;
            if (!evj[q]) keep(cudaEventCreateWithFlags(&evj[q], cudaEventDisableTiming), "cudaEventCreate");
            if (evj[q]) {
                keep(cudaEventRecord(evj[q], ss[q]), "cudaEventRecord(join)");
                keep(cudaStreamWaitEvent(st, evj[q], 0), "cudaStreamWaitEvent(join)");
            } else {
                keep(cudaStreamSynchronize(ss[q]), "cudaStreamSynchronize");   // last resort: wait on the host
            }
        }
        if (d) keep(cudaFreeAsync(d, st), "cudaFreeAsync");
        for (int q = 0; q < kHostStreams; ++q)
            if (ss[q]) keep(cudaStreamDestroy(ss[q]), "cudaStreamDestroy");   // released once their work drains
        if (ev0) keep(cudaEventDestroy(ev0), "cudaEventDestroy");
        for (int q = 0; q < kHostMaxChunks; ++q) {
            if (evh[q]) keep(cudaEventDestroy(evh[q]), "cudaEventDestroy");
            if (evc[q]) keep(cudaEventDestroy(evc[q]), "cudaEventDestroy");
        }
        for (int q = 0; q < kHostStreams; ++q)
            if (evj[q]) keep(cudaEventDestroy(evj[q]), "cudaEventDestroy");
        *this = HostPipe{};
        return rc;
    }
};

// Compact re-encoding of a chunk's schedule for the device->host copy (sdedge_solve_batch_host_compact):
// order as uint16, batch ends as a bit mask (zeroed by the caller).  Grid-stride over n*K elements.
__global__ void pack_kernel(const int32_t* bend, const int32_t* order, long long n, int K, uint16_t* order16,
                            uint32_t* mask)
{
    const int W = (K + 31) / 32;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n * K; i += (long long)gridDim.x * blockDim.x) {
        order16[i] = (uint16_t)order[i];
        const int e = bend[i];
        if (e > 0) atomicOr(mask + (i / K) * W + (e - 1) / 32, 1u << ((e - 1) & 31));
    }
}

int host_pipeline(HostPipe& hp, const sdedge_scenarios* s, int64_t n, const sdedge_params* p, double* out_latency,
                  sdedge_schedule* o, cudaStream_t st, const sdedge_compact_schedule* oc = nullptr)
{
    const size_t K = (size_t)p->K, nn = (size_t)n;
    const size_t bI = nn * K * 4, bD = nn * K * 8, bA = nn * 8, bC = s->coeffs ? nn * 32 : 0;
    const size_t bLat = nn * 24, bS = nn * 4, bW = o->bw_share ? nn * K * 8 : 0;
    size_t off = 0;
    auto take = [&](size_t b) { size_t q = off; off += (b + 255) & ~(size_t)255; return q; };
    const size_t oI = take(bI), oP = take(bD), oG = take(bD), oA = take(bA), oC = take(bC);
    const size_t oLat = take(bLat), oGm = take(bS), oM = take(bS), oBe = take(bI), oOr = take(bI),
                 oW = take(bW), oSt = take(bS);
    const size_t Wm = (K + 31) / 32;
    const size_t oMask = oc ? take(nn * Wm * 4) : 0, oO16 = oc ? take(nn * K * 2) : 0;
    int dev = 0;
    CU(cudaGetDevice(&dev));
    if (int rc2 = ws_alloc(reinterpret_cast<void**>(&hp.d), off, st)) return rc2;
    unsigned char* d = hp.d;
    for (int q = 0; q < kHostStreams; ++q) CU(cudaStreamCreateWithFlags(&hp.ss[q], cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&hp.ev0, cudaEventDisableTiming));
    for (int q = 0; q < kHostMaxChunks; ++q) {
        CU(cudaEventCreateWithFlags(&hp.evh[q], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&hp.evc[q], cudaEventDisableTiming));
    }
    CU(cudaEventRecord(hp.ev0, st));
    for (int q = 0; q < kHostStreams; ++q) CU(cudaStreamWaitEvent(hp.ss[q], hp.ev0, 0));

    const long long nch = std::max(1LL, std::min((long long)kHostMaxChunks, (long long)(n / 32768)));
    const long long chunk = (n + nch - 1) / nch;
    int launches = 0;
    auto h2d = [&](size_t doff, const void* src, size_t row, long long a, long long m, cudaStream_t q) {
        return cudaMemcpyAsync(d + doff + row * a, static_cast<const unsigned char*>(src) + row * a, row * m,
                               cudaMemcpyHostToDevice, q);
    };
    auto d2h = [&](void* dst, size_t doff, size_t row, long long a, long long m, cudaStream_t q) {
        return cudaMemcpyAsync(static_cast<unsigned char*>(dst) + row * a, d + doff + row * a, row * m,
                               cudaMemcpyDeviceToHost, q);
    };
    for (long long c = 0; c < nch; ++c) {
        const long long a = c * chunk, m = std::min(chunk, (long long)n - a);
        if (m <= 0) break;
        cudaStream_t q = hp.ss[0];
        CU(h2d(oI, s->input_len, K * 4, a, m, q));
        CU(h2d(oP, s->tx_power_w, K * 8, a, m, q));
        CU(h2d(oG, s->gain, K * 8, a, m, q));
        CU(h2d(oA, s->alpha, 8, a, m, q));
        if (bC) CU(h2d(oC, s->coeffs, 32, a, m, q));
        CU(cudaEventRecord(hp.evh[c], q));
        q = hp.ss[1 + (c & 1)];
        CU(cudaStreamWaitEvent(q, hp.evh[c], 0));
        sdedge_scenarios ds{reinterpret_cast<int32_t*>(d + oI) + a * K, reinterpret_cast<double*>(d + oP) + a * K,
                            reinterpret_cast<double*>(d + oG) + a * K, reinterpret_cast<double*>(d + oA) + a,
                            bC ? reinterpret_cast<double*>(d + oC) + a * 4 : nullptr};
        sdedge_schedule dsch{reinterpret_cast<int32_t*>(d + oGm) + a, reinterpret_cast<int32_t*>(d + oM) + a,
                             reinterpret_cast<int32_t*>(d + oBe) + a * K, reinterpret_cast<int32_t*>(d + oOr) + a * K,
                             bW ? reinterpret_cast<double*>(d + oW) + a * K : nullptr,
                             reinterpret_cast<int32_t*>(d + oSt) + a, nullptr, nullptr, nullptr};
        sdedge_params pc = *p;
        pc.stream = q;
        if (int rc = solve_device(&ds, m, &pc, reinterpret_cast<double*>(d + oLat) + 3 * a, &dsch)) return rc;
        launches += g_launches;
        if (oc) {                            // re-encode on the device, copy the compact arrays back
            CU(cudaMemsetAsync(d + oMask + Wm * 4 * a, 0, Wm * 4 * m, q));
            const long long blocks = std::min<long long>((m * (long long)K + 255) / 256, 148LL * 16);
            pack_kernel<<<(unsigned)blocks, 256, 0, q>>>(dsch.batch_end, dsch.order, m, (int)K,
                                                          reinterpret_cast<uint16_t*>(d + oO16) + a * K,
                                                          reinterpret_cast<uint32_t*>(d + oMask) + a * Wm);
            CU(cudaGetLastError());
            launches += 1;
        }
        CU(cudaEventRecord(hp.evc[c], q));
        q = hp.ss[3];
        CU(cudaStreamWaitEvent(q, hp.evc[c], 0));
        CU(d2h(out_latency, oLat, 24, a, m, q));
        if (oc) {
            CU(d2h(oc->gamma, oGm, 4, a, m, q));
            CU(d2h(oc->num_batches, oM, 4, a, m, q));
            CU(d2h(oc->batch_end_mask, oMask, Wm * 4, a, m, q));
            CU(d2h(oc->order, oO16, K * 2, a, m, q));
            if (bW) CU(d2h(oc->bw_share, oW, K * 8, a, m, q));
            CU(d2h(oc->status, oSt, 4, a, m, q));
            continue;
        }
        CU(d2h(o->gamma, oGm, 4, a, m, q));
        CU(d2h(o->num_batches, oM, 4, a, m, q));
        CU(d2h(o->batch_end, oBe, K * 4, a, m, q));
        CU(d2h(o->order, oOr, K * 4, a, m, q));
        if (bW) CU(d2h(o->bw_share, oW, K * 8, a, m, q));
        CU(d2h(o->status, oSt, 4, a, m, q));
    }
    g_launches = launches;
    return 0;
}

}  // namespace

// ------------------------------------------------------------ exported C ABI
extern "C" {
#if SDEDGE_DBG
int sdedge_debug_counters(unsigned long long* out)   // development builds: read and clear the event counters
{
    unsigned long long z[16] = {};
    cudaMemcpyFromSymbol(out, g_dbg, sizeof(z));
    cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
    return 0;
}
#endif

int sdedge_abi_version(void) { return SDEDGE_ABI_VERSION; }

const char* sdedge_last_error(void) { return g_err; }

int sdedge_last_launch_count(void) { return g_launches; }

int sdedge_solve_batch(const sdedge_scenarios* s, int64_t n, const sdedge_params* p, double* out_latency,
                       sdedge_schedule* o)
{
    g_err[0] = 0;
    g_launches = 0;
    int rc = validate(s, n, p, out_latency, o);
    if (rc) return rc;
    return solve_device(s, n, p, out_latency, o);
}

int sdedge_solve_batch_host(const sdedge_scenarios* s, int64_t n, const sdedge_params* p, double* out_latency,
                            sdedge_schedule* o)
{
    // Host buffers in, host buffers out.  The batch is cut into <= 16 chunks; all
    // H2D copies go in order on one internal stream, all D2H copies on another,
    // and the solves alternate between two compute streams, chained by events
    // (solve c after H2D c, D2H c after solve c).  So both copy directions run
    // back to back while chunks are solved, and the solves of neighbouring chunks
    // can overlap each other's tail.  The caller's stream is joined at the end
    // (one cudaMemcpyAsync per array and chunk).  On ANY failure after the first
    // allocation the same cleanup runs: the caller's stream waits for everything
    // already queued on the internal streams (so the caller's documented stream
    // sync still covers every DMA touching its buffers), then the device buffer is
    // freed stream-ordered and the streams and events are destroyed.
    g_err[0] = 0;
    g_launches = 0;
    int rc = validate(s, n, p, out_latency, o);
    if (rc) return rc;
    if (n == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    HostPipe hp;
    rc = host_pipeline(hp, s, n, p, out_latency, o, st);
    const int rc2 = hp.finish(st);
    return rc ? rc : rc2;
}

int sdedge_solve_batch_host_compact(const sdedge_scenarios* s, int64_t n, const sdedge_params* p, double* out_latency,
                                    sdedge_compact_schedule* oc)
{
    // sdedge_solve_batch_host with the schedule re-encoded on the device before the copy back
    // (pack_kernel); same chunked pipeline, same cleanup on every path
    g_err[0] = 0;
    g_launches = 0;
    if (!oc) return fail(-1, "null argument");
    if (!oc->gamma || !oc->num_batches || !oc->batch_end_mask || !oc->order || !oc->status)
        return fail(-1, "null argument");
    sdedge_schedule full{oc->gamma, oc->num_batches, reinterpret_cast<int32_t*>(oc->batch_end_mask),
                         reinterpret_cast<int32_t*>(oc->order), oc->bw_share, oc->status, nullptr, nullptr, nullptr};
    int rc = validate(s, n, p, out_latency, &full);   // (the layout pointers only need to be non-null here)
    if (rc) return rc;
    if (n == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    HostPipe hp;
    rc = host_pipeline(hp, s, n, p, out_latency, &full, st, oc);
    const int rc2 = hp.finish(st);
    return rc ? rc : rc2;
}

int sdedge_evaluate_actual(const sdedge_scenarios* s, const int32_t* output_len, int64_t n, const sdedge_params* p,
                           const sdedge_schedule* plan, double* out_t_inf)
{
    g_err[0] = 0;
    g_launches = 0;
    sdedge_schedule dummy{};
    int rc = validate(s, 0, p, nullptr, &dummy);
    if (rc) return rc;
    if (n < 0) return fail(-1, "n < 0");
    if (n == 0) return 0;
    if (!s->input_len || !s->alpha || !output_len || !plan || !plan->gamma || !plan->num_batches ||
        !plan->batch_end || !plan->order || !plan->status || !out_t_inf)
        return fail(-1, "null argument");
    Consts C = make_consts(p);
    Inputs in{s->input_len, s->tx_power_w, s->gain, s->alpha, s->coeffs};
    int dev = 0, nsm = 0, max_smem = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CU(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    int warps = 4;
    while (warps > 1 && (size_t)warps * C.K * sizeof(ActBatch) > 96 * 1024) warps >>= 1;
    const size_t sb = (size_t)warps * C.K * sizeof(ActBatch);
    if (sb > (size_t)max_smem) return fail(-1, "shared memory requirement exceeds the device limit");
    CU(cudaFuncSetAttribute(actual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    long long blocks = std::min<long long>((n + warps - 1) / warps, (long long)nsm * 16);
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    actual_kernel<<<(unsigned)blocks, warps * 32, sb, st>>>(C, in, output_len, plan->gamma, plan->num_batches,
                                                           plan->batch_end, plan->order, plan->status, n,
                                                           out_t_inf);
    CU(cudaGetLastError());
    g_launches = 1;
    return 0;
}

int sdedge_brute_force(const sdedge_scenarios* s, int64_t n, const sdedge_params* p, double* out_t_inf,
                       sdedge_schedule* out)
{
    g_err[0] = 0;
    g_launches = 0;
    sdedge_schedule dummy{};
    int rc = validate(s, 0, p, nullptr, &dummy);
    if (rc) return rc;
    if (n < 0) return fail(-1, "n < 0");
    if (p->K > kBFMaxK) return fail(-1, "brute force needs K <= 20");
    if (p->batching_policy != SDEDGE_BATCH_PROPOSED && p->batching_policy != SDEDGE_BATCH_NO_PIPELINE)
        return fail(-1, "brute force evaluates the pipelined or the no-pipeline cost only");
    if (n == 0) return 0;
    if (!s->input_len || !s->alpha || !out || !out_t_inf || !out->gamma || !out->num_batches ||
        !out->batch_end || !out->order || !out->status)
        return fail(-1, "null argument");
    Consts C = make_consts(p);
    Inputs in{s->input_len, s->tx_power_w, s->gain, s->alpha, s->coeffs};
    int dev = 0, nsm = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    // gamma chunk per CTA item: all gammas of a scenario in one CTA when there are
    // enough scenarios to fill a wave of resident CTAs, else one gamma per item
    const int gc = n >= (long long)nsm * 8 ? C.ng : 1;
    const int nch = (C.ng + gc - 1) / gc;
    const long long items = n * (long long)nch;
    const long long blocks = std::min<long long>(items, (long long)nsm * 8);
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    unsigned char* ws = nullptr;
    const size_t offg = ((size_t)items * sizeof(double) + 255) & ~(size_t)255;
    const size_t offm = offg + (((size_t)items * sizeof(int32_t) + 255) & ~(size_t)255);
    if (int rc2 = ws_alloc(reinterpret_cast<void**>(&ws), offm + (size_t)items * sizeof(unsigned), st)) return rc2;
    double* wsv = reinterpret_cast<double*>(ws);
    int32_t* wsg = reinterpret_cast<int32_t*>(ws + offg);
    unsigned* wsm = reinterpret_cast<unsigned*>(ws + offm);
    bf_item_kernel<<<(unsigned)blocks, kBFWarps * 32, 0, st>>>(
        C, in, items, gc, wsv, wsg, wsm, reinterpret_cast<unsigned long long*>(out->work_counters));
    CU(cudaGetLastError());
    const long long fb = std::min<long long>((n + 3) / 4, (long long)nsm * 16);
    bf_final_kernel<<<(unsigned)fb, 128, 0, st>>>(C, in, n, nch, wsv, wsg, wsm, out_t_inf, out->gamma, out->num_batches,
                                                  out->batch_end, out->order, out->status);
    CU(cudaGetLastError());
    CU(cudaFreeAsync(ws, st));
    g_launches = 2;
    return 0;
}

// ---- multi-GPU gather: the shard ranks store their outputs straight into
// cuda:0's arrays over NVLink through CUDA IPC mappings
int sdedge_ipc_export(const void* dev_ptr, void* handle, uint64_t* offset)
{
    g_err[0] = 0;
    if (!dev_ptr || !handle || !offset) return fail(-1, "null argument");
    using AddrRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CU(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(-2, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (reinterpret_cast<AddrRange>(fn)(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
        return fail(-1, "dev_ptr is not a device allocation");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    memcpy(handle, &h, sizeof(h));
    *offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return 0;
}

int sdedge_ipc_open(const void* handle, uint64_t offset, void** dev_ptr)
{
    g_err[0] = 0;
    if (!handle || !dev_ptr) return fail(-1, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    CU(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = static_cast<unsigned char*>(base) + offset;
    return 0;
}

int sdedge_copy_async(void* dst, const void* src, uint64_t bytes, void* stream)
{
    g_err[0] = 0;
    if ((!dst || !src) && bytes) return fail(-1, "null argument");
    if (bytes) CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
    return 0;
}

int sdedge_ipc_close(void* dev_ptr, uint64_t offset)
{
    g_err[0] = 0;
    if (!dev_ptr) return fail(-1, "null argument");
    CU(cudaIpcCloseMemHandle(static_cast<unsigned char*>(dev_ptr) - offset));
    return 0;
}

int sdedge_kernel_timing(int32_t enable)
{
    g_err[0] = 0;
    g_kt.on = enable != 0;
    g_kt.used = 0;
    return 0;
}

int sdedge_kernel_times(double* ms, int32_t* launches)
{
    g_err[0] = 0;
    if (!ms) return fail(-1, "null argument");
    for (int k = 0; k < 4; ++k) { ms[k] = 0.0; if (launches) launches[k] = 0; }
    for (int q = 0; q < g_kt.used; ++q) {
        CU(cudaEventSynchronize(g_kt.ev[q][1]));
        float t = 0.f;
        CU(cudaEventElapsedTime(&t, g_kt.ev[q][0], g_kt.ev[q][1]));
        ms[g_kt.kind[q]] += t;
        if (launches) ++launches[g_kt.kind[q]];
    }
    return 0;
}

int sdedge_pipe_peak(int32_t fp32, double* ops_per_s, double* elapsed_s)
{
    g_err[0] = 0;
    if (!ops_per_s) return fail(-1, "null ops_per_s");
    int dev = 0, nsm = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int threads = 256, blocks = nsm * 8, iters = fp32 ? 8192 : 2048;
    void* sink = nullptr;
    CU(cudaMalloc(&sink, (size_t)blocks * threads * 8));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    float ms = 0.f;
    for (int rep = 0; rep < 2; ++rep) {   // first pass warms clocks
        CU(cudaEventRecord(e0));
        if (fp32) pipe_peak_kernel<float><<<blocks, threads>>>((float*)sink, iters, 1.0f);
        else pipe_peak_kernel<double><<<blocks, threads>>>((double*)sink, iters, 1.0);
        CU(cudaEventRecord(e1));
        CU(cudaEventSynchronize(e1));
        CU(cudaEventElapsedTime(&ms, e0, e1));
    }
    CU(cudaEventDestroy(e0));
    CU(cudaEventDestroy(e1));
    CU(cudaFree(sink));
    const double ops = (double)blocks * threads * iters * 16.0 * 8.0;
    *ops_per_s = ops / (ms * 1e-3);
    if (elapsed_s) *elapsed_s = ms * 1e-3;
    return 0;
}

}  // extern "C"
