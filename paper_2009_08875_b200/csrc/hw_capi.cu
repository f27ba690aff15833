// hw_capi.cu -- C ABI (include/heatwave_b200.h): context, operator
// orchestration and the device-resident PCG driver.
//
// Each entry point replaces one call site of the reference package
// (/root/reference/pkg/src/heatwave): see the header for the mapping.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/heatwave_b200.h"
#include "hw_common.cuh"

#include "hw_internal.cuh"

using namespace hw;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(e_ == cudaErrorMemoryAllocation ? HWG_ENOMEM : HWG_ECUDA,         \
                        std::string(#call) + ": " + cudaGetErrorString(e_));              \
    } while (0)

#define TRY(expr)                \
    do {                         \
        int rc_ = (expr);        \
        if (rc_ != HWG_OK) return rc_; \
    } while (0)

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct DevBand {           // a temporal factor in CSR on the device
    int32_t *ip = nullptr, *ix = nullptr;
    double *v = nullptr;
    double *tri = nullptr;   // dense (lo, mid, hi) per row (tridiagonal factors)
    TCsr view() const { return TCsr{ip, ix, v}; }
};

struct hwg_ctx {
    hwg_desc d{};
    int dim = 2, J = 0, K = 0, m = 0, nv = 2;
    int mg_reg_ok = 0;                  // every 2D level operator has |beta| <= kRegBetaMax
    int mg_wide = 0;                    // levels (bit l) mg2d_reg runs with its wide thread shape
    int coarse_fast = 1;                // mg2d_coarse below streamed levels: fast arithmetic
    double *cmat1d = nullptr;           // 1D, K >= 6: [op][15][15] level-4 V-cycle operators
    int mg1d_dense = 1;                 // HWG_MG1D_DENSE=0: the level-4..1 sub-cycle (A/B)
    int mg1d_rr = 0;                    // 1D, 7 <= K <= 10, |beta| <= 1/2: mg1d_rr
    int mg1d_rr_minb = 1;               // 1: persistent mg1d_rrp; HWG_RR_MINB=3 / 2: mg1d_rr (A/B)
    double *cmat_rr = nullptr;          // [op][63][64] level-6 V-cycle operators (mg1d_rr)
    int64_t nt = 0, nx = 0, N = 0;     // N = nt * nx (nx: grid points per row)
    int domain = 0;                    // 1: L-shaped (embedded grid, masked quadrant)
    int form = 0;                      // S: 0 five-term (Lemma 2), 1 test-space (Lemma 1)
    int64_t nxu = 0, Nu = 0;           // dof-layout row length / size (= nx, N for domain 0)
    double *cinv = nullptr;            // domain 1: [op][25] level-2 inverses (device)
    double *Xg = nullptr, *Yg = nullptr;   // domain 1: grid-layout operands of full contexts
    int64_t rows_max = 0;              // MG batch capacity (rows)
    bool kernel_only = false;          // distributed-path context (no operator buffers)
    int64_t red_max = 0;               // capacity of the dot partial / tree scratch
    Grid grid{};
    Stencil SM{}, SA{};
    std::vector<double> coef_host;
    std::vector<double> scale;         // wavelet s_j
    double *coef = nullptr;            // device table
    int32_t *row_op_kx = nullptr;      // device: 1 + level_of[r]
    std::vector<int32_t> level_of;
    DevBand At, Mt, L, LT, T, TT, Nn, NT;
    // workspaces
    double *U = nullptr, *MxU = nullptr, *AxU = nullptr, *T12 = nullptr, *G12 = nullptr;
    std::vector<double *> mgX, mgB;    // per level 1..K-1 (2D streaming + coarse)
    double *part = nullptr, *tmp = nullptr, *scal = nullptr;
    int *flag = nullptr;
    double *hscal = nullptr;           // pinned host mirror of scalars
    // PCG vectors (lazy)
    double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    double *fdev = nullptr, *wdev = nullptr;
    cudaStream_t copy_stream = nullptr;   // hwg_solve_host: chunked host -> device copies
    int use_graph = 1;                    // PCG iterations replayed as a CUDA graph
    cudaGraphExec_t graph_exec = nullptr; // one iteration (no recomputation) for graph_w
    cudaStream_t capture_stream = nullptr;  // graphs are captured here (the caller's stream
                                            // may be the legacy default stream)
    const double *graph_w = nullptr;     // the graph bakes in w and the Schur form
    int graph_form = -1;
    int64_t graph_kernels = 0;
    std::vector<cudaEvent_t> copy_events;
    int64_t bytes = 0;
    int64_t launches = 0;
    std::vector<void *> allocs;
    // roofline profiling (hwg_profile_*)
    bool prof = false;
    struct ProfRec { cudaEvent_t a, b; int cls; double bytes; };
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> prof_pool;
    double prof_ms[6] = {0}, prof_bytes[6] = {0};
    int64_t prof_n[6] = {0};
};

// Every entry point runs on its context's device and restores the caller's
// current device on return (contexts on several GPUs in one process).
struct DeviceGuard {
    int prev = -1;
    bool set = false;
    explicit DeviceGuard(const hwg_ctx *c);
    ~DeviceGuard()
    {
        if (set) cudaSetDevice(prev);
    }
};

static cudaEvent_t prof_event(hwg_ctx *c)
{
    if (!c->prof_pool.empty()) {
        cudaEvent_t e = c->prof_pool.back();
        c->prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// drain recorded event pairs into the per-class totals
static void prof_flush(hwg_ctx *c)
{
    for (auto &r : c->prof_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        c->prof_ms[r.cls] += ms;
        c->prof_bytes[r.cls] += r.bytes;
        c->prof_n[r.cls] += 1;
        c->prof_pool.push_back(r.a);
        c->prof_pool.push_back(r.b);
    }
    c->prof_recs.clear();
}

struct ProfScope {
    hwg_ctx *c;
    cudaStream_t st;
    int cls;
    double bytes;
    cudaEvent_t a{}, b{};
    bool on = false;
    ProfScope(hwg_ctx *c_, cudaStream_t s, int k, double by) : c(c_), st(s), cls(k), bytes(by)
    {
        // never inside a stream capture (a caller's CUDA graph): events
        // recorded there cannot be timed
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        on = c->prof && cudaStreamIsCapturing(st, &cs) == cudaSuccess &&
             cs == cudaStreamCaptureStatusNone;
        if (on) {
            if (c->prof_recs.size() > 4096) prof_flush(c);
            a = prof_event(c);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope()
    {
        if (on) {
            b = prof_event(c);
            cudaEventRecord(b, st);
            c->prof_recs.push_back({a, b, cls, bytes});
        }
    }
};

DeviceGuard::DeviceGuard(const hwg_ctx *c)
{
    if (!c || cudaGetDevice(&prev) != cudaSuccess) return;
    if (prev != c->d.device && cudaSetDevice(c->d.device) == cudaSuccess) set = true;
}

static int dalloc(hwg_ctx *c, double **p, int64_t count)
{
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, (size_t)count * sizeof(double));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HWG_ENOMEM, "cudaMalloc of " + std::to_string(count * 8) +
                                    " bytes failed: " + cudaGetErrorString(e));
    }
    c->allocs.push_back(q);
    c->bytes += count * (int64_t)sizeof(double);
    *p = (double *)q;
    return HWG_OK;
}

template <class T>
static int upload(hwg_ctx *c, T **dst, const std::vector<T> &src)
{
    void *q = nullptr;
    CK(cudaMalloc(&q, std::max<size_t>(1, src.size()) * sizeof(T)));
    c->allocs.push_back(q);
    c->bytes += (int64_t)(src.size() * sizeof(T));
    if (!src.empty()) CK(cudaMemcpy(q, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    *dst = (T *)q;
    return HWG_OK;
}

// CSR rows given as (col, value) lists in ascending column order
static int make_band(hwg_ctx *c, DevBand *b, const std::vector<std::vector<std::pair<int, double>>> &rows)
{
    std::vector<int32_t> ip(1, 0), ix;
    std::vector<double> v;
    for (auto &row : rows) {
        for (auto &e : row) {
            ix.push_back(e.first);
            v.push_back(e.second);
        }
        ip.push_back((int32_t)ix.size());
    }
    TRY(upload(c, &b->ip, ip));
    TRY(upload(c, &b->ix, ix));
    TRY(upload(c, &b->v, v));
    // dense triples when every entry lies within one row of the diagonal
    std::vector<double> tri(3 * rows.size(), 0.0);
    bool banded = true;
    for (size_t r = 0; r < rows.size(); ++r)
        for (auto &e : rows[r]) {
            const long d = (long)e.first - (long)r;
            if (d < -1 || d > 1) banded = false;
            else tri[3 * r + (d + 1)] = e.second;
        }
    if (banded) TRY(upload(c, &b->tri, tri));
    return HWG_OK;
}

// temporal.py:82-144 with the values computed by the host (desc->temporal)
static int build_temporal(hwg_ctx *c)
{
    const double *t = c->d.temporal;
    const int n = (int)c->nt;
    const int ne = n - 1;
    using Rows = std::vector<std::vector<std::pair<int, double>>>;
    auto tri = [&](double off_lo, double main, double end, double off_hi, bool drop_zero_main) {
        Rows rows(n);
        for (int i = 0; i < n; ++i) {
            if (i > 0) rows[i].push_back({i - 1, off_lo});
            double dv = (i == 0 || i == n - 1) ? end : main;
            if (!(drop_zero_main && dv == 0.0)) rows[i].push_back({i, dv});
            if (i < n - 1) rows[i].push_back({i + 1, off_hi});
        }
        return rows;
    };
    // M_t = h tridiag(1/6, 2/3, 1/6), ends h/3
    Rows Mt = tri(t[0], t[1], t[2], t[0], false);
    // A_t = tridiag(-1/h, 2/h, -1/h), ends 1/h
    Rows At = tri(t[3], t[4], t[5], t[3], false);
    if (n == 1) {  // J = 0 is not reachable (N_t = 2), kept for safety
        Mt = Rows(1);
        At = Rows(1);
    }
    // L: L[i,i-1] = -1/2, L[i,i+1] = +1/2, L[0,0] = -1/2, L[n-1,n-1] = +1/2
    Rows L(n), LT(n);
    for (int i = 0; i < n; ++i) {
        if (i > 0) L[i].push_back({i - 1, -t[6]});
        if (i == 0) L[i].push_back({0, -t[7]});
        if (i == n - 1) L[i].push_back({i, t[7]});
        if (i < n - 1) L[i].push_back({i + 1, t[6]});
        // L^T[i,k] = L[k,i]
        if (i > 0) LT[i].push_back({i - 1, t[6]});
        if (i == 0) LT[i].push_back({0, -t[7]});
        if (i == n - 1) LT[i].push_back({i, t[7]});
        if (i < n - 1) LT[i].push_back({i + 1, -t[6]});
    }
    // test matrices (2*ne rows): T[2k,k] = -1/sqrt h, T[2k,k+1] = 1/sqrt h,
    // odd rows of T eliminated; N[2k,k] = N[2k,k+1] = sqrt h/2,
    // N[2k+1,k] = -sqrt(3h)/6, N[2k+1,k+1] = +sqrt(3h)/6
    Rows T(2 * ne), Nn(2 * ne), TT(n), NT(n);
    for (int k = 0; k < ne; ++k) {
        T[2 * k] = {{k, -t[8]}, {k + 1, t[8]}};
        Nn[2 * k] = {{k, t[9]}, {k + 1, t[9]}};
        Nn[2 * k + 1] = {{k, -t[10]}, {k + 1, t[10]}};
    }
    for (int i = 0; i < n; ++i) {
        // T^T row i: (2(i-1), +1/sqrt h), (2i, -1/sqrt h)
        if (i > 0) TT[i].push_back({2 * (i - 1), t[8]});
        if (i < ne) TT[i].push_back({2 * i, -t[8]});
        // N^T row i: (2i-2, N[2i-2,i]), (2i-1, N[2i-1,i]), (2i, N[2i,i]), (2i+1, N[2i+1,i])
        if (i > 0) {
            NT[i].push_back({2 * (i - 1), t[9]});
            NT[i].push_back({2 * (i - 1) + 1, t[10]});
        }
        if (i < ne) {
            NT[i].push_back({2 * i, t[9]});
            NT[i].push_back({2 * i + 1, -t[10]});
        }
    }
    TRY(make_band(c, &c->Mt, Mt));
    TRY(make_band(c, &c->At, At));
    TRY(make_band(c, &c->L, L));
    TRY(make_band(c, &c->LT, LT));
    TRY(make_band(c, &c->T, T));
    TRY(make_band(c, &c->TT, TT));
    TRY(make_band(c, &c->Nn, Nn));
    TRY(make_band(c, &c->NT, NT));
    return HWG_OK;
}

// ---------------------------------------------------------------------------
// multigrid driver
// ---------------------------------------------------------------------------
static int64_t level_size(const hwg_ctx *c, int l)
{
    const int64_t m = (1LL << l) - 1;
    return c->dim == 2 ? m * m : m;
}

// X[r] = MG_op(B[r]) for rows [0, rows); row_op: device per-row operator or null
// dot_y (optional): also dot_part[r] = <dot_y row r, X row r>, fused into the
// last finest-level UP pass when that pass runs on mg2d_reg, else by row_dots
// does operator op (or, op = -1, any operator) couple diagonal neighbours on
// level l (c_d != 0)?  The register kernel drops those terms when none does.
static int level_has_diag(const hwg_ctx *c, int l, int op)
{
    const int nops = c->J + 2;
    for (int o = op < 0 ? 0 : op; o < (op < 0 ? nops : op + 1); ++o)
        if (c->coef_host[((size_t)o * (c->K + 1) + l) * HWG_COEF_STRIDE + kCd] != 0.0) return 1;
    return 0;
}

static bool mg_dot_fusable(const hwg_ctx *c)
{
    return c->dim == 2 && c->K >= 6 && c->K <= 11 && c->mg_reg_ok;
}

static int mg_apply(hwg_ctx *c, const double *B, double *X, int64_t rows, int op,
                    const int32_t *row_op, cudaStream_t st, const double *dot_y = nullptr,
                    double *dot_part = nullptr)
{
    const bool fuse = dot_y && mg_dot_fusable(c);
    for (int64_t r0 = 0; r0 < rows; r0 += c->rows_max) {
        const int64_t nr = std::min<int64_t>(c->rows_max, rows - r0);
        const double *Bp = B + r0 * c->nx;
        double *Xp = X + r0 * c->nx;
        const int32_t *ro = row_op ? row_op + r0 : nullptr;
        if (c->dim == 1) {
            Mg1dArgs a{Bp, c->nx, Xp, c->nx, c->coef, c->K + 1, c->K, c->nv, ro, op, nr, c->cmat1d};
            a.cmat_rr = c->cmat_rr;
            a.rr_minb = c->mg1d_rr_minb;
            ProfScope ps(c, st, 5, 16.0 * nr * c->nx);
            CK(c->mg1d_rr ? mg1d_rr_launch(a, st) : mg1d_launch(a, st));
            ++c->launches;
            continue;
        }
        if (c->K <= kCoarseTop2d) {
            MgCoarseArgs a{Bp, c->nx, Xp, c->nx, c->coef, c->K + 1, c->K, c->nv, 1, ro, op, nr,
                           c->domain, c->cinv, 0};
            ProfScope ps(c, st, 4, 16.0 * nr * c->nx);
            CK(mg2d_coarse_launch(a, st));
            ++c->launches;
            continue;
        }
        for (int cyc = 0; cyc < c->nv; ++cyc) {
            for (int l = c->K; l > kCoarseTop2d; --l) {
                MgStreamArgs a{};
                a.B = (l == c->K) ? Bp : c->mgB[l];
                a.ldB = level_size(c, l);
                a.X = (l == c->K) ? Xp : c->mgX[l];
                a.ldX = level_size(c, l);
                a.Bc = c->mgB[l - 1];
                a.ldBc = level_size(c, l - 1);
                a.coef = c->coef;
                a.levels_p1 = c->K + 1;
                a.level = l;
                a.n = (1 << l) - 1;
                a.row_op = ro;
                a.op = op;
                a.zero_start = (l < c->K || cyc == 0) ? 1 : 0;
                a.reg_ok = c->mg_reg_ok;
                a.wide = c->mg_wide;
                a.lshape = c->domain;
                a.diag = level_has_diag(c, l, ro ? -1 : op);
                const double n2 = (double)level_size(c, l), m2 = (double)level_size(c, l - 1);
                ProfScope ps(c, st, l == c->K ? 0 : 2,
                             8.0 * nr * (n2 * (a.zero_start ? 2 : 3) + m2));
                CK(mg2d_stream_launch(a, true, nr, st));
                ++c->launches;
            }
            MgCoarseArgs ca{c->mgB[kCoarseTop2d], level_size(c, kCoarseTop2d),
                            c->mgX[kCoarseTop2d], level_size(c, kCoarseTop2d), c->coef,
                            c->K + 1, kCoarseTop2d, 1, 1, ro, op, nr, c->domain, c->cinv,
                            c->coarse_fast};
            {
                ProfScope ps(c, st, 4, 16.0 * nr * level_size(c, kCoarseTop2d));
                CK(mg2d_coarse_launch(ca, st));
            }
            ++c->launches;
            for (int l = kCoarseTop2d + 1; l <= c->K; ++l) {
                MgStreamArgs a{};
                a.B = (l == c->K) ? Bp : c->mgB[l];
                a.ldB = level_size(c, l);
                a.X = (l == c->K) ? Xp : c->mgX[l];
                a.ldX = level_size(c, l);
                a.Xc = c->mgX[l - 1];
                a.ldXc = level_size(c, l - 1);
                a.coef = c->coef;
                a.levels_p1 = c->K + 1;
                a.level = l;
                a.n = (1 << l) - 1;
                a.row_op = ro;
                a.op = op;
                a.reg_ok = c->mg_reg_ok;
                a.wide = c->mg_wide;
                a.lshape = c->domain;
                a.diag = level_has_diag(c, l, ro ? -1 : op);
                if (fuse && l == c->K && cyc == c->nv - 1) {
                    a.dot_y = dot_y + r0 * c->nx;
                    a.dot_part = dot_part + r0;
                }
                const double n2 = (double)level_size(c, l), m2 = (double)level_size(c, l - 1);
                // b, x0, coarse x in, x out (+ the fused inner product's operand)
                ProfScope ps(c, st, l == c->K ? 1 : 3, 8.0 * nr * (3 * n2 + m2 + (a.dot_y ? n2 : 0)));
                CK(mg2d_stream_launch(a, false, nr, st));
                ++c->launches;
            }
        }
    }
    if (dot_y && !fuse) {
        CK(launch_row_partials(dot_y, X, rows, c->nx, dot_part, st));
        ++c->launches;
    }
    return HWG_OK;
}

// column-wise, so any row layout works: nx = 0 means the grid layout
static int wavelet(hwg_ctx *c, const double *X, double *Y, double *S1, double *S2, bool tr,
                   cudaStream_t st, int64_t nx = 0)
{
    const bool grid = !nx || nx == c->nx;          // grid layout: skip the L's zero quadrant
    CK(wavelet_apply(X, Y, S1, S2, c->J, c->scale.data(), c->nt, nx ? nx : c->nx, tr, st,
                     &c->launches, grid && c->domain ? c->m : 0, c->grid.lm));
    return HWG_OK;
}

// test-space S-hat = W^T (B^T K_Y B + Gamma0) W (system.py:149-180, Lemma 1):
// y = T (M_x U) + N (A_x U) on the 2 2^J test rows, K_Y = O^-1 (x) K_x with
// O = I (temporal.py:141; dividing by 1.0 is exact), then B^T = T^T (x) M_x +
// N^T (x) A_x and the trace row -- the cross-check of the production five-term
// form, in the reference's operation order
static int schur_test_space(hwg_ctx *c, const double *X, double *Y, cudaStream_t st)
{
    const int64_t nt = c->nt, nx = c->nx, N = c->N, ntest = 2 * (nt - 1);
    TRY(wavelet(c, X, c->U, c->T12, c->T12 + N, false, st));
    CK(launch_stencil_rows(c->U, c->MxU, c->AxU, c->grid, c->SM, c->SA, nt, st));
    BandOut y{c->T.view(), c->Nn.view(), c->MxU, c->AxU, c->T12};
    CK(launch_temporal_bands(y, BandOut{}, ntest, nx, st));
    c->launches += 2;
    TRY(mg_apply(c, c->T12, c->G12, ntest, 0, nullptr, st));
    BandOut w1{c->TT.view(), TCsr{nullptr, nullptr, nullptr}, c->G12, nullptr, c->U};
    BandOut w2{c->NT.view(), TCsr{nullptr, nullptr, nullptr}, c->G12, nullptr, c->AxU};
    CK(launch_temporal_bands(w1, w2, nt, nx, st));
    CK(launch_bt_side(c->U, c->AxU, c->MxU, c->G12, c->grid, c->SM, c->SA, nt, st));
    c->launches += 2;
    TRY(wavelet(c, c->G12, Y, c->T12, c->T12 + N, true, st));
    return HWG_OK;
}

// five-term S-hat = W^T S W (system.py:116-147, 182-187)
static int schur(hwg_ctx *c, const double *X, double *Y, cudaStream_t st)
{
    if (c->form == 1) return schur_test_space(c, X, Y, st);
    const int64_t nt = c->nt, N = c->N;
    TRY(wavelet(c, X, c->U, c->T12, c->T12 + N, false, st));
    // t1 = A_t MxU + L^T AxU, t1' = M_t AxU + L MxU (one pass over U); the
    // first row of MxU is kept for the trace term
    CK(launch_bside_fused(c->U, 0, nt, c->T12, c->T12 + N, c->MxU, c->grid, c->SM, c->SA,
                          Tri4{c->At.tri, c->LT.tri, c->Mt.tri, c->L.tri}, 0, nt, nt, st));
    ++c->launches;
    TRY(mg_apply(c, c->T12, c->G12, 2 * nt, 0, nullptr, st));
    CK(launch_bt_side(c->G12, c->G12 + N, c->MxU, c->U, c->grid, c->SM, c->SA, nt, st));
    ++c->launches;
    TRY(wavelet(c, c->U, Y, c->T12, c->T12 + N, true, st));
    return HWG_OK;
}

// K_X = blockdiag[C_l A_x C_l] (system.py:242-276); dot_y (optional): also
// the per-row partials of <dot_y, Y>, fused into the last multigrid pass
// K_X on rows [r0, r0 + nr) only (K_X is row-local)
static int kx_rows(hwg_ctx *c, const double *X, double *Y, int64_t r0, int64_t nr,
                   cudaStream_t st, const double *dot_y, double *dot_part)
{
    const int64_t o = r0 * c->nx;
    TRY(mg_apply(c, X + o, Y + o, nr, 0, c->row_op_kx + r0, st));
    CK(launch_stencil_rows(Y + o, nullptr, c->G12 + o, c->grid, c->SM, c->SA, nr, st));
    ++c->launches;
    TRY(mg_apply(c, c->G12 + o, Y + o, nr, 0, c->row_op_kx + r0, st, dot_y ? dot_y + o : nullptr,
                 dot_part ? dot_part + r0 : nullptr));
    return HWG_OK;
}

static int kx(hwg_ctx *c, const double *X, double *Y, cudaStream_t st,
              const double *dot_y = nullptr, double *dot_part = nullptr)
{
    return kx_rows(c, X, Y, 0, c->nt, st, dot_y, dot_part);
}

static cudaStream_t S(void *s) { return (cudaStream_t)s; }

// dof layout <-> grid layout (domain 1; plain copies otherwise)
static int to_grid(hwg_ctx *c, const double *src, double *dst, int64_t rows, cudaStream_t st)
{
    if (!c->domain) {
        if (src != dst) CK(cudaMemcpyAsync(dst, src, rows * c->nx * sizeof(double), cudaMemcpyDeviceToDevice, st));
        return HWG_OK;
    }
    CK(launch_grid_scatter(src, dst, rows, c->grid, c->nxu, st));
    ++c->launches;
    return HWG_OK;
}

static int from_grid(hwg_ctx *c, const double *src, double *dst, int64_t rows, cudaStream_t st)
{
    if (!c->domain) {
        if (src != dst) CK(cudaMemcpyAsync(dst, src, rows * c->nx * sizeof(double), cudaMemcpyDeviceToDevice, st));
        return HWG_OK;
    }
    CK(launch_grid_gather(src, dst, rows, c->grid, c->nxu, st));
    ++c->launches;
    return HWG_OK;
}

// 1D: the V-cycle from level kMg1dCut (zero start) of every operator as a
// dense matrix, M[op][i][j] = (MG e_i)_j -- computed by the same multigrid
// kernel on unit right-hand sides, so mg1d_reg's dense application is the
// identical linear map (up to rounding)
static int build_coarse_1d(hwg_ctx *c)
{
    if (!c->mg1d_dense) return HWG_OK;
    const int nops = c->J + 2, n = kMg1dCutN;
    const int64_t rows = (int64_t)nops * n;
    std::vector<double> eye((size_t)rows * n, 0.0);
    std::vector<int32_t> ops(rows);
    for (int o = 0; o < nops; ++o)
        for (int i = 0; i < n; ++i) {
            eye[((size_t)o * n + i) * n + i] = 1.0;
            ops[o * n + i] = o;
        }
    double *B = nullptr;
    int32_t *dops = nullptr;
    TRY(upload(c, &B, eye));
    TRY(upload(c, &dops, ops));
    TRY(dalloc(c, &c->cmat1d, rows * n));
    Mg1dArgs a{B, n, c->cmat1d, n, c->coef, c->K + 1, kMg1dCut, 1, dops, 0, rows, nullptr};
    CK(mg1d_launch(a, 0));
    CK(cudaDeviceSynchronize());
    return HWG_OK;
}

// mg1d_rr: the V-cycle from level kRrCut (zero start) of every operator,
// G[op][s][j] = (MG e_s)_j (rows padded to kRrCutLd with zero columns), run
// by the exact shared-memory kernel on unit right-hand sides
static int build_coarse_rr(hwg_ctx *c)
{
    const int nops = c->J + 2, n = kRrCutN;
    const int64_t rows = (int64_t)nops * n;
    std::vector<double> eye((size_t)rows * n, 0.0);
    std::vector<int32_t> ops(rows);
    for (int o = 0; o < nops; ++o)
        for (int i = 0; i < n; ++i) {
            eye[((size_t)o * n + i) * n + i] = 1.0;
            ops[o * n + i] = o;
        }
    double *B = nullptr;
    int32_t *dops = nullptr;
    TRY(upload(c, &B, eye));
    TRY(upload(c, &dops, ops));
    TRY(dalloc(c, &c->cmat_rr, rows * kRrCutLd));
    CK(cudaMemset(c->cmat_rr, 0, sizeof(double) * rows * kRrCutLd));
    Mg1dArgs a{B, n, c->cmat_rr, kRrCutLd, c->coef, c->K + 1, kRrCut, 1, dops, 0, rows, nullptr};
    CK(mg1d_launch(a, 0));
    CK(cudaDeviceSynchronize());
    return HWG_OK;
}

static int ensure_pcg(hwg_ctx *c)
{
    if (c->r) return HWG_OK;
    TRY(dalloc(c, &c->r, c->N));
    TRY(dalloc(c, &c->z, c->N));
    TRY(dalloc(c, &c->p, c->N));
    TRY(dalloc(c, &c->q, c->N));
    return HWG_OK;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char *hwg_last_error(void) { return g_err.c_str(); }
int hwg_version(void) { return 5; }

int hwg_create(const hwg_desc *desc, hwg_ctx **out)
{
    if (!desc || !out) return fail(HWG_EINVAL, "null argument");
    *out = nullptr;
    const hwg_desc &d = *desc;
    if (d.dim != 1 && d.dim != 2) return fail(HWG_EINVAL, "dimension must be 1 or 2 on the GPU path");
    if (d.J < 1 || d.J > 24) return fail(HWG_EINVAL, "J must be in [1, 24]");
    if (d.domain != 0 && d.domain != 1) return fail(HWG_EINVAL, "unknown domain");
    if (d.domain == 1 && d.dim != 2) return fail(HWG_EINVAL, "the L-shaped domain is 2D");
    if (d.domain == 1 && (d.K < 2 || !d.coarse_inv))
        return fail(HWG_EINVAL, "the L-shaped domain needs K >= 2 and the level-2 inverses");
    if (d.K < 1 || (d.dim == 2 && d.K > 11) || (d.dim == 1 && d.K > 10))
        return fail(HWG_EINVAL, d.dim == 2 ? "K must be in [1, 11]" : "K must be in [1, 10]");
    if (d.smooth != 3) return fail(HWG_EINVAL, "the GPU smoother is built for smooth = 3 sweeps");
    if (d.vcycles < 1) return fail(HWG_EINVAL, "vcycles must be >= 1");
    if (!d.coef || !d.stencil_M || !d.stencil_A || !d.temporal || !d.wavelet_scale)
        return fail(HWG_EINVAL, "missing table in descriptor");
    struct Restore {                      // leave the caller's current device as it was
        int prev = -1;
        Restore() { cudaGetDevice(&prev); }
        ~Restore()
        {
            if (prev >= 0) cudaSetDevice(prev);
        }
    } restore_;
    CK(cudaSetDevice(d.device));
    hwg_ctx *c = new hwg_ctx();
    c->d = d;
    c->dim = d.dim;
    c->J = d.J;
    c->K = d.K;
    c->nv = d.vcycles;
    c->m = (1 << d.K) - 1;
    c->nt = (1LL << d.J) + 1;
    c->nx = d.dim == 2 ? (int64_t)c->m * c->m : c->m;
    c->N = c->nt * c->nx;
    c->domain = d.domain;
    const int lm = (c->m - 1) / 2;
    c->nxu = d.domain ? c->nx - (int64_t)(c->m - lm) * (c->m - lm) : c->nx;
    c->Nu = c->nt * c->nxu;
    c->rows_max = d.rows_max > 0 ? d.rows_max : 2 * c->nt;
    c->kernel_only = d.rows_max > 0;
    c->grid = Grid{d.dim, c->m, c->nx, d.domain ? lm : (1 << 30)};
    c->SM = Stencil{d.stencil_M[0], d.stencil_M[1], d.stencil_M[2], d.stencil_M[3]};
    c->SA = Stencil{d.stencil_A[0], d.stencil_A[1], d.stencil_A[2], d.stencil_A[3]};
    c->scale.assign(d.wavelet_scale, d.wavelet_scale + d.J);
    const int nops = d.J + 2;
    c->coef_host.assign(d.coef, d.coef + (size_t)nops * (d.K + 1) * HWG_COEF_STRIDE);
    // mg2d_reg thread shapes are a property of the context (the global time
    // axis), never of a call's batch: results do not depend on how rows are
    // batched or split over time slabs.  Few temporal rows leave each SM one
    // or two warps of a level <= 9 pass; the wide shapes halve a thread's
    // points (hw_mg2d_reg.cu, profiles/r02/mg_wide_sweep.txt)
    {
        const int64_t n_t = ((int64_t)1 << d.J) + 1;
        if (n_t <= kWideWarps) c->mg_wide |= (1 << 7) | (1 << 8);
        if (2 * n_t <= kWideWarps) c->mg_wide |= 1 << 9;
        if (d.domain && n_t <= 148) c->mg_wide |= 1 << 10;
    }
    c->mg_reg_ok = 1;
    for (int op = 0; op < nops; ++op)
        for (int l = 1; l <= d.K; ++l) {
            const double *cf = &c->coef_host[((size_t)op * (d.K + 1) + l) * HWG_COEF_STRIDE];
            const double b = cf[kCy] * cf[kInv];
            if (!(fabs(b) <= kRegBetaMax)) c->mg_reg_ok = 0;
        }
    if (const char *ev = getenv("HWG_MG_REG"))      // A/B switch for measurements
        if (ev[0] == '0') c->mg_reg_ok = 0;
        else if (ev[0] == '4' && c->mg_reg_ok) c->mg_reg_ok = 2;   // P = 4 at n = 1023
        else if (ev[0] == '5' && c->mg_reg_ok) c->mg_reg_ok = 3;   // P = 4 for UP at n = 1023
    if (const char *ev = getenv("HWG_COARSE_EXACT"))        // A/B switch for measurements
        if (ev[0] == '1') c->coarse_fast = 0;
    if (const char *ev = getenv("HWG_MG1D_DENSE"))          // A/B switch for measurements
        if (ev[0] == '0') c->mg1d_dense = 0;
    // 1D register-resident hierarchy: its truncated lane carries need |beta| <= 1/2
    // on every level (always true for alpha A + mu M, alpha > 0, mu >= 0)
    if (d.dim == 1 && d.K >= kRrCut + 1 && d.K <= 10) {
        c->mg1d_rr = 1;
        for (int op = 0; op < nops; ++op)
            for (int l = kRrCut + 1; l <= d.K; ++l) {
                const double *cf = &c->coef_host[((size_t)op * (d.K + 1) + l) * HWG_COEF_STRIDE];
                if (!(fabs(cf[kCy] * cf[kInv]) <= 0.5)) c->mg1d_rr = 0;
            }
    }
    if (const char *ev = getenv("HWG_MG1D"))                // A/B: 1 = mg1d_reg
        if (ev[0] == '1') c->mg1d_rr = 0;
    if (const char *ev = getenv("HWG_RR_MINB"))
        if (ev[0] == '2' || ev[0] == '3') c->mg1d_rr_minb = ev[0] - '0';
    if (const char *ev = getenv("HWG_GRAPH"))               // A/B switch for measurements
        if (ev[0] == '0') c->use_graph = 0;
    // streamed levels without mg2d_reg: mg2d_stream covers n <= 1023 and has no mask
    if (!c->mg_reg_ok && d.dim == 2 && d.K > kCoarseTop2d && (d.K > 10 || d.domain)) {
        delete c;
        return fail(HWG_EINVAL, "level operators with |c_y / c_0| > 0.2726 are supported on the "
                                "square with K <= 10 only");
    }
    int rc;
#define GO(x)                      \
    do {                           \
        rc = (x);                  \
        if (rc != HWG_OK) {        \
            hwg_destroy(c);        \
            return rc;             \
        }                          \
    } while (0)
    GO(upload(c, &c->coef, c->coef_host));
    if (c->domain) {
        std::vector<double> ci(d.coarse_inv, d.coarse_inv + (size_t)nops * 25);
        GO(upload(c, &c->cinv, ci));
    }
    c->level_of.assign(c->nt, 0);
    for (int j = 1; j <= d.J; ++j)
        for (int64_t r = (1LL << (j - 1)) + 1; r <= (1LL << j); ++r) c->level_of[r] = j;
    std::vector<int32_t> ops(c->nt);
    for (int64_t r = 0; r < c->nt; ++r) ops[r] = 1 + c->level_of[r];
    GO(upload(c, &c->row_op_kx, ops));
    GO(build_temporal(c));
    if (d.dim == 1 && d.K > kMg1dCut + 1) GO(build_coarse_1d(c));
    if (c->mg1d_rr) GO(build_coarse_rr(c));
    if (!c->kernel_only) {
        GO(dalloc(c, &c->U, c->N));
        GO(dalloc(c, &c->MxU, c->N));
        GO(dalloc(c, &c->AxU, c->N));
        GO(dalloc(c, &c->T12, 2 * c->N));
        GO(dalloc(c, &c->G12, 2 * c->N));
        if (c->domain) {
            GO(dalloc(c, &c->Xg, c->N));
            GO(dalloc(c, &c->Yg, c->N));
        }
    }
    c->mgX.assign(d.K + 1, nullptr);
    c->mgB.assign(d.K + 1, nullptr);
    if (d.dim == 2 && d.K > kCoarseTop2d) {
        for (int l = kCoarseTop2d; l < d.K; ++l) {
            GO(dalloc(c, &c->mgX[l], c->rows_max * level_size(c, l)));
            GO(dalloc(c, &c->mgB[l], c->rows_max * level_size(c, l)));
        }
    }
    c->red_max = std::max<int64_t>(c->rows_max, c->nt) + 8;   // dot partials / tree scratch
    GO(dalloc(c, &c->part, c->red_max));
    GO(dalloc(c, &c->tmp, c->red_max));
    GO(dalloc(c, &c->scal, 16));
    {
        void *q = nullptr;
        if (cudaMalloc(&q, sizeof(int)) != cudaSuccess) {
            hwg_destroy(c);
            return fail(HWG_ENOMEM, "flag alloc");
        }
        c->allocs.push_back(q);
        c->flag = (int *)q;
        if (cudaMallocHost((void **)&c->hscal, 16 * sizeof(double)) != cudaSuccess) {
            hwg_destroy(c);
            return fail(HWG_ENOMEM, "pinned alloc");
        }
    }
#undef GO
    *out = c;
    return HWG_OK;
}

int hwg_profile_enable(hwg_ctx *c, int enable)
{
    DeviceGuard dg_(c);
    if (!c) return fail(HWG_EINVAL, "null context");
    prof_flush(c);
    for (int k = 0; k < 6; ++k) {
        c->prof_ms[k] = c->prof_bytes[k] = 0.0;
        c->prof_n[k] = 0;
    }
    c->prof = enable != 0;
    return HWG_OK;
}

int hwg_profile_read(hwg_ctx *c, int kclass, double *ms, double *bytes, int64_t *launches)
{
    DeviceGuard dg_(c);
    if (!c || kclass < 0 || kclass >= 6) return fail(HWG_EINVAL, "bad profile class");
    prof_flush(c);
    if (ms) *ms = c->prof_ms[kclass];
    if (bytes) *bytes = c->prof_bytes[kclass];
    if (launches) *launches = c->prof_n[kclass];
    return HWG_OK;
}

int hwg_destroy(hwg_ctx *c)
{
    DeviceGuard dg_(c);
    if (!c) return HWG_OK;
    prof_flush(c);
    for (cudaEvent_t e : c->prof_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : c->copy_events) cudaEventDestroy(e);
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (void *p : c->allocs) cudaFree(p);
    if (c->hscal) cudaFreeHost(c->hscal);
    delete c;
    return HWG_OK;
}

int64_t hwg_workspace_bytes(const hwg_ctx *c) { return c ? c->bytes : 0; }
int64_t hwg_launch_count(const hwg_ctx *c) { return c ? c->launches : 0; }

int hwg_wavelet(hwg_ctx *c, const double *X, double *Y, int transpose, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y) return fail(HWG_EINVAL, "null argument");
    if (c->kernel_only) return fail(HWG_EINVAL, "kernel-only (distributed) context");
    if (X == Y) return fail(HWG_EINVAL, "wavelet input and output may not alias");
    TRY(wavelet(c, X, Y, c->T12, c->T12 + c->N, transpose != 0, S(stream), c->nxu));
    return HWG_OK;
}

int hwg_spatial(hwg_ctx *c, int which, const double *X, double *Y, int64_t rows, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || rows < 0) return fail(HWG_EINVAL, "bad argument");
    cudaStream_t st = S(stream);
    if (!c->domain || c->kernel_only) {          // kernel contexts: grid layout
        CK(launch_stencil_rows(X, which == 0 ? Y : nullptr, which == 0 ? nullptr : Y, c->grid,
                               c->SM, c->SA, rows, st));
        ++c->launches;
        return HWG_OK;
    }
    for (int64_t r0 = 0; r0 < rows; r0 += 2 * c->nt) {   // dof layout via the T12 / G12 scratch
        const int64_t nr = std::min<int64_t>(2 * c->nt, rows - r0);
        TRY(to_grid(c, X + r0 * c->nxu, c->T12, nr, st));
        CK(launch_stencil_rows(c->T12, which == 0 ? c->G12 : nullptr, which == 0 ? nullptr : c->G12,
                               c->grid, c->SM, c->SA, nr, st));
        ++c->launches;
        TRY(from_grid(c, c->G12, Y + r0 * c->nxu, nr, st));
    }
    return HWG_OK;
}

int hwg_schur_apply(hwg_ctx *c, const double *X, double *Y, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y) return fail(HWG_EINVAL, "null argument");
    if (c->kernel_only) return fail(HWG_EINVAL, "kernel-only (distributed) context");
    if (!c->domain) return schur(c, X, Y, S(stream));
    TRY(to_grid(c, X, c->Xg, c->nt, S(stream)));
    TRY(schur(c, c->Xg, c->Yg, S(stream)));
    return from_grid(c, c->Yg, Y, c->nt, S(stream));
}

int hwg_kx_apply(hwg_ctx *c, const double *X, double *Y, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y) return fail(HWG_EINVAL, "null argument");
    if (c->kernel_only) return fail(HWG_EINVAL, "kernel-only (distributed) context");
    if (X == Y) return fail(HWG_EINVAL, "K_X input and output may not alias");
    if (!c->domain) return kx(c, X, Y, S(stream));
    TRY(to_grid(c, X, c->Xg, c->nt, S(stream)));
    TRY(kx(c, c->Xg, c->Yg, S(stream)));
    return from_grid(c, c->Yg, Y, c->nt, S(stream));
}

int hwg_set_schur_form(hwg_ctx *c, int form)
{
    DeviceGuard dg_(c);
    if (!c || (form != 0 && form != 1)) return fail(HWG_EINVAL, "form must be 0 (five-term) or 1 (test-space)");
    if (form != c->form && c->graph_exec) {   // the captured iteration applies the old form
        cudaGraphExecDestroy(c->graph_exec);
        c->graph_exec = nullptr;
        c->graph_w = nullptr;
    }
    c->form = form;
    return HWG_OK;
}

int hwg_grid_scatter(hwg_ctx *c, const double *X, double *Y, int64_t rows, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || rows < 0) return fail(HWG_EINVAL, "bad argument");
    if (X == Y && c->domain) return fail(HWG_EINVAL, "layout conversion may not alias");
    return to_grid(c, X, Y, rows, S(stream));
}

int hwg_grid_gather(hwg_ctx *c, const double *X, double *Y, int64_t rows, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || rows < 0) return fail(HWG_EINVAL, "bad argument");
    if (X == Y && c->domain) return fail(HWG_EINVAL, "layout conversion may not alias");
    return from_grid(c, X, Y, rows, S(stream));
}

int hwg_mg_rows(hwg_ctx *c, int32_t op, const int32_t *op_host, const double *B, double *X,
                int64_t rows, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !B || !X || rows < 0) return fail(HWG_EINVAL, "bad argument");
    if (B == X) return fail(HWG_EINVAL, "MG input and output may not alias");
    if (op < 0 || op > c->J + 1) return fail(HWG_EKEY, "no multigrid operator " + std::to_string(op));
    int32_t *dops = nullptr;
    if (op_host) {
        std::vector<int32_t> ops(op_host, op_host + rows);
        for (int32_t o : ops)
            if (o < 0 || o > c->J + 1) return fail(HWG_EKEY, "no multigrid operator " + std::to_string(o));
        CK(cudaMallocAsync((void **)&dops, std::max<int64_t>(rows, 1) * sizeof(int32_t), S(stream)));
        CK(cudaMemcpyAsync(dops, ops.data(), rows * sizeof(int32_t), cudaMemcpyHostToDevice, S(stream)));
    }
    int rc = HWG_OK;
    if (!c->domain || c->kernel_only) {
        rc = mg_apply(c, B, X, rows, op, dops, S(stream));
    } else {                                   // dof layout via the T12 / G12 scratch
        for (int64_t r0 = 0; r0 < rows && rc == HWG_OK; r0 += 2 * c->nt) {
            const int64_t nr = std::min<int64_t>(2 * c->nt, rows - r0);
            rc = to_grid(c, B + r0 * c->nxu, c->T12, nr, S(stream));
            if (rc == HWG_OK) rc = mg_apply(c, c->T12, c->G12, nr, op, dops ? dops + r0 : nullptr, S(stream));
            if (rc == HWG_OK) rc = from_grid(c, c->G12, X + r0 * c->nxu, nr, S(stream));
        }
    }
    if (dops) cudaFreeAsync(dops, S(stream));
    return rc;
}

int hwg_rhs(hwg_ctx *c, const double *F, const double *load, const double *u0proj,
            double *fhat, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !fhat) return fail(HWG_EINVAL, "null argument");
    if (c->kernel_only) return fail(HWG_EINVAL, "kernel-only (distributed) context");
    cudaStream_t st = S(stream);
    const int64_t nt = c->nt, nx = c->nx, N = c->N, ntest = 2 * (nt - 1);
    double *const fout = fhat;
    if (c->domain) {                       // dof-layout inputs -> grid layout
        if (F) {
            TRY(to_grid(c, F, c->Xg, nt, st));
            F = c->Xg;
        } else if (load) {
            TRY(to_grid(c, load, c->T12, ntest, st));
            load = c->T12;
        }
        fhat = c->Yg;
    }
    // g part: W^T (T^T (x) M_x + N^T (x) A_x) K_Y y, y = (N (x) M_x) F
    if (F || load) {
        const double *y = load;
        if (F) {
            CK(launch_stencil_rows(F, c->MxU, nullptr, c->grid, c->SM, c->SA, nt, st));
            BandOut o1{c->Nn.view(), TCsr{nullptr, nullptr, nullptr}, c->MxU, nullptr, c->T12};
            BandOut o2{};
            CK(launch_temporal_bands(o1, o2, ntest, nx, st));
            c->launches += 2;
            y = c->T12;
        }
        TRY(mg_apply(c, y, c->G12, ntest, 0, nullptr, st));      // K_Y = O^-1 (x) K_x, O = I
        BandOut o1{c->TT.view(), TCsr{nullptr, nullptr, nullptr}, c->G12, nullptr, c->U};
        BandOut o2{c->NT.view(), TCsr{nullptr, nullptr, nullptr}, c->G12, nullptr, c->AxU};
        CK(launch_temporal_bands(o1, o2, nt, nx, st));
        CK(launch_bt_side(c->U, c->AxU, nullptr, c->MxU, c->grid, c->SM, c->SA, nt, st));
        c->launches += 2;
        TRY(wavelet(c, c->MxU, fhat, c->U, c->AxU, true, st));
    } else {
        CK(cudaMemsetAsync(fhat, 0, N * sizeof(double), st));
    }
    if (u0proj) {
        CK(cudaMemsetAsync(c->T12, 0, N * sizeof(double), st));
        TRY(to_grid(c, u0proj, c->T12, 1, st));
        TRY(wavelet(c, c->T12, c->G12, c->U, c->AxU, true, st));
        CK(launch_add(fhat, c->G12, fhat, N, st));
        ++c->launches;
    }
    if (c->domain) TRY(from_grid(c, fhat, fout, nt, st));
    return HWG_OK;
}

int hwg_dot(hwg_ctx *c, const double *X, const double *Y, int64_t rows, double *result_host,
            void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || !result_host || rows < 0 || rows > c->rows_max)
        return fail(HWG_EINVAL, "bad argument");
    cudaStream_t st = S(stream);
    CK(launch_dot(X, Y, rows, c->kernel_only ? c->nx : c->nxu, c->part, c->tmp, c->scal + 8, st,
                  &c->launches));
    CK(cudaMemcpyAsync(c->hscal + 8, c->scal + 8, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *result_host = c->hscal[8];
    return HWG_OK;
}

}  // extern "C"

// One PCG iteration without residual recomputation (solver.py:212-256):
// q = S p, p.q, alpha, r -= alpha q, z = K_X r with r.z fused, beta, then
// w += alpha p and p = z + beta p in one pass; the four scalars are copied to
// the pinned host mirror.  Everything is stream-ordered and device-resident,
// so the sequence can be captured as a CUDA graph.
static int enqueue_iteration(hwg_ctx *c, double *w, cudaStream_t st)
{
    const int64_t N = c->N, nt = c->nt, nx = c->nx;
    TRY(schur(c, c->p, c->q, st));
    CK(launch_dot(c->p, c->q, nt, nx, c->part, c->tmp, c->scal + 1, st, &c->launches));
    CK(launch_pcg_alpha(c->scal, st));
    CK(launch_update_wr(w, c->r, c->p, c->q, c->scal, N, 0, 1, st));
    c->launches += 2;
    TRY(kx(c, c->r, c->z, st, c->r, c->part));
    CK(launch_tree(c->part, nt, c->tmp, c->scal + 2, st));
    ++c->launches;
    CK(cudaMemcpyAsync(c->hscal + 1, c->scal + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(launch_pcg_beta(c->scal, st));
    CK(launch_update_wp(w, c->p, c->z, c->scal, N, 1, st));
    c->launches += 2;
    CK(cudaMemcpyAsync(c->hscal + 3, c->scal + 3, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    return HWG_OK;
}

// the iteration as an instantiated CUDA graph (captured once per w buffer):
// ~300 dependent launches become one graph launch
static int iteration_graph(hwg_ctx *c, double *w)
{
    if (c->graph_exec && c->graph_w == w && c->graph_form == c->form) return HWG_OK;
    if (c->graph_exec) {
        cudaGraphExecDestroy(c->graph_exec);
        c->graph_exec = nullptr;
    }
    if (!c->capture_stream) CK(cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking));
    cudaStream_t cs = c->capture_stream;
    const int64_t l0 = c->launches;
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    const int rc = enqueue_iteration(c, w, cs);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cs, &g);
    const int64_t kernels = c->launches - l0;           // counted at each replay instead
    c->launches = l0;
    if (rc != HWG_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    CK(e);
    const cudaError_t ei = cudaGraphInstantiate(&c->graph_exec, g, 0);
    cudaGraphDestroy(g);
    CK(ei);
    c->graph_w = w;
    c->graph_form = c->form;
    c->graph_kernels = kernels;
    return HWG_OK;
}

// f arriving in row chunks: chunk k (rows [k rows, (k+1) rows)) is in place
// once ev[k] has completed (hwg_solve_host's pipelined host -> device copy)
struct StagedInput {
    int n = 0;
    int64_t rows = 0;
    const cudaEvent_t *ev = nullptr;
};

// PCG on grid-layout f, w (hwg_pcg converts dof-layout operands)
static int pcg_core(hwg_ctx *c, const double *f, double *w, double epsilon, double rtol,
                    int32_t max_iterations, int32_t recompute_every, hwg_pcg_stats *st_out,
                    cudaStream_t st, const StagedInput *staged = nullptr)
{
    TRY(ensure_pcg(c));
    const int64_t N = c->N, nt = c->nt, nx = c->nx;
    hwg_pcg_stats dummy{};
    hwg_pcg_stats &out = st_out ? *st_out : dummy;
    out.iterations = 0;
    out.ms_schur = out.ms_precond = out.ms_vector = out.ms_total = 0.0;
    auto push = [&](double *arr, int k, double v) {
        if (arr && k < out.capacity) arr[k] = v;
    };
    cudaEvent_t ev[8];
    for (auto &e : ev) CK(cudaEventCreate(&e));
    struct Guard {
        cudaEvent_t *e;
        ~Guard() { for (int i = 0; i < 8; ++i) cudaEventDestroy(e[i]); }
    } guard{ev};
    CK(cudaEventRecord(ev[0], st));
    CK(cudaMemsetAsync(w, 0, N * sizeof(double), st));
    // zero right-hand side returns immediately (solver.py:196-198)
    CK(cudaMemsetAsync(c->flag, 0, sizeof(int), st));
    int hflag = 0;
    if (staged && staged->n > 1) {
        // r = f and z = K_X r chunk by chunk as the rows arrive (K_X is
        // row-local), overlapping the host -> device copy of the later rows
        CK(cudaEventRecord(ev[1], st));
        for (int k = 0; k < staged->n; ++k) {
            const int64_t r0 = k * staged->rows, nr = std::min(staged->rows, nt - r0);
            CK(cudaStreamWaitEvent(st, staged->ev[k], 0));
            CK(launch_any_nonzero(f + r0 * nx, nr * nx, c->flag, st));
            CK(cudaMemcpyAsync(c->r + r0 * nx, f + r0 * nx, nr * nx * sizeof(double),
                               cudaMemcpyDeviceToDevice, st));
            ++c->launches;
            TRY(kx_rows(c, c->r, c->z, r0, nr, st, c->r, c->part));
        }
        CK(cudaEventRecord(ev[2], st));
        CK(cudaMemcpyAsync(&hflag, c->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!hflag) {
            push(out.residual_norms, 0, 0.0);
            out.epsilon_used = epsilon;
            return HWG_OK;
        }
    } else {
        CK(launch_any_nonzero(f, N, c->flag, st));
        ++c->launches;
        CK(cudaMemcpyAsync(&hflag, c->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!hflag) {
            push(out.residual_norms, 0, 0.0);
            out.epsilon_used = epsilon;
            return HWG_OK;
        }
        CK(cudaMemcpyAsync(c->r, f, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CK(cudaEventRecord(ev[1], st));
        TRY(kx(c, c->r, c->z, st, c->r, c->part));       // r.z fused into K_X's last pass
        CK(cudaEventRecord(ev[2], st));
    }
    CK(launch_tree(c->part, nt, c->tmp, c->scal + 0, st));
    ++c->launches;
    CK(cudaMemcpyAsync(c->hscal, c->scal, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev[1], ev[2]));
    out.ms_precond += ms;
    double rho = c->hscal[0];
    push(out.residual_norms, 0, std::sqrt(std::max(rho, 0.0)));
    const double eps = rtol > 0 ? rtol * std::sqrt(std::max(rho, 0.0)) : epsilon;
    out.epsilon_used = eps;
    if (rho <= eps * eps) {
        CK(cudaEventRecord(ev[7], st));
        CK(cudaEventSynchronize(ev[7]));
        CK(cudaEventElapsedTime(&ms, ev[0], ev[7]));
        out.ms_total = ms;
        return HWG_OK;
    }
    CK(cudaMemcpyAsync(c->p, c->z, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    const bool graphs = c->use_graph && !c->prof;      // profiling events need plain launches
    for (int k = 1; k <= max_iterations; ++k) {
      const bool recompute = (k % recompute_every) == 0;
      if (graphs && !recompute) {
        TRY(iteration_graph(c, w));                      // (re)captured when w changes
        CK(cudaGraphLaunch(c->graph_exec, st));
        c->launches += c->graph_kernels;
        CK(cudaEventRecord(ev[6], st));
        CK(cudaEventSynchronize(ev[6]));
      } else {
        CK(cudaEventRecord(ev[1], st));
        TRY(schur(c, c->p, c->q, st));
        CK(cudaEventRecord(ev[2], st));
        CK(launch_dot(c->p, c->q, nt, nx, c->part, c->tmp, c->scal + 1, st, &c->launches));
        CK(launch_pcg_alpha(c->scal, st));
        // r -= alpha q now; w += alpha p is deferred into the p update below
        // (one pass over p), except before a residual recomputation, which
        // needs the current w
        CK(launch_update_wr(w, c->r, c->p, c->q, c->scal, N, recompute ? 1 : 0, recompute ? 0 : 1, st));
        c->launches += 2;
        CK(cudaEventRecord(ev[3], st));
        if (recompute) {
            TRY(schur(c, w, c->z, st));
            CK(launch_sub(f, c->z, c->r, N, st));
            ++c->launches;
        }
        CK(cudaEventRecord(ev[4], st));
        TRY(kx(c, c->r, c->z, st, c->r, c->part));       // r.z fused into K_X's last pass
        CK(cudaEventRecord(ev[5], st));
        CK(launch_tree(c->part, nt, c->tmp, c->scal + 2, st));
        ++c->launches;
        CK(cudaMemcpyAsync(c->hscal + 1, c->scal + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(launch_pcg_beta(c->scal, st));
        CK(launch_update_wp(w, c->p, c->z, c->scal, N, recompute ? 0 : 1, st));
        c->launches += 2;
        CK(cudaMemcpyAsync(c->hscal + 3, c->scal + 3, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ev[6], st));
        CK(cudaEventSynchronize(ev[6]));
        float a = 0, b = 0, cc = 0, dd = 0;
        CK(cudaEventElapsedTime(&a, ev[1], ev[2]));
        CK(cudaEventElapsedTime(&b, ev[2], ev[3]));
        CK(cudaEventElapsedTime(&cc, ev[3], ev[4]));
        CK(cudaEventElapsedTime(&dd, ev[4], ev[5]));
        out.ms_schur += a + cc;
        out.ms_vector += b;
        out.ms_precond += dd;
      }
        const double pq = c->hscal[1], rho_new = c->hscal[2];
        const double alpha = c->hscal[3], beta = c->hscal[4];
        if (!(pq > 0)) {
            char buf[128];
            snprintf(buf, sizeof buf, "operator lost positive definiteness (p^T S p = %g)", pq);
            return fail(HWG_ENOTSPD, buf);
        }
        push(out.alphas, k - 1, alpha);
        push(out.betas, k - 1, beta);
        push(out.residual_norms, k, std::sqrt(std::max(rho_new, 0.0)));
        out.iterations = k;
        if (rho_new <= eps * eps) {
            CK(cudaEventRecord(ev[7], st));
            CK(cudaEventSynchronize(ev[7]));
            CK(cudaEventElapsedTime(&ms, ev[0], ev[7]));
            out.ms_total = ms;
            return HWG_OK;
        }
    }
    CK(cudaEventRecord(ev[7], st));
    CK(cudaEventSynchronize(ev[7]));
    CK(cudaEventElapsedTime(&ms, ev[0], ev[7]));
    out.ms_total = ms;
    char buf[160];
    snprintf(buf, sizeof buf, "PCG did not reach tolerance %g within %d iterations", eps,
             max_iterations);
    return fail(HWG_EMAXIT, buf);
}

extern "C" {

int hwg_pcg(hwg_ctx *c, const double *f, double *w, double epsilon, double rtol,
            int32_t max_iterations, int32_t recompute_every, hwg_pcg_stats *st_out, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !f || !w) return fail(HWG_EINVAL, "null argument");
    if (c->kernel_only) return fail(HWG_EINVAL, "kernel-only (distributed) context");
    if (!(epsilon > 0) && !(rtol > 0)) return fail(HWG_EINVAL, "tolerance must be positive");
    if (max_iterations < 0 || recompute_every < 1) return fail(HWG_EINVAL, "bad iteration limits");
    cudaStream_t st = S(stream);
    if (!c->domain)
        return pcg_core(c, f, w, epsilon, rtol, max_iterations, recompute_every, st_out, st);
    TRY(to_grid(c, f, c->Xg, c->nt, st));
    const int rc = pcg_core(c, c->Xg, c->Yg, epsilon, rtol, max_iterations, recompute_every,
                            st_out, st);
    if (rc != HWG_OK && rc != HWG_EMAXIT) return rc;
    const std::string msg = g_err;
    TRY(from_grid(c, c->Yg, w, c->nt, st));
    if (rc != HWG_OK) g_err = msg;
    return rc;
}

int hwg_solve_host(hwg_ctx *c, const double *fhat_host, double *u_host, double epsilon,
                   double rtol, int32_t max_iterations, int32_t recompute_every,
                   hwg_pcg_stats *stats, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !fhat_host || !u_host) return fail(HWG_EINVAL, "null argument");
    if (c->kernel_only) return fail(HWG_EINVAL, "kernel-only (distributed) context");
    cudaStream_t st = S(stream);
    if (!(epsilon > 0) && !(rtol > 0)) return fail(HWG_EINVAL, "tolerance must be positive");
    if (max_iterations < 0 || recompute_every < 1) return fail(HWG_EINVAL, "bad iteration limits");
    if (!c->fdev) {
        TRY(dalloc(c, &c->fdev, c->N));
        TRY(dalloc(c, &c->wdev, c->N));
    }
    // large problems: copy f-hat in row chunks on a second stream and start
    // the (row-local) initial K_X on each chunk as it lands
    StagedInput staged;
    // >= 256 rows per chunk (a one-wave K_X batch at least) and <= 8 chunks
    const int64_t chunk_rows = std::max<int64_t>(256, (c->nt + 7) / 8);
    if (!c->domain && c->N >= (int64_t)1 << 26 && c->nt > chunk_rows) {
        if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        const int n = (int)((c->nt + chunk_rows - 1) / chunk_rows);
        while ((int)c->copy_events.size() < n + 1) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->copy_events.push_back(e);
        }
        CK(cudaEventRecord(c->copy_events[n], st));       // earlier work on fdev done
        CK(cudaStreamWaitEvent(c->copy_stream, c->copy_events[n], 0));
        for (int k = 0; k < n; ++k) {
            const int64_t r0 = k * chunk_rows, nr = std::min(chunk_rows, c->nt - r0);
            CK(cudaMemcpyAsync(c->fdev + r0 * c->nx, fhat_host + r0 * c->nx,
                               nr * c->nx * sizeof(double), cudaMemcpyHostToDevice, c->copy_stream));
            CK(cudaEventRecord(c->copy_events[k], c->copy_stream));
        }
        staged = StagedInput{n, chunk_rows, c->copy_events.data()};
    } else {
        CK(cudaMemcpyAsync(c->fdev, fhat_host, c->Nu * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    const double *f = c->fdev;
    if (c->domain) {                          // dof layout -> grid layout (in place is not
        TRY(to_grid(c, c->fdev, c->Xg, c->nt, st));   // allowed: via Xg)
        f = c->Xg;
    }
    int rc = pcg_core(c, f, c->wdev, epsilon, rtol, max_iterations, recompute_every, stats, st,
                      staged.n > 1 ? &staged : nullptr);
    if (rc != HWG_OK && rc != HWG_EMAXIT) return rc;
    const std::string msg = g_err;
    TRY(wavelet(c, c->wdev, c->U, c->T12, c->T12 + c->N, false, st));
    const double *u = c->U;
    if (c->domain) {
        TRY(from_grid(c, c->U, c->fdev, c->nt, st));
        u = c->fdev;
    }
    CK(cudaMemcpyAsync(u_host, u, c->Nu * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (rc != HWG_OK) g_err = msg;
    return rc;
}

// ---- time-slab building blocks --------------------------------------------
int hwg_syn_stage(hwg_ctx *c, int j, const double *C, int64_t c0, const double *Dw, int64_t d0,
                  const double *Dhalo, double *Y, int64_t f0, int64_t nf, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !C || !Dw || !Y || j < 1 || j > c->J || nf < 0) return fail(HWG_EINVAL, "bad argument");
    CK(launch_syn_stage(j, c->scale[j - 1], C, c0, Dw, d0, Dhalo, Y, f0, nf, c->nx, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_ana_stage(hwg_ctx *c, int j, const double *X, int64_t x0, double *C, int64_t c0,
                  int64_t nc, double *Dw, int64_t d0, int64_t nd, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || (nc && !C) || (nd && !Dw) || j < 1 || j > c->J || nc < 0 || nd < 0)
        return fail(HWG_EINVAL, "bad argument");
    CK(launch_ana_stage(j, c->scale[j - 1], X, x0, C, c0, nc, Dw, d0, nd, c->nx, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_bside_rows(hwg_ctx *c, const double *U, int64_t u0, int64_t nu, double *T1, double *T2,
                   int64_t r0, int64_t nr, double *E0, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !U || !T1 || !T2 || nr < 0 || r0 < 0 || r0 + nr > c->nt) return fail(HWG_EINVAL, "bad argument");
    if (u0 > (r0 > 0 ? r0 - 1 : 0) || u0 + nu < (r0 + nr < c->nt ? r0 + nr + 1 : r0 + nr))
        return fail(HWG_EINVAL, "U does not cover the rows the temporal bands need");
    if (nr == 0) return HWG_OK;
    CK(launch_bside_fused(U, u0, nu, T1, T2, r0 == 0 ? E0 : nullptr, c->grid, c->SM, c->SA,
                          Tri4{c->At.tri, c->LT.tri, c->Mt.tri, c->L.tri}, r0, nr, c->nt,
                          S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_bt_rows(hwg_ctx *c, const double *G1, const double *G2, const double *E0, double *out,
                int64_t rows, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !G1 || !G2 || !out || rows < 0) return fail(HWG_EINVAL, "bad argument");
    if (rows == 0) return HWG_OK;
    CK(launch_bt_side(G1, G2, E0, out, c->grid, c->SM, c->SA, rows, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_mg_rows_dev(hwg_ctx *c, const int32_t *ops, const double *B, double *X, int64_t rows,
                    void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !ops || !B || !X || rows < 0) return fail(HWG_EINVAL, "bad argument");
    if (B == X) return fail(HWG_EINVAL, "MG input and output may not alias");
    if (rows == 0) return HWG_OK;
    return mg_apply(c, B, X, rows, 0, ops, S(stream));
}

int hwg_mg_rows_dev_dot(hwg_ctx *c, const int32_t *ops, const double *B, double *X, int64_t rows,
                        const double *Y, double *part, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !ops || !B || !X || !Y || !part || rows < 0) return fail(HWG_EINVAL, "bad argument");
    if (B == X) return fail(HWG_EINVAL, "MG input and output may not alias");
    if (rows == 0) return HWG_OK;
    return mg_apply(c, B, X, rows, 0, ops, S(stream), Y, part);
}

int hwg_row_partials(hwg_ctx *c, const double *X, const double *Y, int64_t rows, double *part,
                     void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || !part || rows < 0) return fail(HWG_EINVAL, "bad argument");
    CK(launch_row_partials(X, Y, rows, c->nx, part, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_tree_sum(hwg_ctx *c, const double *part, int64_t n, double *result, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !part || !result || n < 0 || n + 4 > c->red_max) return fail(HWG_EINVAL, "bad argument");
    CK(launch_tree(part, n, c->tmp, result, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_axpy(hwg_ctx *c, double a, const double *X, double *Y, int64_t n, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || n < 0) return fail(HWG_EINVAL, "bad argument");
    CK(launch_axpy(a, X, Y, n, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_xpay(hwg_ctx *c, double a, const double *X, double *Y, int64_t n, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || n < 0) return fail(HWG_EINVAL, "bad argument");
    CK(launch_xpay(a, X, Y, n, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_pcg_scalar(hwg_ctx *c, int step, double *scal, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !scal || (step != 0 && step != 1)) return fail(HWG_EINVAL, "bad argument");
    CK(step == 0 ? launch_pcg_alpha(scal, S(stream)) : launch_pcg_beta(scal, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_pcg_update_wr(hwg_ctx *c, double *w, double *r, const double *p, const double *q,
                      const double *scal, int64_t n, int do_w, int do_r, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !scal || n < 0 || (do_w && (!w || !p)) || (do_r && (!r || !q)))
        return fail(HWG_EINVAL, "bad argument");
    if (n == 0 || (!do_w && !do_r)) return HWG_OK;
    CK(launch_update_wr(w, r, p, q, scal, n, do_w ? 1 : 0, do_r ? 1 : 0, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_pcg_update_wp(hwg_ctx *c, double *w, double *p, const double *z, const double *scal,
                      int64_t n, int do_w, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !p || !z || !scal || n < 0 || (do_w && !w)) return fail(HWG_EINVAL, "bad argument");
    if (n == 0) return HWG_OK;
    CK(launch_update_wp(w, p, z, scal, n, do_w ? 1 : 0, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_sub(hwg_ctx *c, const double *f, const double *t, double *r, int64_t n, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !f || !t || !r || n < 0) return fail(HWG_EINVAL, "bad argument");
    if (n == 0) return HWG_OK;
    CK(launch_sub(f, t, r, n, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_any_nonzero(hwg_ctx *c, const double *X, int64_t n, int32_t *flag, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !flag || n < 0) return fail(HWG_EINVAL, "bad argument");
    if (n == 0) return HWG_OK;
    CK(launch_any_nonzero(X, n, (int *)flag, S(stream)));
    ++c->launches;
    return HWG_OK;
}

int hwg_temporal_rows(hwg_ctx *c, int band, const double *X, int64_t x0, double *Y, int64_t r0,
                      int64_t nr, void *stream)
{
    DeviceGuard dg_(c);
    if (!c || !X || !Y || nr < 0 || r0 < 0) return fail(HWG_EINVAL, "bad argument");
    const DevBand *bands[8] = {&c->Mt, &c->At, &c->L, &c->LT, &c->T, &c->TT, &c->Nn, &c->NT};
    if (band < 0 || band > 7) return fail(HWG_EINVAL, "unknown temporal band");
    const int64_t rows = (band == 4 || band == 6) ? 2 * (c->nt - 1) : c->nt;
    if (r0 + nr > rows) return fail(HWG_EINVAL, "row range outside the band");
    CK(launch_temporal_rows(bands[band]->view(), X, x0, Y, r0, nr, c->nx, S(stream)));
    ++c->launches;
    return HWG_OK;
}

}  // extern "C"
