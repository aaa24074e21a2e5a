// engine.cu -- the slot engine and the C ABI (include/bhpp.h).
//
// An Engine<T, B> owns the device state of B query slots (node-major,
// slot-minor) and drives rounds: K1 prep -> K2/K2b V pull -> K3/K3b U pull ->
// K4 control -> K5/K6 finalize + top-k.  Query control lives on the device
// (K4), so the host only launches rounds and polls one flag every few rounds;
// finished slots are refilled from the batch queue inside K4.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>

#include "control.cuh"
#include "kernels.cuh"
#include "topk.cuh"
#include <nvtx3/nvToolsExt.h>

#include "small.cuh"
#include "frontier.cuh"

namespace bh {
// BH_TRACE_E2E diagnostics: host timestamps (us) of the stages of a host-pointer batch
static double g_tstamp[8];
static inline double host_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace bh
namespace bh {

bh_graph *graph_create(int64_t, int64_t, int64_t, const int64_t *, const int32_t *, const double *,
                       const int64_t *, const int32_t *, const double *, const double *, const double *,
                       int32_t, int32_t);
void graph_free_arrays(bh_graph *g);

static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches += n; }

static thread_local std::string t_err;

template <typename X>
static X *dalloc(size_t count) {
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, count * sizeof(X)));
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        throw std::bad_alloc();
    }
    if (e != cudaSuccess) throw CudaError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return (X *)p;
}

// ---------------------------------------------------------------------------
// small utility kernels
// Slot column s of a [n][B] state array to / from a caller-order vector
// (perm: store -> caller index, null for the identity).
template <typename T>
__global__ void k_col_get(const T *X, int B, int s, int64_t n, const int32_t *perm, double *out) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        out[perm ? perm[u] : u] = (double)X[u * B + s];
}
template <typename T>
__global__ void k_col_set(T *X, int B, int s, int64_t n, const int32_t *perm, const double *in) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        X[u * B + s] = (T)in[perm ? perm[u] : u];
}

// Launch a round kernel with programmatic stream serialization (PDL) and,
// optionally, an L2 access-policy window (persisting hub slab of the operand).
template <typename... KArgs, typename... Args>
static void launch_pdl_win(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                           const cudaAccessPolicyWindow *win, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (win && win->num_bytes > 0) {
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow = *win;
        cfg.numAttrs = 2;
    }
    BH_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BH_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

static int grid1d(int64_t n, int threads = 256, int cap = 148 * 16) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap));
}

// ---------------------------------------------------------------------------
struct RunSpec {
    int32_t job = BH_JOB_BHPP;
    int64_t n_q = 0;
    const int32_t *sources = nullptr;  // device
    const int32_t *tie = nullptr;      // device or null
    double alpha = 0.15, lam = 1.0, eps_b = 1e-6, eps_f = 1e-6;
    int32_t power_t = 0;
    int64_t init_np = 0;
    const double *x0 = nullptr;          // device [n_q][n_u] (POWER)
    const double *ledger_r = nullptr;    // device [n_u] (PI_PUSH, slot 0)
    const double *ledger_est = nullptr;  // device [n_u] (PI_PUSH, slot 0)
    int32_t k = 0, exclude = 0, want_scores = 0;
    int32_t *topk_idx = nullptr;  // device
    double *topk_score = nullptr;
    bh_trace *trace = nullptr;
    double *scores = nullptr;
    bh_round_hook hook = nullptr;
    void *hook_user = nullptr;
    bool async = false;  // graph path only: enqueue and return (finish() completes)
};

static std::atomic<int> g_profiling{0};
// push_engine._SCATTER_LIMIT (push_engine.py:44): a round runs in frontier form when
// the pushed rows touch at most this fraction of |E| (bh_set_scatter_limit)
static std::atomic<double> g_scatter_limit{0.01};
static double scatter_limit() { return g_scatter_limit.load(); }

struct EngineBase {
    virtual ~EngineBase() = default;
    bh_run_stats stats{};
    virtual void run(const RunSpec &rs, cudaStream_t st) = 0;
    virtual void finish() = 0;  // completes an async run
    virtual void read_ledger(int s, double *r_u_dev, double *est_dev, cudaStream_t st) = 0;
    virtual void slot_state(int s, Slot *out, cudaStream_t st) = 0;
    int nslots = 0;
    int k_cap = 0;
};

// Merge-path partition of one pull side into n_warps contiguous edge ranges
// balanced on (edges + ROWCOST * rows), boundaries snapped to row starts where
// the row is short; rows cut by a boundary get one partial
// slot per warp touching them (SURVEY.md sec. 7 hard part 3: hub rows of
// ~1e6 edges must not serialise).
struct SidePlan {
    WarpWork *work = nullptr;
    CutRow *cuts = nullptr;
    int32_t *cut_count = nullptr;
    int32_t n_warps = 0, n_cuts = 0, n_parts = 0;
    int grid = 1;
    int threads = PULL_THREADS;  // block size of the dense pull
    int front_grid = 1;          // 256-thread blocks covering the same n_warps (frontier pulls)
    void free_all() {
        cudaFree(work);
        cudaFree(cuts);
        cudaFree(cut_count);
        work = nullptr;
        cuts = nullptr;
        cut_count = nullptr;
    }
};

static void build_plan(const Side &sd, int64_t n_e, int n_warps, SidePlan &pl, int64_t row_cost) {
    const int64_t ROWCOST = row_cost;
    const std::vector<int64_t> &ip = sd.h_indptr;
    const int64_t n = sd.n_rows;
    const int64_t total = n_e + ROWCOST * n;
    const int64_t snap = std::max<int64_t>(32, n_e / std::max(1, n_warps) / 8);
    std::vector<int64_t> eb((size_t)n_warps + 1);
    eb[0] = 0;
    eb[n_warps] = n_e;
    for (int w = 1; w < n_warps; w++) {
        const int64_t d = (int64_t)((__int128)total * w / n_warps);
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (ip[mid] + ROWCOST * mid <= d) lo = mid; else hi = mid - 1;
        }
        int64_t e = lo >= n ? n_e : std::min(std::max(d - ROWCOST * lo, ip[lo]), ip[lo + 1]);
        // a boundary inside a short row moves to the nearer row start: only rows that are long
        // against a warp's range (hubs) are cut, so most warps skip the cut protocol (two
        // fences and an atomic per cut) at the cost of at most snap / 2 edges of imbalance
        if (lo < n && ip[lo + 1] - ip[lo] <= snap) e = (e - ip[lo] < ip[lo + 1] - e) ? ip[lo] : ip[lo + 1];
        eb[w] = std::max(e, eb[w - 1]);
    }
    std::vector<WarpWork> work((size_t)n_warps);
    std::vector<CutRow> cuts;
    int32_t parts = 0;
    auto add_part = [&](int64_t row, int32_t &ci, int32_t &pi) {
        if (cuts.empty() || cuts.back().row != (int32_t)row) cuts.push_back({(int32_t)row, 0, parts, 0});
        ci = (int32_t)cuts.size() - 1;
        pi = parts++;
        cuts.back().n_parts++;
    };
    for (int w = 0; w < n_warps; w++) {
        WarpWork &wk = work[w];
        wk.e0 = eb[w];
        wk.e1 = eb[w + 1];
        wk.cut0 = wk.part0 = wk.cut1 = wk.part1 = -1;
        wk.r0 = 0;
        wk.pad = 0;
        if (wk.e0 >= wk.e1) continue;
        const int64_t r0 = std::upper_bound(ip.begin(), ip.end(), wk.e0) - ip.begin() - 1;
        const int64_t rl = std::upper_bound(ip.begin(), ip.end(), wk.e1 - 1) - ip.begin() - 1;
        wk.r0 = (int32_t)r0;
        if (ip[r0] < wk.e0 || ip[r0 + 1] > wk.e1) add_part(r0, wk.cut0, wk.part0);
        if (rl != r0 && ip[rl + 1] > wk.e1) add_part(rl, wk.cut1, wk.part1);
    }
    pl.n_warps = n_warps;
    pl.n_cuts = (int32_t)cuts.size();
    pl.n_parts = parts;
    pl.work = dalloc<WarpWork>(work.size());
    BH_CUDA(cudaMemcpy(pl.work, work.data(), work.size() * sizeof(WarpWork), cudaMemcpyHostToDevice));
    pl.cuts = dalloc<CutRow>(std::max<size_t>(1, cuts.size()));
    if (!cuts.empty()) BH_CUDA(cudaMemcpy(pl.cuts, cuts.data(), cuts.size() * sizeof(CutRow), cudaMemcpyHostToDevice));
    pl.cut_count = dalloc<int32_t>(std::max<size_t>(1, cuts.size()));
    BH_CUDA(cudaMemset(pl.cut_count, 0, std::max<size_t>(1, cuts.size()) * sizeof(int32_t)));
}

template <typename T, int B>
struct Engine final : EngineBase {
    static constexpr bool WIDE = B >= 32;
    bh_graph *g;
    T *R = nullptr, *P = nullptr, *XV = nullptr, *Y = nullptr;
    T *EST = nullptr;      // estimates, storage type (fp32 mode: fp32, SURVEY 8(d)'s s bytes)
    double *OUTS = nullptr;
    Slot *slots = nullptr;
    Finish *fins = nullptr;
    Control *ctl = nullptr;
    Control *h_ctl = nullptr;
    Partials part{};
    double *scratch = nullptr;
    uint64_t *cand_key = nullptr;
    int64_t *cand_idx = nullptr;
    double *hook_r = nullptr, *hook_est = nullptr;
    int32_t *chunk_done = nullptr;
    std::vector<cudaEvent_t> evpool;
    SidePlan plan_v, plan_u;
    // K-F frontier rounds (frontier.cuh): control block, K1's pushed-node flags,
    // row bitmaps, work items and split-row partials per side
    FrontCtl *front = nullptr;
    FrontCtl *h_front = nullptr;
    uint8_t *flag_u = nullptr;
    FrontPiece *hub_pieces = nullptr;
    int64_t n_hub_pieces = 0;
    uint32_t *bits_v = nullptr, *bits_u = nullptr;
    FrontItem *items_v = nullptr, *items_u = nullptr;
    double *fscr_v = nullptr, *fscr_u = nullptr;
    int32_t *pcnt_v = nullptr, *pcnt_u = nullptr;
    int grid_front = 1;
    cudaGraphConditionalHandle fcond{};
    int use_fcond = 0;  // K1 sets the graph's IF/ELSE condition (capture of the batch graph)
    // Frontier rounds are compiled into a run when the scatter limit allows them
    // and the block is narrow (B <= FRONT_MAX_B) or the limit forces them (>= 1):
    // for 32+ slots in mixed phases the union frontier is dense in practically
    // every round (a slot in power iteration makes it all of U), and the per-round
    // decision (K1's flags + ticket, the IF/ELSE node) costs ~8 % at c2.
    static constexpr int FRONT_MAX_B = 16;
    bool front_on = false;
    // L2 residency of the gathered operands' hub slabs (store rows [0, h) of P for
    // the V pull, of XV for the U pull; degree-ordered store): empty windows
    // unless the operands outgrow L2 (BH_L2_PERSIST_MB overrides the carve-out)
    cudaAccessPolicyWindow win_v{}, win_u{};
    // one batch = one CUDA graph: a WHILE node around one round, condition set by K4
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaStream_t cap_stream = nullptr;
    std::vector<unsigned char> graph_key;
    int fin_chunk = SEL_ITEMS * TOPK_THREADS, n_chunks = 1;  // one register-cached select per chunk
    int grid_elem = 1, grid_comb = 1, grid_k5 = 1;  // K1 / K1a grids (one resident wave each)

    // Elementwise K1 / K1a geometry (nodes in flight per thread, blocks per SM),
    // measured at c2 on B200 (profiles/r01_pull_variants.md): fp32 K1 one node
    // per thread at 4 blocks/SM, K1a software-pipelined at 3 blocks/SM; fp64 two
    // nodes per thread at 2 blocks/SM.  The same geometry is at least as fast in
    // the HBM regime (c3: 4-8 nodes per thread measured equal or slower,
    // profiles/r02_store_ab.md), so there is one geometry per dtype.
    using ElemFn = void (*)(ElemArgs<T>);
    ElemFn push_kernel() const {
        if (front_on) {
            if constexpr (sizeof(T) == 4 && B >= 32) return k_push<B, T, 1, 4, false, true>;
            else return k_push<B, T, 2, 2, false, true>;
        }
        if constexpr (sizeof(T) == 4 && B >= 32) return k_push<B, T, 1, 4>;
        else return k_push<B, T, 2, 2>;
    }
    static ElemFn combine_kernel() {
        if constexpr (sizeof(T) == 4 && B >= 32) return k_combine<B, T, 1, 3, true>;
        else return k_combine<B, T, 2, 2>;
    }

    // Dense pulls.  B < 32: k_pull_small.  B >= 32: the row-flag pull k_pull_rf on the
    // store's flagged edge stream; k_pull_sw (row-pointer walk, SwPipe's default geometry)
    // serves stores without that stream (a caller's graph with an empty row) and BH_PULL=sw.
    using PullFn = void (*)(PullArgs<T>);
    template <int SIDE>
    static PullFn sw_kernel() {
        if constexpr (!WIDE) return k_pull_small<B, T, SIDE>;
        else return k_pull_sw<B, T, SIDE>;
    }
    // Row-flag pull geometries, measured on one B200 (profiles/r02_rf_pull.md): 8 rows in
    // flight per warp; 8-byte lanes (64 fp32 slots) run four blocks of 7 warps per SM (72
    // registers), 16-byte lanes three blocks of 8 (80), 32-byte lanes two blocks of 8.
    // BH_RF_GEO="v,u" overrides per side for A/B runs.
    static constexpr int RF_GEOS = 3;
    template <int SIDE>
    static PullFn rf_kernel(int geo) {
        if constexpr (!WIDE) {
            return nullptr;
        } else {
            switch (geo) {
                case 0: return k_pull_rf<B, T, SIDE, 8, 3>;
                case 1: return k_pull_rf<B, T, SIDE, 8, 2>;
                default: return k_pull_rf<B, T, SIDE, 8, 4, 7>;
            }
        }
    }
    static int rf_warps(int geo) { return geo == 2 ? 7 : PULL_WARPS; }
    bool use_rf = false;
    int rf_geo[2] = {0, 0};
    PullFn pull_kernel(int side) const {
        if (use_rf) return side == SIDE_V ? rf_kernel<SIDE_V>(rf_geo[0]) : rf_kernel<SIDE_U>(rf_geo[1]);
        return side == SIDE_V ? sw_kernel<SIDE_V>() : sw_kernel<SIDE_U>();
    }

    explicit Engine(bh_graph *graph) : g(graph) {
        this->nslots = B;
        const int64_t nu = g->n_u, nv = g->n_v;
        R = dalloc<T>(nu * B);
        P = dalloc<T>(nu * B);
        Y = dalloc<T>(nu * B);
        XV = dalloc<T>(nv * B);
        EST = dalloc<T>(nu * B);
        OUTS = dalloc<double>(nu * B);
        slots = dalloc<Slot>(B);
        fins = dalloc<Finish>(B);
        ctl = dalloc<Control>(1);
        BH_CUDA(cudaMallocHost(&h_ctl, sizeof(Control)));
        BH_CUDA(cudaMemset(R, 0, nu * B * sizeof(T)));
        BH_CUDA(cudaMemset(P, 0, nu * B * sizeof(T)));
        BH_CUDA(cudaMemset(Y, 0, nu * B * sizeof(T)));
        BH_CUDA(cudaMemset(XV, 0, nv * B * sizeof(T)));
        BH_CUDA(cudaMemset(EST, 0, nu * B * sizeof(T)));
        BH_CUDA(cudaMemset(ctl, 0, sizeof(Control)));
        int sms = 148;
        BH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
        setup_l2_windows(nu, nv);
        // dense pull selection: the row-flag pull when the store has the flagged edge
        // stream (no empty row); BH_PULL=sw keeps the row-pointer pull (A/B)
        use_rf = WIDE && g->U.ecv && g->V.ecv;
        if (const char *m = getenv("BH_PULL")) use_rf = use_rf && strcmp(m, "sw") != 0;
        if (use_rf) {
            constexpr int LB = (B / 32) * (int)sizeof(T);
            rf_geo[0] = rf_geo[1] = LB <= 8 ? 2 : (LB <= 16 ? 0 : 1);  // 8-byte lanes: 4 blocks of 7 warps; 16: 3 of 8; 32: 2 of 8
            if (const char *m = getenv("BH_RF_GEO")) {  // "v,u"
                int gv = rf_geo[0], gu = rf_geo[1];
                const int k = sscanf(m, "%d,%d", &gv, &gu);
                if (k == 1) gu = gv;
                if (k >= 1) {
                    rf_geo[0] = std::min(std::max(gv, 0), RF_GEOS - 1);
                    rf_geo[1] = std::min(std::max(gu, 0), RF_GEOS - 1);
                }
            }
        }
        for (int side = 0; side < 2; side++) {
            const Side &sd = side == SIDE_V ? g->V : g->U;
            SidePlan &pl = side == SIDE_V ? plan_v : plan_u;
            PullFn fn = pull_kernel(side);
            const int wpb = use_rf ? rf_warps(rf_geo[side]) : PULL_WARPS;
            pl.threads = wpb * 32;
            int occ = 1;
            BH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, pl.threads, 0));
            occ = std::max(1, occ);
            // one resident wave of warps, fewer if the side is tiny
            int64_t grid = (int64_t)occ * sms;
            const int64_t want = (g->n_e + 2 * sd.n_rows) / 64 / wpb + 1;
            grid = std::max<int64_t>(1, std::min(grid, want));
            pl.grid = (int)grid;
            pl.front_grid = (int)((grid * wpb + PULL_WARPS - 1) / PULL_WARPS);
            // cost of a row in edges: a V-pull emit also counts n_p (measured at c2, rows of 10 / 20
            // edges, profiles/r02_rf_pull.md: V 2 -> 3 gains 1.3 %, U 2 -> 1 gains 2 %; 0 and >= 4
            // lose 4-30 %)
            build_plan(sd, g->n_e, (int)grid * wpb, pl, use_rf ? (side == SIDE_V ? 3 : 1) : 2);
        }
        {  // one resident wave of the elementwise kernels
            int occ_p = 1, occ_c = 1;
            BH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, push_kernel(), ELEM_THREADS, 0));
            BH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, combine_kernel(), ELEM_THREADS, 0));
            grid_elem = grid1d(nu * (B / ElemGeo<B>::EV), ELEM_THREADS, std::max(1, occ_p) * sms);
            grid_comb = grid1d(nu * (B / ElemGeo<B>::EV), ELEM_THREADS, std::max(1, occ_c) * sms);
        }
        n_chunks = (int)((nu + fin_chunk - 1) / fin_chunk);
        grid_k5 = (int)std::min<int64_t>((int64_t)n_chunks * std::min(B, 16), 16 * sms);
        part.rows_k1 = grid_elem;
        part.rows_k2 = plan_v.n_warps;
        part.rows_k3 = grid_comb;
        part.cnt = dalloc<int64_t>((size_t)grid_elem * B);
        part.np_u = dalloc<int64_t>((size_t)grid_elem * B);
        part.lmass = dalloc<double>((size_t)grid_elem * B);
        BH_CUDA(cudaMemset(part.lmass, 0, (size_t)grid_elem * B * sizeof(double)));
        part.np_v = dalloc<int64_t>((size_t)plan_v.n_warps * B);
        part.any = dalloc<int32_t>((size_t)part.rows_k3 * B);
        part.sum = dalloc<double>((size_t)part.rows_k3 * B);
        part.wsum = dalloc<double>((size_t)part.rows_k3 * B);
        BH_CUDA(cudaMemset(part.np_v, 0, (size_t)plan_v.n_warps * B * sizeof(int64_t)));
        BH_CUDA(cudaMemset(part.cnt, 0, (size_t)grid_elem * B * sizeof(int64_t)));
        BH_CUDA(cudaMemset(part.np_u, 0, (size_t)grid_elem * B * sizeof(int64_t)));
        const int64_t parts = std::max<int64_t>(1, std::max(plan_u.n_parts, plan_v.n_parts));
        scratch = dalloc<double>((size_t)parts * B);
        hook_r = dalloc<double>(nu);
        hook_est = dalloc<double>(nu);
        chunk_done = dalloc<int32_t>(MAX_B);
        BH_CUDA(cudaMemset(chunk_done, 0, MAX_B * sizeof(int32_t)));
        {  // frontier buffers (FRONT_CHUNK-edge items; a split row of d edges has <= 2 d / CHUNK parts)
            const int64_t ne = g->n_e, chunks = ne / FRONT_CHUNK + 2, parts = 2 * chunks;
            front = dalloc<FrontCtl>(1);
            BH_CUDA(cudaMallocHost(&h_front, sizeof(FrontCtl)));
            BH_CUDA(cudaMemset(front, 0, sizeof(FrontCtl)));
            flag_u = dalloc<uint8_t>(nu);
            BH_CUDA(cudaMemset(flag_u, 0, nu));
            std::vector<FrontPiece> pcs;  // hub U rows cut into FRONT_WALK-edge claim pieces
            for (int64_t r = 0; r < nu; r++) {
                const int64_t e0 = g->U.h_indptr[r], e1 = g->U.h_indptr[r + 1];
                if (e1 - e0 <= FRONT_WALK) continue;
                for (int64_t e = e0; e < e1; e += FRONT_WALK) pcs.push_back({e, std::min(e1, e + FRONT_WALK), (int32_t)r, 0});
            }
            n_hub_pieces = (int64_t)pcs.size();
            hub_pieces = dalloc<FrontPiece>(std::max<size_t>(1, pcs.size()));
            if (!pcs.empty())
                BH_CUDA(cudaMemcpy(hub_pieces, pcs.data(), pcs.size() * sizeof(FrontPiece), cudaMemcpyHostToDevice));
            bits_v = dalloc<uint32_t>((nv + 31) / 32);
            bits_u = dalloc<uint32_t>((nu + 31) / 32);
            BH_CUDA(cudaMemset(bits_v, 0, ((nv + 31) / 32) * 4));
            BH_CUDA(cudaMemset(bits_u, 0, ((nu + 31) / 32) * 4));
            // item slots: rows + hub chunks, at most doubled by the per-warp allocation
            // chunks (an abandoned chunk is at least half used), plus one open chunk per
            // warp of the claim kernels
            grid_front = 4 * sms;
            const int64_t open = (int64_t)FRONT_ITEM_CHUNK * grid_front * 8 + FRONT_ITEM_CHUNK;
            items_v = dalloc<FrontItem>(2 * (nv + chunks) + open);
            items_u = dalloc<FrontItem>(2 * (nu + chunks) + open);
            fscr_v = dalloc<double>((size_t)parts * B);
            fscr_u = dalloc<double>((size_t)parts * B);
            pcnt_v = dalloc<int32_t>(parts);
            pcnt_u = dalloc<int32_t>(parts);
            BH_CUDA(cudaMemset(pcnt_v, 0, parts * 4));
            BH_CUDA(cudaMemset(pcnt_u, 0, parts * 4));
        }
    }

    void setup_l2_windows(int64_t nu, int64_t nv) {
        int l2 = 0, maxp = 0, maxwin = 0;
        BH_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device));
        BH_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, g->device));
        BH_CUDA(cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, g->device));
        const double row = (double)B * sizeof(T);
        const double operands = row * (double)(nu + nv);
        // Off by default: at c3 the carve-out slowed K1 / K1a by 35 % and gained
        // the pulls 2-5 %, a net loss (profiles/r02_store_ab.md); opt-in with
        // BH_L2_PERSIST_MB (a carve-out of that size, shared by the two windows)
        double mb = 0.0;
        (void)operands;
        if (const char *m = getenv("BH_L2_PERSIST_MB")) mb = atof(m);
        if (!g->relabeled || mb <= 0 || maxp <= 0 || maxwin <= 0) return;
        const size_t carve = std::min<size_t>((size_t)maxp, (size_t)(mb * 1048576.0));
        // the carve-out is shared by the two windows (one per pull), in proportion
        // to the operands' sizes but at most their whole size
        const double fu = (double)nu / (double)(nu + nv);
        auto make = [&](cudaAccessPolicyWindow &w, void *base, int64_t rows, double share) {
            const size_t full = (size_t)(row * (double)rows);
            size_t bytes = std::min<size_t>({full, (size_t)maxwin, (size_t)(share * (double)carve)});
            w.base_ptr = base;
            w.num_bytes = bytes;
            w.hitRatio = 1.0f;
            w.hitProp = cudaAccessPropertyPersisting;
            w.missProp = cudaAccessPropertyStreaming;
        };
        make(win_v, P, nu, fu);
        make(win_u, XV, nv, 1.0 - fu);
        size_t cur = 0;
        BH_CUDA(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
        if (cur < carve) BH_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
        l2_carve = carve;
    }
    size_t l2_carve = 0;

    ~Engine() override {
        cudaFree(R); cudaFree(P); cudaFree(Y); cudaFree(XV); cudaFree(EST); cudaFree(OUTS);
        cudaFree(slots); cudaFree(fins); cudaFree(ctl); cudaFreeHost(h_ctl);
        cudaFree(part.cnt); cudaFree(part.np_u); cudaFree(part.np_v); cudaFree(part.lmass);
        cudaFree(part.any); cudaFree(part.sum); cudaFree(part.wsum);
        cudaFree(scratch); cudaFree(cand_key); cudaFree(cand_idx);
        cudaFree(hook_r); cudaFree(hook_est); cudaFree(chunk_done);
        cudaFree(front); cudaFreeHost(h_front); cudaFree(flag_u); cudaFree(hub_pieces); cudaFree(bits_v); cudaFree(bits_u);
        cudaFree(items_v); cudaFree(items_u); cudaFree(fscr_v); cudaFree(fscr_u); cudaFree(pcnt_v); cudaFree(pcnt_u);
        plan_u.free_all();
        plan_v.free_all();
        for (auto e : evpool) cudaEventDestroy(e);
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (graph) cudaGraphDestroy(graph);
        if (cap_stream) cudaStreamDestroy(cap_stream);
    }

    cudaEvent_t ev(size_t i) {
        while (evpool.size() <= i) {
            cudaEvent_t e;
            BH_CUDA(cudaEventCreate(&e));
            evpool.push_back(e);
        }
        return evpool[i];
    }

    void ensure_cand(int k) {
        if (k <= k_cap) return;
        cudaFree(cand_key);
        cudaFree(cand_idx);
        cand_key = dalloc<uint64_t>((size_t)B * n_chunks * k);
        cand_idx = dalloc<int64_t>((size_t)B * n_chunks * k);
        k_cap = k;
    }

    PullArgs<T> pull_args(int side, double alpha) {
        const double one_minus_alpha = 1.0 - alpha;
        PullArgs<T> a{};
        const Side &sd = side == SIDE_V ? g->V : g->U;
        const SidePlan &pl = side == SIDE_V ? plan_v : plan_u;
        a.indptr = sd.indptr;
        a.n_rows = sd.n_rows;
        a.indices = sd.indices;
        a.vals = (const T *)sd.vals;
        a.work = pl.work;
        a.cuts = pl.cuts;
        a.cut_count = pl.cut_count;
        a.scratch = scratch;
        a.n_warps = pl.n_warps;
        a.X = side == SIDE_V ? P : XV;
        a.Y = side == SIDE_V ? XV : Y;
        a.slots = slots;
        a.active = &ctl->active;
        a.np_v = part.np_v;
        a.one_minus_alpha = one_minus_alpha;
        a.ecv = sd.ecv;
        return a;
    }

    void launch_pull(int side, const PullArgs<T> &a, cudaStream_t st) {
        const SidePlan &pl = side == SIDE_V ? plan_v : plan_u;
        launch_pdl_win(pull_kernel(side), pl.grid, pl.threads, 0, st, side == SIDE_V ? &win_v : &win_u, a);
    }

    ElemArgs<T> elem_args(const RunSpec &rs) {
        ElemArgs<T> ea{};
        ea.n_u = g->n_u;
        ea.R = R;
        ea.P = P;
        ea.Y = Y;
        ea.EST = EST;
        ea.deg_u = g->U.deg;
        ea.ws_u = g->ws_u;
        ea.inv_ws_u = g->inv_ws_u;
        ea.x0 = rs.x0;
        ea.perm_u = g->U.perm;
        ea.slots = slots;
        ea.active = &ctl->active;
        ea.part = part;
        ea.alpha = rs.alpha;
        ea.front = front_on ? front : nullptr;
        ea.flag_u = front_on ? flag_u : nullptr;
        ea.fcond = fcond;
        ea.use_fcond = use_fcond;
        return ea;
    }

    FrontArgs front_args() const {
        FrontArgs fa{};
        fa.f = front;
        fa.active = &ctl->active;
        fa.B = B;
        fa.elem_bytes = (int)sizeof(T);
        fa.n_u = g->n_u;
        fa.n_v = g->n_v;
        fa.n_e = g->n_e;
        fa.u_ptr = g->U.indptr;
        fa.v_ptr = g->V.indptr;
        fa.u_col = g->U.indices;
        fa.v_col = g->V.indices;
        fa.flag_u = flag_u;
        fa.hub_pieces = hub_pieces;
        fa.n_hub_pieces = n_hub_pieces;
        fa.bits_v = bits_v;
        fa.bits_u = bits_u;
        fa.items_v = items_v;
        fa.items_u = items_u;
        fa.XV = XV;
        fa.Y = Y;
        return fa;
    }

    FrontPullArgs<T> front_pull_args(int side, double alpha) const {
        FrontPullArgs<T> a{};
        const Side &sd = side == SIDE_V ? g->V : g->U;
        a.f = front;
        a.active = &ctl->active;
        a.indptr = sd.indptr;
        a.indices = sd.indices;
        a.vals = (const T *)sd.vals;
        a.items = side == SIDE_V ? items_v : items_u;
        a.X = side == SIDE_V ? P : XV;
        a.Y = side == SIDE_V ? XV : Y;
        a.scratch = side == SIDE_V ? fscr_v : fscr_u;
        a.pcnt = side == SIDE_V ? pcnt_v : pcnt_u;
        a.slots = slots;
        a.np_v = part.np_v;
        a.n_warps = plan_v.n_warps;
        a.scale = side == SIDE_V ? 1.0 - alpha : 1.0;
        return a;
    }

    // The V / U halves of a frontier round (Fa Fb Fc | Fd Fe + the dense U pull
    // when the U half is dense), each kernel gated on FrontCtl.
    void launch_front_v(double alpha, cudaStream_t st) {
        const FrontArgs fa = front_args();
        launch_pdl(k_front_reset, grid_front, 256, 0, st, fa);
        launch_pdl(k_front_mark<SIDE_V>, grid_front, 256, 0, st, fa);
        launch_pdl(k_front_pull<B, T, SIDE_V>, plan_v.front_grid, PULL_THREADS, 0, st, front_pull_args(SIDE_V, alpha));
        count_launch(3);
        stats.launches += 3;
    }
    void launch_front_u(double alpha, cudaStream_t st) {
        const FrontArgs fa = front_args();
        launch_pdl(k_front_mark<SIDE_U>, grid_front, 256, 0, st, fa);
        launch_pdl(k_front_pull<B, T, SIDE_U>, plan_u.front_grid, PULL_THREADS, 0, st, front_pull_args(SIDE_U, alpha));
        PullArgs<T> pu = pull_args(SIDE_U, alpha);
        pu.active = &front->gate_udense;
        launch_pull(SIDE_U, pu, st);
        count_launch(3);
        stats.launches += 3;
    }
    void launch_dense(int side, double alpha, cudaStream_t st) {
        PullArgs<T> pa = pull_args(side, alpha);
        if (front_on) pa.active = &front->gate_dense;
        launch_pull(side, pa, st);
        count_launch(1);
        stats.launches += 1;
    }

    // One round: K5 (the slots K4 finished last round) | K1 K2 K3 K1a | K4.  In the
    // batch graph K5 sits under an IF node on a branch parallel to K1..K1a (a finished
    // slot is refilled one round later, so nothing else touches its columns meanwhile),
    // and the pulls under an IF/ELSE node set by K1 (frontier / dense).  Eagerly, both
    // forms are launched and gate themselves.
    void launch_round(const RunSpec &rs, const ControlArgs &ca, const FinalArgs<T> &fa, cudaStream_t st,
                      int64_t round, bool prof, bool with_k5 = true, bool with_k4 = true) {
        const size_t e0 = (size_t)round * 7;
        const ElemArgs<T> ea = elem_args(rs);
        if (prof) BH_CUDA(cudaEventRecord(ev(e0), st));
        if (with_k5) {
            launch_pdl(k_finalize<T>, grid_k5, TOPK_THREADS, 0, st, fa);
            count_launch(1);
            stats.launches += 1;
        }
        if (prof) BH_CUDA(cudaEventRecord(ev(e0 + 1), st));
        launch_pdl(push_kernel(), grid_elem, ELEM_THREADS, 0, st, ea);
        if (prof) BH_CUDA(cudaEventRecord(ev(e0 + 2), st));
        if (front_on) launch_front_v(rs.alpha, st);
        launch_dense(SIDE_V, rs.alpha, st);
        if (prof) BH_CUDA(cudaEventRecord(ev(e0 + 3), st));
        if (front_on) launch_front_u(rs.alpha, st);
        launch_dense(SIDE_U, rs.alpha, st);
        if (prof) BH_CUDA(cudaEventRecord(ev(e0 + 4), st));
        launch_pdl(combine_kernel(), grid_comb, ELEM_THREADS, 0, st, ea);
        if (prof) BH_CUDA(cudaEventRecord(ev(e0 + 5), st));
        if (with_k4) launch_pdl(k_control, B, CONTROL_THREADS, 0, st, ca);
        if (prof) BH_CUDA(cudaEventRecord(ev(e0 + 6), st));
        const int n = 2 + (with_k4 ? 1 : 0);
        count_launch(n);
        stats.launches += n;
        BH_CUDA(cudaGetLastError());
    }


    void collect_profile(int64_t rounds) {
        // events per round: K5 | K1 | K2 | K3 | K1a | K4
        double t[6] = {0, 0, 0, 0, 0, 0};
        for (int64_t r = 0; r < rounds; r++) {
            for (int j = 0; j < 6; j++) {
                float ms = 0.f;
                BH_CUDA(cudaEventElapsedTime(&ms, ev((size_t)r * 7 + j), ev((size_t)r * 7 + j + 1)));
                t[j] += ms;
            }
        }
        stats.ms_prep = t[1] + t[4];
        stats.ms_vpull = t[2];
        stats.ms_upull = t[3];
        stats.ms_control = t[0] + t[5];
        stats.profiled = 1;
    }

    // (Re)build the batch graph when the round's kernel arguments change.
    void ensure_graph(const RunSpec &rs, ControlArgs ca, const FinalArgs<T> &fa) {
        // explicit field-wise key (struct padding is not part of it)
        std::vector<unsigned char> key;
        auto put = [&key](const auto &v) {
            const unsigned char *p = reinterpret_cast<const unsigned char *>(&v);
            key.insert(key.end(), p, p + sizeof(v));
        };
        put(rs.job); put(rs.n_q); put(rs.sources); put(rs.tie); put(rs.alpha); put(rs.lam); put(rs.eps_b);
        put(rs.eps_f); put(rs.power_t); put(rs.init_np); put(rs.x0); put(rs.ledger_r); put(rs.ledger_est);
        put(rs.k); put(rs.exclude); put(rs.want_scores); put(rs.topk_idx); put(rs.topk_score); put(rs.trace);
        put(rs.scores);
        put(ca.budget_scale); put(ca.log_decay); put(ca.max_rounds); put(ca.sources); put(ca.tie_skip);
        put(fa.cand_key); put(fa.cand_idx); put(fa.out_scores); put(fa.chunk_done); put(front_on);
        if (graph_exec && key == graph_key) return;
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (graph) cudaGraphDestroy(graph);
        graph_exec = nullptr;
        graph = nullptr;
        if (!cap_stream) BH_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
        BH_CUDA(cudaGraphCreate(&graph, 0));
        cudaGraphConditionalHandle h;
        BH_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        BH_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        ca.use_cond = 1;
        ca.cond = h;
        // K5 (finalize of the slots the previous round's K4 finished) under an IF node
        // set by K4, on a branch parallel to K1..K1a; K4 waits for both
        cudaGraphConditionalHandle hf;
        BH_CUDA(cudaGraphConditionalHandleCreate(&hf, body, 0, cudaGraphCondAssignDefault));
        ca.use_fin_cond = 1;
        ca.fin_cond = hf;
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hf;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t if_node;
        BH_CUDA(cudaGraphAddNode(&if_node, body, nullptr, 0, &ip));
        cudaGraph_t if_body = ip.conditional.phGraph_out[0];
        cudaGraph_t captured;
        BH_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, if_body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        k_finalize<T><<<grid_k5, TOPK_THREADS, 0, cap_stream>>>(fa);
        BH_CUDA(cudaGetLastError());
        BH_CUDA(cudaStreamEndCapture(cap_stream, &captured));
        const int64_t launches0 = stats.launches, counted0 = g_launches.load();
        if (!front_on) {  // body: K1 -> K2 -> K3 -> K1a -> K4 (PDL chain; K4 also waits for the K5 branch)
            BH_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal));
            launch_round(rs, ca, fa, cap_stream, 0, false, /*with_k5=*/false, /*with_k4=*/false);
            BH_CUDA(cudaStreamUpdateCaptureDependencies(cap_stream, &if_node, 1, cudaStreamAddCaptureDependencies));
            launch_pdl(k_control, B, CONTROL_THREADS, 0, cap_stream, ca);
            BH_CUDA(cudaGetLastError());
            BH_CUDA(cudaStreamEndCapture(cap_stream, &captured));
        } else {
            // body: K1 -> IF/ELSE (frontier pulls | dense pulls, condition set by K1's last
            // block) -> K1a -> K4 (K4 also waits for the K5 branch)
            BH_CUDA(cudaGraphConditionalHandleCreate(&fcond, body, 0, cudaGraphCondAssignDefault));
            use_fcond = 1;
            const ElemArgs<T> ea = elem_args(rs);
            use_fcond = 0;
            BH_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            launch_pdl(push_kernel(), grid_elem, ELEM_THREADS, 0, cap_stream, ea);
            BH_CUDA(cudaGetLastError());
            cudaStreamCaptureStatus cst;
            const cudaGraphNode_t *deps = nullptr;
            size_t n_deps = 0;
            BH_CUDA(cudaStreamGetCaptureInfo(cap_stream, &cst, nullptr, nullptr, &deps, &n_deps));
            if (n_deps != 1) throw CudaError("batch graph: K1 capture has no single node");
            const cudaGraphNode_t k1_node = deps[0];
            BH_CUDA(cudaStreamEndCapture(cap_stream, &captured));
            cudaGraphNodeParams pp = {};
            pp.type = cudaGraphNodeTypeConditional;
            pp.conditional.handle = fcond;
            pp.conditional.type = cudaGraphCondTypeIf;
            pp.conditional.size = 2;  // [0] frontier (condition 1), [1] dense (else)
            cudaGraphNode_t pull_node;
            BH_CUDA(cudaGraphAddNode(&pull_node, body, &k1_node, 1, &pp));
            BH_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, pp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal));
            launch_front_v(rs.alpha, cap_stream);
            launch_front_u(rs.alpha, cap_stream);
            BH_CUDA(cudaGetLastError());
            BH_CUDA(cudaStreamEndCapture(cap_stream, &captured));
            BH_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, pp.conditional.phGraph_out[1], nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal));
            launch_dense(SIDE_V, rs.alpha, cap_stream);
            launch_dense(SIDE_U, rs.alpha, cap_stream);
            BH_CUDA(cudaGetLastError());
            BH_CUDA(cudaStreamEndCapture(cap_stream, &captured));
            BH_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, body, &pull_node, nullptr, 1, cudaStreamCaptureModeThreadLocal));
            combine_kernel()<<<grid_comb, ELEM_THREADS, 0, cap_stream>>>(ea);  // after a conditional node: plain edge
            BH_CUDA(cudaStreamUpdateCaptureDependencies(cap_stream, &if_node, 1, cudaStreamAddCaptureDependencies));
            launch_pdl(k_control, B, CONTROL_THREADS, 0, cap_stream, ca);
            BH_CUDA(cudaGetLastError());
            BH_CUDA(cudaStreamEndCapture(cap_stream, &captured));
        }
        // after the loop: K5 for the slots the last round finished
        BH_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, graph, &node, nullptr, 1, cudaStreamCaptureModeThreadLocal));
        k_finalize<T><<<grid_k5, TOPK_THREADS, 0, cap_stream>>>(fa);
        BH_CUDA(cudaGetLastError());
        BH_CUDA(cudaStreamEndCapture(cap_stream, &captured));
        stats.launches = launches0;
        count_launch((int)(counted0 - g_launches.load()));  // captured, not launched (finish() counts them)
        BH_CUDA(cudaGraphInstantiate(&graph_exec, graph, 0));
        graph_key = key;
    }

    void run(const RunSpec &rs, cudaStream_t st) override {
        if (rs.k > TOPK_MAX) throw InvalidArg("k exceeds the device top-k limit (1024) of bh_query_batch");
        if (rs.k > 0) ensure_cand(rs.k);
        BH_CUDA(cudaMemsetAsync(slots, 0, sizeof(Slot) * B, st));
        Control c0{};
        c0.active = 1;
        c0.n_q = (int32_t)rs.n_q;
        *h_ctl = c0;
        BH_CUDA(cudaMemcpyAsync(ctl, h_ctl, sizeof(Control), cudaMemcpyHostToDevice, st));
        {  // frontier control: every XV / Y row is stale, the scatter limit of this run
            const double lim = scatter_limit();
            front_on = lim >= 0.0 && (B <= FRONT_MAX_B || lim >= 1.0);
            const int64_t li =
                lim < 0.0 ? -1 : (lim * (double)g->n_e >= 9.0e18 ? INT64_MAX : (int64_t)(lim * (double)g->n_e));
            k_front_begin<<<1, 1, 0, st>>>(front, li);
            count_launch();
            BH_CUDA(cudaGetLastError());
        }

        ControlArgs ca{};
        ca.slots = slots;
        ca.fin = fins;
        ca.ctl = ctl;
        ca.part = part;
        ca.sources = rs.sources;
        ca.inv_u = g->U.inv;
        ca.trace = rs.trace;
        ca.tie_skip = rs.tie;
        ca.ws_u = g->ws_u;
        ca.n_u = g->n_u;
        ca.alpha = rs.alpha;
        ca.lam = rs.lam;
        ca.eps_b = rs.eps_b;
        ca.eps_f = rs.eps_f;
        ca.budget_scale = 2.0 * (double)g->n_e;
        ca.log_decay = std::log(1.0 / (1.0 - rs.alpha));
        ca.job = rs.job;
        ca.power_t = rs.power_t;
        ca.init_np = rs.init_np;
        ca.B = B;
        ca.first = 1;
        k_control<<<B, CONTROL_THREADS, 0, st>>>(ca);
        count_launch();
        BH_CUDA(cudaGetLastError());
        ca.first = 0;
        if (rs.job == BH_JOB_PI_PUSH) {  // seed ledger into slot 0 (query 0 -> slot 0)
            k_col_set<T><<<grid1d(g->n_u), 256, 0, st>>>(R, B, 0, g->n_u, g->U.perm, rs.ledger_r);
            k_col_set<T><<<grid1d(g->n_u), 256, 0, st>>>(EST, B, 0, g->n_u, g->U.perm, rs.ledger_est);
            count_launch(2);
        }

        FinalArgs<T> fa{};
        fa.n_u = g->n_u;
        fa.B = B;
        fa.k = rs.k;
        fa.exclude = rs.exclude;
        fa.want_scores = rs.want_scores;
        fa.chunk = fin_chunk;
        fa.n_chunks = n_chunks;
        fa.EST = EST;
        fa.P = P;
        fa.ws_u = g->ws_u;
        fa.perm_u = g->U.perm;
        fa.alpha = rs.alpha;
        fa.fin = fins;
        fa.ctl = ctl;
        fa.outs = OUTS;
        fa.out_scores = rs.scores;
        fa.cand_key = cand_key;
        fa.cand_idx = cand_idx;
        fa.topk_idx = rs.topk_idx;
        fa.topk_score = rs.topk_score;
        fa.trace = rs.trace;
        fa.chunk_done = chunk_done;

        const int poll = rs.hook ? 1 : 8;
        const bool prof = g_profiling.load() != 0;
        stats = bh_run_stats{};
        stats.slots = B;
        stats.launches = 1;
        ca.max_rounds = 100000000;
        if (!rs.hook && !prof && !getenv("BH_NO_GRAPH")) {
            g_tstamp[3] = host_us();
            ensure_graph(rs, ca, fa);
            g_tstamp[4] = host_us();
            BH_CUDA(cudaGraphLaunch(graph_exec, st));
            g_tstamp[5] = host_us();
            BH_CUDA(cudaMemcpyAsync(h_ctl, ctl, sizeof(Control), cudaMemcpyDeviceToHost, st));
            BH_CUDA(cudaMemcpyAsync(h_front, front, sizeof(FrontCtl), cudaMemcpyDeviceToHost, st));
            pending = st;
            if (!rs.async) finish();
            return;
        }
        int32_t last_seq = 0;
        std::vector<double> hr, he;
        const int64_t max_rounds = 100000000;
        for (int64_t round = 0; round < max_rounds;) {
            for (int i = 0; i < poll; i++, round++) {
                launch_round(rs, ca, fa, st, round, prof);
                if (rs.hook) {
                    Slot s0;
                    slot_state(0, &s0, st);
                    if (s0.push_seq != last_seq && s0.last_phase >= 0) {
                        last_seq = s0.push_seq;
                        hr.resize(g->n_u);
                        he.resize(g->n_u);
                        read_ledger(0, hook_r, hook_est, st);
                        BH_CUDA(cudaMemcpyAsync(hr.data(), hook_r, g->n_u * sizeof(double), cudaMemcpyDeviceToHost, st));
                        BH_CUDA(cudaMemcpyAsync(he.data(), hook_est, g->n_u * sizeof(double), cudaMemcpyDeviceToHost, st));
                        BH_CUDA(cudaStreamSynchronize(st));
                        rs.hook(rs.hook_user, s0.last_phase, s0.last_rounds, hr.data(), he.data(), s0.n_p);
                    }
                }
            }
            BH_CUDA(cudaMemcpyAsync(h_ctl, ctl, sizeof(Control), cudaMemcpyDeviceToHost, st));
            BH_CUDA(cudaStreamSynchronize(st));
            if (!h_ctl->active && h_ctl->n_fin == 0) {
                check_error();
                stats.rounds = h_ctl->rounds_active;
                BH_CUDA(cudaMemcpy(h_front, front, sizeof(FrontCtl), cudaMemcpyDeviceToHost));
                stats.frontier_rounds = h_front->rounds_front;
                stats.frontier_u_rounds = h_front->rounds_ufront;
                if (prof) collect_profile(round);
                return;
            }
        }
        throw CudaError("query batch did not terminate");
    }

    cudaStream_t pending = nullptr;

    void check_error() const {
        if (h_ctl->error == 2) throw InvalidArg("node index out of range");
        if (h_ctl->error) throw CudaError("query batch did not terminate");
    }

    void finish() override {
        if (!pending) return;
        cudaStream_t st = pending;
        pending = nullptr;
        BH_CUDA(cudaStreamSynchronize(st));
        check_error();
        stats.rounds = h_ctl->rounds_active;
        // graph path: K5 only in the rounds where a slot finished (IF node)
        // K1 K1a K4 every round, the two dense pulls or the six frontier kernels
        const int64_t rounds = h_ctl->rounds_active, fr = front_on ? h_front->rounds_front : 0;
        const int64_t n_launch = 3 * rounds + 2 * (rounds - fr) + 6 * fr + h_ctl->fin_rounds;
        stats.launches += n_launch;
        stats.frontier_rounds = fr;
        stats.frontier_u_rounds = h_front->rounds_ufront;
        count_launch((int)n_launch);
    }

    void read_ledger(int s, double *r_dev, double *est_dev, cudaStream_t st) override {
        k_col_get<T><<<grid1d(g->n_u), 256, 0, st>>>(R, B, s, g->n_u, g->U.perm, r_dev);
        k_col_get<T><<<grid1d(g->n_u), 256, 0, st>>>(EST, B, s, g->n_u, g->U.perm, est_dev);
        count_launch(2);
        BH_CUDA(cudaGetLastError());
    }

    void slot_state(int s, Slot *out, cudaStream_t st) override {
        BH_CUDA(cudaMemcpyAsync(out, slots + s, sizeof(Slot), cudaMemcpyDeviceToHost, st));
        BH_CUDA(cudaStreamSynchronize(st));
    }
};

// ---------------------------------------------------------------------------
// Small-graph path (small.cuh): one CTA per query, the whole state machine in
// one launch.  Used for BHPP jobs without a round hook when the per-query
// state fits in shared memory.
static bool small_disabled() {
    static const bool off = getenv("BH_NO_SMALL") != nullptr && atoi(getenv("BH_NO_SMALL")) != 0;
    return off;
}

template <typename T>
struct SmallEngine final : EngineBase {
    bh_graph *g;
    SmallPlan plan;
    double *led_r = nullptr, *led_est = nullptr;  // single-query ledger (caller order)
    cudaStream_t pending = nullptr;
    int32_t *h_err = nullptr;

    // Row slices of one side for CL ranks, balanced on edges + rows; then each
    // rank's work items (rows in chunks of <= SMALL_CHUNK edges, longest first).
    static void build_side(const Side &sd, int cl, std::vector<int32_t> &slice, std::vector<SmallItem> &items,
                           std::vector<int32_t> &ioff, std::vector<SmallSplit> &split, std::vector<int32_t> &soff,
                           int32_t &n_parts) {
        const int64_t n = sd.n_rows, E = sd.h_indptr[n];
        const int64_t total = E + 2 * n;
        slice.assign(cl + 1, 0);
        slice[cl] = (int32_t)n;
        for (int r = 1; r < cl; r++) {
            const int64_t target = total * r / cl;
            int64_t lo = slice[r - 1], hi = n;
            while (lo < hi) {  // first row whose cost prefix reaches the target
                const int64_t mid = (lo + hi) / 2;
                if (sd.h_indptr[mid] + 2 * mid < target) lo = mid + 1; else hi = mid;
            }
            slice[r] = (int32_t)lo;
        }
        items.clear();
        split.clear();
        ioff.assign(cl + 1, 0);
        soff.assign(cl + 1, 0);
        int32_t parts = 0;
        for (int r = 0; r < cl; r++) {
            const size_t first = items.size();
            for (int64_t row = slice[r]; row < slice[r + 1]; row++) {
                const int64_t e0 = sd.h_indptr[row], d = sd.h_indptr[row + 1] - e0;
                if (d <= SMALL_CHUNK) {
                    items.push_back({(int32_t)row, (int32_t)d, e0, -1, 0});
                    continue;
                }
                const int32_t np = (int32_t)((d + SMALL_CHUNK - 1) / SMALL_CHUNK);
                split.push_back({(int32_t)row, parts, np, 0});
                for (int32_t c = 0; c < np; c++)
                    items.push_back({(int32_t)row, (int32_t)std::min<int64_t>(SMALL_CHUNK, d - (int64_t)c * SMALL_CHUNK),
                                     e0 + (int64_t)c * SMALL_CHUNK, parts + c, 0});
                parts += np;
            }
            std::stable_sort(items.begin() + first, items.end(),
                             [](const SmallItem &x, const SmallItem &y) { return x.len > y.len; });
            ioff[r + 1] = (int32_t)items.size();
            soff[r + 1] = (int32_t)split.size();
        }
        n_parts = parts;
    }

    template <class X>
    static X *upload(const std::vector<X> &v) {
        X *d = dalloc<X>(std::max<size_t>(1, v.size()));
        if (!v.empty()) BH_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice));
        return d;
    }

    static size_t smem_for(const bh_graph *g, int32_t parts) {
        return SmallSmem<T>::bytes(g->n_u, g->n_v, parts);
    }

    // cluster size: BH_SMALL_CL (1, 2, 4, 8, 16), default 8 (portable)
    static int cluster_size() {
        const char *m = getenv("BH_SMALL_CL");
        const int v = m ? atoi(m) : 8;
        return (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) ? v : 8;
    }

    explicit SmallEngine(bh_graph *graph) : g(graph) {
        this->nslots = 1;
        plan.cl = cluster_size();
        std::vector<int32_t> us, vs, iu, iv, su, sv;
        std::vector<SmallItem> itu, itv;
        std::vector<SmallSplit> spu, spv;
        build_side(g->V, plan.cl, vs, itv, iv, spv, sv, plan.n_parts_v);
        build_side(g->U, plan.cl, us, itu, iu, spu, su, plan.n_parts_u);
        plan.items_v = upload(itv);
        plan.items_u = upload(itu);
        plan.split_v = upload(spv);
        plan.split_u = upload(spu);
        std::vector<int32_t> offs;
        for (auto *v : {&us, &vs, &iu, &iv, &su, &sv}) offs.insert(offs.end(), v->begin(), v->end());
        plan.offs = upload(offs);
        plan.smem = smem_for(g, std::max(plan.n_parts_v, plan.n_parts_u));
        for (int r = 0; r < plan.cl; r++) {
            plan.cap_ev = std::max<int32_t>(plan.cap_ev, (int32_t)(g->V.h_indptr[vs[r + 1]] - g->V.h_indptr[vs[r]]));
            plan.cap_eu = std::max<int32_t>(plan.cap_eu, (int32_t)(g->U.h_indptr[us[r + 1]] - g->U.h_indptr[us[r]]));
            plan.cap_iv = std::max<int32_t>(plan.cap_iv, iv[r + 1] - iv[r]);
            plan.cap_iu = std::max<int32_t>(plan.cap_iu, iu[r + 1] - iu[r]);
        }
        // one process-wide ceiling for the kernel (a per-graph value would break the
        // launches of other graphs' engines): everything the opt-in limit leaves
        cudaFuncAttributes fa{};
        BH_CUDA(cudaFuncGetAttributes(&fa, k_small_query<T>));
        int optin = 0;
        BH_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
        const int ceiling = optin - (int)fa.sharedSizeBytes;
        if ((int64_t)plan.smem > ceiling) throw CudaError("small path: shared memory plan exceeds the device limit");
        {  // stage each rank's graph slice in shared memory when it fits beside the state
            const size_t st = SmallSmem<T>::staged(plan.cap_ev, plan.cap_eu, plan.cap_iv, plan.cap_iu);
            if (plan.smem + st <= (size_t)ceiling && !getenv("BH_SMALL_NOSTAGE")) {
                plan.stage = 1;
                plan.smem += st;
            }
        }
        BH_CUDA(cudaFuncSetAttribute(k_small_query<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, ceiling));
        if (plan.cl > 8) BH_CUDA(cudaFuncSetAttribute(k_small_query<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)plan.cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)plan.cl);
        cfg.blockDim = dim3(SMALL_THREADS);
        cfg.dynamicSmemBytes = plan.smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        BH_CUDA(cudaOccupancyMaxActiveClusters(&clusters, k_small_query<T>, &cfg));
        if (clusters < 1) throw CudaError("small path: no resident cluster");
        plan.cluster_cap = clusters;
        plan.error = dalloc<int32_t>(1);
        plan.ctl = dalloc<Control>(1);
        led_r = dalloc<double>(g->n_u);
        led_est = dalloc<double>(g->n_u);
        BH_CUDA(cudaMallocHost(&h_err, 2 * sizeof(int32_t)));
    }
    ~SmallEngine() override {
        plan.free_all();
        cudaFree(led_r);
        cudaFree(led_est);
        if (h_err) cudaFreeHost(h_err);
    }

    // Eligible graphs: the state of one query fits in a CTA's shared memory.
    static bool fits(const bh_graph *g) {
        if (small_disabled() || g->n_e > 4000000) return false;
        int64_t parts = 0;
        for (const Side *sd : {&g->U, &g->V}) {
            int64_t p = 0;
            for (int64_t r = 0; r < sd->n_rows; r++) {
                const int64_t d = sd->h_indptr[r + 1] - sd->h_indptr[r];
                if (d > SMALL_CHUNK) p += (d + SMALL_CHUNK - 1) / SMALL_CHUNK;
            }
            parts = std::max(parts, p);
        }
        const size_t static_smem = sizeof(SelectSmem) + TOPK_MAX * 16 + 1024 + sizeof(Slot) + sizeof(Finish);
        return smem_for(g, (int32_t)parts) + static_smem <= 200 * 1024;
    }

    void run(const RunSpec &rs, cudaStream_t st) override {
        if (rs.k > TOPK_MAX) throw InvalidArg("k exceeds the device top-k limit (1024) of bh_query_batch");
        SmallArgs<T> a{};
        a.n_u = g->n_u;
        a.n_v = g->n_v;
        a.n_e = g->n_e;
        a.u_ptr = g->U.indptr;
        a.v_ptr = g->V.indptr;
        a.u_col = g->U.indices;
        a.v_col = g->V.indices;
        a.u_val = (const T *)g->U.vals;
        a.v_val = (const T *)g->V.vals;
        a.deg_u = g->U.deg;
        a.ws_u = g->ws_u;
        a.inv_ws_u = g->inv_ws_u;
        a.perm_u = g->U.perm;
        const int cl = plan.cl;
        a.u_slice = plan.offs;
        a.v_slice = plan.offs + (cl + 1);
        a.iu_off = plan.offs + 2 * (cl + 1);
        a.iv_off = plan.offs + 3 * (cl + 1);
        a.su_off = plan.offs + 4 * (cl + 1);
        a.sv_off = plan.offs + 5 * (cl + 1);
        a.items_v = plan.items_v;
        a.items_u = plan.items_u;
        a.split_v = plan.split_v;
        a.split_u = plan.split_u;
        a.n_parts_v = plan.n_parts_v;
        a.n_parts_u = plan.n_parts_u;
        a.stage = plan.stage;
        a.cap_ev = plan.cap_ev;
        a.cap_eu = plan.cap_eu;
        a.cap_iv = plan.cap_iv;
        a.cap_iu = plan.cap_iu;
        ControlArgs &ca = a.ca;
        ca.ctl = plan.ctl;
        ca.sources = rs.sources;
        ca.inv_u = g->U.inv;
        ca.trace = rs.trace;
        ca.tie_skip = rs.tie;
        ca.ws_u = g->ws_u;
        ca.n_u = g->n_u;
        ca.alpha = rs.alpha;
        ca.lam = rs.lam;
        ca.eps_b = rs.eps_b;
        ca.eps_f = rs.eps_f;
        ca.budget_scale = 2.0 * (double)g->n_e;
        ca.log_decay = std::log(1.0 / (1.0 - rs.alpha));
        ca.job = rs.job;
        a.n_q = (int32_t)rs.n_q;
        a.k = rs.k;
        a.exclude = rs.exclude;
        a.want_scores = rs.want_scores;
        a.topk_idx = rs.topk_idx;
        a.topk_score = rs.topk_score;
        a.trace = rs.trace;
        a.scores = rs.want_scores ? rs.scores : nullptr;
        a.ledger_r = rs.n_q == 1 ? led_r : nullptr;
        a.ledger_est = rs.n_q == 1 ? led_est : nullptr;
        a.max_rounds = 100000000;
        a.error = plan.error;
        BH_CUDA(cudaMemsetAsync(plan.error, 0, sizeof(int32_t), st));
        BH_CUDA(cudaMemsetAsync(plan.ctl, 0, sizeof(Control), st));
        const int n_clusters = (int)std::max<int64_t>(1, std::min<int64_t>(rs.n_q, plan.cluster_cap));
        unsigned long long *prof = nullptr;
        if (getenv("BH_SMALL_PROF")) {
            prof = dalloc<unsigned long long>(8);
            BH_CUDA(cudaMemsetAsync(prof, 0, 64, st));
        }
        a.prof = prof;
        {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)cl;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3((unsigned)(n_clusters * cl));
            cfg.blockDim = dim3(SMALL_THREADS);
            cfg.dynamicSmemBytes = plan.smem;
            cfg.stream = st;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            BH_CUDA(cudaLaunchKernelEx(&cfg, k_small_query<T>, a));
        }
        if (prof) {
            unsigned long long h[8];
            BH_CUDA(cudaMemcpyAsync(h, prof, 64, cudaMemcpyDeviceToHost, st));
            BH_CUDA(cudaStreamSynchronize(st));
            fprintf(stderr, "small-path cycles: K1 %llu sync1 %llu Vpull %llu sync2 %llu Upull %llu K1a+sums %llu sync3+K4 %llu\n",
                    h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
            cudaFree(prof);
        }
        count_launch();
        BH_CUDA(cudaGetLastError());
        BH_CUDA(cudaMemcpyAsync(h_err, plan.error, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        BH_CUDA(cudaMemcpyAsync(h_err + 1, &plan.ctl->error, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        stats = bh_run_stats{};
        stats.slots = 1;
        stats.launches = 1;
        pending = st;
        if (!rs.async) finish();
    }
    void finish() override {
        if (!pending) return;
        cudaStream_t st = pending;
        pending = nullptr;
        BH_CUDA(cudaStreamSynchronize(st));
        if (h_err[1] == 2) throw InvalidArg("node index out of range");
        if (h_err[0]) throw CudaError("query batch did not terminate");
    }
    void read_ledger(int, double *r_dev, double *est_dev, cudaStream_t st) override {
        BH_CUDA(cudaMemcpyAsync(r_dev, led_r, g->n_u * sizeof(double), cudaMemcpyDeviceToDevice, st));
        BH_CUDA(cudaMemcpyAsync(est_dev, led_est, g->n_u * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    void slot_state(int, Slot *, cudaStream_t) override { throw CudaError("small path has no round hook"); }
};

// ---------------------------------------------------------------------------
struct EngineCache {
    std::map<int, std::unique_ptr<EngineBase>> by_b;
    std::unique_ptr<EngineBase> small;  // small-graph path (one CTA per query), when eligible
    int small_ok = -1;                  // -1 unknown, 0 not eligible, 1 eligible
    EngineBase *last = nullptr;
    EngineBase *pending = nullptr;  // engine of an un-finished BH_QUERY_ASYNC batch
    cudaStream_t stream = nullptr;
    // host-call staging buffers
    int32_t *d_src = nullptr, *d_tie = nullptr;
    int64_t cap_q = 0, cap_tie = 0;
    int32_t *d_tk_idx = nullptr;
    double *d_tk_sc = nullptr;
    int64_t cap_tk = 0, cap_tks = 0;
    bh_trace *d_trace = nullptr;
    int64_t cap_tr = 0;
    double *d_scores = nullptr;
    int64_t cap_sc = 0;
    double *d_vec_a = nullptr, *d_vec_b = nullptr;
    int64_t cap_vec = 0;
    unsigned char *h_stage = nullptr;  // pinned staging for the host-pointer inputs and outputs
    size_t cap_stage = 0;
    ~EngineCache() {
        by_b.clear();
        small.reset();
        if (h_stage) cudaFreeHost(h_stage);
        cudaFree(d_src); cudaFree(d_tie); cudaFree(d_tk_idx); cudaFree(d_tk_sc);
        cudaFree(d_trace); cudaFree(d_scores); cudaFree(d_vec_a); cudaFree(d_vec_b);
        if (stream) cudaStreamDestroy(stream);
    }
};

template <typename X>
static void grow(X *&p, int64_t &cap, int64_t need) {
    if (need <= cap) return;
    cudaFree(p);
    p = dalloc<X>((size_t)need);
    cap = need;
}

static EngineCache &cache_of(bh_graph *g) {
    if (!g->engines) {
        auto *c = new EngineCache();
        BH_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        g->engines = c;
    }
    return *(EngineCache *)g->engines;
}

template <typename T>
static EngineBase *make_engine(bh_graph *g, int B) {
    switch (B) {
        case 1: return new Engine<T, 1>(g);
        case 4: return new Engine<T, 4>(g);
        case 16: return new Engine<T, 16>(g);
        case 32: return new Engine<T, 32>(g);
        case 64: return new Engine<T, 64>(g);
        case 128: return new Engine<T, 128>(g);
        default: throw InvalidArg("slots must be one of 1, 4, 16, 32, 64, 128");
    }
}

static int auto_slots(bh_graph *g, int64_t n_q) {
    // 128 slots once the batch fills them: per-round cost grows sub-linearly in B
    // (c5 on B200: 2189 q/s at 64 slots, 2625 at 128)
    int b = n_q <= 1 ? 1 : n_q <= 4 ? 4 : n_q <= 16 ? 16 : n_q <= 32 ? 32 : n_q <= 64 ? 64 : 128;
    // an engine of that width exists: no device-memory query (cudaMemGetInfo goes to
    // the driver and was measured stalling a call by up to 100 ms on a busy host)
    if (cache_of(g).by_b.count(b)) return b;
    // keep the per-slot state within a fraction of device memory: step down
    // through the engine widths, never below one slot
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        static const int widths[] = {128, 64, 32, 16, 4, 1};
        const int s = g->dtype == BH_DTYPE_F32 ? 4 : 8;
        const double per_slot = (double)g->n_u * (5.0 * s + 8) + (double)g->n_v * s;  // R P Y EST XV + OUTS
        for (int w : widths) {
            if (w > b) continue;
            b = w;
            if ((double)w * per_slot <= 0.6 * (double)free_b) break;
        }
    }
    return b;
}

static EngineBase &engine_for(bh_graph *g, int B) {
    EngineCache &c = cache_of(g);
    auto it = c.by_b.find(B);
    if (it != c.by_b.end()) return *it->second;
    EngineBase *e = g->dtype == BH_DTYPE_F32 ? make_engine<float>(g, B) : make_engine<double>(g, B);
    c.by_b[B].reset(e);
    return *e;
}

// The small-graph engine of g, or null when g's state does not fit a CTA.
static EngineBase *small_engine(bh_graph *g) {
    EngineCache &c = cache_of(g);
    if (c.small_ok < 0) {
        const bool ok = g->dtype == BH_DTYPE_F32 ? SmallEngine<float>::fits(g) : SmallEngine<double>::fits(g);
        c.small_ok = ok ? 1 : 0;
    }
    if (!c.small_ok || small_disabled()) return nullptr;
    if (!c.small) {
        if (g->dtype == BH_DTYPE_F32) c.small.reset(new SmallEngine<float>(g));
        else c.small.reset(new SmallEngine<double>(g));
    }
    return c.small.get();
}

static void check_params(double alpha, double eps_b, double eps_f, double lam) {
    if (!(alpha > 0.0 && alpha < 1.0)) throw InvalidArg("alpha must lie strictly between 0 and 1");
    if (!(eps_b > 0.0) || !(eps_f > 0.0)) throw InvalidArg("epsilon shares must be positive");
    if (!(lam > 0.0)) throw InvalidArg("lam must be positive");
}

}  // namespace bh

// ===========================================================================
// C ABI
using namespace bh;

template <class F>
static int guarded(F &&f) {
    try {
        f();
        return BH_OK;
    } catch (const FallbackNeeded &) {
        t_err = "input needs the reference-semantics parser";
        return BH_EFALLBACK;
    } catch (const InvalidArg &e) {
        t_err = e.what();
        return BH_EINVAL;
    } catch (const std::bad_alloc &) {
        t_err = "device or host allocation failed";
        return BH_ENOMEM;
    } catch (const CudaError &e) {
        t_err = e.what();
        return BH_ECUDA;
    } catch (const std::exception &e) {
        t_err = e.what();
        return BH_ECUDA;
    }
}

// bh_stream_gate: hold the stream until the host sets *flag (at most ~5 s, so
// a caller that synchronises on the gated stream before releasing it stalls
// instead of hanging).
__global__ void k_gate(const int32_t *flag) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*(volatile const int32_t *)flag == 0) {
        __nanosleep(256);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 5000000000ull) break;
    }
}

extern "C" {

const char *bh_last_error(void) { return t_err.c_str(); }
static_assert(sizeof(bh_trace) == 96, "bh_trace layout (include/bhpp.h)");
static_assert(sizeof(bh_run_stats) == 80, "bh_run_stats layout (include/bhpp.h)");
int bh_version(void) { return 3; }
int64_t bh_kernel_launches(void) { return g_launches.load(); }

int bh_csr_build(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *edge_u, const int64_t *edge_v,
                 const double *edge_w, int64_t *u_indptr, int32_t *u_indices, double *u_weights,
                 int64_t *v_indptr, int32_t *v_indices, double *v_weights, double *ws_u, double *ws_v,
                 int32_t device) {
    int dup = 0;
    const int rc = guarded([&] {
        if (!edge_u || !edge_v || !edge_w || !u_indptr || !u_indices || !u_weights || !v_indptr || !v_indices ||
            !v_weights || !ws_u || !ws_v)
            throw InvalidArg("null argument");
        dup = csr_build(n_u, n_v, n_e, edge_u, edge_v, edge_w, u_indptr, u_indices, u_weights, v_indptr, v_indices,
                        v_weights, ws_u, ws_v, device);
    });
    if (rc == BH_OK && dup) {
        t_err = "duplicate edge passed to constructor";
        return BH_EDUP;
    }
    return rc;
}

struct bh_edge_list {
    bh::EdgeListResult r;
};

int bh_edge_list_parse(const char *buf, int64_t len, const char *delim, int64_t delim_len, int32_t has_default,
                       double default_weight, bh_edge_list **out, int64_t *err_line) {
    return guarded([&] {
        if (!out || (!buf && len > 0) || len < 0) throw InvalidArg("null argument");
        if (delim && delim_len <= 0) throw InvalidArg("empty delimiter");
        *out = nullptr;
        if (err_line) *err_line = 0;
        auto *el = new bh_edge_list();
        el->r = bh::parse_edge_list(buf, len, delim, delim_len, has_default != 0, default_weight);
        if (el->r.status != bh::PARSE_OK) {
            if (err_line) *err_line = el->r.err_line;
            delete el;
            throw FallbackNeeded();
        }
        *out = el;
    });
}

int bh_edge_list_sizes(const bh_edge_list *el, int64_t *n_u, int64_t *n_v, int64_t *u_bytes, int64_t *v_bytes,
                       int64_t *n_e) {
    return guarded([&] {
        if (!el || !n_u || !n_v || !u_bytes || !v_bytes || !n_e) throw InvalidArg("null argument");
        *n_u = (int64_t)el->r.u_labels.size();
        *n_v = (int64_t)el->r.v_labels.size();
        int64_t bu = 0, bv = 0;
        for (const auto &x : el->r.u_labels) bu += (int64_t)x.size();
        for (const auto &x : el->r.v_labels) bv += (int64_t)x.size();
        *u_bytes = bu;
        *v_bytes = bv;
        *n_e = (int64_t)el->r.ew.size();
    });
}

int bh_edge_list_export(const bh_edge_list *el, char *u_blob, int64_t *u_ends, char *v_blob, int64_t *v_ends,
                        int64_t *edge_u, int64_t *edge_v, double *edge_w) {
    return guarded([&] {
        if (!el || !u_ends || !v_ends || !edge_u || !edge_v || !edge_w) throw InvalidArg("null argument");
        auto put = [](const std::vector<std::string> &labs, char *blob, int64_t *ends) {
            int64_t o = 0;
            for (size_t i = 0; i < labs.size(); i++) {
                if (!labs[i].empty()) std::memcpy(blob + o, labs[i].data(), labs[i].size());
                o += (int64_t)labs[i].size();
                ends[i] = o;
            }
        };
        put(el->r.u_labels, u_blob, u_ends);
        put(el->r.v_labels, v_blob, v_ends);
        const size_t n = el->r.ew.size();
        std::memcpy(edge_u, el->r.eu.data(), n * sizeof(int64_t));
        std::memcpy(edge_v, el->r.ev.data(), n * sizeof(int64_t));
        std::memcpy(edge_w, el->r.ew.data(), n * sizeof(double));
    });
}

void bh_edge_list_free(bh_edge_list *el) { delete el; }

int bh_alias_create(bh_graph *g, const double *u_prob, const int64_t *u_alias, const double *v_prob,
                    const int64_t *v_alias, bh_alias **out) {
    return guarded([&] {
        if (!g || !u_prob || !u_alias || !v_prob || !v_alias || !out) throw InvalidArg("null argument");
        std::lock_guard<std::mutex> lock(g->mu);
        *out = bh::alias_create(g, u_prob, u_alias, v_prob, v_alias);
    });
}

int bh_alias_build(int64_t n_rows, int64_t n_e, const int64_t *indptr, const double *weights, int32_t device,
                   double *prob, int64_t *alias) {
    return guarded([&] {
        if (!indptr || !weights || !prob || !alias) throw InvalidArg("null argument");
        if (n_rows <= 0 || n_e < 0 || indptr[0] != 0 || indptr[n_rows] != n_e) throw InvalidArg("corrupt CSR offsets");
        if (n_e > 0) alias_build(n_rows, n_e, indptr, weights, device, prob, alias);
    });
}

int bh_monte_carlo(const bh_alias *a, int64_t source, double alpha, int64_t first, int64_t n, uint64_t seed,
                   int64_t *counts) {
    return guarded([&] {
        if (!a || !counts) throw InvalidArg("null argument");
        if (!(alpha > 0.0 && alpha < 1.0)) throw InvalidArg("alpha must lie strictly between 0 and 1");
        if (source < 0 || source >= a->g->n_u) throw InvalidArg("node index out of range");
        if (n < 0 || first < 0) throw InvalidArg("bad walk range");
        std::lock_guard<std::mutex> lock(a->g->mu);
        bh::mc_walks(a, source, alpha, first, n, seed, counts);
    });
}

void bh_alias_destroy(bh_alias *a) {
    if (!a) return;
    cudaSetDevice(a->device);
    delete a;
}

int bh_query_wait(bh_graph *g) {
    return guarded([&] {
        if (!g) throw InvalidArg("null argument");
        std::lock_guard<std::mutex> lock(g->mu);
        BH_CUDA(cudaSetDevice(g->device));
        EngineCache &c = cache_of(g);
        g_tstamp[0] = host_us();
        EngineBase *e = c.pending;
        c.pending = nullptr;
        if (e) e->finish();
    });
}

int bh_stream_gate(void *stream, const int32_t *flag) {
    return guarded([&] {
        if (!flag) throw InvalidArg("null argument");
        k_gate<<<1, 1, 0, (cudaStream_t)stream>>>(flag);
        count_launch();
        BH_CUDA(cudaGetLastError());
    });
}

int bh_set_profiling(int32_t on) {
    g_profiling = on ? 1 : 0;
    return BH_OK;
}

int bh_set_scatter_limit(double fraction) {
    if (std::isnan(fraction)) return BH_EINVAL;
    g_scatter_limit = fraction;
    return BH_OK;
}

int bh_last_run_stats(bh_graph *g, bh_run_stats *out) {
    return guarded([&] {
        if (!g || !out) throw InvalidArg("null argument");
        std::lock_guard<std::mutex> lock(g->mu);
        EngineCache &c = cache_of(g);
        *out = c.last ? c.last->stats : bh_run_stats{};
    });
}

int bh_graph_create(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *u_indptr, const int32_t *u_indices,
                    const double *u_weights, const int64_t *v_indptr, const int32_t *v_indices,
                    const double *v_weights, const double *ws_u, const double *ws_v, int32_t device,
                    int32_t dtype, bh_graph **out) {
    return guarded([&] {
        if (!out) throw InvalidArg("out is null");
        *out = graph_create(n_u, n_v, n_e, u_indptr, u_indices, u_weights, v_indptr, v_indices, v_weights, ws_u,
                            ws_v, device, dtype);
    });
}

void bh_graph_destroy(bh_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    delete (EngineCache *)g->engines;
    g->engines = nullptr;
    graph_free_arrays(g);
    delete g;
}

int bh_graph_get_info(const bh_graph *g, bh_graph_info *out) {
    return guarded([&] {
        if (!g || !out) throw InvalidArg("null argument");
        out->n_u = g->n_u;
        out->n_v = g->n_v;
        out->n_e = g->n_e;
        out->dtype = g->dtype;
        out->device = g->device;
        out->device_bytes = g->device_bytes;
        int64_t mu = 0, mv = 0;
        for (int64_t r = 0; r < g->n_u; r++) mu = std::max(mu, g->U.h_indptr[r + 1] - g->U.h_indptr[r]);
        for (int64_t r = 0; r < g->n_v; r++) mv = std::max(mv, g->V.h_indptr[r + 1] - g->V.h_indptr[r]);
        out->max_deg_u = mu;
        out->max_deg_v = mv;
    });
}

int bh_query_batch(bh_graph *g, const bh_query_params *p, const int32_t *sources, int64_t n_q,
                   const int32_t *tie_skip, int32_t *topk_idx, double *topk_score, bh_trace *trace,
                   double *scores, void *stream) {
    struct NvtxRange {  // one NVTX range per batch (nsys / ncu --nvtx)
        NvtxRange() { nvtxRangePushA("bh_query_batch"); }
        ~NvtxRange() { nvtxRangePop(); }
    } nvtx_range;
    const double t_entry =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    return guarded([&] {
        if (!g || !p || !trace) throw InvalidArg("null argument");
        if (n_q < 0 || n_q > (1LL << 31) - 1) throw InvalidArg("bad query count");
        if (n_q == 0) return;
        check_params(p->alpha, p->eps_b, p->eps_f, p->lam);
        if (p->k < 0) throw InvalidArg("k must be nonnegative");
        std::lock_guard<std::mutex> lock(g->mu);
        BH_CUDA(cudaSetDevice(g->device));
        EngineCache &c = cache_of(g);
        g_tstamp[0] = host_us();
        if (c.pending) {  // an async batch not yet waited for: complete it first
            EngineBase *e0 = c.pending;
            c.pending = nullptr;
            e0->finish();
        }
        cudaStream_t st = stream ? (cudaStream_t)stream : c.stream;
        EngineBase *sm = p->slots > 0 ? nullptr : small_engine(g);
        const int B = sm ? 1 : p->slots > 0 ? p->slots : auto_slots(g, n_q);
        EngineBase &e = sm ? *sm : engine_for(g, B);
        c.last = &e;
        RunSpec rs{};
        rs.job = BH_JOB_BHPP;
        rs.n_q = n_q;
        rs.alpha = p->alpha;
        rs.lam = p->lam;
        rs.eps_b = p->eps_b;
        rs.eps_f = p->eps_f;
        rs.k = p->k;
        rs.exclude = p->exclude_query;
        rs.want_scores = p->want_scores && scores;
        if (p->on_device) {
            rs.async = (p->flags & BH_QUERY_ASYNC) != 0;
            c.pending = rs.async ? &e : nullptr;
            rs.sources = sources;
            rs.tie = tie_skip;
            rs.topk_idx = topk_idx;
            rs.topk_score = topk_score;
            rs.trace = trace;
            rs.scores = scores;
            e.run(rs, st);
            return;
        }
        // host pointers: validate, stage in, run, stage out.  Inputs and outputs go
        // through one pinned staging buffer (a pageable H2D copy would synchronise the
        // stream first), the outputs copied device -> pinned right behind the batch on
        // the stream: one synchronisation, no host turnaround between the batch and its copies.
        for (int64_t i = 0; i < n_q; i++)
            if (sources[i] < 0 || sources[i] >= g->n_u) throw InvalidArg("node index out of range");
        grow(c.d_src, c.cap_q, n_q);
        if (tie_skip) grow(c.d_tie, c.cap_tie, n_q);
        grow(c.d_trace, c.cap_tr, n_q);
        rs.sources = c.d_src;
        rs.tie = tie_skip ? c.d_tie : nullptr;
        rs.trace = c.d_trace;
        if (p->k > 0 && topk_idx) {
            grow(c.d_tk_idx, c.cap_tk, n_q * p->k);
            grow(c.d_tk_sc, c.cap_tks, n_q * p->k);
            rs.topk_idx = c.d_tk_idx;
            rs.topk_score = c.d_tk_sc;
        }
        if (rs.want_scores) {
            grow(c.d_scores, c.cap_sc, n_q * g->n_u);
            rs.scores = c.d_scores;
        }
        const size_t b_in = n_q * sizeof(int32_t) * (tie_skip ? 2 : 1);
        const size_t b_tr = n_q * sizeof(bh_trace);
        const size_t b_ti = rs.topk_idx ? n_q * p->k * sizeof(int32_t) : 0;
        const size_t b_ts = rs.topk_idx && topk_score ? n_q * p->k * sizeof(double) : 0;
        const size_t b_sc = rs.want_scores ? n_q * g->n_u * sizeof(double) : 0;  // large: copied directly
        const size_t off_tr = (b_in + 15) / 16 * 16;
        const size_t need = off_tr + b_tr + b_ti + b_ts;
        if (need > c.cap_stage) {
            if (c.h_stage) cudaFreeHost(c.h_stage);
            c.h_stage = nullptr;
            c.cap_stage = 0;
            BH_CUDA(cudaMallocHost(&c.h_stage, need));
            c.cap_stage = need;
        }
        g_tstamp[1] = host_us();
        int32_t *h_src = reinterpret_cast<int32_t *>(c.h_stage);
        std::memcpy(h_src, sources, n_q * sizeof(int32_t));
        BH_CUDA(cudaMemcpyAsync(c.d_src, h_src, n_q * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        if (tie_skip) {
            std::memcpy(h_src + n_q, tie_skip, n_q * sizeof(int32_t));
            BH_CUDA(cudaMemcpyAsync(c.d_tie, h_src + n_q, n_q * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        }
        unsigned char *h_tr = c.h_stage + off_tr, *h_ti = h_tr + b_tr, *h_ts = h_ti + b_ti;
        rs.async = true;
        // BH_TRACE_E2E=1: host-path phase times on stderr (diagnostic)
        static const bool trace_e2e = getenv("BH_TRACE_E2E") != nullptr;
        cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};
        auto now_us = [] {
            return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
        };
        double th[4] = {t_entry, 0, 0, 0};
        g_tstamp[2] = host_us();
        if (trace_e2e) {
            for (auto &x : tev) BH_CUDA(cudaEventCreate(&x));
            BH_CUDA(cudaEventRecord(tev[0], st));
        }
        e.run(rs, st);
        if (trace_e2e) BH_CUDA(cudaEventRecord(tev[1], st));
        th[1] = now_us();
        BH_CUDA(cudaMemcpyAsync(h_tr, c.d_trace, b_tr, cudaMemcpyDeviceToHost, st));
        if (b_ti) BH_CUDA(cudaMemcpyAsync(h_ti, c.d_tk_idx, b_ti, cudaMemcpyDeviceToHost, st));
        if (b_ts) BH_CUDA(cudaMemcpyAsync(h_ts, c.d_tk_sc, b_ts, cudaMemcpyDeviceToHost, st));
        if (b_sc) BH_CUDA(cudaMemcpyAsync(scores, c.d_scores, b_sc, cudaMemcpyDeviceToHost, st));
        if (trace_e2e) BH_CUDA(cudaEventRecord(tev[2], st));
        th[2] = now_us();
        e.finish();  // synchronises the stream (graph path), checks termination
        BH_CUDA(cudaStreamSynchronize(st));
        th[3] = now_us();
        if (trace_e2e) {
            float d_graph = 0.f, d_out = 0.f;
            BH_CUDA(cudaEventElapsedTime(&d_graph, tev[0], tev[1]));
            BH_CUDA(cudaEventElapsedTime(&d_out, tev[1], tev[2]));
            fprintf(stderr, "[bh e2e] host: entry to launch %.1f us (lock %.1f, setup %.1f, inputs %.1f, run %.1f, graph %.1f, "
                    "launch %.1f), copies enqueued %.1f us, wait %.1f us; device: batch %.3f ms, outputs %.3f ms\n",
                    th[1] - th[0], g_tstamp[0] - th[0], g_tstamp[1] - g_tstamp[0], g_tstamp[2] - g_tstamp[1],
                    g_tstamp[3] - g_tstamp[2], g_tstamp[4] - g_tstamp[3], g_tstamp[5] - g_tstamp[4], th[2] - th[1],
                    th[3] - th[2], d_graph, d_out);
            for (auto &x : tev) cudaEventDestroy(x);
        }
        std::memcpy(trace, h_tr, b_tr);
        if (b_ti) std::memcpy(topk_idx, h_ti, b_ti);
        if (b_ts) std::memcpy(topk_score, h_ts, b_ts);
    });
}

int bh_push_run(bh_graph *g, int32_t job, int32_t source, double alpha, double lam, double eps_b, double eps_f,
                int32_t tie_skip, double *residue_u, double *estimate, int64_t *n_p, double *scores,
                bh_trace *trace, bh_round_hook hook, void *user) {
    struct NvtxRange {
        NvtxRange() { nvtxRangePushA("bh_push_run"); }
        ~NvtxRange() { nvtxRangePop(); }
    } nvtx_range;
    return guarded([&] {
        if (!g || !trace) throw InvalidArg("null argument");
        if (job < BH_JOB_BHPP || job > BH_JOB_PI_PUSH) throw InvalidArg("bad job");
        if (!(alpha > 0.0 && alpha < 1.0)) throw InvalidArg("alpha must lie strictly between 0 and 1");
        if (source < 0 || source >= g->n_u) throw InvalidArg("node index out of range");
        if (job != BH_JOB_PI_PUSH && !(eps_b > 0.0)) throw InvalidArg("epsilon_b must be positive");
        if ((job == BH_JOB_PI_PUSH || job == BH_JOB_BHPP) && !(eps_f > 0.0)) throw InvalidArg("epsilon_f must be positive");
        if ((job == BH_JOB_PI_PUSH || job == BH_JOB_BHPP) && !(lam > 0.0)) throw InvalidArg("lam must be positive");
        std::lock_guard<std::mutex> lock(g->mu);
        BH_CUDA(cudaSetDevice(g->device));
        EngineCache &c = cache_of(g);
        g_tstamp[0] = host_us();
        cudaStream_t st = c.stream;
        EngineBase *sm = job == BH_JOB_BHPP && !hook ? small_engine(g) : nullptr;
        EngineBase &e = sm ? *sm : engine_for(g, 1);
        c.last = &e;
        const int64_t nu = g->n_u;
        grow(c.d_src, c.cap_q, 1);
        grow(c.d_trace, c.cap_tr, 1);
        if (c.cap_vec < nu) {
            cudaFree(c.d_vec_a);
            cudaFree(c.d_vec_b);
            c.d_vec_a = dalloc<double>(nu);
            c.d_vec_b = dalloc<double>(nu);
            c.cap_vec = nu;
        }
        grow(c.d_scores, c.cap_sc, nu);
        BH_CUDA(cudaMemcpyAsync(c.d_src, &source, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        RunSpec rs{};
        rs.job = job;
        rs.n_q = 1;
        rs.sources = c.d_src;
        int32_t tie_h = tie_skip;
        grow(c.d_tie, c.cap_tie, 1);
        BH_CUDA(cudaMemcpyAsync(c.d_tie, &tie_h, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        rs.tie = c.d_tie;
        rs.alpha = alpha;
        rs.lam = lam > 0 ? lam : 1.0;
        rs.eps_b = eps_b > 0 ? eps_b : 1.0;
        rs.eps_f = eps_f > 0 ? eps_f : 1.0;
        rs.trace = c.d_trace;
        rs.want_scores = 1;
        rs.scores = c.d_scores;
        rs.hook = hook;
        rs.hook_user = user;
        if (job == BH_JOB_PI_PUSH) {
            BH_CUDA(cudaMemcpyAsync(c.d_vec_a, residue_u, nu * sizeof(double), cudaMemcpyHostToDevice, st));
            BH_CUDA(cudaMemcpyAsync(c.d_vec_b, estimate, nu * sizeof(double), cudaMemcpyHostToDevice, st));
            rs.ledger_r = c.d_vec_a;
            rs.ledger_est = c.d_vec_b;
            rs.init_np = *n_p;
        }
        e.run(rs, st);
        BH_CUDA(cudaStreamSynchronize(st));
        // ledger out (slot 0)
        e.read_ledger(0, c.d_vec_a, c.d_vec_b, st);
        BH_CUDA(cudaMemcpyAsync(residue_u, c.d_vec_a, nu * sizeof(double), cudaMemcpyDeviceToHost, st));
        BH_CUDA(cudaMemcpyAsync(estimate, c.d_vec_b, nu * sizeof(double), cudaMemcpyDeviceToHost, st));
        BH_CUDA(cudaMemcpyAsync(trace, c.d_trace, sizeof(bh_trace), cudaMemcpyDeviceToHost, st));
        if (scores && (job == BH_JOB_BHPP || job == BH_JOB_PI_PUSH))
            BH_CUDA(cudaMemcpyAsync(scores, c.d_scores, nu * sizeof(double), cudaMemcpyDeviceToHost, st));
        BH_CUDA(cudaStreamSynchronize(st));
        *n_p = job == BH_JOB_SS_PUSH || job == BH_JOB_SELECTIVE ? trace->n_p_b : trace->n_p_f;
    });
}

int bh_power_iteration(bh_graph *g, const double *start, int64_t n_vec, double alpha, int32_t t, double *out) {
    return guarded([&] {
        if (!g || !start || !out) throw InvalidArg("null argument");
        if (!(alpha > 0.0 && alpha < 1.0)) throw InvalidArg("alpha must lie strictly between 0 and 1");
        if (t < 0) throw InvalidArg("iteration count must be nonnegative");
        if (n_vec <= 0) return;
        std::lock_guard<std::mutex> lock(g->mu);
        BH_CUDA(cudaSetDevice(g->device));
        EngineCache &c = cache_of(g);
        g_tstamp[0] = host_us();
        cudaStream_t st = c.stream;
        const int64_t nu = g->n_u;
        const int B = auto_slots(g, n_vec);
        EngineBase &e = engine_for(g, B);
        grow(c.d_src, c.cap_q, n_vec);
        std::vector<int32_t> zeros((size_t)n_vec, 0);
        BH_CUDA(cudaMemcpyAsync(c.d_src, zeros.data(), n_vec * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        grow(c.d_trace, c.cap_tr, n_vec);
        double *d_x0 = dalloc<double>((size_t)n_vec * nu);
        double *d_out = dalloc<double>((size_t)n_vec * nu);
        try {
            BH_CUDA(cudaMemcpyAsync(d_x0, start, n_vec * nu * sizeof(double), cudaMemcpyHostToDevice, st));
            RunSpec rs{};
            rs.job = BH_JOB_POWER;
            rs.n_q = n_vec;
            rs.sources = c.d_src;
            rs.alpha = alpha;
            rs.power_t = t;
            rs.x0 = d_x0;
            rs.trace = c.d_trace;
            rs.want_scores = 1;
            rs.scores = d_out;
            e.run(rs, st);
            BH_CUDA(cudaMemcpyAsync(out, d_out, n_vec * nu * sizeof(double), cudaMemcpyDeviceToHost, st));
            BH_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cudaFree(d_x0);
            cudaFree(d_out);
            throw;
        }
        cudaFree(d_x0);
        cudaFree(d_out);
    });
}

int bh_topk(const double *scores, int64_t n, int64_t k, int64_t exclude, int64_t *out_idx, double *out_score,
            int64_t *out_count) {
    return guarded([&] {
        if (!scores || !out_idx || !out_score || !out_count) throw InvalidArg("null argument");
        if (k <= 0) throw InvalidArg("k must be positive");
        *out_count = 0;
        if (n <= 0) return;
        cudaStream_t st = nullptr;
        double *dx = dalloc<double>(n);
        int64_t *didx = nullptr, *dcnt = nullptr;
        double *dsc = nullptr;
        uint64_t *ck = nullptr;
        int64_t *ci = nullptr;
        void *tmp = nullptr;
        auto cleanup = [&] {
            cudaFree(dx); cudaFree(didx); cudaFree(dcnt); cudaFree(dsc); cudaFree(ck); cudaFree(ci); cudaFree(tmp);
        };
        try {
            BH_CUDA(cudaMemcpyAsync(dx, scores, n * sizeof(double), cudaMemcpyHostToDevice, st));
            const int64_t kk = std::min(k, n);
            if (kk <= TOPK_MAX) {
                const int64_t chunk = SEL_ITEMS * TOPK_THREADS;
                const int64_t nch = (n + chunk - 1) / chunk;
                ck = dalloc<uint64_t>(nch * kk);
                ci = dalloc<int64_t>(nch * kk);
                didx = dalloc<int64_t>(kk);
                dsc = dalloc<double>(kk);
                dcnt = dalloc<int64_t>(1);
                k_vec_topk_chunks<<<(unsigned)nch, TOPK_THREADS, 0, st>>>(dx, n, kk, exclude, chunk, ck, ci);
                k_vec_topk_merge<<<1, TOPK_THREADS, 0, st>>>(nch * kk, kk, ck, ci, didx, dsc, dcnt);
                count_launch(2);
                BH_CUDA(cudaGetLastError());
                int64_t m = 0;
                BH_CUDA(cudaMemcpyAsync(&m, dcnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
                BH_CUDA(cudaStreamSynchronize(st));
                BH_CUDA(cudaMemcpy(out_idx, didx, m * sizeof(int64_t), cudaMemcpyDeviceToHost));
                BH_CUDA(cudaMemcpy(out_score, dsc, m * sizeof(double), cudaMemcpyDeviceToHost));
                *out_count = m;
            } else {
                // large k: stable radix sort of (order key desc, index) pairs
                uint64_t *keys_in = dalloc<uint64_t>(n), *keys_out = dalloc<uint64_t>(n);
                int64_t *v_in = dalloc<int64_t>(n), *v_out = dalloc<int64_t>(n);
                std::vector<int64_t> iota((size_t)n);
                std::vector<uint64_t> hk((size_t)n);
                for (int64_t i = 0; i < n; i++) {
                    iota[i] = i;
                    uint64_t b;
                    std::memcpy(&b, &scores[i], 8);
                    hk[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
                }
                BH_CUDA(cudaMemcpy(keys_in, hk.data(), n * 8, cudaMemcpyHostToDevice));
                BH_CUDA(cudaMemcpy(v_in, iota.data(), n * 8, cudaMemcpyHostToDevice));
                size_t tb = 0;
                cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, keys_in, keys_out, v_in, v_out, (int)n);
                tmp = dalloc<char>(tb);
                cub::DeviceRadixSort::SortPairsDescending(tmp, tb, keys_in, keys_out, v_in, v_out, (int)n);
                count_launch(4);
                BH_CUDA(cudaGetLastError());
                std::vector<int64_t> order((size_t)n);
                BH_CUDA(cudaMemcpy(order.data(), v_out, n * 8, cudaMemcpyDeviceToHost));
                cudaFree(keys_in); cudaFree(keys_out); cudaFree(v_in); cudaFree(v_out);
                int64_t m = 0;
                for (int64_t i = 0; i < n && m < k; i++) {
                    if (order[i] == exclude) continue;
                    out_idx[m] = order[i];
                    out_score[m] = scores[order[i]];
                    m++;
                }
                *out_count = m;
            }
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
