// mpjacobi.cu -- host orchestration and the C ABI of include/mpjacobi.h.
//
// Alg. 3 as a sequence of device stages, one private stream per
// call (event-joined to the caller's stream so the legacy stream works and the
// sweep can be captured into a CUDA graph):
//   a0 symmetrise A, ||A||_F                        k_util
//   a1 fp32 Jacobi on fl32(A) -> Z                  jacobi_run<float>
//   a2 Q = CGS2(Z)                                  k_orth (+ DMMA GEMMs)
//   a3 T = Q^T A Q, symmetrised; V = Q              k_gemm, k_util
//   a4-a8 fp64 Jacobi sweeps on (T, V)              jacobi_run<double>
//   a10 Lambda = sort(diag T), V permuted           k_util
// The only host<->device traffic inside the loop is the 8-byte ||off(T)||_F
// read once per sweep for the stop test.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>
#include <cstring>
#include <string>
#include <vector>

#include "mpj_device.cuh"
#include "mpj_internal.h"

namespace mpj {

// multi-GPU (k_mg.cu)
mpj_status mg_eig(bool mixed, const double *A, int64_t n, int64_t lda, double *Lambda, double *V, int64_t ldv,
                  int *sweeps_out, const void *nccl_id, int rank, int nranks, int emulate, cudaStream_t user,
                  const mpj_config &cfg, mpj_report &rep, double *h_pin);

// SVD (k_svd.cu)
size_t svd_workspace(int64_t m, int64_t n);
mpj_status svd_run(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U, int64_t ldu,
                   double *V, int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes, cudaStream_t st,
                   const mpj_config &cfg, mpj_report &r, double *h_pin, bool a_dev, bool out_dev,
                   const float *Zin, bool zin_dev, float *Zout, bool zout_dev, int64_t ldz);

mpj_status svd_mg_run(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U, int64_t ldu,
                      double *V, int64_t ldv, int *sweeps, const void *nccl_id, int rank, int nranks, int emulate,
                      cudaStream_t st, const mpj_config &cfg, mpj_report &r, double *h_pin);

// Block-variant entry (k_block.cu).
template <typename R>
mpj_status block_sweep(R *T, int64_t ldt, R *V, int64_t ldv, int vrows, const DevSched &S, R nu,
                       int rule, unsigned long long *cnt, void *scratch, cudaStream_t st, bool first_sweep,
                       int max_brounds, int max_inner);
template <typename R>
size_t block_scratch_bytes(int np, int b);

namespace {
thread_local std::string g_err;
thread_local long long g_launches = 0;
}  // namespace

void set_error(const std::string &msg) { g_err = msg; }
void count_launch(long long k) { g_launches += k; }

cudaError_t smem_optin(const void *func, size_t bytes, int threads, int *per_sm)
{
    // the attribute is a per-(function, device) MAXIMUM: only ever raised, so a
    // launch with any size set before stays valid (a cache keyed by size alone
    // would skip re-raising it after a smaller size lowered it)
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> attr;
    static std::map<std::tuple<const void *, int, size_t, int>, int> occ_tab;   // -> CTAs per SM
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    auto ak = std::make_pair(func, dev);
    auto ai = attr.find(ak);
    if (ai == attr.end() || ai->second < bytes) {
        e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return e;
        attr[ak] = bytes;
    }
    auto key = std::make_tuple(func, dev, bytes, threads);
    auto it = occ_tab.find(key);
    if (it == occ_tab.end()) {
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, bytes);
        if (e != cudaSuccess) return e;
        it = occ_tab.emplace(key, std::max(1, occ)).first;
    }
    if (per_sm) *per_sm = it->second;
    return cudaSuccess;
}

// ---- kernel timing ---------------------------------------------------------
namespace {
struct ProfRec { double sec = 0; long long n = 0; };
bool g_prof = false;
std::map<std::string, ProfRec> g_prof_tab;
struct Pending { std::string name; cudaEvent_t a, b; };
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_ev_pool;
cudaEvent_t ev_get()
{
    if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
}
}  // namespace
bool prof_on() { return g_prof; }
void prof_mark(const char *name, cudaStream_t st, bool begin)
{
    if (!g_prof) return;
    cudaEvent_t e = ev_get();
    cudaEventRecord(e, st);
    if (begin) g_pending.push_back(Pending{name, e, nullptr});
    else {
        for (auto it = g_pending.rbegin(); it != g_pending.rend(); ++it)
            if (!it->b && it->name == name) { it->b = e; return; }
        g_ev_pool.push_back(e);
    }
}
void prof_add(const std::string &name, long long n)
{
    if (g_prof) g_prof_tab[name].n += n;
}
void prof_flush()
{
    for (auto &p : g_pending) {
        if (p.b) {
            float ms = 0.f;
            if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
                ProfRec &r = g_prof_tab[p.name];
                r.sec += ms * 1e-3; r.n += 1;
            }
            g_ev_pool.push_back(p.b);
        }
        g_ev_pool.push_back(p.a);
    }
    g_pending.clear();
}

// ---------------------------------------------------------------------------
// Ordering (reading R1), an implementation independent of oracle/.
// GVL round-robin ("music"): slot 0 of the top row is fixed; everybody else
// moves one place around the table each round.
// ---------------------------------------------------------------------------
int padded_n(int64_t n, int b)
{
    const int64_t w = 2 * (int64_t)b;
    return (int)(((n + w - 1) / w) * w);
}

static void rotate_table(std::vector<int> &top, std::vector<int> &bot)
{
    const int m = (int)top.size();
    if (m < 2) return;
    std::vector<int> t2(m), b2(m);
    t2[0] = top[0];
    t2[1] = bot[0];
    for (int k = 2; k < m; ++k) t2[k] = top[k - 1];
    for (int k = 0; k < m - 1; ++k) b2[k] = bot[k + 1];
    b2[m - 1] = top[m - 1];
    top.swap(t2);
    bot.swap(b2);
}

void build_schedule(int64_t n, int b, HostSchedule &hs)
{
    hs.n = (int)n;
    hs.b = b;
    hs.np = padded_n(n, b);
    hs.nb = hs.np / b;
    hs.mb = hs.nb / 2;
    hs.rounds = hs.np - 1;
    hs.bsched.clear();
    hs.lsched.clear();
    std::vector<int> top(hs.mb), bot(hs.mb);
    for (int k = 0; k < hs.mb; ++k) { top[k] = 2 * k; bot[k] = 2 * k + 1; }
    for (int R = 0; R < hs.nb - 1; ++R) {
        for (int k = 0; k < hs.mb; ++k) hs.bsched.push_back(make_int2(top[k], bot[k]));
        rotate_table(top, bot);
    }
    if (b > 1) {
        const int hb = b / 2;
        std::vector<int> lt(hb), lb(hb);
        for (int k = 0; k < hb; ++k) { lt[k] = 2 * k; lb[k] = 2 * k + 1; }
        for (int s = 0; s < b - 1; ++s) {
            for (int k = 0; k < hb; ++k) hs.lsched.push_back(make_int2(lt[k], lb[k]));
            rotate_table(lt, lb);
        }
    }
}

// ---------------------------------------------------------------------------
// Workspace arena (256-byte aligned bump allocator; a NULL base measures).
// ---------------------------------------------------------------------------
struct Arena {
    char *base = nullptr;
    size_t off = 0, cap = 0;
    template <typename T>
    T *take(size_t count)
    {
        off = (off + 255) & ~(size_t)255;
        T *p = base ? (T *)(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

static int auto_b(int64_t n)
{
    // b = 32 (2b = 64 tiles) from n = 32 up (n <= 64 is padded to one 64 x 64
    // block pair: a sweep is one K3 + one K4 launch); smaller b only below
    if (n >= 32) return 32;
    int b = (int)((n + 3) / 4) * 2;     // about n/2, even
    return std::max(1, std::min(32, b));
}

static int resolve_b(int64_t n, const mpj_config *cfg)
{
    int b = (cfg && cfg->block_b > 0) ? cfg->block_b : auto_b(n);
    return b;
}

static int resolve_variant(int np, int b, const mpj_config *cfg)
{
    int v = cfg ? cfg->variant : MPJ_VARIANT_AUTO;
    // block variant whenever the b = 32 kernels apply: at n_p = 64 one block pair
    // makes a sweep one K3 launch (all 63 rounds in shared memory) plus the V update
    if (v == MPJ_VARIANT_AUTO) v = (np >= 64 && b == 32) ? MPJ_VARIANT_BLOCK : MPJ_VARIANT_SCALAR;
    if ((v == MPJ_VARIANT_BLOCK || v == MPJ_VARIANT_BLOCK_FULL) && b != 32) v = MPJ_VARIANT_SCALAR;   // b = 32 kernels
    return v;
}
static bool is_block(int v) { return v == MPJ_VARIANT_BLOCK || v == MPJ_VARIANT_BLOCK_FULL; }
constexpr int kMaxInner = 30;     // inner sweeps of the classic block Jacobi (reading R26)

// ---------------------------------------------------------------------------
// Per-call stream context: private stream joined to the caller's stream.
// ---------------------------------------------------------------------------
struct CtxCache {            // per-thread, created once: no per-call allocation or sync
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    double *h_pin = nullptr;
    int dev = -1;
};
static thread_local CtxCache g_ctx;

struct Ctx {
    cudaStream_t user = nullptr, st = nullptr;
    cudaEvent_t ev = nullptr;
    double *h_pin = nullptr;   // pinned host scalars
    bool open_ = false;
    mpj_status open(void *stream)
    {
        user = (cudaStream_t)stream;
        int dev = 0;
        MPJ_CK(cudaGetDevice(&dev));
        if (g_ctx.st == nullptr || g_ctx.dev != dev) {
            // keep stream-ordered allocations (library-owned workspaces) cached in the
            // device's default pool instead of trimming it at every synchronisation
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            MPJ_CK(cudaStreamCreateWithFlags(&g_ctx.st, cudaStreamNonBlocking));
            MPJ_CK(cudaEventCreateWithFlags(&g_ctx.ev, cudaEventDisableTiming));
            MPJ_CK(cudaMallocHost(&g_ctx.h_pin, 64 * sizeof(double)));
            g_ctx.dev = dev;
        }
        st = g_ctx.st; ev = g_ctx.ev; h_pin = g_ctx.h_pin;
        MPJ_CK(cudaEventRecord(ev, user));
        MPJ_CK(cudaStreamWaitEvent(st, ev, 0));
        open_ = true;
        return MPJ_OK;
    }
    mpj_status close()
    {
        if (open_) {
            cudaEventRecord(ev, st);
            cudaStreamWaitEvent(user, ev, 0);
            cudaStreamSynchronize(st);
            open_ = false;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error(std::string("CUDA: ") + cudaGetErrorString(e));
            return MPJ_ERR_CUDA;
        }
        return MPJ_OK;
    }
    ~Ctx() { close(); }
};

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st;
    explicit Timer(cudaStream_t s) : st(s)
    {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
    }
    double stop()
    {
        float ms = 0.f;
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        return ms * 1e-3;
    }
    ~Timer()
    {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

// ---------------------------------------------------------------------------
// The Jacobi loop (Alg. 2 / Alg. 3 steps 4-11) on padded n_p x n_p T, V.
// ---------------------------------------------------------------------------
template <typename R>
struct JacobiBufs {
    int2 *pq;
    R *t, *s, *u;
    unsigned long long *cnt;
    double *part, *off;
    int2 *bsched, *lsched;
    void *block_scratch;
    R *Tn;          // scalar variant: the other T buffer of the fused round kernel
    int *pos;       // scalar variant: row -> (slot, is q)
};

template <typename R>
static void carve_jacobi(Arena &ar, int np, int b, int variant, JacobiBufs<R> &jb)
{
    const int h = np / 2;
    jb.pq = ar.take<int2>(h);
    jb.t = ar.take<R>(h);
    jb.s = ar.take<R>(h);
    jb.u = ar.take<R>(h);
    jb.cnt = ar.take<unsigned long long>(4);
    jb.part = ar.take<double>(kRedBlocks);
    jb.off = ar.take<double>(4);
    const int nb = np / b;
    jb.bsched = ar.take<int2>((size_t)std::max(nb - 1, 1) * std::max(nb / 2, 1));
    jb.lsched = ar.take<int2>((size_t)std::max(b - 1, 1) * std::max(b / 2, 1));
    jb.block_scratch = is_block(variant) ? ar.take<char>(block_scratch_bytes<R>(np, b)) : nullptr;
    jb.Tn = (variant == MPJ_VARIANT_SCALAR) ? ar.take<R>((size_t)np * np) : nullptr;
    jb.pos = ar.take<int>(np);
}

// the scalar round kernels: K1 + fused K2/K3 (coalesced, out of place into the
// other T buffer; default) or K1 + K2 + K3 in place (MPJ_SCALAR_FUSED=0, A/B)
static bool scalar_fused()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MPJ_SCALAR_FUSED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// Instantiated graphs of one scalar-variant sweep, reused across calls with
// the same buffers and parameters (instantiating one cost ~170 us + ~100 us
// to destroy per call: a fifth of an n = 32 EVD).  Kernel arguments are
// baked into a graph, so the key holds every pointer and scalar it captures.
struct SweepGraphKey {
    int dev, np, rule, rounds, fused, rsize;
    double nu;
    const void *ptr[11];
    bool operator==(const SweepGraphKey &o) const
    {
        return dev == o.dev && np == o.np && rule == o.rule && rounds == o.rounds && fused == o.fused &&
               rsize == o.rsize && std::memcmp(&nu, &o.nu, sizeof(nu)) == 0 &&
               std::memcmp(ptr, o.ptr, sizeof(ptr)) == 0;
    }
};
struct SweepGraph {
    SweepGraphKey key;
    cudaGraphExec_t exec;
    long long kernels;
};
static std::mutex g_sweep_graph_mu;
static std::vector<SweepGraph> g_sweep_graphs;   // most recent last; at most 16 kept

struct JacobiOut {
    int sweeps = 0;
    long long rotations = 0;
    double hist[64] = {0};
    long long rot_hist[64] = {0};   // rotations applied in sweep k+1
    int nhist = 0;
};

template <typename R>
static mpj_status jacobi_run(Ctx &cx, R *T, R *V, int n, int b, int variant, double tol, R nu,
                             int rule, int max_sweeps, int64_t max_rounds, JacobiBufs<R> &jb,
                             JacobiOut &out)
{
    cudaStream_t st = cx.st;
    HostSchedule hs;
    build_schedule(n, b, hs);
    const int np = hs.np, h = np / 2;
    DevSched ds;
    ds.bsched = jb.bsched; ds.lsched = jb.lsched; ds.b = b; ds.nb = hs.nb; ds.np = np; ds.rounds = hs.rounds;
    if (!hs.bsched.empty())
        MPJ_CK(cudaMemcpyAsync(jb.bsched, hs.bsched.data(), hs.bsched.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    if (!hs.lsched.empty())
        MPJ_CK(cudaMemcpyAsync(jb.lsched, hs.lsched.data(), hs.lsched.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    MPJ_CK(cudaMemsetAsync(jb.cnt, 0, sizeof(unsigned long long), st));

    cudaGraphExec_t gexec = nullptr;
    long long graph_kernels = 0;
    const bool use_graph = (variant == MPJ_VARIANT_SCALAR) && max_rounds < 0;
    int64_t rounds_done = 0;
    int sweeps = 0;
    mpj_status status = MPJ_ERR_NOCONV;
    unsigned long long rot_prev = 0;
    for (;;) {
        launch_norm<R>(T, np, np, np, true, jb.part, jb.off, st);
        MPJ_CK(cudaMemcpyAsync(cx.h_pin, jb.off, sizeof(double), cudaMemcpyDeviceToHost, st));
        MPJ_CK(cudaMemcpyAsync(cx.h_pin + 1, jb.cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        MPJ_CK(cudaStreamSynchronize(st));
        const double off = cx.h_pin[0];
        unsigned long long rot_now = 0;
        std::memcpy(&rot_now, cx.h_pin + 1, sizeof(rot_now));
        if (sweeps >= 1 && sweeps <= 64) out.rot_hist[sweeps - 1] = (long long)(rot_now - rot_prev);
        rot_prev = rot_now;
        if (sweeps < 64) { out.hist[sweeps] = off; out.nhist = sweeps + 1; }
        if (!std::isfinite(off)) { set_error("non-finite off-norm"); status = MPJ_ERR_NONFINITE; break; }
        if (off <= tol) { status = MPJ_OK; break; }
        if (sweeps >= max_sweeps) { status = MPJ_ERR_NOCONV; break; }
        if (max_rounds >= 0 && rounds_done >= max_rounds) { status = MPJ_OK; break; }
        ++sweeps;
        if (is_block(variant)) {
            // block round 0 holds 2b - 1 scalar rounds (b - 1 intra-block + b
            // cross), every later one b (reading R1); a round limit must fall
            // on a block-round boundary
            int nbr = hs.nb - 1;
            int64_t used = hs.rounds;
            if (max_rounds >= 0 && max_rounds - rounds_done < hs.rounds) {
                const int64_t left = max_rounds - rounds_done;
                int k = 0;
                used = 0;
                while (k < nbr) {
                    const int64_t c = k == 0 ? 2 * b - 1 : b;
                    if (used + c > left) break;
                    used += c;
                    ++k;
                }
                if (used != left) {
                    set_error("max_rounds must end on a block-round boundary (2b-1, then +b)");
                    return MPJ_ERR_INVALID;
                }
                nbr = k;
            }
            MPJ_TRY(block_sweep<R>(T, np, V, np, np, ds, nu, rule, jb.cnt, jb.block_scratch, st, sweeps == 1,
                                   nbr, variant == MPJ_VARIANT_BLOCK_FULL ? kMaxInner : 0));
            rounds_done += used;
        } else {
            // scalar rounds; the fused kernel writes T into the other buffer, so a
            // sweep (an odd number of rounds) ends with one copy back
            const bool fused = scalar_fused();
            auto sweep_rounds = [&](int r0, int r1) {
                R *cur = T, *nxt = jb.Tn;
                for (int r = r0; r < r1; ++r) {
                    launch_round_params<R>(cur, np, ds, r, nu, rule, jb.pq, jb.t, jb.s, jb.u, jb.cnt, st, jb.pos);
                    if (fused) {
                        launch_round_apply_fused_oop<R>(cur, nxt, np, V, np, np, np, jb.pq, jb.pos, jb.t, jb.s, jb.u,
                                                        st);
                        std::swap(cur, nxt);
                    } else {
                        launch_round_apply<R>(cur, np, jb.pq, jb.t, jb.s, jb.u, h, st);
                        launch_round_apply_v<R>(V, np, np, jb.pq, jb.s, jb.u, h, st);
                    }
                }
                if (cur != T) MPJ_CK_VOID(cudaMemcpyAsync(T, cur, (size_t)np * np * sizeof(R), cudaMemcpyDeviceToDevice, st));
            };
            if (use_graph) {
                // the cache lock is held from the lookup to the launch: a cached
                // exec is never evicted (at most 16 are kept; beyond that a call
                // instantiates its own and destroys it after its final sync)
                SweepGraphKey key;
                std::memset(&key, 0, sizeof(key));
                cudaGetDevice(&key.dev);
                key.np = np; key.rule = rule; key.rounds = hs.rounds; key.fused = fused ? 1 : 0;
                key.rsize = (int)sizeof(R); key.nu = (double)nu;
                const void *ptrs[11] = {T, V, jb.Tn, jb.pq, jb.pos, jb.t, jb.s, jb.u, jb.cnt, jb.bsched, jb.lsched};
                std::memcpy(key.ptr, ptrs, sizeof(ptrs));
                std::unique_lock<std::mutex> lk(g_sweep_graph_mu);
                cudaGraphExec_t ge = gexec;
                if (!ge)
                    for (auto &e : g_sweep_graphs)
                        if (e.key == key) { ge = e.exec; graph_kernels = e.kernels; break; }
                if (!ge) {
                    cudaGraph_t g;
                    const long long l0 = g_launches;
                    MPJ_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                    sweep_rounds(0, hs.rounds);
                    MPJ_CK(cudaStreamEndCapture(st, &g));
                    graph_kernels = g_launches - l0;
                    g_launches = l0;
                    MPJ_CK(cudaGraphInstantiate(&ge, g, 0));
                    cudaGraphDestroy(g);
                    if (g_sweep_graphs.size() < 16) g_sweep_graphs.push_back({key, ge, graph_kernels});
                    else gexec = ge;                 // this call's own exec (destroyed below)
                }
                MPJ_CK(cudaGraphLaunch(ge, st));
                lk.unlock();
                count_launch(graph_kernels);
                rounds_done += hs.rounds;
            } else {
                int r1 = hs.rounds;
                if (max_rounds >= 0) r1 = (int)std::min<int64_t>(r1, max_rounds - rounds_done);
                sweep_rounds(0, r1);
                rounds_done += r1;
            }
        }
    }
    unsigned long long rot = 0;
    MPJ_CK(cudaMemcpyAsync(cx.h_pin, jb.cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    if (gexec) cudaGraphExecDestroy(gexec);   // an uncached exec of this call (the cache was full)
    std::memcpy(&rot, cx.h_pin, sizeof(rot));
    out.sweeps = sweeps;
    out.rotations = (long long)rot;
    MPJ_CK(cudaGetLastError());
    return status;
}

// ---------------------------------------------------------------------------
// Host/device pointer handling for the end-to-end entry points.
// ---------------------------------------------------------------------------
static bool is_device_ptr(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static mpj_status copy2d(void *dst, int64_t ldd, const void *src, int64_t lds, int64_t rows, int64_t cols,
                         size_t esz, cudaMemcpyKind kind, cudaStream_t st)
{
    if (rows <= 0 || cols <= 0) return MPJ_OK;
    MPJ_CK(cudaMemcpy2DAsync(dst, ldd * esz, src, lds * esz, rows * esz, cols, kind, st));
    return MPJ_OK;
}

// ---------------------------------------------------------------------------
// Alg. 3 / Alg. 2 drivers
// ---------------------------------------------------------------------------
struct EigPlan {
    int n, b, np, variant;
    void *symqr_ws;
    double *Asym, *T, *V, *W;
    float *T32, *V32;
    double *red_part, *red_out;
    int *flag, *rank;
    double *lam;
    void *orth_ws;
    JacobiBufs<double> j64;
    JacobiBufs<float> j32;
};

static void carve_eig(Arena &ar, int64_t n, const mpj_config *cfg, EigPlan &p)
{
    p.n = (int)n;
    p.b = resolve_b(n, cfg);
    p.np = padded_n(n, p.b);
    p.variant = resolve_variant(p.np, p.b, cfg);
    const size_t nn = (size_t)p.np * p.np;
    p.Asym = ar.take<double>(nn);
    p.T = ar.take<double>(nn);
    p.V = ar.take<double>(nn);
    p.W = ar.take<double>(nn);
    p.T32 = ar.take<float>(nn);
    p.V32 = ar.take<float>(nn);
    p.red_part = ar.take<double>(kRedBlocks);
    p.red_out = ar.take<double>(4);
    p.flag = ar.take<int>(4);
    p.rank = ar.take<int>(p.np);
    p.lam = ar.take<double>(p.np);
    p.orth_ws = ar.take<char>((cfg && cfg->orth == MPJ_ORTH_HOUSEHOLDER) ? hqr_workspace(p.np, p.np)
                                                                           : orth_workspace(p.np));
    p.symqr_ws = ar.take<char>(symqr_workspace(p.np));
    carve_jacobi<double>(ar, p.np, p.b, p.variant, p.j64);
    carve_jacobi<float>(ar, p.np, p.b, p.variant, p.j32);
}

static mpj_status read_scalar(Ctx &cx, const double *d, double &out)
{
    MPJ_CK(cudaMemcpyAsync(cx.h_pin, d, sizeof(double), cudaMemcpyDeviceToHost, cx.st));
    MPJ_CK(cudaStreamSynchronize(cx.st));
    out = cx.h_pin[0];
    return MPJ_OK;
}

// Low-stage stop tolerance factor (reading R12): max(10, 1.25 sqrt(n)) unless set.
double eps_low_factor(const mpj_config &cfg, int64_t n)
{
    if (cfg.eps_low_factor > 0) return cfg.eps_low_factor;
    return std::max(10.0, 1.25 * std::sqrt((double)n));
}

static const double kOmega = 1.1102230246251565e-16;    // 2^-53
static const double kUpsilon = 5.9604644775390625e-08;  // 2^-24

static mpj_status eig_impl(bool mixed, const double *A, int64_t n, int64_t lda, double *Lambda,
                           double *V, int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes,
                           void *stream, const mpj_config *cfg_in, mpj_report *rep,
                           const float *Zin = nullptr, float *Zout = nullptr, int64_t ldz = 0)
{
    g_err.clear();
    if (n < 1 || lda < n || ldv < n || !A || !Lambda || !V || ((Zin || Zout) && ldz < n)) {
        set_error("mpjacobi_eig: invalid argument");
        return MPJ_ERR_INVALID;
    }
    if (n > (1 << 20)) { set_error("n too large"); return MPJ_ERR_INVALID; }
    mpj_config cfg;
    if (cfg_in) cfg = *cfg_in; else mpj_config_default_eig(&cfg);
    const int b = resolve_b(n, &cfg);
    if (b < 1 || (b > 1 && (b & 1))) { set_error("block_b must be 1 or even"); return MPJ_ERR_INVALID; }

    Ctx cx;
    MPJ_TRY(cx.open(stream));
    Timer t_all(cx.st);
    const long long l0 = g_launches;

    // n <= 64 with the default configuration and device buffers: the
    // single-CTA kernels of the batched path run the same Alg. 3 (symmetric-QR
    // step 1, Cholesky-QR step 2, Q^T A Q, the fp64 sweeps of the one 64 x 64
    // block pair) in one launch pair, where the general path needs ~50
    // launches and a host round trip per sweep (n = 32: 0.40 vs 0.85 ms).
    // MPJ_SMALL_BATCHED=0 turns it off.
    static const bool small_batched = !(getenv("MPJ_SMALL_BATCHED") && getenv("MPJ_SMALL_BATCHED")[0] == '0');
    if (mixed && small_batched && n <= 64 && !Zin && !Zout && cfg.variant == MPJ_VARIANT_AUTO &&
        (cfg.low_solver == MPJ_LOW_SYMQR || cfg.low_solver == MPJ_LOW_AUTO)) {
        // host buffers or leading dimensions other than n are staged (the same kernels either way)
        const bool a_d = is_device_ptr(A) && lda == n, l_d = is_device_ptr(Lambda), v_d = is_device_ptr(V) && ldv == n;
        double *stg = nullptr;
        MPJ_CK(cudaMallocAsync(&stg, (size_t)(2 * n * n + n) * sizeof(double) + 2 * sizeof(int), cx.st));
        double *Ad = a_d ? const_cast<double *>(A) : stg, *Vd = v_d ? V : stg + n * n, *Ld = l_d ? Lambda : stg + 2 * n * n;
        int *dsw = (int *)(stg + 2 * n * n + n);
        MPJ_CK(cudaMemsetAsync(dsw, 0, 2 * sizeof(int), cx.st));
        mpj_status s = MPJ_OK;
        if (!a_d)
            s = copy2d(Ad, n, A, lda, n, n, sizeof(double),
                       is_device_ptr(A) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, cx.st);
        if (s == MPJ_OK) s = batched_evd(Ad, n, 1, Ld, Vd, dsw, dsw + 1, nullptr, nullptr, cx.st, cfg);
        if (s == MPJ_OK || s == MPJ_ERR_NOCONV) {   // NOCONV: the last iterate is written, as on the general path
            mpj_status c2 = MPJ_OK;
            if (!v_d)
                c2 = copy2d(V, ldv, Vd, n, n, n, sizeof(double),
                            is_device_ptr(V) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, cx.st);
            if (c2 == MPJ_OK && !l_d && cudaMemcpyAsync(Lambda, Ld, n * sizeof(double), cudaMemcpyDeviceToHost,
                                                        cx.st) != cudaSuccess)
                c2 = MPJ_ERR_CUDA;
            if (c2 != MPJ_OK) s = c2;
        }
        int hsw[2] = {0, 0};
        cudaMemcpyAsync(cx.h_pin, dsw, 2 * sizeof(int), cudaMemcpyDeviceToHost, cx.st);
        cudaFreeAsync(stg, cx.st);
        cudaStreamSynchronize(cx.st);
        std::memcpy(hsw, cx.h_pin, sizeof(hsw));
        mpj_report r;
        std::memset(&r, 0, sizeof(r));
        r.n_padded = 64;
        r.block_b = 32;
        r.variant = MPJ_VARIANT_BLOCK;
        r.sweeps = hsw[0];
        r.sweeps_low = hsw[1];
        r.t_total = t_all.stop();
        r.launches = g_launches - l0;
        if (rep) *rep = r;
        if (sweeps) *sweeps = hsw[0];
        mpj_status c = cx.close();
        return s != MPJ_OK ? s : c;
    }

    Arena ar;
    EigPlan p;
    carve_eig(ar, n, &cfg, p);   // measure
    const size_t need = ar.off + 256;
    void *own = nullptr;
    if (!workspace) {
        MPJ_CK(cudaMallocAsync(&own, need, cx.st));
        workspace = own;
    } else if (ws_bytes < need) {
        set_error("workspace too small");
        return MPJ_ERR_NOMEM;
    }
    ar = Arena();
    ar.base = (char *)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
    carve_eig(ar, n, &cfg, p);
    const int np = p.np;
    mpj_report r;
    std::memset(&r, 0, sizeof(r));
    r.n_padded = np;
    r.block_b = p.b;
    r.variant = p.variant;

    auto finish = [&](mpj_status s) -> mpj_status {
        if (own) cudaFreeAsync(own, cx.st);
        r.t_total = t_all.stop();
        r.launches = g_launches - l0;
        if (rep) *rep = r;
        mpj_status c = cx.close();
        return s != MPJ_OK ? s : c;
    };
    // every error exit below releases the workspace and fills rep (finish)
#define MPJ_CKF(expr)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));              \
            return finish(MPJ_ERR_CUDA);                                                \
        }                                                                               \
    } while (0)
#define MPJ_TRYF(expr)                                                                  \
    do {                                                                                \
        mpj_status s_ = (expr);                                                         \
        if (s_ != MPJ_OK) return finish(s_);                                            \
    } while (0)

    // a0: stage A (host or device) into T, symmetrise into Asym, check finite, ||A||_F
    const bool a_dev = is_device_ptr(A);
    {
        mpj_status s;
        if (a_dev) s = copy2d(p.T, np, A, lda, n, n, sizeof(double), cudaMemcpyDeviceToDevice, cx.st);
        else s = copy2d(p.T, np, A, lda, n, n, sizeof(double), cudaMemcpyHostToDevice, cx.st);
        if (s != MPJ_OK) return finish(s);
    }
    cudaMemsetAsync(p.flag, 0, sizeof(int), cx.st);
    launch_check_finite(p.T, np, (int)n, (int)n, p.flag, cx.st);
    launch_symmetrize(p.T, np, (int)n, p.Asym, np, np, cx.st);
    launch_norm<double>(p.Asym, np, np, np, false, p.red_part, p.red_out, cx.st);
    MPJ_CKF(cudaMemcpyAsync(cx.h_pin, p.red_out, sizeof(double), cudaMemcpyDeviceToHost, cx.st));
    MPJ_CKF(cudaMemcpyAsync(cx.h_pin + 1, p.flag, sizeof(int), cudaMemcpyDeviceToHost, cx.st));
    MPJ_CKF(cudaStreamSynchronize(cx.st));
    const double normA = cx.h_pin[0];
    int bad = 0;
    std::memcpy(&bad, cx.h_pin + 1, sizeof(int));
    if (bad) { set_error("input has NaN/Inf"); return finish(MPJ_ERR_NONFINITE); }
    r.norm_a = normA;

    mpj_status s = MPJ_OK;
    if (mixed) {
        // a1: low-precision stage (reading R12) -- or the caller's Z
        Timer tl(cx.st);
        if (Zin) {
            MPJ_CKF(cudaMemsetAsync(p.V32, 0, (size_t)np * np * sizeof(float), cx.st));
            MPJ_TRYF(copy2d(p.V32, np, Zin, ldz, n, n, sizeof(float),
                            is_device_ptr(Zin) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, cx.st));
            r.status_low = MPJ_OK;
        } else if (cfg.low_solver != MPJ_LOW_JACOBI) {
            // "symmetric QR factorization in low precision" (reading R12')
            launch_copy_pad<double, float>(p.Asym, np, np, np, p.T32, np, np, np, cx.st);
            MPJ_TRYF(low_evd_symqr(p.T32, np, (int)n, p.V32, np, p.W, np, p.T, p.V, p.symqr_ws, cx.st));
            r.status_low = MPJ_OK;
        } else {
            launch_copy_pad<double, float>(p.Asym, np, np, np, p.T32, np, np, np, cx.st);
            MPJ_CKF(cudaMemsetAsync(p.V32, 0, (size_t)np * np * sizeof(float), cx.st));
            launch_identity<float>(p.V32, np, (int)n, (int)n, cx.st);
            launch_norm<float>(p.T32, np, np, np, false, p.red_part, p.red_out, cx.st);
            double nA32 = 0;
            MPJ_TRYF(read_scalar(cx, p.red_out, nA32));
            JacobiOut jo;
            mpj_status sl = jacobi_run<float>(cx, p.T32, p.V32, (int)n, p.b, p.variant,
                                              eps_low_factor(cfg, n) * kUpsilon * nA32,
                                              (float)(cfg.nu_low_factor * kUpsilon), cfg.stop_rule,
                                              cfg.max_sweeps_low, -1, p.j32, jo);
            if (sl != MPJ_OK && sl != MPJ_ERR_NOCONV) return finish(sl);
            r.sweeps_low = jo.sweeps;
            r.rotations_low = jo.rotations;
            r.status_low = sl;
            for (int k = 0; k < jo.nhist && k < 64; ++k) r.off_hist_low[k] = jo.hist[k];
        }
        if (Zout)
            MPJ_TRYF(copy2d(Zout, ldz, p.V32, np, n, n, sizeof(float),
                            is_device_ptr(Zout) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, cx.st));
        r.t_low = tl.stop();

        // a2: Q = orth(Z), Z = fp64(V32) (n x n real block)
        Timer to(cx.st);
        launch_copy_pad<float, double>(p.V32, np, (int)n, (int)n, p.W, np, (int)n, (int)n, cx.st);
        MPJ_CKF(cudaMemsetAsync(p.V, 0, (size_t)np * np * sizeof(double), cx.st));
        if (cfg.orth == MPJ_ORTH_HOUSEHOLDER) {
            s = orth_householder(p.W, np, p.V, np, n, n, p.orth_ws, cx.st);
        } else {
            // MPJ_ORTH_AUTO: the fixed-point Cholesky QR (R10b) up to n = 2048, CGS above;
            // it declines (NOCONV) when Z is not orthogonal enough, and CGS runs
            s = MPJ_ERR_NOCONV;
            if (cfg.orth == MPJ_ORTH_SERIES || (cfg.orth == MPJ_ORTH_AUTO && n <= 2048))
                s = orth_series(p.W, np, p.V, np, n, cx.st);
            if (s == MPJ_ERR_NOCONV) s = orth_cgs2(p.W, np, p.V, np, n, n, p.orth_ws, cx.st);
        }
        if (s != MPJ_OK) return finish(s);
        r.t_orth = to.stop();

        // a3: T = Q^T A Q (W = A Q, T = Q^T W), symmetrised (reading R11)
        Timer tp(cx.st);
        MPJ_CKF(cudaMemsetAsync(p.T, 0, (size_t)np * np * sizeof(double), cx.st));
        launch_dgemm(false, false, n, n, n, 1.0, p.Asym, np, p.V, np, 0.0, p.W, np, cx.st);
        // T is symmetric: only its upper tiles are formed, then mirrored (reading R11)
        launch_dgemm(true, false, n, n, n, 1.0, p.V, np, p.W, np, 0.0, p.T, np, cx.st, nullptr, 0, true);
        launch_symmetrize_inplace(p.T, np, (int)n, cx.st, true);
        launch_norm<double>(p.T, np, np, np, true, p.red_part, p.red_out, cx.st);
        MPJ_TRYF(read_scalar(cx, p.red_out, r.off0));
        r.t_precond = tp.stop();
    } else {
        MPJ_CKF(cudaMemcpyAsync(p.T, p.Asym, (size_t)np * np * sizeof(double), cudaMemcpyDeviceToDevice, cx.st));
        MPJ_CKF(cudaMemsetAsync(p.V, 0, (size_t)np * np * sizeof(double), cx.st));
        launch_identity<double>(p.V, np, (int)n, (int)n, cx.st);
        launch_norm<double>(p.T, np, np, np, true, p.red_part, p.red_out, cx.st);
        MPJ_TRYF(read_scalar(cx, p.red_out, r.off0));
    }

    // a4-a8: fp64 sweeps
    {
        Timer tj(cx.st);
        JacobiOut jo;
        s = jacobi_run<double>(cx, p.T, p.V, (int)n, p.b, p.variant, cfg.eps_factor * kOmega * normA,
                               cfg.nu_factor * kOmega, cfg.stop_rule, cfg.max_sweeps, -1, p.j64, jo);
        r.sweeps = jo.sweeps;
        r.rotations = jo.rotations;
        r.status = s;
        for (int k = 0; k < jo.nhist && k < 64; ++k) r.off_hist[k] = jo.hist[k];
        for (int k = 0; k < 64; ++k) r.rot_hist[k] = jo.rot_hist[k];
        r.t_jacobi = tj.stop();
        if (s != MPJ_OK && s != MPJ_ERR_NOCONV) return finish(s);
    }
    if (sweeps) *sweeps = r.sweeps;

    // a10: extraction (stable descending)
    {
        Timer te(cx.st);
        const bool l_dev = is_device_ptr(Lambda), v_dev = is_device_ptr(V);
        double *lam_d = l_dev ? Lambda : p.lam;
        double *v_d = v_dev ? V : p.W;
        const int64_t ldvo = v_dev ? ldv : np;
        launch_extract_evd(p.T, np, p.V, np, (int)n, (int)n, lam_d, v_d, ldvo, p.rank, cx.st);
        if (!l_dev) MPJ_CKF(cudaMemcpyAsync(Lambda, p.lam, n * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
        if (!v_dev) {
            mpj_status c = copy2d(V, ldv, p.W, np, n, n, sizeof(double), cudaMemcpyDeviceToHost, cx.st);
            if (c != MPJ_OK) return finish(c);
        }
        MPJ_CKF(cudaStreamSynchronize(cx.st));
        r.t_extract = te.stop();
    }
    return finish(s);
#undef MPJ_CKF
#undef MPJ_TRYF
}

template <typename R>
static mpj_status jacobi_impl(R *T, int64_t ldt, R *V, int64_t ldv, int64_t n, double tol, double nu,
                              int max_sweeps, int64_t max_rounds, int *sweeps, long long *rotations,
                              double *hist, void *stream, const mpj_config *cfg)
{
    g_err.clear();
    if (n < 1 || ldt < n || ldv < n || !T || !V) { set_error("invalid argument"); return MPJ_ERR_INVALID; }
    const int b = resolve_b(n, cfg);
    if (b < 1 || (b > 1 && (b & 1))) { set_error("block_b must be 1 or even"); return MPJ_ERR_INVALID; }
    const int np = padded_n(n, b);
    const int variant = resolve_variant(np, b, cfg);
    const int rule = cfg ? cfg->stop_rule : 0;
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    Arena ar;
    JacobiBufs<R> jb;
    R *Tp, *Vp;
    auto carve = [&]() {
        Tp = ar.take<R>((size_t)np * np);
        Vp = ar.take<R>((size_t)np * np);
        carve_jacobi<R>(ar, np, b, variant, jb);
    };
    carve();
    void *own = nullptr;
    MPJ_CK(cudaMallocAsync(&own, ar.off + 256, cx.st));
    ar = Arena();
    ar.base = (char *)(((uintptr_t)own + 255) & ~(uintptr_t)255);
    carve();
    launch_copy_pad<R, R>(T, ldt, (int)n, (int)n, Tp, np, np, np, cx.st);
    launch_copy_pad<R, R>(V, ldv, (int)n, (int)n, Vp, np, np, np, cx.st);
    JacobiOut jo;
    mpj_status s = jacobi_run<R>(cx, Tp, Vp, (int)n, b, variant, tol, (R)nu, rule, max_sweeps, max_rounds,
                                 jb, jo);
    if (s == MPJ_OK || s == MPJ_ERR_NOCONV) {
        launch_copy_pad<R, R>(Tp, np, (int)n, (int)n, T, ldt, (int)n, (int)n, cx.st);
        launch_copy_pad<R, R>(Vp, np, (int)n, (int)n, V, ldv, (int)n, (int)n, cx.st);
    }
    cudaFreeAsync(own, cx.st);
    if (sweeps) *sweeps = jo.sweeps;
    if (rotations) *rotations = jo.rotations;
    if (hist) for (int k = 0; k < 64; ++k) hist[k] = k < jo.nhist ? jo.hist[k] : 0.0;
    mpj_status c = cx.close();
    return s != MPJ_OK ? s : c;
}

}  // namespace mpj

// ===========================================================================
// C ABI
// ===========================================================================
using namespace mpj;

extern "C" {

void mpj_config_default_eig(mpj_config *c)
{
    if (!c) return;
    c->eps_factor = 0.1;
    c->nu_factor = 20.0;
    c->eps_low_factor = 0.0;   /* reading R12: max(10, 1.25 sqrt(n)) */
    c->nu_low_factor = 20.0;
    c->early_stop_ratio = 0.0;
    c->max_sweeps = 60;
    c->max_sweeps_low = 60;
    c->stop_rule = 0;
    c->variant = MPJ_VARIANT_AUTO;
    c->block_b = 0;
    c->low_solver = MPJ_LOW_AUTO;
    c->orth = MPJ_ORTH_AUTO;
}

void mpj_config_default_svd(mpj_config *c)
{
    if (!c) return;
    mpj_config_default_eig(c);
    c->nu_factor = 1.0;
    c->nu_low_factor = 1.0;
    c->early_stop_ratio = 2e-4;
    c->eps_low_factor = 10.0;   /* SPEC's 10 upsilon: measured best for Alg. 5 (DESIGN R12) */
}

const char *mpjacobi_last_error(void) { return g_err.c_str(); }
void mpjacobi_profile_enable(int on) { mpj::g_prof = on != 0; }
void mpjacobi_profile_reset(void)
{
    mpj::prof_flush();
    mpj::g_prof_tab.clear();
}
void mpjacobi_profile_get(const char *kernel, double *seconds, long long *launches)
{
    mpj::prof_flush();
    auto it = mpj::g_prof_tab.find(kernel ? kernel : "");
    if (seconds) *seconds = it == mpj::g_prof_tab.end() ? 0.0 : it->second.sec;
    if (launches) *launches = it == mpj::g_prof_tab.end() ? 0 : it->second.n;
}
long long mpjacobi_launch_count(void) { return g_launches; }

size_t mpjacobi_eig_workspace(int64_t n, const mpj_config *cfg)
{
    if (n < 1) return 0;
    mpj_config c;
    if (cfg) c = *cfg; else mpj_config_default_eig(&c);
    Arena ar;
    EigPlan p;
    carve_eig(ar, n, &c, p);
    return ar.off + 256;
}

mpj_status mpjacobi_eig(const double *A, int64_t n, int64_t lda, double *Lambda, double *V, int64_t ldv,
                        int *sweeps, void *workspace, size_t ws_bytes, void *stream, const mpj_config *cfg,
                        mpj_report *rep)
{
    return eig_impl(true, A, n, lda, Lambda, V, ldv, sweeps, workspace, ws_bytes, stream, cfg, rep);
}

mpj_status mpjacobi_eig_z(const double *A, int64_t n, int64_t lda, const float *Z_in, float *Z_out, int64_t ldz,
                          double *Lambda, double *V, int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes,
                          void *stream, const mpj_config *cfg, mpj_report *rep)
{
    return eig_impl(true, A, n, lda, Lambda, V, ldv, sweeps, workspace, ws_bytes, stream, cfg, rep, Z_in, Z_out,
                    ldz);
}

mpj_status mpjacobi_eig_plain(const double *A, int64_t n, int64_t lda, double *Lambda, double *V,
                              int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes, void *stream,
                              const mpj_config *cfg, mpj_report *rep)
{
    return eig_impl(false, A, n, lda, Lambda, V, ldv, sweeps, workspace, ws_bytes, stream, cfg, rep);
}

mpj_status mpjacobi_jacobi_f64(double *T, int64_t ldt, double *V, int64_t ldv, int64_t n, double tol,
                               double nu, int max_sweeps, int64_t max_rounds, int *sweeps,
                               long long *rotations, double *hist, void *stream, const mpj_config *cfg)
{
    return jacobi_impl<double>(T, ldt, V, ldv, n, tol, nu, max_sweeps, max_rounds, sweeps, rotations, hist,
                               stream, cfg);
}

mpj_status mpjacobi_jacobi_f32(float *T, int64_t ldt, float *V, int64_t ldv, int64_t n, double tol,
                               double nu, int max_sweeps, int64_t max_rounds, int *sweeps,
                               long long *rotations, double *hist, void *stream, const mpj_config *cfg)
{
    return jacobi_impl<float>(T, ldt, V, ldv, n, tol, nu, max_sweeps, max_rounds, sweeps, rotations, hist,
                              stream, cfg);
}

mpj_status mpjacobi_orth(const double *Z, double *Q, int64_t n, void *stream)
{
    g_err.clear();
    if (n < 1 || !Z || !Q) { set_error("invalid argument"); return MPJ_ERR_INVALID; }
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    void *ws = nullptr;
    MPJ_CK(cudaMallocAsync(&ws, orth_workspace(n), cx.st));
    mpj_status s = orth_cgs2(Z, n, Q, n, n, n, ws, cx.st);
    cudaFreeAsync(ws, cx.st);
    mpj_status c = cx.close();
    return s != MPJ_OK ? s : c;
}

mpj_status mpjacobi_orth_series(const double *Z, double *Q, int64_t n, void *stream)
{
    g_err.clear();
    if (n < 1 || !Z || !Q) { set_error("invalid argument"); return MPJ_ERR_INVALID; }
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    mpj_status s = orth_series(Z, n, Q, n, n, cx.st);
    if (s == MPJ_ERR_NOCONV) set_error("orth_series: ||Z^T Z - I||_F > 1e-4");
    mpj_status c = cx.close();
    return s != MPJ_OK ? s : c;
}

mpj_status mpjacobi_orth_householder(const double *Z, double *Q, int64_t n, void *stream)
{
    g_err.clear();
    if (n < 1 || !Z || !Q) { set_error("invalid argument"); return MPJ_ERR_INVALID; }
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    void *ws = nullptr;
    MPJ_CK(cudaMallocAsync(&ws, hqr_workspace(n, n), cx.st));
    mpj_status s = orth_householder(Z, n, Q, n, n, n, ws, cx.st);
    cudaFreeAsync(ws, cx.st);
    mpj_status c = cx.close();
    return s != MPJ_OK ? s : c;
}

mpj_status mpjacobi_precond(const double *A, const double *Q, double *T, int64_t n, void *stream)
{
    g_err.clear();
    if (n < 1 || !A || !Q || !T) { set_error("invalid argument"); return MPJ_ERR_INVALID; }
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    double *W = nullptr;
    MPJ_CK(cudaMallocAsync(&W, (size_t)n * n * sizeof(double), cx.st));
    launch_dgemm(false, false, n, n, n, 1.0, A, n, Q, n, 0.0, W, n, cx.st);
    launch_dgemm(true, false, n, n, n, 1.0, Q, n, W, n, 0.0, T, n, cx.st, nullptr, 0, true);
    launch_symmetrize_inplace(T, n, (int)n, cx.st, true);
    cudaFreeAsync(W, cx.st);
    return cx.close();
}

mpj_status mpjacobi_dgemm(int transa, const double *A, const double *B, double *C, int64_t m, int64_t n,
                          int64_t k, void *stream)
{
    g_err.clear();
    if (m < 0 || n < 0 || k < 0 || !A || !B || !C) { set_error("invalid argument"); return MPJ_ERR_INVALID; }
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    const size_t se = dgemm_scratch_elems(m, n);
    double *scr = nullptr;
    MPJ_CK(cudaMallocAsync(&scr, se * sizeof(double), cx.st));
    launch_dgemm(transa != 0, false, m, n, k, 1.0, A, transa ? k : m, B, k, 0.0, C, m, cx.st, scr, se);
    cudaFreeAsync(scr, cx.st);
    return cx.close();
}

}  // extern "C"

// ---------------------------------------------------------------------------
// multi-GPU entry point (kernels in k_mg.cu)
mpj_status mpjacobi_eig_mg(const double *A, int64_t n, int64_t lda, double *Lambda, double *V, int64_t ldv,
                           int *sweeps, const void *nccl_id, int rank, int nranks, int emulate_ranks, void *stream,
                           const mpj_config *cfg_in, mpj_report *rep)
{
    using namespace mpj;
    set_error("");
    const int G = nccl_id ? nranks : std::max(1, emulate_ranks);
    if (n < 1 || lda < n || ldv < n || !A || !Lambda || !V || G < 1 || (nccl_id && (rank < 0 || rank >= nranks))) {
        set_error("mpjacobi_eig_mg: invalid argument");
        return MPJ_ERR_INVALID;
    }
    mpj_config cfg;
    if (cfg_in) cfg = *cfg_in; else mpj_config_default_eig(&cfg);
    if (cfg.block_b != 0 && cfg.block_b != 32) { set_error("mpjacobi_eig_mg: block_b must be 32"); return MPJ_ERR_INVALID; }
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    const long long l0 = mpjacobi_launch_count();
    Timer t_all(cx.st);
    mpj_report r;
    std::memset(&r, 0, sizeof(r));
    mpj_status s = mg_eig(true, A, n, lda, Lambda, V, ldv, sweeps, nccl_id, rank, nranks, emulate_ranks, cx.st, cfg,
                          r, cx.h_pin);
    r.t_total = t_all.stop();
    r.launches = mpjacobi_launch_count() - l0;
    if (rep) *rep = r;
    mpj_status c = cx.close();
    return s != MPJ_OK ? s : c;
}

// SVD entry points (kernels in k_svd.cu)
// ---------------------------------------------------------------------------
extern "C" {
size_t mpjacobi_svd_workspace(int64_t m, int64_t n, const mpj_config *)
{
    if (m < 1 || n < 1 || m < n) return 0;
    return mpj::svd_workspace(m, n);
}

static mpj_status svd_impl(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U,
                           int64_t ldu, double *V, int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes,
                           void *stream, const mpj_config *cfg_in, mpj_report *rep, const float *Zin, float *Zout,
                           int64_t ldz)
{
    using namespace mpj;
    set_error("");
    if (n < 1 || m < n || lda < m || ldu < m || ldv < n || !A || !Sigma || !U || !V || ((Zin || Zout) && ldz < n)) {
        set_error("mpjacobi_svd: need m >= n >= 1, lda, ldu >= m, ldv >= n (ldz >= n), non-NULL buffers");
        return MPJ_ERR_INVALID;
    }
    mpj_config cfg;
    if (cfg_in) cfg = *cfg_in; else mpj_config_default_svd(&cfg);
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    const long long l0 = mpjacobi_launch_count();
    Timer t_all(cx.st);
    mpj_report r;
    std::memset(&r, 0, sizeof(r));
    const bool a_dev = is_device_ptr(A);
    const bool out_dev = is_device_ptr(U) && is_device_ptr(V) && is_device_ptr(Sigma);
    mpj_status s = svd_run(A, m, n, lda, Sigma, U, ldu, V, ldv, sweeps, workspace, ws_bytes, cx.st, cfg, r,
                           cx.h_pin, a_dev, out_dev, Zin, is_device_ptr(Zin), Zout, is_device_ptr(Zout), ldz);
    r.t_total = t_all.stop();
    r.launches = mpjacobi_launch_count() - l0;
    if (rep) *rep = r;
    mpj_status c = cx.close();
    return s != MPJ_OK ? s : c;
}

mpj_status mpjacobi_svd(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U, int64_t ldu,
                        double *V, int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes, void *stream,
                        const mpj_config *cfg, mpj_report *rep)
{
    return svd_impl(A, m, n, lda, Sigma, U, ldu, V, ldv, sweeps, workspace, ws_bytes, stream, cfg, rep, nullptr,
                    nullptr, 0);
}

mpj_status mpjacobi_svd_mg(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U,
                           int64_t ldu, double *V, int64_t ldv, int *sweeps, const void *nccl_id, int rank,
                           int nranks, int emulate_ranks, void *stream, const mpj_config *cfg_in, mpj_report *rep)
{
    using namespace mpj;
    set_error("");
    const int G = nccl_id ? nranks : std::max(1, emulate_ranks);
    if (n < 1 || m < n || lda < m || ldu < m || ldv < n || !A || !Sigma || !U || !V || G < 1 ||
        (nccl_id && (rank < 0 || rank >= nranks)) || !is_device_ptr(U) || !is_device_ptr(V) ||
        !is_device_ptr(Sigma)) {
        set_error("mpjacobi_svd_mg: need m >= n >= 1, lda, ldu >= m, ldv >= n, DEVICE Sigma / U / V");
        return MPJ_ERR_INVALID;
    }
    mpj_config cfg;
    if (cfg_in) cfg = *cfg_in; else mpj_config_default_svd(&cfg);
    Ctx cx;
    MPJ_TRY(cx.open(stream));
    const long long l0 = mpjacobi_launch_count();
    Timer t_all(cx.st);
    mpj_report r;
    std::memset(&r, 0, sizeof(r));
    mpj_status s = svd_mg_run(A, m, n, lda, Sigma, U, ldu, V, ldv, sweeps, nccl_id, rank, nranks, emulate_ranks,
                              cx.st, cfg, r, cx.h_pin);
    r.t_total = t_all.stop();
    r.launches = mpjacobi_launch_count() - l0;
    if (rep) *rep = r;
    mpj_status c = cx.close();
    return s != MPJ_OK ? s : c;
}

mpj_status mpjacobi_svd_z(const double *A, int64_t m, int64_t n, int64_t lda, const float *Z_in, float *Z_out,
                          int64_t ldz, double *Sigma, double *U, int64_t ldu, double *V, int64_t ldv, int *sweeps,
                          void *workspace, size_t ws_bytes, void *stream, const mpj_config *cfg, mpj_report *rep)
{
    return svd_impl(A, m, n, lda, Sigma, U, ldu, V, ldv, sweeps, workspace, ws_bytes, stream, cfg, rep, Z_in, Z_out,
                    ldz);
}
}
