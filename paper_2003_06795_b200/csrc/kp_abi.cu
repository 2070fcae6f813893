// C-ABI entry points of libkp.so (declared in include/kp_abi.h): validation,
// config-space enumeration, family dispatch, the timing loop (K4), the
// per-problem sweep, and runtime selection through the generated
// decision-tree headers (K5).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kp_internal.cuh"
#include "simt_registry.h"
#include "tc_registry.h"
#include "skinny_registry.h"
#include "generated/selectors.h"

namespace kp {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

kp_status fail(kp_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

void note_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

kp_status check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return KP_OK;
    return fail(KP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------- K1 scheduling --
static std::atomic<int> g_schedule{1};
int simt_schedule() { return g_schedule.load(std::memory_order_relaxed); }

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cached[dev] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 1;
    }
    return cached[dev];
}

kp_status sk_reserve(uint32_t n, SkFlags* out) {
    static std::mutex mu;
    static uint32_t* rings[64] = {nullptr};
    static uint32_t next_slot[64] = {0};
    static uint32_t next_epoch[64] = {0};
    if (n == 0 || n > KP_SK_RING / 4) return fail(KP_ERR_UNSUPPORTED, "stream-K grid too large");
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
        return fail(KP_ERR_CUDA, "stream-K: no current device");
    std::lock_guard<std::mutex> lock(mu);
    if (!rings[dev]) {
        void* ptr = nullptr;
        if (cudaMalloc(&ptr, KP_SK_RING * sizeof(uint32_t)) != cudaSuccess)
            return check_launch("stream-K flag ring cudaMalloc");
        if (cudaMemset(ptr, 0, KP_SK_RING * sizeof(uint32_t)) != cudaSuccess)
            return check_launch("stream-K flag ring cudaMemset");
        rings[dev] = static_cast<uint32_t*>(ptr);
    }
    if (++next_epoch[dev] == 0) ++next_epoch[dev];  // 0 is the ring's initial value
    out->flags = rings[dev];
    out->base = next_slot[dev];
    out->epoch = next_epoch[dev];
    next_slot[dev] = (next_slot[dev] + n) & KP_SK_RING_MASK;
    return KP_OK;
}

// ---------------------------------------------------------- config space --
// Canonical order of dataset.all_configs() (reference dataset.py:119-126):
// lexicographic over (acc, row_tile, col_tile, (wg_rows, wg_cols)).
static const uint32_t kTiles[4] = {1, 2, 4, 8};
static const uint32_t kWorkGroups[10][2] = {{1, 64}, {1, 128}, {8, 8},  {8, 16}, {8, 32},
                                            {16, 8}, {16, 16}, {32, 8}, {64, 1}, {128, 1}};

static int tile_index(uint32_t v) {
    for (int i = 0; i < 4; ++i)
        if (kTiles[i] == v) return i;
    return -1;
}
static int wg_index(uint32_t r, uint32_t c) {
    for (int i = 0; i < 10; ++i)
        if (kWorkGroups[i][0] == r && kWorkGroups[i][1] == c) return i;
    return -1;
}

static bool paper_domain(const kp_config& c) {
    return tile_index(c.acc) >= 0 && tile_index(c.row_tile) >= 0 && tile_index(c.col_tile) >= 0 &&
           wg_index(c.wg_rows, c.wg_cols) >= 0;
}

static kp_config paper_config(int idx) {
    const int wg = idx % 10, ct = (idx / 10) % 4, rt = (idx / 40) % 4, acc = idx / 160;
    return kp_config{kTiles[acc], kTiles[rt], kTiles[ct], kWorkGroups[wg][0], kWorkGroups[wg][1]};
}

// ------------------------------------------------------------ validation --
static kp_status to_problem(const kp_gemm_desc* d, const void* A, const void* B, float* C,
                            GemmProblem* g) {
    if (!d) return fail(KP_ERR_INVALID_ARG, "null gemm descriptor");
    if (!A || !B || !C) return fail(KP_ERR_INVALID_ARG, "null operand pointer");
    if (d->batch < 1 || d->m < 1 || d->k < 1 || d->n < 1) {
        char buf[160];
        snprintf(buf, sizeof buf, "problem dims must be >= 1, got batch=%lld m=%lld k=%lld n=%lld",
                 (long long)d->batch, (long long)d->m, (long long)d->k, (long long)d->n);
        return fail(KP_ERR_BAD_SHAPE, buf);
    }
    if (d->m > 0x7fffffffLL || d->n > 0x7fffffffLL || d->k > 0x7fffffffLL)
        return fail(KP_ERR_BAD_SHAPE, "m, k, n must fit in int32");
    const bool ta = d->trans_a != 0, tb = d->trans_b != 0;
    if (d->lda < (ta ? d->m : d->k)) return fail(KP_ERR_BAD_SHAPE, "lda too small");
    if (d->ldb < (tb ? d->k : d->n)) return fail(KP_ERR_BAD_SHAPE, "ldb too small");
    if (d->ldc < d->n) return fail(KP_ERR_BAD_SHAPE, "ldc too small");
    if (d->batch > 1 && (d->stride_a < 0 || d->stride_b < 0 || d->stride_c < d->m * d->ldc))
        return fail(KP_ERR_BAD_SHAPE, "bad batch strides (C batches must not overlap)");
    g->batch = d->batch; g->m = d->m; g->n = d->n; g->k = d->k;
    g->ta = ta; g->tb = tb;
    g->lda = d->lda; g->ldb = d->ldb; g->ldc = d->ldc;
    g->sa = d->batch > 1 ? d->stride_a : 0;
    g->sb = d->batch > 1 ? d->stride_b : 0;
    g->sc = d->batch > 1 ? d->stride_c : 0;
    g->alpha = d->alpha; g->beta = d->beta;
    g->A = A; g->B = B; g->C = C;
    return KP_OK;
}

#ifdef KP_LEAN
// Lean library (the paper's deployment build): only the kernels named by the
// compiled selectors exist; generated/simt_lean.cu provides the dispatch.
namespace simt {
kp_status lean_dispatch(const kp_config& c, int layout, const GemmProblem& g, cudaStream_t s);
}
#else
static const simt::LaunchFn kSimt[16] = {
    simt::KP_SIMT_FN(1, 1), simt::KP_SIMT_FN(1, 2), simt::KP_SIMT_FN(1, 4), simt::KP_SIMT_FN(1, 8),
    simt::KP_SIMT_FN(2, 1), simt::KP_SIMT_FN(2, 2), simt::KP_SIMT_FN(2, 4), simt::KP_SIMT_FN(2, 8),
    simt::KP_SIMT_FN(4, 1), simt::KP_SIMT_FN(4, 2), simt::KP_SIMT_FN(4, 4), simt::KP_SIMT_FN(4, 8),
    simt::KP_SIMT_FN(8, 1), simt::KP_SIMT_FN(8, 2), simt::KP_SIMT_FN(8, 4), simt::KP_SIMT_FN(8, 8),
};
#endif

static kp_status valid_config(kp_family fam, const kp_config& c) {
    if (fam == KP_F32_SIMT) {
        if (!paper_domain(c)) {
            char buf[160];
            snprintf(buf, sizeof buf, "config (%u,%u,%u,%u,%u) outside the 640-point domain", c.acc,
                     c.row_tile, c.col_tile, c.wg_rows, c.wg_cols);
            return fail(KP_ERR_INVALID_CONFIG, buf);
        }
        return KP_OK;
    }
    if (fam == KP_TF32_TC || fam == KP_BF16_TC) return tc::valid(fam, c);
    return fail(KP_ERR_INVALID_ARG, "unknown kernel family");
}

// The all-zero config names the small-M path (KP_SKINNY_CONFIG in kp_abi.h).
static bool is_skinny(const kp_config& c) {
    return c.acc == 0 && c.row_tile == 0 && c.col_tile == 0 && c.wg_rows == 0 && c.wg_cols == 0;
}

static kp_status run(kp_family fam, const kp_config& c, const GemmProblem& g, cudaStream_t s) {
    if (is_skinny(c)) return skinny::launch(fam, g, s);
    if (fam == KP_F32_SIMT) {
        const int layout = (g.ta ? 2 : 0) + (g.tb ? 1 : 0);
#ifdef KP_LEAN
        return simt::lean_dispatch(c, layout, g, s);
#else
        return kSimt[tile_index(c.acc) * 4 + tile_index(c.row_tile)](int(c.col_tile), layout, g,
                                                                      int(c.wg_rows), int(c.wg_cols), s);
#endif
    }
    return tc::launch(fam, c, g, s);
}

// ---------------------------------------------------------------- timing --
struct EventPool {
    std::vector<cudaEvent_t> ev;
    ~EventPool() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    kp_status ensure(size_t n) {
        while (ev.size() < n) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return check_launch("cudaEventCreate");
            ev.push_back(e);
        }
        return KP_OK;
    }
};
static thread_local EventPool g_events;

static kp_status time_one(kp_family fam, const kp_config& c, const GemmProblem& g, int warmup,
                          int reps, double min_sample_ns, double max_cell_ns, double* out,
                          cudaStream_t s, double hopeless_ns = 0.0) {
    if (reps < 1) return fail(KP_ERR_INVALID_ARG, "reps must be >= 1");
    kp_status st;
    if ((st = g_events.ensure(2 * size_t(reps) + 2)) != KP_OK) return st;
    cudaEvent_t* ev = g_events.ev.data();
    // one timed launch sizes the samples and doubles as the cold launch (its
    // first-launch costs only make the sizing conservative)
    cudaEventRecord(ev[0], s);
    if ((st = run(fam, c, g, s)) != KP_OK) return st;
    cudaEventRecord(ev[1], s);
    if (cudaEventSynchronize(ev[1]) != cudaSuccess) return check_launch("warm-up sync");
    float one_ms = 0.f;
    cudaEventElapsedTime(&one_ms, ev[0], ev[1]);
    const double one_ns = std::max(1.0, double(one_ms) * 1e6);
    if (hopeless_ns > 0.0 && one_ns > hopeless_ns) {  // sweep: far off the best so far
        *out = one_ns;
        return KP_OK;
    }
    int nreps = reps;
    bool budget_hit = false;
    if (max_cell_ns > 0.0 && one_ns * reps > max_cell_ns) {
        nreps = std::max(1, int(max_cell_ns / one_ns));
        budget_hit = true;
    }
    if (!budget_hit)
        for (int w = 1; w < warmup; ++w)
            if ((st = run(fam, c, g, s)) != KP_OK) return st;
    const int inner = int(std::min(4096.0, std::max(1.0, std::ceil(min_sample_ns / one_ns))));
    for (int r = 0; r < nreps; ++r) {
        cudaEventRecord(ev[2 + 2 * r], s);
        for (int i = 0; i < inner; ++i)
            if ((st = run(fam, c, g, s)) != KP_OK) return st;
        cudaEventRecord(ev[3 + 2 * r], s);
    }
    if (cudaEventSynchronize(ev[1 + 2 * nreps]) != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        return fail(KP_ERR_CUDA, std::string("timing sync: ") + cudaGetErrorString(e));
    }
    std::vector<double> per;
    per.reserve(nreps);
    for (int r = 0; r < nreps; ++r) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[2 + 2 * r], ev[3 + 2 * r]);
        per.push_back(double(ms) * 1e6 / inner);
    }
    std::sort(per.begin(), per.end());
    *out = (nreps % 2) ? per[nreps / 2] : 0.5 * (per[nreps / 2 - 1] + per[nreps / 2]);
    return KP_OK;
}

}  // namespace kp

using namespace kp;

// ================================================================ C ABI ===
extern "C" {

int32_t kp_abi_version(void) { return KP_ABI_VERSION; }

int32_t kp_num_configs(kp_family family) {
    if (family == KP_F32_SIMT) return 640;
    if (family == KP_TF32_TC || family == KP_BF16_TC) return tc::num_configs(family);
    return 0;
}

kp_status kp_config_at(kp_family family, int32_t index, kp_config* out) {
    if (!out) return fail(KP_ERR_INVALID_ARG, "null output");
    if (index < 0 || index >= kp_num_configs(family))
        return fail(KP_ERR_INVALID_ARG, "config index out of range");
    if (family == KP_F32_SIMT) {
        *out = paper_config(index);
        return KP_OK;
    }
    return tc::config_at(family, index, out);
}

kp_status kp_config_valid(kp_family family, kp_config cfg) { return valid_config(family, cfg); }

int32_t kp_set_schedule(int32_t mode) {
    if (mode < 0 || mode > 2) return -1;
    return g_schedule.exchange(mode);
}

int32_t kp_set_tc_split(int32_t mode) { return tc::set_split_mode(mode); }

int32_t kp_set_skinny(int32_t mode) { return skinny::set_mode(mode); }

kp_status kp_gemm_skinny(kp_family family, const kp_gemm_desc* desc, const void* A,
                         const void* B, float* C, void* stream) {
    kp_status st;
    GemmProblem g;
    if ((st = to_problem(desc, A, B, C, &g)) != KP_OK) return st;
    return skinny::launch(family, g, static_cast<cudaStream_t>(stream));
}

kp_status kp_gemm(kp_family family, kp_config cfg, const kp_gemm_desc* desc, const void* A,
                  const void* B, float* C, void* stream) {
    kp_status st;
    if (!is_skinny(cfg) && (st = valid_config(family, cfg)) != KP_OK) return st;
    GemmProblem g;
    if ((st = to_problem(desc, A, B, C, &g)) != KP_OK) return st;
    return run(family, cfg, g, static_cast<cudaStream_t>(stream));
}

kp_status kp_gemm_time(kp_family family, kp_config cfg, const kp_gemm_desc* desc, const void* A,
                       const void* B, float* C, int32_t warmup, int32_t reps, double min_sample_ns,
                       double max_cell_ns, double* runtime_ns, void* stream) {
    kp_status st;
    if (!runtime_ns) return fail(KP_ERR_INVALID_ARG, "null runtime output");
    if (!is_skinny(cfg) && (st = valid_config(family, cfg)) != KP_OK) return st;
    GemmProblem g;
    if ((st = to_problem(desc, A, B, C, &g)) != KP_OK) return st;
    return time_one(family, cfg, g, warmup, reps, min_sample_ns, max_cell_ns, runtime_ns,
                    static_cast<cudaStream_t>(stream));
}

kp_status kp_sweep_problem_ex(kp_family family, const kp_config* cfgs, int32_t n_cfgs,
                              const kp_gemm_desc* desc, const void* A, const void* B, float* C,
                              int32_t warmup, int32_t reps, double min_sample_ns,
                              double max_cell_ns, int32_t flags, double* runtime_ns, void* stream) {
    if (!cfgs || !runtime_ns || n_cfgs < 0) return fail(KP_ERR_INVALID_ARG, "bad sweep arguments");
    if (flags & ~int32_t(KP_SWEEP_EARLY_EXIT)) return fail(KP_ERR_INVALID_ARG, "unknown sweep flags");
    kp_status st;
    GemmProblem g;
    if ((st = to_problem(desc, A, B, C, &g)) != KP_OK) return st;
    for (int32_t i = 0; i < n_cfgs; ++i)
        if (!is_skinny(cfgs[i]) && (st = valid_config(family, cfgs[i])) != KP_OK) return st;
    // With KP_SWEEP_EARLY_EXIT, a config whose first launch is both over 1 ms
    // and 8x the best median of this call so far keeps that single timing: it
    // normalises below 0.125 either way and the extra launches would dominate
    // the sweep. Callers timing only part of a problem's configs clear the
    // flag, so every cell gets the same statistic as in a whole-problem call.
    const bool early = (flags & KP_SWEEP_EARLY_EXIT) != 0;
    double best = 0.0;
    for (int32_t i = 0; i < n_cfgs; ++i) {
        const double hopeless = early && best > 0.0 ? std::max(1e6, 8.0 * best) : 0.0;
        st = time_one(family, cfgs[i], g, warmup, reps, min_sample_ns, max_cell_ns,
                      runtime_ns + i, static_cast<cudaStream_t>(stream), hopeless);
        if (st == KP_OK && (best == 0.0 || runtime_ns[i] < best)) best = runtime_ns[i];
        if (st != KP_OK) {
            char buf[96];
            snprintf(buf, sizeof buf, " [config #%d (%u,%u,%u,%u,%u)]", i, cfgs[i].acc,
                     cfgs[i].row_tile, cfgs[i].col_tile, cfgs[i].wg_rows, cfgs[i].wg_cols);
            g_last_error += buf;
            return st;
        }
    }
    return KP_OK;
}

kp_status kp_sweep_problem(kp_family family, const kp_config* cfgs, int32_t n_cfgs,
                           const kp_gemm_desc* desc, const void* A, const void* B, float* C,
                           int32_t warmup, int32_t reps, double min_sample_ns, double max_cell_ns,
                           double* runtime_ns, void* stream) {
    return kp_sweep_problem_ex(family, cfgs, n_cfgs, desc, A, B, C, warmup, reps, min_sample_ns,
                               max_cell_ns, KP_SWEEP_EARLY_EXIT, runtime_ns, stream);
}

kp_status kp_select_ex(kp_family family, int32_t trans_a, int32_t trans_b, int64_t batch,
                       int64_t m, int64_t k, int64_t n, kp_config* out) {
    if (!out) return fail(KP_ERR_INVALID_ARG, "null output");
    if (m < 1 || k < 1 || n < 1 || batch < 1) return fail(KP_ERR_BAD_SHAPE, "problem dims must be >= 1");
    // batch 1: the plain selector; batch > 1: the strided-batched selector
    // whose dataset batch is closest in log scale, else the plain one
    const KpSelectorEntry* best = nullptr;
    double best_d = 0.0;
    for (int i = 0; i < kp_num_selectors; ++i) {
        const KpSelectorEntry& e = kp_selectors[i];
        if (!e.fn || e.family != int(family) || e.trans_a != (trans_a != 0) ||
            e.trans_b != (trans_b != 0))
            continue;
        if ((batch == 1) != (e.batch == 1)) {
            if (batch == 1 || best) continue;  // plain problems never take a batched tree
            best = &e;                          // batched problem: plain tree as fallback
            best_d = 1e30;
            continue;
        }
        if (e.batch == batch) { best = &e; break; }  // exact (always so for batch 1)
        const double d = std::fabs(std::log(double(e.batch)) - std::log(double(batch)));
        if (!best || d < best_d) { best = &e; best_d = d; }
    }
    if (!best)
        return fail(KP_ERR_UNSUPPORTED, "no selector compiled in for this family / transpose variant");
    *out = best->fn(m, k, n);
    return KP_OK;
}

kp_status kp_select(kp_family family, int32_t trans_a, int32_t trans_b, int64_t m, int64_t k,
                    int64_t n, kp_config* out) {
    return kp_select_ex(family, trans_a, trans_b, 1, m, k, n, out);
}

kp_status kp_auto_config(kp_family family, int32_t trans_a, int32_t trans_b, int64_t batch,
                         int64_t m, int64_t k, int64_t n, kp_config* out) {
    if (!out) return fail(KP_ERR_INVALID_ARG, "null output");
    kp_status st = kp_select_ex(family, trans_a, trans_b, batch, m, k, n, out);
    if (st != KP_OK) return st;
    GemmProblem g{};
    g.batch = batch; g.m = m; g.k = k; g.n = n;
    if (skinny::eligible(family, g)) *out = kp_config{0, 0, 0, 0, 0};
    return KP_OK;
}

kp_status kp_gemm_auto(kp_family family, const kp_gemm_desc* desc, const void* A, const void* B,
                       float* C, void* stream, kp_config* chosen) {
    if (!desc) return fail(KP_ERR_INVALID_ARG, "null gemm descriptor");
    kp_config cfg;
    kp_status st = kp_select_ex(family, desc->trans_a, desc->trans_b, desc->batch, desc->m, desc->k,
                                desc->n, &cfg);
    if (st != KP_OK) return st;
    GemmProblem g;
    if ((st = to_problem(desc, A, B, C, &g)) != KP_OK) return st;
    if (skinny::eligible(family, g)) {  // small-M (FC) shapes: the HBM-streaming path
        if (chosen) *chosen = kp_config{0, 0, 0, 0, 0};
        return skinny::launch(family, g, static_cast<cudaStream_t>(stream));
    }
    if (chosen) *chosen = cfg;
    return kp_gemm(family, cfg, desc, A, B, C, stream);
}

const char* kp_status_string(kp_status status) {
    switch (status) {
        case KP_OK: return "ok";
        case KP_ERR_INVALID_CONFIG: return "invalid config";
        case KP_ERR_BAD_SHAPE: return "bad shape";
        case KP_ERR_ALIGNMENT: return "alignment";
        case KP_ERR_UNSUPPORTED: return "unsupported";
        case KP_ERR_CUDA: return "cuda error";
        case KP_ERR_INVALID_ARG: return "invalid argument";
    }
    return "unknown status";
}

const char* kp_last_error(void) { return g_last_error.c_str(); }

int64_t kp_launch_count(void) { return g_launches.load(); }

kp_status kp_device_info(int32_t device, int32_t* sm_count, int32_t* sm_clock_khz, int32_t* cc) {
    int v = 0, major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
        return check_launch("cudaDeviceGetAttribute");
    if (sm_count) *sm_count = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, device) != cudaSuccess)
        return check_launch("cudaDeviceGetAttribute");
    if (sm_clock_khz) *sm_clock_khz = v;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (cc) *cc = major * 10 + minor;
    return KP_OK;
}

}  // extern "C"
