// lk_api.cu — host side of the C-ABI (include/lanekit_b200.h): context,
// device buffers, host-built exact tables, CUDA-graph replay, hooks.
//
// Host code here is compiled with -ffp-contract=off so the tables it builds
// with glibc's exp (the same libm the reference links) are bit-identical to
// what the reference computes inline (preprocess.hpp:47-50).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <tuple>
#include <random>
#include <string>
#include <vector>

#include "../../include/lanekit_b200.h"
#include "lk_kernels.h"

using lkg::Dev;
using lkg::FrameAux;
using lkg::LaunchPlan;

namespace {

thread_local std::string g_err;

lk_status fail(lk_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define CU(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(LK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

const char* kStageNames[12] = {
    "block statistics", "left disparity",      "right disparity",
    "consistency check", "v-disparity accumulation", "road path extraction",
    "road profile fit",  "road mask",           "bilateral smoothing",
    "edge detection",    "vanishing point estimation", "lane detection",
};  // pipeline.hpp:101-116

// config.hpp:124-152 (same checks, same messages)
const char* config_problem(const lk_config& c) {
    if (c.rho < 1) return "rho must be >= 1";
    if (c.tau < 0) return "tau must be >= 0";
    if (c.d_max < 1) return "d_max must be >= 1";
    if (c.tr_lrc < 0) return "tr_lrc must be >= 0";
    if (!(c.sigma_floor > 0)) return "sigma_floor must be > 0";
    if (c.lambda_y < 0) return "lambda_y must be >= 0";
    if (!(c.tr_y > 0)) return "tr_y must be > 0";
    if (!(c.eps_y > 0 && c.eps_y <= 1)) return "eps_y must be in (0, 1]";
    if (c.varpi < 0) return "varpi must be >= 0";
    if (!(c.sigma_s > 0)) return "sigma_s must be > 0";
    if (!(c.sigma_r > 0)) return "sigma_r must be > 0";
    if (c.bf_window < 1 || c.bf_window % 2 == 0) return "bf_window must be odd and >= 1";
    if (c.sobel_threshold < 0) return "sobel_threshold must be >= 0";
    if (c.chi < 0) return "chi must be >= 0";
    if (!(c.rho_vote > 0)) return "rho_vote must be > 0";
    if (c.lambda_x < 0) return "lambda_x must be >= 0";
    if (!(c.tr_x > 0)) return "tr_x must be > 0";
    if (!(c.eps_x > 0 && c.eps_x <= 1)) return "eps_x must be in (0, 1]";
    if (!(c.sigma_g > 0)) return "sigma_g must be > 0";
    if (c.nu < 0) return "nu must be >= 0";
    if (c.varsigma < 0) return "varsigma must be >= 0";
    if (c.lambda_g < 0) return "lambda_g must be >= 0";
    if (c.xi < 0) return "xi must be >= 0";
    if (!std::isnan(c.tr_lpv) && !(c.tr_lpv < 0)) return "tr_lpv must be negative (or auto)";
    if (c.min_lane_sep < 0) return "min_lane_sep must be >= 0";
    if (c.threads < 1) return "threads must be >= 1";
    return nullptr;
}

constexpr int kMaxIter = 200;  // pipeline.hpp:198, 244
constexpr int kMaxBranches = 16;      // concurrent frame ranges (streams) per batch
constexpr int kMinBranchFrames = 16;  // smallest range worth a branch
constexpr int kH2dChunksDefault = 12; // host-fed batches: copy/compute pipeline depth
constexpr int kBranchesDefault = 8;   // device-resident batches: concurrent frame ranges

}  // namespace

struct lk_ctx {
    int device = 0;
    uint32_t flags = 0;
    int max_batch = 0;
    lk_config cfg{};
    Dev d{};
    LaunchPlan lp{};
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[13] = {};
    int branches = 1;
    cudaStream_t side[kMaxBranches - 1] = {};
    cudaEvent_t fork = nullptr, join[kMaxBranches - 1] = {};
    cudaEvent_t copied[kMaxBranches] = {};   // host-fed pipeline: chunk k's inputs are resident
    int h2d_chunks = kMaxBranches;           // host-fed batches: copy/compute pipeline depth
    std::map<std::tuple<long, int, int>, cudaGraphExec_t> range_graphs;  // (f0, n, timed|stereo)
    int timed_frames = 0;
    bool timed = false;
    std::vector<void*> allocs;
    std::map<int, cudaGraphExec_t> graphs;
    uint8_t* in_grey = nullptr;  // the (left) grey
    uint8_t* in_disp = nullptr;  // the disparity (stereo: written by stage 4)
    uint8_t* in_right = nullptr; // stereo contexts: the right grey
    bool run_stereo = false;     // the batch being enqueued runs stages 1-4 first
    int slot = 0;                // input slot the captured graphs read (streaming API)
    // streaming API (lk_submit_batch / lk_wait_batch): two input slots
    uint8_t* slot_grey[2] = {};
    uint8_t* slot_disp[2] = {};
    uint8_t* slot_right[2] = {};  // stereo submits: the right grey (slot 0 = in_right)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t slot_copied[2] = {}, slot_free[2] = {}, slot_done[2] = {};
    struct Pending {
        int slot, n;
        lk_frame_report* reports;
    };
    Pending pending[2];
    int n_pending = 0, next_slot = 0;
    bool last_stereo = false;
    int last_n = 0;
    // Road-row copy of streamed grey (lk_submit_batch, fast path): a front pass
    // (stages 5-7 of the batch into scratch buffers, on front_stream) yields
    // each frame's first grey row read downstream; only rows from the batch's
    // smallest such row down are copied. h2d_dma counts every H2D byte moved.
    bool road_copy = true;
    bool front_ready = false;
    Dev front{};
    LaunchPlan front_lp{};
    cudaStream_t front_stream = nullptr;
    cudaEvent_t front_done[kMaxBranches] = {};
    cudaEvent_t disp_copied[kMaxBranches] = {};
    int road_chunks = 2;  // frame chunks of the road-row copy (LK_ROAD_CHUNKS)
    double road_saved = 1.0;  // fraction of the grey the last road-row copy skipped
    unsigned road_probe = 0;
    int* d_rows = nullptr;  // [max_batch] first grey row per frame (H: none)
    int* h_rows = nullptr;  // pinned copy
    unsigned long long h2d_dma = 0;

    template <typename T>
    lk_status alloc(T** p, size_t count) {
        void* q = nullptr;
        const size_t bytes = count * sizeof(T);
        if (bytes) {
            cudaError_t e = cudaMalloc(&q, bytes);
            if (e != cudaSuccess)
                return fail(LK_ERR_CUDA, "cudaMalloc(" + std::to_string(bytes) +
                                             " B): " + cudaGetErrorString(e));
            allocs.push_back(q);
        }
        *p = static_cast<T*>(q);
        return LK_OK;
    }
};

extern "C" {

int lk_abi_version(void) { return LK_ABI_VERSION; }

const char* lk_last_error(void) { return g_err.c_str(); }

const char* lk_stage_name(int stage) {
    return (stage >= 1 && stage <= 12) ? kStageNames[stage - 1] : "";
}

void lk_config_default(lk_config* c) {  // config.hpp:16-46
    std::memset(c, 0, sizeof *c);
    c->rho = 3;
    c->tau = 1;
    c->d_max = 64;
    c->tr_lrc = 3;
    c->sigma_floor = 1e-4;
    c->lambda_y = 30.0;
    c->tr_y = 4.0;
    c->eps_y = 0.99;
    c->varpi = 3.0;
    c->sigma_s = 300.0;
    c->sigma_r = 0.3;
    c->bf_window = 11;
    c->sobel_threshold = 100.0;
    c->chi = 25;
    c->rho_vote = 1.0;
    c->lambda_x = 10.0;
    c->tr_x = 16.0;
    c->eps_x = 0.99;
    c->sigma_g = 3.5;
    c->nu = 1;
    c->varsigma = 3;
    c->lambda_g = 1.0;
    c->xi = 0.5;
    c->tr_lpv = std::numeric_limits<double>::quiet_NaN();
    c->min_lane_sep = 20;
    c->rng_seed = 1;
    c->paper_sign = 0;
    c->threads = 1;
}

lk_status lk_validate_config(const lk_config* c) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null config");
    if (const char* m = config_problem(*c)) return fail(LK_ERR_CONFIG, std::string("config: ") + m);
    return LK_OK;
}

lk_status lk_frame_message(const lk_frame_report* rep, char* buf, size_t len) {
    if (!rep || !buf || !len) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    static const char* texts[] = {
        "",
        "empty input image",
        "v-disparity histogram is empty; no road surface evidence",
        "ransac: fewer points than the sample size",
        "ransac: no sample produced a fit",
        "road profile: singular V_py derivative at row ",
        "sobel: image smaller than the kernel",
        "vanishing-point accumulator is empty; no lane edge evidence",
        "m1: image smaller than the kernel",
        "stereo pair dimensions differ",
    };
    if (rep->status == 0) {
        buf[0] = 0;
        return LK_OK;
    }
    const int st = (int)rep->failed_stage, m = (int)rep->msg;
    std::string text = (m >= 0 && m <= 9) ? texts[m] : "unknown failure";
    if (m == LK_MSG_SINGULAR_VPY) text += std::to_string(rep->err_row);
    std::snprintf(buf, len, "stage %d (%s): %s", st, lk_stage_name(st), text.c_str());
    return LK_OK;
}

lk_status lk_create(lk_ctx** out, int device, const lk_config* cfg, int width, int height,
                    int max_batch, uint32_t flags) {
    if (!out || !cfg) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (lk_status s = lk_validate_config(cfg)) return s;
    if (width <= 0 || height <= 0)
        return fail(LK_ERR_INVALID_ARGUMENT, "stage 1 (block statistics): empty input image");
    if (width > 65535 || height > 32767)
        return fail(LK_ERR_INVALID_ARGUMENT, "frame dimensions exceed 65535 x 32767");
    if (max_batch < 1) return fail(LK_ERR_INVALID_ARGUMENT, "max_batch must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(LK_ERR_NO_DEVICE, "no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(LK_ERR_NO_DEVICE, "device index out of range");
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(LK_ERR_NO_DEVICE, std::string("lanekit_b200 needs sm_100 (Blackwell); got ") +
                                          prop.name);
    CU(cudaSetDevice(device));

    auto* c = new lk_ctx();
    c->device = device;
    c->flags = flags;
    c->max_batch = max_batch;
    c->cfg = *cfg;
    Dev& d = c->d;
    const int W = width, H = height, B = max_batch;
    d.W = W;
    d.H = H;
    d.d_max = cfg->d_max;
    d.D1 = cfg->d_max + 1;
    d.px = (size_t)W * H;
    d.ext_lo = -(int)std::llround(cfg->xi * W);          // vanish.hpp:24-26
    d.ext_cols = (int)std::llround((2 * cfg->xi + 1) * W);  // vanish.hpp:28-30
    d.rho = (cfg->bf_window - 1) / 2;                     // pipeline.hpp:220
    d.win = 2 * d.rho + 1;
    d.words_per_row = (W + 31) / 32;
    d.hooks = (flags & LK_FLAG_HOOKS) ? 1 : 0;
    d.lambda_y = cfg->lambda_y;
    d.tr_y = cfg->tr_y;
    d.eps_y = cfg->eps_y;
    d.varpi = cfg->varpi;
    d.rho_vote = cfg->rho_vote;
    d.lambda_x = cfg->lambda_x;
    d.tr_x = cfg->tr_x;
    d.eps_x = cfg->eps_x;
    d.sigma_g = cfg->sigma_g;
    d.lambda_g = cfg->lambda_g;
    d.tr_lpv = cfg->tr_lpv;
    d.chi = cfg->chi;
    d.nu = cfg->nu;
    d.varsigma = cfg->varsigma;
    d.min_lane_sep = cfg->min_lane_sep;
    d.paper_sign = cfg->paper_sign ? 1 : 0;
    d.max_iter = kMaxIter;
    for (int oi = 0; oi < 11; ++oi) {  // offsets {0, -1, 1, -2, 2, ...}: dp.hpp:43-51 scan order
        const int off = (oi & 1) ? -((oi + 1) >> 1) : (oi >> 1);
        d.upen[oi] = d.paper_sign ? cfg->lambda_x * off : cfg->lambda_x * std::abs(off);
        d.upk[oi] = d.upen[oi] < 1e8 && d.upen[oi] > -1e8 ? (int)d.upen[oi] * 16 + oi : 0;
    }
    {  // both selection paths are exact; the switch only trades a pass for a gather
        const char* e = std::getenv("LK_P99_L2_MIN");
        d.p99_l2_min = e ? (unsigned)std::strtoul(e, nullptr, 10) : 65536u;
    }
    if (d.ext_cols < 1) {
        delete c;
        return fail(LK_ERR_CONFIG, "extended column axis is empty");
    }
    if (flags & LK_FLAG_STEREO) {  // run_pipeline's stage-1 checks (pipeline.hpp:121-126)
        const char* why = nullptr;
        if (W <= 2 * cfg->rho || H <= 2 * cfg->rho)
            why = "stage 1 (block statistics): image smaller than the matching block";
        else if (cfg->rho < 1 || cfg->rho > 5)
            why = "stereo: block radius rho must be 1..5 on the GPU";
        else if (cfg->d_max > 255)
            why = "stereo: d_max must be <= 255 (u8 disparity maps)";
        if (why) {
            delete c;
            return fail(LK_ERR_INVALID_ARGUMENT, why);
        }
        d.stereo = 1;
        d.srho = cfg->rho;
        d.tau = cfg->tau;
        d.tr_lrc = cfg->tr_lrc;
        d.sigma_floor = cfg->sigma_floor;
    }
    const int C = d.ext_cols, D1 = d.D1;

    // ---- exact host tables (glibc exp, as the reference evaluates them)
    const int win = d.win, rho = d.rho;
    std::vector<double> ws((size_t)win * win), wr(256 * 256), val(256);
    const double inv_s2 = 1.0 / (cfg->sigma_s * cfg->sigma_s);  // preprocess.hpp:36-37
    const double inv_r2 = 1.0 / (cfg->sigma_r * cfg->sigma_r);
    for (int dj = -rho; dj <= rho; ++dj)
        for (int di = -rho; di <= rho; ++di) {
            const double ds = static_cast<double>(di) * di + static_cast<double>(dj) * dj;
            ws[(size_t)(dj + rho) * win + (di + rho)] = std::exp(-ds * inv_s2);
        }
    for (int k = 0; k < 256; ++k) val[k] = k / 255.0;  // image_io.hpp:147
    for (int kc = 0; kc < 256; ++kc)
        for (int kv = 0; kv < 256; ++kv) {
            const double dr = val[kv] - val[kc];
            wr[kc * 256 + kv] = std::exp(-dr * dr * inv_r2);
        }
    // smallest s with !(sqrt(s) < t): the edge test of preprocess.hpp:109
    // made sqrt-free and exact (sqrt is correctly rounded and monotone)
    {
        const double t = cfg->sobel_threshold / 255.0;
        auto pass = [&](double s) { return !(std::sqrt(s) < t); };
        uint64_t lo = 0, hi = 0x7ff0000000000000ULL;  // +0 .. +inf
        if (pass(0.0)) {
            d.sobel_s_star = 0.0;
        } else {
            while (hi - lo > 1) {
                const uint64_t mid = lo + (hi - lo) / 2;
                double m;
                std::memcpy(&m, &mid, 8);
                if (pass(m))
                    hi = mid;
                else
                    lo = mid;
            }
            std::memcpy(&d.sobel_s_star, &hi, 8);
        }
    }
    d.sobel_s_star_lo = (float)d.sobel_s_star;
    if ((double)d.sobel_s_star_lo > d.sobel_s_star)
        d.sobel_s_star_lo = std::nextafter(d.sobel_s_star_lo, -std::numeric_limits<float>::infinity());
    std::vector<uint64_t> rng((size_t)kMaxIter * 5);
    {
        std::mt19937_64 eng(cfg->rng_seed);  // ransac.hpp:44
        for (auto& x : rng) x = eng();
    }

    lk_status s = LK_OK;
    auto A = [&](auto** p, size_t n) {
        if (s == LK_OK) s = c->alloc(p, n);
    };
    double *d_ws, *d_wr, *d_val;
    float2* d_nt = nullptr;
    std::vector<float2> need_tab;
    uint64_t* d_rng;
    A(&d_ws, ws.size());
    A(&d_wr, wr.size());
    A(&d_val, val.size());
    A(&d_rng, rng.size());
    A(&c->in_grey, (size_t)B * d.px + 16);  // +16: k_refine_exact reads rows as whole words
    A(&c->in_disp, (size_t)B * d.px + 16);  // +16: k_vdisparity stages 16-byte aligned spans
    if (d.stereo) {
        A(&c->in_right, (size_t)B * d.px);
        A(&d.sat, (size_t)B * 4 * d.px);
        A(&d.mu_l, (size_t)B * d.px);
        A(&d.sig_l, (size_t)B * d.px);
        A(&d.mu_r, (size_t)B * d.px);
        A(&d.sig_r, (size_t)B * d.px);
        A(&d.disp_l, (size_t)B * d.px);
        A(&d.disp_r, (size_t)B * d.px);
    }
    A(&d.rep, (size_t)B);
    A(&d.aux, (size_t)B);
    A(&c->lp.vhistT, (size_t)B * H * D1);
    A(&d.vpath, (size_t)B * D1 * 2);
    A(&d.beta_inl, (size_t)B * D1 * 2);
    A(&d.vpy, (size_t)B * H);
    A(&d.vsing, (size_t)B * H);
    A(&d.fv, (size_t)B * H);
    A(&d.vpx, (size_t)B * H);
    A(&d.smoothed, (size_t)B * d.px);
    A(&d.ebits, (size_t)B * H * d.words_per_row);
    d.n_seg = (W + lkg::SB_TW - 1) / lkg::SB_TW;
    A(&d.seg_cnt, (size_t)B * H * d.n_seg);
    A(&d.seg_off, (size_t)B * H * d.n_seg);
    A(&d.row_off, (size_t)B * (H + 1));
    A(&d.e_uv, (size_t)B * d.px);
    A(&d.e_gx, (size_t)B * d.px);
    A(&d.e_gy, (size_t)B * d.px);
    A(&d.e_th, (size_t)B * d.px);
    A(&d.e_wg, (size_t)B * d.px);
    A(&d.e_col, (size_t)B * d.px);
    A(&d.uchoice, (size_t)B * H * C);
    A(&d.upath, (size_t)B * H * 2);
    A(&d.gamma_inl, (size_t)B * H * 2);
    A(&d.m1, (size_t)B * d.px);
    A(&d.p99hist, (size_t)B * 2048);
    A(&d.p99hist2, (size_t)B * 4096);
    A(&d.p99cand, (size_t)B * d.px);
    A(&d.energy, (size_t)B * C);
    A(&d.mrange, (size_t)B * H);
    A(&d.track_np, (size_t)B * C);
    A(&d.e_touch, (size_t)B * C);
    int sort_cap = 1;
    while (sort_cap < C / 2 + 2) sort_cap <<= 1;
    d.lane_cap = sort_cap;
    A(&d.lanes, (size_t)B * d.lane_cap);
    if (d.hooks) {
        A(&d.mask, (size_t)B * d.px);
        A(&d.gx, (size_t)B * d.px);
        A(&d.gy, (size_t)B * d.px);
        A(&d.mag, (size_t)B * d.px);
        A(&d.theta, (size_t)B * d.px);
        A(&d.acc, (size_t)B * H * C);
        A(&d.m0, (size_t)B * d.px);
        A(&d.polylines, (size_t)B * d.lane_cap * H);
    }
    if (s != LK_OK) {
        lk_destroy(c);
        return s;
    }
    d.ws = d_ws;
    d.wr = d_wr;
    d.val = d_val;
    d.rng = d_rng;
    d.grey = c->in_grey;
    d.disp = c->in_disp;
    d.right = c->in_right;
    d.disp_out = d.stereo ? c->in_disp : nullptr;
    if (!d.hooks) d.vchoice = nullptr;

    // ---- shared-memory plan
    LaunchPlan& lp = c->lp;
    const size_t vp_base = (size_t)2 * H * 8;
    lp.vpath_choice_smem = vp_base + (size_t)D1 * H <= 160 * 1024;
    lp.vpath_smem = vp_base + (lp.vpath_choice_smem ? (size_t)D1 * H : 0);
    if (!lp.vpath_choice_smem) A(&d.vchoice, (size_t)B * D1 * H);
    lp.vdisp_smem = lkg::vdisparity_smem(W, D1);
    lp.road_smem = (size_t)(8 * D1 + 2) * 4 + (size_t)4 * D1 * 8 + 16;  // tbuf: (K+1) rows
    lp.bf_smem = (size_t)(256 + win * win) * 8 +
                 (size_t)(lkg::BF_TH + 2 * rho) * (lkg::BF_TW + 2 * rho) + 16;
    {
        const size_t twh = lkg::BT_W + 10, thh = lkg::BT_H + 10, npx = twh * thh;
        const size_t tri = (size_t)lkg::BT_TRI_N * (lkg::BT_TRI_N + 1) / 2;
        const char* m = std::getenv("LK_BILATERAL_MODE");
        lp.bt_mode = m ? std::atoi(m) : 0;
        const bool table = lp.bt_mode == 0 || lp.bt_mode == 3;
        lp.bt_smem = (table ? tri * 8 : 0) + npx * 8 + npx * 4 + 2 * 256 * 4 + npx + 256 + 16;
        if (win == 11)
            for (int i = 0; i < 121; ++i) lp.ws.w[i] = ws[i];
    }
    // Certified fast front end (lk_fastpath.cu): throughput mode only (hooks
    // export exact maps), 11x11 window, and a weight range whose FP32 error
    // budget holds (exponent of the smallest weight <= 20; default 11.1).
    {
        const double xmax = 50.0 * inv_s2 + inv_r2;
        lp.fast_front = win == 11 && !d.hooks && !(flags & LK_FLAG_EXACT) && xmax <= 20.0 &&
                        lkg::prescreen_threads(W) <= 768 &&
                        lkg::prescreen_smem(W, lkg::prescreen_threads(W)) <= 200 * 1024;
        d.n_stile = ((W + lkg::SB_TW - 1) / lkg::SB_TW) * ((H + lkg::SB_TH - 1) / lkg::SB_TH);
        d.need_cap = d.n_stile * (lkg::SB_TW + 2) * (lkg::SB_TH + 2);  // every ring pixel of every tile
        lp.refine_ctas = 8;
        lp.decide_ctas = 32;
        // certified pre-screen constants (lk_fastpath.cu), each
        // rounded toward the safe side
        auto up = [](double x) {
            float y = (float)x;
            return (double)y < x ? std::nextafter(y, INFINITY) : y;
        };
        double wmin = 1.0;
        for (double w : ws) wmin = std::min(wmin, w);
        const double iw = 1.0 / wmin * (1.0 + 1e-12);
        lp.ps.kappa = up(inv_r2);
        lp.ps.inv_wmin = up(iw);
        lp.ps.ew = up(iw - 1.0);
        {  // sup over 0 < x <= 1 of (1 - exp(-kappa x^2)) / x; |f'| <= 2 kappa bounds the gap
            const double h = 1e-5;
            double fm = 0.0;
            for (double x = h; x <= 1.0 + h / 2; x += h)
                fm = std::max(fm, (1.0 - std::exp(-inv_r2 * x * x)) / x);
            lp.ps.fmax = up(fm + 2.0 * inv_r2 * h + 1e-9);
        }
        lp.ps.c1 = up(1.0 / (121.0 * 255.0));
        lp.ps.c2 = up(1.0 / (121.0 * 255.0 * 255.0));
        lp.ps.s_star_lo = d.sobel_s_star_lo;
        lp.fast_width = W;
        for (int j = 0; j < 11; ++j)
            for (int i = 0; i < 11; ++i)
                lp.nbf.S[j * 11 + i] = (float)(win == 11 ? ws[(size_t)j * 11 + i] : 0.0);
        need_tab.resize(511);
        for (int i = 0; i < 511; ++i) {
            const double dl = i - 255, r = std::exp(-(dl / 255.0) * (dl / 255.0) * inv_r2);
            need_tab[i] = make_float2((float)r, (float)(r * dl));
        }
        if (lp.fast_front) {
            A(&d.smoothed_f, (size_t)B * d.px);
            A(&d.pbits, (size_t)B * H * d.words_per_row);
            A(&d.fneed, (size_t)B * d.px);
            A(&d_nt, need_tab.size());
            A(&d.need, (size_t)B * d.need_cap);
            A(&d.need_cnt, (size_t)B);
            A(&d.ctile, (size_t)B * d.n_stile);
            A(&d.ctile_cnt, (size_t)B);
        }
    }
    // u-path DP shape: 512 threads (2 CTAs / SM) up to 4096 extended columns,
    // else 1024 threads; SP consecutive states per thread (0 = strided fallback)
    lp.upath_nt = C <= 512 * 8 ? 512 : 1024;
    {
        // vote columns staged in shared memory (2 B each): 8 K votes keep two
        // 512-thread CTAs per SM; a 1024-thread DP runs alone on its SM and
        // takes as many as fit (a hi-res frame has ~15 K; unstaged, the band
        // slide waits on a global load every stage)
        const size_t base = (size_t)(2 * C + 32) * 8 + (size_t)2 * C * 4 + (size_t)2 * H * 4 +
                            (size_t)lkg::BT_CHUNK * (2 * lkg::BT_SPAN + 1) + 8 +
                            (size_t)(H + 1) * 4 + 16;
        size_t cap = lkg::K4_VOTE_CAP;
        if (lp.upath_nt == 1024) {
            const size_t room = prop.sharedMemPerBlockOptin > base + 2048
                                    ? (prop.sharedMemPerBlockOptin - base - 2048) / 2 : 0;
            cap = std::max(cap, std::min(room, (size_t)32768) & ~(size_t)15);
        }
        d.vote_cap = (int)cap;
        lp.vanish_smem = base + cap * 2;
    }
    {
        // SP consecutive states per thread over NT/32 - 1 warps: the last warp
        // holds no states and slides the band counts alone (k_vanish's product
        // loop; measured 419 -> 382 us KITTI, 1348 -> 1093 us hi-res against
        // warp 0 sliding beside its DP). Without room for it, every warp.
        const int nt = lp.upath_nt;
        int sp = (C + nt - 33) / (nt - 32);
        if (sp == 7) sp = 8;
        if (sp > 8) {
            sp = (C + nt - 1) / nt;
            if (sp == 7) sp = 8;
        }
        if (nt == 1024 && sp < 5) sp = 5;
        lp.upath_sp = sp > 8 ? 0 : sp;
    }
    lp.gamma_smem = (size_t)(GAMMA_NW + 4) * H * 4 + 8 + (size_t)6 * H * 8 + 16 +  // px, pv, NW+2 lists, basis rows
                    (size_t)kMaxIter * 5 * 8;                                     // + the staged draws
    lp.m_tile_h = 16;
    auto m_bytes = [&](int th) {
        const size_t GH = th + 2 + 2 * cfg->varsigma, GW = lkg::M_TW + 2 + 2 * cfg->nu;
        const size_t MH = th + 2, MW = lkg::M_TW + 2;
        return (GH * GW + MH * MW) * 8 + 2048 * 4;
    };
    while (lp.m_tile_h > 1 && m_bytes(lp.m_tile_h) > 96 * 1024) lp.m_tile_h /= 2;
    lp.m_smem = m_bytes(lp.m_tile_h);
    d.m_tile_shift = 0;
    while ((1 << d.m_tile_shift) < lp.m_tile_h) ++d.m_tile_shift;
    d.m_ntx = (W + lkg::M_TW - 1) / lkg::M_TW;
    d.m_nty = (H + lp.m_tile_h - 1) / lp.m_tile_h;
    A(&d.m1_nz, (size_t)B * d.m_ntx * d.m_nty);
    A(&d.wg_nz, (size_t)B * d.m_ntx * d.m_nty);
    lp.collect_blocks = 32;
    lp.sort_cap = sort_cap;
    lp.select_smem = (size_t)sort_cap * 12 + (size_t)((C + 31) / 32) * 8 + 16;  // + certificate bits
    const size_t smem_cap = prop.sharedMemPerBlockOptin;
    if (lp.vdisp_smem > smem_cap || lp.vpath_smem > smem_cap || lp.road_smem > smem_cap || lp.bf_smem > smem_cap || lp.bt_smem > smem_cap ||
        lp.vanish_smem > smem_cap || lp.gamma_smem > smem_cap || lp.m_smem > smem_cap || lp.select_smem > smem_cap) {
        lk_destroy(c);
        return fail(LK_ERR_CONFIG, "frame geometry / window sizes exceed shared memory");
    }
    if (s != LK_OK) {
        lk_destroy(c);
        return s;
    }
    cudaError_t e = lkg::configure_kernels(lp);
    lp.need_ctas = lkg::need_bilateral_ctas(prop.multiProcessorCount);
    if (const char* nc = std::getenv("LK_NEED_CTAS")) lp.need_ctas = std::max(1, std::atoi(nc));
    if (e == cudaSuccess && d.stereo) {
        if (lkg::stereo_smem(d) > smem_cap) {
            lk_destroy(c);
            return fail(LK_ERR_CONFIG, "stereo: frame width exceeds the shared-memory row window");
        }
        e = lkg::configure_stereo(d);
    }
    if (e == cudaSuccess) {  // texture view of the exact weight table (TEX-pipe gathers)
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = d_wr;
        rd.res.linear.desc = cudaCreateChannelDesc<int2>();
        rd.res.linear.sizeInBytes = wr.size() * 8;
        cudaTextureDesc td{};
        td.readMode = cudaReadModeElementType;
        cudaTextureObject_t tex = 0;
        e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
        d.wr_tex = tex;
    }
    if (e == cudaSuccess) e = cudaMemcpy(d_ws, ws.data(), ws.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_wr, wr.data(), wr.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_val, val.data(), val.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_rng, rng.data(), rng.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && d_nt)
        e = cudaMemcpy(d_nt, need_tab.data(), need_tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
    d.need_tab = d_nt;
    if (e == cudaSuccess) {
        const char* r = std::getenv("LK_ROAD_COPY");  // 0: streamed grey is copied whole
        c->road_copy = !(r && std::atoi(r) == 0);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    for (int i = 0; i < 13 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
    {
        const char* b = std::getenv("LK_BRANCHES");
        c->branches = b ? std::atoi(b) : kBranchesDefault;
        if (c->branches < 1) c->branches = 1;
        if (c->branches > kMaxBranches) c->branches = kMaxBranches;
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
    {
        const char* k = std::getenv("LK_H2D_CHUNKS");
        c->h2d_chunks = k ? std::atoi(k) : kH2dChunksDefault;
        if (c->h2d_chunks < 1) c->h2d_chunks = 1;
        if (c->h2d_chunks > kMaxBranches) c->h2d_chunks = kMaxBranches;
    }
    for (int i = 0; i < kMaxBranches - 1 && e == cudaSuccess; ++i) {
        e = cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join[i], cudaEventDisableTiming);
    }
    for (int i = 0; i < kMaxBranches && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&c->copied[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        lk_destroy(c);
        return fail(LK_ERR_CUDA, std::string("context setup: ") + cudaGetErrorString(e));
    }
    *out = c;
    return LK_OK;
}

lk_status lk_destroy(lk_ctx* c) {
    if (!c) return LK_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    for (int k = 0; k < 2; ++k)
        for (cudaEvent_t e : {c->slot_copied[k], c->slot_free[k], c->slot_done[k]})
            if (e) cudaEventDestroy(e);
    if (c->front_stream) {
        cudaStreamSynchronize(c->front_stream);
        cudaStreamDestroy(c->front_stream);
    }
    for (int k = 0; k < kMaxBranches; ++k) {
        if (c->front_done[k]) cudaEventDestroy(c->front_done[k]);
        if (c->disp_copied[k]) cudaEventDestroy(c->disp_copied[k]);
    }
    if (c->h_rows) cudaFreeHost(c->h_rows);
    for (auto& kv : c->range_graphs) cudaGraphExecDestroy(kv.second);
    for (cudaEvent_t e : c->copied)
        if (e) cudaEventDestroy(e);
    if (c->d.wr_tex) cudaDestroyTextureObject((cudaTextureObject_t)c->d.wr_tex);
    for (cudaEvent_t e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->fork) cudaEventDestroy(c->fork);
    for (int i = 0; i < kMaxBranches - 1; ++i) {
        if (c->join[i]) cudaEventDestroy(c->join[i]);
        if (c->side[i]) {
            cudaStreamSynchronize(c->side[i]);
            cudaStreamDestroy(c->side[i]);
        }
    }
    for (void* p : c->allocs) cudaFree(p);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return LK_OK;
}

void* lk_stream(lk_ctx* c) { return c ? (void*)c->stream : nullptr; }

static int branch_count(const lk_ctx* c, int n);

int lk_launches_per_batch(lk_ctx* c) {
    return c ? (lkg::launches_per_batch(c->d, c->lp) + (c->last_stereo ? lkg::stereo_launches() : 0)) *
                   branch_count(c, c->last_n ? c->last_n : c->max_batch)
             : 0;
}

int lk_timed_frames(lk_ctx* c) { return c ? c->timed_frames : 0; }

lk_status lk_device_inputs(lk_ctx* c, uint8_t** grey, uint8_t** disparity) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    if (grey) *grey = c->in_grey;
    if (disparity) *disparity = c->in_disp;
    return LK_OK;
}

// View of frames [f0, f0 + ...) of every frame-major buffer: the same kernels
// run on a sub-batch without knowing it (layouts are frame-major throughout).
static void view_of(const Dev& d, const LaunchPlan& dlp, size_t f0, Dev& v, LaunchPlan& lp) {
    v = d;
    lp = dlp;
    const size_t H = d.H, px = d.px, C = d.ext_cols, D1 = d.D1;
    auto sh = [&](auto& p, size_t per) {
        if (p) p += f0 * per;
    };
    sh(v.grey, px);
    sh(v.disp, px);
    sh(v.right, px);
    sh(v.sat, 4 * px);
    sh(v.mu_l, px);
    sh(v.sig_l, px);
    sh(v.mu_r, px);
    sh(v.sig_r, px);
    sh(v.disp_l, px);
    sh(v.disp_r, px);
    sh(v.disp_out, px);
    sh(v.rep, 1);
    sh(v.aux, 1);
    sh(lp.vhistT, H * D1);
    sh(v.vchoice, D1 * H);
    sh(v.vpath, D1 * 2);
    sh(v.beta_inl, D1 * 2);
    sh(v.vpy, H);
    sh(v.vsing, H);
    sh(v.fv, H);
    sh(v.vpx, H);
    sh(v.smoothed, px);
    sh(v.smoothed_f, px);
    sh(v.pbits, H * d.words_per_row);
    sh(v.fneed, px);
    sh(v.need, (size_t)d.need_cap);
    sh(v.need_cnt, 1);
    sh(v.ctile, (size_t)d.n_stile);
    sh(v.ctile_cnt, 1);
    sh(v.ebits, H * d.words_per_row);
    sh(v.seg_cnt, H * d.n_seg);
    sh(v.seg_off, H * d.n_seg);
    sh(v.row_off, H + 1);
    sh(v.e_uv, px);
    sh(v.e_gx, px);
    sh(v.e_gy, px);
    sh(v.e_th, px);
    sh(v.e_wg, px);
    sh(v.e_col, px);
    sh(v.uchoice, H * C);
    sh(v.upath, H * 2);
    sh(v.gamma_inl, H * 2);
    sh(v.m1, px);
    sh(v.m1_nz, (size_t)d.m_ntx * d.m_nty);
    sh(v.wg_nz, (size_t)d.m_ntx * d.m_nty);
    sh(v.p99hist, 2048);
    sh(v.p99hist2, 4096);
    sh(v.p99cand, px);
    sh(v.energy, C);
    sh(v.mrange, H);
    sh(v.track_np, C);
    sh(v.e_touch, C);
    sh(v.lanes, (size_t)d.lane_cap);
    sh(v.polylines, (size_t)d.lane_cap * H);
    sh(v.mask, px);
    sh(v.gx, px);
    sh(v.gy, px);
    sh(v.mag, px);
    sh(v.theta, px);
    sh(v.acc, H * C);
    sh(v.m0, px);
}

static void frame_view(const lk_ctx* c, size_t f0, Dev& v, LaunchPlan& lp) {
    view_of(c->d, c->lp, f0, v, lp);
}

static lk_status enqueue_range(lk_ctx* c, size_t f0, int n, cudaStream_t st, cudaEvent_t* ev) {
    Dev d;
    LaunchPlan lp;
    frame_view(c, f0, d, lp);
    CU(cudaMemsetAsync(d.rep, 0, (size_t)n * sizeof(lk_frame_report), st));
    CU(cudaMemsetAsync(d.aux, 0, (size_t)n * sizeof(FrameAux), st));
    if (std::isnan(d.tr_lpv)) {
        CU(cudaMemsetAsync(d.p99hist, 0, (size_t)n * 2048 * sizeof(unsigned), st));
        CU(cudaMemsetAsync(d.p99hist2, 0, (size_t)n * 4096 * sizeof(unsigned), st));
    }
    if (c->run_stereo) CU(lkg::launch_stereo(d, n, st, ev));
    CU(lkg::launch_pipeline(d, lp, n, st, ev, !c->run_stereo));
    return LK_OK;
}

// Graph mode splits the batch into up to kMaxBranches frame ranges captured
// on forked streams: one range's latency-bound per-frame kernels (DP,
// RANSAC, selection) then overlap another range's throughput-bound
// bilateral/Sobel passes instead of leaving most SMs idle. Stage events
// time branch 0 (lk_timed_frames frames).
static int branch_count(const lk_ctx* c, int n) {
    if (c->flags & LK_FLAG_NO_GRAPH) return 1;
    int b = c->branches;
    while (b > 1 && n / b < kMinBranchFrames) --b;
    return b;
}

static lk_status enqueue_direct(lk_ctx* c, int n, bool timed) {
    const int nb = branch_count(c, n);
    if (nb == 1) {
        c->timed_frames = n;
        return enqueue_range(c, 0, n, c->stream, timed ? c->ev : nullptr);
    }
    CU(cudaEventRecord(c->fork, c->stream));
    size_t f0 = 0;
    for (int b = 0; b < nb; ++b) {
        const int nf = n / nb + (b < n % nb);
        cudaStream_t st = b == 0 ? c->stream : c->side[b - 1];
        if (b) CU(cudaStreamWaitEvent(st, c->fork, 0));
        if (b == 0) c->timed_frames = nf;
        if (lk_status s = enqueue_range(c, f0, nf, st, (timed && b == 0) ? c->ev : nullptr)) return s;
        f0 += nf;
    }
    for (int b = 1; b < nb; ++b) {
        CU(cudaEventRecord(c->join[b - 1], c->side[b - 1]));
        CU(cudaStreamWaitEvent(c->stream, c->join[b - 1], 0));
    }
    return LK_OK;
}

// Replays (capturing on first use) the graph of frames [f0, f0 + n) on st.
static lk_status launch_range_graph(lk_ctx* c, size_t f0, int n, cudaStream_t st, bool timed) {
    const auto key = std::make_tuple((long)f0, n, (timed ? 1 : 0) | (c->run_stereo ? 2 : 0));
    auto it = c->range_graphs.find(key);
    if (it == c->range_graphs.end()) {
        cudaGraph_t g;
        CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        lk_status s = enqueue_range(c, f0, n, st, timed ? c->ev : nullptr);
        cudaError_t e = cudaStreamEndCapture(st, &g);
        if (s != LK_OK) return s;
        if (e != cudaSuccess) return fail(LK_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        cudaGraphExec_t ex;
        e = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(LK_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        it = c->range_graphs.emplace(key, ex).first;
    }
    CU(cudaGraphLaunch(it->second, st));
    return LK_OK;
}

// Host-fed batch: the frames are split into up to h2d_chunks ranges on the
// context's streams. Range k's host->device copy starts when range k-1's
// copy is done (the copies share the link), and range k's graph starts as
// soon as its own inputs are resident, so copies overlap the compute of the
// ranges before them instead of preceding the whole batch.
// Input slot 0 of the streaming API is the buffer the direct entry points
// (lk_run_batch, lk_enqueue, ...) read. Once streaming has started, every batch
// that reads slot 0 marks it free only after its kernels, so a later submit's
// copy into slot 0 cannot overwrite the inputs of a batch still running.
static lk_status release_slot0(lk_ctx* c) {
    if (c->copy_stream && c->slot == 0) CU(cudaEventRecord(c->slot_free[0], c->stream));
    return LK_OK;
}

static lk_status run_host_pipelined(lk_ctx* c, const uint8_t* grey, const uint8_t* disp, int n) {
    uint8_t* second = c->run_stereo ? c->in_right : c->in_disp;  // right grey or disparity
    int nk = c->h2d_chunks;
    while (nk > 1 && n / nk < kMinBranchFrames) --nk;
    const size_t px = c->d.px;
    c->last_n = n;
    c->timed = true;
    c->last_stereo = c->run_stereo;
    CU(cudaEventRecord(c->fork, c->stream));
    size_t f0 = 0;
    for (int k = 0; k < nk; ++k) {
        const int nf = n / nk + (k < n % nk);
        cudaStream_t st = k == 0 ? c->stream : c->side[k - 1];
        if (k) CU(cudaStreamWaitEvent(st, c->copied[k - 1], 0));
        CU(cudaMemcpyAsync(c->in_grey + f0 * px, grey + f0 * px, (size_t)nf * px,
                           cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(second + f0 * px, disp + f0 * px, (size_t)nf * px,
                           cudaMemcpyHostToDevice, st));
        c->h2d_dma += 2 * (unsigned long long)nf * px;
        CU(cudaEventRecord(c->copied[k], st));
        if (k == 0) c->timed_frames = nf;
        if (c->flags & LK_FLAG_NO_GRAPH) {
            if (lk_status s = enqueue_range(c, f0, nf, st, k == 0 ? c->ev : nullptr)) return s;
        } else if (lk_status s = launch_range_graph(c, f0, nf, st, k == 0)) {
            return s;
        }
        f0 += nf;
    }
    for (int k = 1; k < nk; ++k) {
        CU(cudaEventRecord(c->join[k - 1], c->side[k - 1]));
        CU(cudaStreamWaitEvent(c->stream, c->join[k - 1], 0));
    }
    return release_slot0(c);
}

static lk_status enqueue_graph(lk_ctx* c, int n);

static lk_status enqueue_mode(lk_ctx* c, int n) {
    CU(cudaSetDevice(c->device));
    c->last_n = n;
    c->last_stereo = c->run_stereo;
    c->timed = true;
    const lk_status s = (c->flags & LK_FLAG_NO_GRAPH) ? enqueue_direct(c, n, true)
                                                      : enqueue_graph(c, n);
    if (s != LK_OK) return s;
    return release_slot0(c);
}

static lk_status enqueue_graph(lk_ctx* c, int n) {
    const int key = 4 * n + 2 * c->slot + (c->run_stereo ? 1 : 0);
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        cudaGraph_t g;
        CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        lk_status s = enqueue_direct(c, n, true);
        cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        if (s != LK_OK) return s;
        if (e != cudaSuccess) return fail(LK_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
        cudaGraphExec_t ex;
        e = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(LK_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        it = c->graphs.emplace(key, ex).first;
    }
    CU(cudaGraphLaunch(it->second, c->stream));
    return LK_OK;
}

lk_status lk_enqueue(lk_ctx* c, int n) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    if (n < 1 || n > c->max_batch) return fail(LK_ERR_INVALID_ARGUMENT, "batch size out of range");
    c->run_stereo = false;
    return enqueue_mode(c, n);
}

// ---- streaming: batch k+1's host->device copy (copy stream) overlaps batch
// k's kernels (context stream). Two input slots; the kernels of consecutive
// batches stay ordered on the context stream (they share intermediates).
lk_status lk_wait_batch(lk_ctx* c) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    if (c->n_pending == 0) return fail(LK_ERR_INVALID_ARGUMENT, "no submitted batch to wait for");
    const lk_ctx::Pending p = c->pending[0];
    if (cudaError_t e = cudaEventSynchronize(c->slot_done[p.slot]); e != cudaSuccess) {
        c->n_pending = 0;  // the stream is broken: no submitted batch can be reported
        return fail(LK_ERR_CUDA, std::string("lk_wait_batch: ") + cudaGetErrorString(e));
    }
    c->pending[0] = c->pending[1];
    --c->n_pending;
    bool any = false;
    if (p.reports)
        for (int i = 0; i < p.n; ++i) {
            p.reports[i].rng_seed = c->cfg.rng_seed;
            any |= p.reports[i].status != 0;
        }
    return any ? LK_ERR_FRAME : LK_OK;
}

// First streaming use: the second input slot, the copy stream, slot events.
static lk_status ensure_streaming(lk_ctx* c) {
    if (c->copy_stream) return LK_OK;
    if (lk_status s = c->alloc(&c->slot_grey[1], (size_t)c->max_batch * c->d.px + 16)) return s;
    if (lk_status s = c->alloc(&c->slot_disp[1], (size_t)c->max_batch * c->d.px + 16)) return s;
    c->slot_grey[0] = c->in_grey;
    c->slot_disp[0] = c->in_disp;
    CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        CU(cudaEventCreateWithFlags(&c->slot_copied[k], cudaEventDisableTiming));
        // timing-enabled: a copy stream waiting on a DisableTiming event recorded
        // after a graph launch was measured to serialise with the next batch
        CU(cudaEventCreate(&c->slot_free[k]));
        CU(cudaEventCreateWithFlags(&c->slot_done[k], cudaEventDisableTiming));
        CU(cudaEventRecord(c->slot_free[k], c->stream));
    }
    return LK_OK;
}

// First road-row copy: scratch outputs for the front pass (stages 5-7:
// reports, v-disparity, v-path, beta inliers, V_py, f(v), mask row ranges;
// the v-path choices in global memory so its CTAs need 6 KB of shared memory
// and start beside the running batch), its stream (highest priority) and the
// per-frame first-row array.
static lk_status ensure_front(lk_ctx* c) {
    if (c->front_ready) return LK_OK;
    const size_t B = c->max_batch, H = c->d.H, D1 = c->d.D1;
    c->front = c->d;
    c->front_lp = c->lp;
    Dev& f = c->front;
    lk_status s = LK_OK;
    auto A = [&](auto** p, size_t n) {
        if (s == LK_OK) s = c->alloc(p, n);
    };
    A(&f.rep, B);
    A(&f.aux, B);
    A(&c->front_lp.vhistT, B * H * D1);
    A(&f.vpath, B * D1 * 2);
    A(&f.beta_inl, B * D1 * 2);
    A(&f.vpy, B * H);
    A(&f.vsing, B * H);
    A(&f.fv, B * H);
    A(&f.mrange, B * H);
    A(&f.vchoice, B * D1 * H);
    A(&c->d_rows, B);
    if (s != LK_OK) return s;
    c->front_lp.vpath_choice_smem = 0;
    c->front_lp.vpath_smem = (size_t)2 * H * 8;
    CU(cudaMallocHost((void**)&c->h_rows, B * sizeof(int)));
    int least = 0, greatest = 0;
    CU(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CU(cudaStreamCreateWithPriority(&c->front_stream, cudaStreamNonBlocking, greatest));
    for (int k = 0; k < kMaxBranches; ++k) {
        CU(cudaEventCreateWithFlags(&c->front_done[k], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->disp_copied[k], cudaEventDisableTiming));
    }
    if (const char* r = std::getenv("LK_ROAD_CHUNKS"))
        c->road_chunks = std::max(1, std::min(kMaxBranches, std::atoi(r)));
    c->front_ready = true;
    return LK_OK;
}

// Device-resident stream (BASELINE config 5): the pipeline over the frames
// already in the input buffers (lk_device_inputs) plus the asynchronous
// read-back of their reports, queued like lk_submit_batch (lk_wait_batch).
// Batch k+1's kernels follow batch k's report copy on the context stream, so
// the host consumes batch k's records while batch k+1 runs.
lk_status lk_submit_resident(lk_ctx* c, int n, lk_frame_report* reports) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    if (n < 1 || n > c->max_batch) return fail(LK_ERR_INVALID_ARGUMENT, "batch size out of range");
    CU(cudaSetDevice(c->device));
    if (lk_status s = ensure_streaming(c)) return s;
    if (c->n_pending == 2) {  // at most two batches in flight
        const lk_status s = lk_wait_batch(c);
        if (s != LK_OK && s != LK_ERR_FRAME) return s;
    }
    const int sl = c->next_slot;  // completion-event slot (the inputs stay in slot 0)
    c->next_slot ^= 1;
    c->slot = 0;
    c->run_stereo = false;
    if (lk_status s = enqueue_mode(c, n)) return s;
    if (reports)
        CU(cudaMemcpyAsync(reports, c->d.rep, (size_t)n * sizeof(lk_frame_report),
                           cudaMemcpyDeviceToHost, c->stream));
    CU(cudaEventRecord(c->slot_done[sl], c->stream));
    c->pending[c->n_pending++] = {sl, n, reports};
    return LK_OK;
}

// Streaming submit shared by the mono (grey + disparity) and stereo (left +
// right) entry points: the copy goes to one of two input slots on the copy
// stream, the kernels wait for it, and the next submit's copy overlaps them.
static lk_status submit(lk_ctx* c, const uint8_t* a, const uint8_t* b, int n,
                        lk_frame_report* reports, bool stereo) {
    if (!c || !a || !b) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    if (stereo && !c->d.stereo)
        return fail(LK_ERR_INVALID_ARGUMENT, "context was created without LK_FLAG_STEREO");
    if (n < 1 || n > c->max_batch) return fail(LK_ERR_INVALID_ARGUMENT, "batch size out of range");
    CU(cudaSetDevice(c->device));
    if (lk_status s = ensure_streaming(c)) return s;
    if (stereo && !c->slot_right[0]) {
        if (lk_status s = c->alloc(&c->slot_right[1], (size_t)c->max_batch * c->d.px)) return s;
        c->slot_right[0] = c->in_right;
    }
    if (c->n_pending == 2) {  // at most two batches in flight
        const lk_status s = lk_wait_batch(c);
        if (s != LK_OK && s != LK_ERR_FRAME) return s;
    }
    const int sl = c->next_slot;
    c->next_slot ^= 1;
    const size_t bytes = (size_t)n * c->d.px;
    uint8_t* second = stereo ? c->slot_right[sl] : c->slot_disp[sl];
    // (the front pass and the wait pay off only when the horizon is low enough:
    // after a batch that skipped < 15 % of its grey rows, whole frames again,
    // re-probing every 16th batch)
    const bool road = !stereo && c->road_copy && c->lp.fast_front && !c->d.hooks &&
                      (c->road_saved >= 0.15 || (++c->road_probe & 15) == 0);
    if (road)
        if (lk_status s = ensure_front(c)) return s;
    // inputs into the slot once the batch that last read it has finished
    CU(cudaStreamWaitEvent(c->copy_stream, c->slot_free[sl], 0));
    if (!road) {
        CU(cudaMemcpyAsync(c->slot_grey[sl], a, bytes, cudaMemcpyHostToDevice, c->copy_stream));
        CU(cudaMemcpyAsync(second, b, bytes, cudaMemcpyHostToDevice, c->copy_stream));
        c->h2d_dma += 2 * (unsigned long long)bytes;
    } else {
        // Road-row copy: the disparity first; stages 5-7 of this batch on the
        // front stream give each frame's first grey row read by stages 8-12
        // (horizon - 1 - rho: the mask is empty above the horizon,
        // preprocess.hpp:18); the host waits for them (the previous batch keeps
        // computing) and copies the rows from the batch's smallest one down.
        // Rows above it stay stale in the slot and are never read.
        // In frame chunks, so chunk k's grey copy is queued while chunk k+1's
        // stages 5-7 run and the link does not wait for them.
        const size_t px = c->d.px;
        int nk = c->road_chunks;
        while (nk > 1 && n / nk < 4) --nk;
        cudaStream_t fs = c->front_stream;
        for (int k = 0, f0 = 0; k < nk; ++k) {
            const int nf = n / nk + (k < n % nk);
            CU(cudaMemcpyAsync(second + (size_t)f0 * px, b + (size_t)f0 * px, (size_t)nf * px,
                               cudaMemcpyHostToDevice, c->copy_stream));
            CU(cudaEventRecord(c->disp_copied[k], c->copy_stream));
            CU(cudaStreamWaitEvent(fs, c->disp_copied[k], 0));
            Dev fd;
            LaunchPlan flp;
            view_of(c->front, c->front_lp, (size_t)f0, fd, flp);
            fd.disp = second + (size_t)f0 * px;
            CU(cudaMemsetAsync(fd.rep, 0, (size_t)nf * sizeof(lk_frame_report), fs));
            CU(cudaMemsetAsync(fd.aux, 0, (size_t)nf * sizeof(FrameAux), fs));
            CU(lkg::launch_road_front(fd, flp, nf, c->d_rows + f0, fs));
            CU(cudaMemcpyAsync(c->h_rows + f0, c->d_rows + f0, (size_t)nf * sizeof(int),
                               cudaMemcpyDeviceToHost, fs));
            CU(cudaEventRecord(c->front_done[k], fs));
            f0 += nf;
        }
        unsigned long long copied = 0;
        for (int k = 0, f0 = 0; k < nk; ++k) {
            const int nf = n / nk + (k < n % nk);
            CU(cudaEventSynchronize(c->front_done[k]));
            int r0 = c->d.H;
            for (int i = f0; i < f0 + nf; ++i) r0 = std::min(r0, c->h_rows[i]);
            if (r0 < c->d.H) {
                const size_t off = (size_t)f0 * px + (size_t)r0 * c->d.W, w = px - (size_t)r0 * c->d.W;
                CU(cudaMemcpy2DAsync(c->slot_grey[sl] + off, px, a + off, px, w, (size_t)nf,
                                     cudaMemcpyHostToDevice, c->copy_stream));
                c->h2d_dma += (unsigned long long)w * nf;
                copied += (unsigned long long)w * nf;
            }
            f0 += nf;
        }
        c->h2d_dma += bytes;
        c->road_saved = 1.0 - (double)copied / (double)bytes;
    }
    CU(cudaEventRecord(c->slot_copied[sl], c->copy_stream));
    // kernels on the slot (graphs are keyed by slot), then the reports. A
    // stereo batch's stage 4 writes the context's disparity buffer as before.
    CU(cudaStreamWaitEvent(c->stream, c->slot_copied[sl], 0));
    const uint8_t* g0 = c->d.grey;
    const uint8_t* d0 = c->d.disp;
    const uint8_t* r0 = c->d.right;
    c->d.grey = c->slot_grey[sl];
    if (stereo)
        c->d.right = second;
    else
        c->d.disp = second;
    c->slot = sl;
    c->run_stereo = stereo;
    const lk_status s = enqueue_mode(c, n);
    c->d.grey = g0;
    c->d.disp = d0;
    c->d.right = r0;
    c->slot = 0;
    c->run_stereo = false;
    if (s != LK_OK) return s;
    CU(cudaEventRecord(c->slot_free[sl], c->stream));
    if (reports)
        CU(cudaMemcpyAsync(reports, c->d.rep, (size_t)n * sizeof(lk_frame_report),
                           cudaMemcpyDeviceToHost, c->stream));
    CU(cudaEventRecord(c->slot_done[sl], c->stream));
    c->pending[c->n_pending++] = {sl, n, reports};
    return LK_OK;
}

lk_status lk_submit_batch(lk_ctx* c, const uint8_t* grey, const uint8_t* disparity, int n,
                          lk_frame_report* reports) {
    return submit(c, grey, disparity, n, reports, false);
}

lk_status lk_submit_stereo_batch(lk_ctx* c, const uint8_t* left, const uint8_t* right, int n,
                                 lk_frame_report* reports) {
    return submit(c, left, right, n, reports, true);
}

lk_status lk_enqueue_stereo(lk_ctx* c, int n) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    if (!c->d.stereo) return fail(LK_ERR_INVALID_ARGUMENT, "context was created without LK_FLAG_STEREO");
    if (n < 1 || n > c->max_batch) return fail(LK_ERR_INVALID_ARGUMENT, "batch size out of range");
    c->run_stereo = true;
    return enqueue_mode(c, n);
}

lk_status lk_stereo_inputs(lk_ctx* c, uint8_t** left, uint8_t** right) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    if (!c->d.stereo) return fail(LK_ERR_INVALID_ARGUMENT, "context was created without LK_FLAG_STEREO");
    if (left) *left = c->in_grey;
    if (right) *right = c->in_right;
    return LK_OK;
}

lk_status lk_synchronize(lk_ctx* c) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    CU(cudaStreamSynchronize(c->stream));
    return LK_OK;
}

lk_status lk_fetch_reports(lk_ctx* c, lk_frame_report* reports, int n) {
    if (!c || !reports) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    if (n < 1 || n > c->max_batch) return fail(LK_ERR_INVALID_ARGUMENT, "batch size out of range");
    CU(cudaMemcpyAsync(reports, c->d.rep, (size_t)n * sizeof(lk_frame_report),
                       cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    bool any = false;
    for (int i = 0; i < n; ++i) {
        reports[i].rng_seed = c->cfg.rng_seed;
        any |= reports[i].status != 0;
    }
    return any ? LK_ERR_FRAME : LK_OK;
}

lk_status lk_run_batch(lk_ctx* c, const uint8_t* grey, const uint8_t* disparity, int n,
                       lk_mem where, lk_frame_report* reports) {
    if (!c || !grey || !disparity) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    if (n < 1 || n > c->max_batch) return fail(LK_ERR_INVALID_ARGUMENT, "batch size out of range");
    CU(cudaSetDevice(c->device));
    const size_t bytes = (size_t)n * c->d.px;
    c->run_stereo = false;
    if (where == LK_MEM_HOST) {
        if (lk_status s = run_host_pipelined(c, grey, disparity, n)) return s;
    } else {
        if (grey != c->in_grey)
            CU(cudaMemcpyAsync(c->in_grey, grey, bytes, cudaMemcpyDeviceToDevice, c->stream));
        if (disparity != c->in_disp)
            CU(cudaMemcpyAsync(c->in_disp, disparity, bytes, cudaMemcpyDeviceToDevice, c->stream));
        if (lk_status s = lk_enqueue(c, n)) return s;
    }
    if (reports) return lk_fetch_reports(c, reports, n);
    CU(cudaStreamSynchronize(c->stream));
    return LK_OK;
}

lk_status lk_run_stereo_batch(lk_ctx* c, const uint8_t* left, const uint8_t* right, int n,
                              lk_mem where, lk_frame_report* reports) {
    if (!c || !left || !right) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->d.stereo) return fail(LK_ERR_INVALID_ARGUMENT, "context was created without LK_FLAG_STEREO");
    if (n < 1 || n > c->max_batch) return fail(LK_ERR_INVALID_ARGUMENT, "batch size out of range");
    CU(cudaSetDevice(c->device));
    const size_t bytes = (size_t)n * c->d.px;
    c->run_stereo = true;
    if (where == LK_MEM_HOST) {
        if (lk_status s = run_host_pipelined(c, left, right, n)) return s;
    } else {
        if (left != c->in_grey)
            CU(cudaMemcpyAsync(c->in_grey, left, bytes, cudaMemcpyDeviceToDevice, c->stream));
        if (right != c->in_right)
            CU(cudaMemcpyAsync(c->in_right, right, bytes, cudaMemcpyDeviceToDevice, c->stream));
        if (lk_status s = enqueue_mode(c, n)) return s;
    }
    if (reports) return lk_fetch_reports(c, reports, n);
    CU(cudaStreamSynchronize(c->stream));
    return LK_OK;
}

lk_status lk_stage_times(lk_ctx* c, float ms[13]) {
    if (!c || !ms) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    for (int i = 0; i < 13; ++i) ms[i] = 0.f;
    if (!c->timed) return fail(LK_ERR_UNAVAILABLE, "no batch has run yet");
    CU(cudaStreamSynchronize(c->stream));
    int prev = 0;
    for (int st = c->last_stereo ? 1 : 5; st <= 12; ++st) {  // [st] = end of stage st
        CU(cudaEventElapsedTime(&ms[st], c->ev[prev], c->ev[st]));
        prev = st;
    }
    CU(cudaEventElapsedTime(&ms[0], c->ev[0], c->ev[12]));
    return LK_OK;
}

lk_status lk_get_stage(lk_ctx* c, int frame, int stage, void* dst, size_t capacity,
                       size_t* needed) {
    if (!c) return fail(LK_ERR_INVALID_ARGUMENT, "null context");
    if (frame < 0 || frame >= c->last_n) return fail(LK_ERR_INVALID_ARGUMENT, "frame out of range");
    if (stage < 0 || stage >= LK_STAGE_COUNT) return fail(LK_ERR_INVALID_ARGUMENT, "unknown stage");
    CU(cudaSetDevice(c->device));
    CU(cudaStreamSynchronize(c->stream));
    const Dev& d = c->d;
    lk_frame_report rep;
    CU(cudaMemcpy(&rep, d.rep + frame, sizeof rep, cudaMemcpyDeviceToHost));
    static const int produced_by[LK_STAGE_COUNT] = {5,  6,  7,  7,  7,  8,  9,  10, 10,
                                                    10, 10, 10, 11, 11, 11, 11, 11, 12,
                                                    12, 12, 12, 12, 1,  1,  2,  3,  4};
    if (stage >= LK_STAGE_STATS_MU && !c->last_stereo)
        return fail(LK_ERR_UNAVAILABLE, "stage 1-4 hooks need a stereo batch (lk_run_stereo_batch)");
    if (rep.status != 0 && rep.failed_stage <= produced_by[stage])
        return fail(LK_ERR_UNAVAILABLE, "stage not reached: the frame failed earlier");
    const bool hook_only = stage == LK_STAGE_MASK || stage == LK_STAGE_GX || stage == LK_STAGE_GY ||
                           stage == LK_STAGE_MAG || stage == LK_STAGE_THETA ||
                           stage == LK_STAGE_VPX_ACC || stage == LK_STAGE_M0 ||
                           stage == LK_STAGE_POLYLINES;
    if (hook_only && !d.hooks) return fail(LK_ERR_UNAVAILABLE, "hook needs LK_FLAG_HOOKS");
    if (stage == LK_STAGE_SMOOTHED && c->lp.fast_front)
        return fail(LK_ERR_UNAVAILABLE,
                    "SMOOTHED is exact only around edges on the fast path: use LK_FLAG_HOOKS "
                    "or LK_FLAG_EXACT");
    const size_t px = d.px, H = d.H, C = d.ext_cols, D1 = d.D1;
    const size_t rows = (size_t)(d.H - rep.horizon);
    const size_t f = (size_t)frame;
    const int n_edges = (int)rep.edge_pixels;
    std::vector<char> buf;
    auto grab = [&](const void* src, size_t bytes) -> lk_status {
        buf.resize(bytes);
        if (bytes) CU(cudaMemcpy(buf.data(), src, bytes, cudaMemcpyDeviceToHost));
        return LK_OK;
    };
    lk_status s = LK_OK;
    switch (stage) {
        case LK_STAGE_STATS_MU: s = grab(d.mu_l + f * px, px * 8); break;
        case LK_STAGE_STATS_SIGMA: s = grab(d.sig_l + f * px, px * 8); break;
        case LK_STAGE_DISP_LEFT: s = grab(d.disp_l + f * px, px); break;
        case LK_STAGE_DISP_RIGHT: s = grab(d.disp_r + f * px, px); break;
        case LK_STAGE_DISPARITY: s = grab(d.disp_out + f * px, px); break;
        case LK_STAGE_VDISPARITY: {  // stored transposed [D1][H] for the v-path DP
            s = grab(c->lp.vhistT + f * H * D1, H * D1 * 4);
            if (s != LK_OK) break;
            std::vector<char> t(buf.size());
            const int32_t* src = reinterpret_cast<const int32_t*>(buf.data());
            int32_t* dst = reinterpret_cast<int32_t*>(t.data());
            for (size_t v = 0; v < H; ++v)
                for (size_t k = 0; k < D1; ++k) dst[v * D1 + k] = src[k * H + v];
            buf.swap(t);
            break;
        }
        case LK_STAGE_VPATH: s = grab(d.vpath + f * D1 * 2, D1 * 8); break;
        case LK_STAGE_BETA_INLIERS:
            s = grab(d.beta_inl + f * D1 * 2, (size_t)rep.beta_inlier_count * 8);
            break;
        case LK_STAGE_VPY: s = grab(d.vpy + f * H, H * 8); break;
        case LK_STAGE_VPY_SINGULAR: s = grab(d.vsing + f * H, H); break;
        case LK_STAGE_MASK: s = grab(d.mask + f * px, px); break;
        case LK_STAGE_SMOOTHED: s = grab(d.smoothed + f * px, px * 8); break;
        case LK_STAGE_GX: s = grab(d.gx + f * px, px * 8); break;
        case LK_STAGE_GY: s = grab(d.gy + f * px, px * 8); break;
        case LK_STAGE_MAG: s = grab(d.mag + f * px, px * 8); break;
        case LK_STAGE_THETA: s = grab(d.theta + f * px, px * 8); break;
        case LK_STAGE_EDGES:
        case LK_STAGE_VOTES: {
            std::vector<int32_t> uv(n_edges), col(n_edges);
            std::vector<double> gx(n_edges), gy(n_edges), th(n_edges);
            if (n_edges) {
                CU(cudaMemcpy(uv.data(), d.e_uv + f * px, n_edges * 4, cudaMemcpyDeviceToHost));
                CU(cudaMemcpy(col.data(), d.e_col + f * px, n_edges * 4, cudaMemcpyDeviceToHost));
                CU(cudaMemcpy(gx.data(), d.e_gx + f * px, n_edges * 8, cudaMemcpyDeviceToHost));
                CU(cudaMemcpy(gy.data(), d.e_gy + f * px, n_edges * 8, cudaMemcpyDeviceToHost));
                CU(cudaMemcpy(th.data(), d.e_th + f * px, n_edges * 8, cudaMemcpyDeviceToHost));
            }
            if (stage == LK_STAGE_EDGES) {
                std::vector<lk_edge> e(n_edges);
                for (int i = 0; i < n_edges; ++i)
                    e[i] = {uv[i] & 0xffff, uv[i] >> 16, gx[i], gy[i], th[i]};
                buf.assign((char*)e.data(), (char*)e.data() + e.size() * sizeof(lk_edge));
            } else {
                std::vector<lk_vote> v;
                for (int i = 0; i < n_edges; ++i)
                    if (col[i] != lkg::kSkipCol) v.push_back({uv[i] & 0xffff, uv[i] >> 16, col[i]});
                buf.assign((char*)v.data(), (char*)v.data() + v.size() * sizeof(lk_vote));
            }
            break;
        }
        case LK_STAGE_VPX_ACC: s = grab(d.acc + f * H * C, rows * C * 8); break;
        case LK_STAGE_UPATH: s = grab(d.upath + f * H * 2, rows * 8); break;
        case LK_STAGE_GAMMA_INLIERS:
            s = grab(d.gamma_inl + f * H * 2, (size_t)rep.gamma_inlier_count * 8);
            break;
        case LK_STAGE_VPX: s = grab(d.vpx + f * H, H * 8); break;
        case LK_STAGE_M0: s = grab(d.m0 + f * px, px * 8); break;
        case LK_STAGE_M1: {
            s = grab(d.m1 + f * px, px * 8);
            if (s != LK_OK || d.hooks) break;
            // without hooks only the non-zero tiles on rows >= horizon - varsigma - 1 are written
            std::vector<uint8_t> nz((size_t)d.m_nty * d.m_ntx);
            CU(cudaMemcpy(nz.data(), d.m1_nz + f * nz.size(), nz.size(), cudaMemcpyDeviceToHost));
            double* m = (double*)buf.data();
            for (int v = 0; v < d.H; ++v)
                for (int u = 0; u < d.W; ++u)
                    if (v < (int)rep.horizon - d.varsigma - 1 ||
                        !nz[(v >> d.m_tile_shift) * d.m_ntx + (u / lkg::M_TW)])
                        m[(size_t)v * d.W + u] = 0.0;
            break;
        }
        case LK_STAGE_ENERGY: s = grab(d.energy + f * C, C * 8); break;
        case LK_STAGE_LANES:
            s = grab(d.lanes + f * d.lane_cap, (size_t)rep.lane_count * sizeof(lk_lane));
            break;
        case LK_STAGE_POLYLINES: {
            const size_t nl = (size_t)rep.lane_count;
            buf.resize(nl * rows * 8);
            for (size_t k = 0; k < nl; ++k)
                CU(cudaMemcpy(buf.data() + k * rows * 8, d.polylines + (f * d.lane_cap + k) * H,
                              rows * 8, cudaMemcpyDeviceToHost));
            break;
        }
    }
    if (s != LK_OK) return s;
    if (needed) *needed = buf.size();
    if (dst) {
        if (capacity < buf.size()) return fail(LK_ERR_INVALID_ARGUMENT, "destination too small");
        if (!buf.empty()) std::memcpy(dst, buf.data(), buf.size());
    }
    return LK_OK;
}

// Pinned host memory for end-to-end (host-fed) runs.
lk_status lk_h2d_bytes(lk_ctx* c, unsigned long long* bytes) {
    if (!c || !bytes) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    *bytes = c->h2d_dma;
    return LK_OK;
}

lk_status lk_host_alloc(void** p, size_t bytes) {
    if (!p) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    CU(cudaMallocHost(p, bytes));
    return LK_OK;
}

lk_status lk_host_free(void* p) {
    CU(cudaFreeHost(p));
    return LK_OK;
}

// Layout check for bindings: sizes of the ABI structs.
void lk_abi_sizes(size_t* out) {
    out[0] = sizeof(lk_config);
    out[1] = sizeof(lk_frame_report);
    out[2] = sizeof(lk_scene_params);
    out[3] = sizeof(lk_edge);
    out[4] = sizeof(lk_vote);
    out[5] = sizeof(lk_lane);
}

}  // extern "C"

namespace lkg {
cudaError_t fp64_probe(int sms, double* ops_per_s);
}

extern "C" lk_status lk_measure_fp64(int device, double* ops_per_s) {
    if (!ops_per_s) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    CU(cudaSetDevice(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    CU(lkg::fp64_probe(prop.multiProcessorCount, ops_per_s));
    return LK_OK;
}

extern "C" lk_status lk_fast_path_error(lk_ctx* c, double* max_abs_error) {
    if (!c || !max_abs_error) return fail(LK_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->lp.fast_front || c->last_n < 1)
        return fail(LK_ERR_UNAVAILABLE, "no fast-path batch has run on this context");
    CU(cudaSetDevice(c->device));
    double* scratch = nullptr;
    CU(cudaMalloc(&scratch, sizeof(double)));
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(double), c->stream);
    if (e == cudaSuccess) {
        // the pipeline computes s~ only near the road mask: recompute every tile
        lkg::launch_fast_bilateral(c->d, c->lp, c->last_n, c->stream, 1);
        lkg::launch_exact_bilateral(c->d, c->lp, c->last_n, c->stream);  // every pixel, exact
        e = lkg::fast_error(c->d, c->last_n, c->stream, scratch);
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(max_abs_error, scratch, sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(scratch);
    if (e != cudaSuccess) return fail(LK_ERR_CUDA, std::string("fast path check: ") + cudaGetErrorString(e));
    return LK_OK;
}
