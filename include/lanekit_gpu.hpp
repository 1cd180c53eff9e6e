// lanekit_gpu.hpp — header-only C++ shim over the C-ABI for callers that use
// the reference's own types (lanekit::GrayImage, lanekit::DisparityMap,
// lanekit::PipelineConfig; image.hpp:11-36, config.hpp:16-46).
//
//   lanekit_gpu::Result r = lanekit_gpu::run_from_disparity(left, disparity, cfg);
//   r.report.lane_count;  r.lanes();  r.stage<double>(LK_STAGE_M1);  ...
//
// mirrors stages 5-12 of lanekit::run_pipeline (pipeline.hpp:184-270) with the
// disparity injected, throwing lanekit_gpu::StageError with the reference's
// "stage N (name): msg" text (common.hpp:18-24) when a stage fails. The grey
// image must hold 8-bit values k/255.0 exactly (what read_png_gray produces,
// image_io.hpp:147); anything else is rejected rather than silently rounded.
// Templated on the image/config types so this header needs no lanekit headers.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lanekit_b200.h"

namespace lanekit_gpu {

struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};

struct StageError : Error {  // lanekit::StageError (common.hpp:18-24)
    int stage;
    std::string stage_name;
    StageError(int st, std::string name, const std::string& msg)
        : Error(msg), stage(st), stage_name(std::move(name)) {}
};

inline void check(lk_status s) {
    if (s != LK_OK) throw Error(lk_last_error());
}

template <typename Cfg>
lk_config to_lk_config(const Cfg& c) {  // field for field, config.hpp:16-46
    lk_config o;
    lk_config_default(&o);
    o.rho = c.rho;
    o.tau = c.tau;
    o.d_max = c.d_max;
    o.tr_lrc = c.tr_lrc;
    o.sigma_floor = c.sigma_floor;
    o.lambda_y = c.lambda_y;
    o.tr_y = c.tr_y;
    o.eps_y = c.eps_y;
    o.varpi = c.varpi;
    o.sigma_s = c.sigma_s;
    o.sigma_r = c.sigma_r;
    o.bf_window = c.bf_window;
    o.sobel_threshold = c.sobel_threshold;
    o.chi = c.chi;
    o.rho_vote = c.rho_vote;
    o.lambda_x = c.lambda_x;
    o.tr_x = c.tr_x;
    o.eps_x = c.eps_x;
    o.sigma_g = c.sigma_g;
    o.nu = c.nu;
    o.varsigma = c.varsigma;
    o.lambda_g = c.lambda_g;
    o.xi = c.xi;
    o.tr_lpv = c.tr_lpv;
    o.min_lane_sep = c.min_lane_sep;
    o.rng_seed = c.rng_seed;
    o.paper_sign = c.paper_sign ? 1 : 0;
    o.threads = c.threads;
    return o;
}

class Context {  // one per host thread; owns device buffers and CUDA graphs
  public:
    Context(int width, int height, const lk_config& cfg, int max_batch = 1, int device = 0,
            uint32_t flags = LK_FLAG_HOOKS) {
        lk_ctx* c = nullptr;
        check(lk_create(&c, device, &cfg, width, height, max_batch, flags));
        ctx_.reset(c);
    }
    lk_ctx* get() const { return ctx_.get(); }

  private:
    struct Del {
        void operator()(lk_ctx* c) const { lk_destroy(c); }
    };
    std::unique_ptr<lk_ctx, Del> ctx_;
};

struct Result {  // PipelineReport + lazily copied PipelineResult members
    lk_frame_report report{};
    std::shared_ptr<Context> ctx;
    int frame = 0;

    template <typename T>
    std::vector<T> stage(lk_stage id) const {
        size_t need = 0;
        check(lk_get_stage(ctx->get(), frame, id, nullptr, 0, &need));
        std::vector<T> v(need / sizeof(T));
        if (need) check(lk_get_stage(ctx->get(), frame, id, v.data(), need, &need));
        return v;
    }
    std::vector<lk_lane> lanes() const { return stage<lk_lane>(LK_STAGE_LANES); }
};

namespace detail {
template <typename Gray, typename Disp>
void check_inputs(const Gray& left, const Disp& disparity) {
    if (left.width == 0 || left.height == 0 || disparity.width == 0 || disparity.height == 0)
        throw StageError(1, lk_stage_name(1), "stage 1 (block statistics): empty input image");
    if (left.width != disparity.width || left.height != disparity.height)
        throw StageError(1, lk_stage_name(1),
                         "stage 1 (block statistics): stereo pair dimensions differ");
}

// k/255.0 grey -> u8 k (rejecting any other value), int disparity -> u8
template <typename Gray, typename Disp>
void to_u8(const Gray& left, const Disp& disparity, uint8_t* g, uint8_t* d) {
    const size_t n = static_cast<size_t>(left.width) * left.height;
    for (size_t i = 0; i < n; ++i) {
        const double x = left.data[i];
        const long k = std::lround(x * 255.0);
        if (k < 0 || k > 255 || k / 255.0 != x)
            throw Error("lanekit_gpu: grey value is not an 8-bit level k/255.0");
        g[i] = static_cast<uint8_t>(k);
        const int dv = disparity.data[i];
        if (dv < 0 || dv > 255) throw Error("lanekit_gpu: disparity outside 0..255");
        d[i] = static_cast<uint8_t>(dv);
    }
}

inline void throw_if_failed(const lk_frame_report& rep) {
    if (rep.status != 0) {
        char buf[256];
        lk_frame_message(&rep, buf, sizeof buf);
        const int st = static_cast<int>(rep.failed_stage);
        throw StageError(st, lk_stage_name(st), buf);
    }
}
}  // namespace detail

// The drop-in for a caller that runs frame after frame (lanedet detect, a
// video loop): the context, its device buffers, pinned staging and captured
// CUDA graph are built once, so a call costs the frame's copies and kernels.
// A Result's hooks read the context's buffers: they stay valid until the next
// run() on the same Pipeline.
class Pipeline {
  public:
    template <typename Cfg>
    Pipeline(int width, int height, const Cfg& cfg, int device = 0,
             uint32_t flags = LK_FLAG_HOOKS)
        : w_(width), h_(height) {
        const lk_config c = to_lk_config(cfg);
        check(lk_validate_config(&c));
        ctx_ = std::make_shared<Context>(width, height, c, 1, device, flags);
        void* g = nullptr;
        void* d = nullptr;
        check(lk_host_alloc(&g, static_cast<size_t>(width) * height));
        check(lk_host_alloc(&d, static_cast<size_t>(width) * height));
        g_.reset(static_cast<uint8_t*>(g));
        d_.reset(static_cast<uint8_t*>(d));
    }

    template <typename Gray, typename Disp>
    Result run(const Gray& left, const Disp& disparity) {
        detail::check_inputs(left, disparity);
        if (left.width != w_ || left.height != h_)
            throw Error("lanekit_gpu: frame size differs from the Pipeline's");
        detail::to_u8(left, disparity, g_.get(), d_.get());
        Result r;
        r.ctx = ctx_;
        const lk_status s = lk_run_batch(ctx_->get(), g_.get(), d_.get(), 1, LK_MEM_HOST, &r.report);
        if (s != LK_OK && s != LK_ERR_FRAME) check(s);
        detail::throw_if_failed(r.report);
        return r;
    }

  private:
    struct HostDel {
        void operator()(uint8_t* p) const { lk_host_free(p); }
    };
    int w_, h_;
    std::shared_ptr<Context> ctx_;
    std::unique_ptr<uint8_t, HostDel> g_, d_;
};

// Stages 5-12 on one frame; `left` is a GrayImage-like (width, height,
// data of k/255.0), `disparity` a DisparityMap-like (ints, 0 = invalid).
// One-shot: builds a context for the call (use Pipeline to reuse one).
template <typename Gray, typename Disp, typename Cfg>
Result run_from_disparity(const Gray& left, const Disp& disparity, const Cfg& cfg,
                          int device = 0) {
    detail::check_inputs(left, disparity);
    Pipeline p(left.width, left.height, cfg, device);
    return p.run(left, disparity);
}

}  // namespace lanekit_gpu
