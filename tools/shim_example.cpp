// shim_example.cpp — a reference-typed caller of the GPU path through
// include/lanekit_gpu.hpp. With -DWITH_LANEKIT it uses the reference's own
// lanekit::GrayImage / DisparityMap / PipelineConfig (image.hpp, config.hpp),
// otherwise structurally identical local stand-ins (the GPU box has no
// /root/reference). Prints the lanes or the StageError; exit 0 on either.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lanekit_gpu.hpp"

#ifdef WITH_LANEKIT
#include "lanekit/config.hpp"
#include "lanekit/image.hpp"
using GrayImage = lanekit::GrayImage;
using DisparityMap = lanekit::DisparityMap;
using PipelineConfig = lanekit::PipelineConfig;
#else
template <typename T>
struct Image {
    int width = 0, height = 0;
    std::vector<T> data;
    Image(int w, int h, T v) : width(w), height(h), data(static_cast<size_t>(w) * h, v) {}
};
using GrayImage = Image<double>;
using DisparityMap = Image<int>;
struct PipelineConfig {
    int rho = 3, tau = 1, d_max = 64, tr_lrc = 3;
    double sigma_floor = 1e-4, lambda_y = 30, tr_y = 4, eps_y = 0.99, varpi = 3, sigma_s = 300,
           sigma_r = 0.3;
    int bf_window = 11;
    double sobel_threshold = 100;
    int chi = 25;
    double rho_vote = 1, lambda_x = 10, tr_x = 16, eps_x = 0.99, sigma_g = 3.5;
    int nu = 1, varsigma = 3;
    double lambda_g = 1, xi = 0.5, tr_lpv = __builtin_nan("");
    int min_lane_sep = 20;
    unsigned long long rng_seed = 1;
    bool paper_sign = false;
    int threads = 1;
};
#endif

int main(int argc, char** argv) {
    lk_scene_params p;
    lk_scene_default(&p);
    p.width = 1242;
    p.height = 375;
    p.beta[0] = -15.0;
    p.beta[1] = 0.15;
    p.beta[2] = 1e-4;
    p.gamma[0] = 621.0;
    p.gamma[1] = -0.10;
    p.gamma[2] = 2.5e-4;
    p.d_max = 255;
    p.n_lanes = 2;
    p.lane_bottoms[0] = 0.30 * 1242;
    p.lane_bottoms[1] = 0.62 * 1242;
    p.noise_sigma = 0.02;
    p.rng_seed = 5;
    std::vector<uint8_t> g(1242 * 375), d(1242 * 375);
    if (lk_synth_scene(&p, g.data(), nullptr, d.data(), nullptr) != LK_OK) return 2;
    GrayImage left(1242, 375, 0.0);
    DisparityMap disp(1242, 375, 0);
    for (size_t i = 0; i < g.size(); ++i) {
        left.data[i] = g[i] / 255.0;
        disp.data[i] = d[i];
    }
    PipelineConfig cfg;
    try {
        const lanekit_gpu::Result r = lanekit_gpu::run_from_disparity(left, disp, cfg);
        std::printf("lanes:");
        for (const lk_lane& l : r.lanes()) std::printf(" %d", l.bottom_col);
        std::printf("\n");
    } catch (const lanekit_gpu::StageError& e) {
        std::printf("StageError %d: %s\n", e.stage, e.what());
    } catch (const lanekit_gpu::Error& e) {
        std::printf("Error: %s\n", e.what());
        return 0;
    }
    // --latency N: the drop-in's per-frame latency with the context reused
    // (lanekit_gpu::Pipeline), host frame in -> lanes out, N calls
    if (argc == 3 && std::strcmp(argv[1], "--latency") == 0) {
        const int n = std::atoi(argv[2]);
        lanekit_gpu::Pipeline pipe(1242, 375, cfg);
        std::vector<double> ms;
        bool same = true;
        for (int i = 0; i < n + 5; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            const lanekit_gpu::Result r = pipe.run(left, disp);
            const auto t1 = std::chrono::steady_clock::now();
            same &= r.report.lane_count == 2 && r.report.lane_bottom_col[0] == 767 &&
                    r.report.lane_bottom_col[1] == 370;
            if (i >= 5) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
        }
        std::sort(ms.begin(), ms.end());
        std::printf("{\"batch1_latency_ms\": {\"median\": %.4f, \"p99\": %.4f, \"min\": %.4f, "
                    "\"calls\": %d, \"lanes_identical\": %s}}\n",
                    ms[ms.size() / 2], ms[std::min(ms.size() - 1, ms.size() * 99 / 100)], ms[0], n,
                    same ? "true" : "false");
    }
    return 0;
}
