// lk_oracle.hpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// CPU restatement of stages 5-12 of lanekit's run_pipeline
// (/root/reference/proj/include/lanekit/pipeline.hpp:184-270) with the
// disparity map injected. Every function cites the reference file:line it
// restates. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
// leg may load this code. Built with -O3 -ffp-contract=off and no -march
// (the reference's Release flags never contract to FMA, CMakeLists.txt:8-10).
//
// Parity pin: oracle/_ref builds the UNMODIFIED reference headers (with a
// stand-in for the absent Eigen3, oracle/eigen_standin/) behind the same C API;
// tests/test_oracle_vs_ref.py and the committed tests/golden/ fixtures check
// this restatement against it bit for bit.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "../include/lanekit_b200.h"

namespace orc {

using Real = double;
inline constexpr Real kPi = 3.14159265358979323846;  // common.hpp:11

// A failed stage: stage number + lk_msg id (+ row for the singular V_py case).
struct Fail {
    int stage;
    int msg;
    int row;
};

// Solver-level failure inside a fit (lanekit::Error thrown by a fit function).
struct FitError {};

using Pt = std::pair<int, int>;  // (axis coordinate, row), as the reference's points

// All intermediates of one frame (PipelineResult, pipeline.hpp:69-99).
struct Result {
    lk_frame_report rep{};
    int W = 0, H = 0, D1 = 0, ext_lo = 0, ext_cols = 0;
    std::vector<int32_t> vdisp;      // [H][D1]
    std::vector<Pt> vpath;           // (d, v)
    std::vector<Pt> beta_inliers;
    std::vector<Real> vpy;           // [H]
    std::vector<uint8_t> vpy_singular;
    std::vector<uint8_t> mask;       // [H][W]
    std::vector<Real> smoothed, gx, gy, mag, theta;  // [H][W]
    std::vector<lk_edge> edges;
    std::vector<lk_vote> votes;
    std::vector<Real> acc;           // [rows][ext_cols]
    std::vector<Pt> upath;           // (ext col, v)
    std::vector<Pt> gamma_inliers;
    std::vector<Real> vpx;           // [H]
    std::vector<Real> m0, m1;        // [H][W]
    std::vector<Real> energy;        // [ext_cols]
    std::vector<lk_lane> lanes;
    std::vector<Real> polylines;     // [lanes][rows], NaN = truncated
};

void run_frame(const uint8_t* grey, const uint8_t* disp, int W, int H, const lk_config& cfg,
               Result& r);

// ---- unit-level restatements exposed for the kernel parity tests
Real dp_min_path(int stages, int states, const Real* data /*[stages][states]*/,
                 const int* offsets, int n_off, const Real* pen_by_offset_index,
                 std::vector<int>& path);
bool fit_parabola(const std::vector<Pt>& pts, Real out[3]);
bool fit_quartic(const std::vector<Pt>& pts, Real kappa, Real v_normalizer, Real out[5],
                 Real* s_out);
struct RansacOut {
    Real model[5] = {0, 0, 0, 0, 0};
    Real s = 0;  // quartic v_normalizer
    std::vector<Pt> inliers;
    int iterations = 0;
    Real fraction = 0;
    bool degraded = false;
};
// kind 3 = parabola (ransac_beta), 5 = quartic (ransac_gamma). Throws Fail{0,msg,0}.
RansacOut ransac(int kind, const std::vector<Pt>& pts, Real tol, Real eps, int max_iter,
                 uint64_t seed);
Real piecewise_weight(Real theta_e, Real theta_vp, Real sigma_g);
void lane_track(Real u_bottom, const Real* vpx, const Real* vpy, int v_top, int v_max,
                Real* track);
Real auto_lane_threshold(const Real* m1, int W, int H, int v_top, int v_max);

}  // namespace orc
