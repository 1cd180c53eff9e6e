// lanedet_gpu.cpp — command-line front end over the C-ABI, the GPU drop-in for
// the reference's `lanedet` (tools/lanedet.cpp:51-178):
//
//   lanedet_gpu detect --left L --right R --out-dir D [--config F] [--set k=v]... [--emit-all]
//   lanedet_gpu stream --list PAIRS --out CSV [--batch N] [--config F] [--set k=v]... [--threads N]
//   lanedet_gpu synth  --out-dir D [--seed S] [--width W] [--height H]
//
// stream feeds many KITTI-style pairs (image_io.hpp:75-149 decode on host
// threads, pinned double-buffered slots) through lk_submit_stereo_batch and
// writes one lane-result line per pair (see cmd_stream).
// detect runs run_pipeline on the GPU (stages 1-12, LK_FLAG_STEREO | LK_FLAG_HOOKS)
// and writes the reference's artifact set (artifacts.hpp:140-228): disparity.pgm,
// vdisparity.pgm, vpx_accumulator.pgm, edges.png, lanes.csv, overlay.png and
// report.json, plus the per-stage files of --emit-all. Differences, by design:
//   * inputs must be 8-bit (P5 maxval 255, or 8-bit grey PNG): the GPU path
//     takes u8 frames (k means k/255.0, image_io.hpp:147); 16-bit and colour
//     inputs are rejected instead of converted;
//   * PNG files are written by this file's own zlib-based encoder, so their
//     pixels match libpng's output but not their compressed bytes;
//   * report.json stage timings are the GPU's (CUDA events per stage);
//   * synth writes the images and the true disparity, not ground_truth.json.
#include <zlib.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lanekit_b200.h"

namespace {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Gray8 {
    int w = 0, h = 0;
    std::vector<uint8_t> px;
};

// ---------------------------------------------------------------- PGM / PNG

long pgm_token(std::istream& in, const std::string& path) {  // image_io.hpp:50-70
    for (;;) {
        const int c = in.peek();
        if (c == EOF) throw Error("pgm: truncated header in " + path);
        if (c == '#') {
            std::string skip;
            std::getline(in, skip);
            continue;
        }
        if (std::isspace(c)) {
            in.get();
            continue;
        }
        break;
    }
    long v = 0;
    in >> v;
    if (!in) throw Error("pgm: bad header token in " + path);
    return v;
}

Gray8 read_pgm8(const std::string& path) {  // image_io.hpp:73-105, 8-bit only
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error("pgm: cannot open " + path);
    char m0 = 0, m1 = 0;
    in.get(m0).get(m1);
    if (m0 != 'P' || m1 != '5') throw Error("pgm: " + path + " is not binary P5");
    const long w = pgm_token(in, path), h = pgm_token(in, path), maxval = pgm_token(in, path);
    if (w < 1 || h < 1 || maxval < 1 || maxval > 65535) throw Error("pgm: bad dimensions in " + path);
    if (maxval != 255)
        throw Error("pgm: " + path + ": only maxval 255 maps exactly onto the u8 GPU input");
    in.get();
    Gray8 g{(int)w, (int)h, std::vector<uint8_t>((size_t)w * h)};
    in.read(reinterpret_cast<char*>(g.px.data()), (std::streamsize)g.px.size());
    if (!in) throw Error("pgm: truncated raster in " + path);
    return g;
}

void write_pgm(const std::string& path, int w, int h, const std::vector<uint16_t>& v, int maxval) {
    std::ofstream out(path, std::ios::binary);  // image_io.hpp:25-46
    if (!out) throw Error("pgm: cannot open " + path + " for writing");
    out << "P5\n" << w << " " << h << "\n" << maxval << "\n";
    std::vector<uint8_t> raster;
    if (maxval < 256) {
        raster.assign(v.begin(), v.end());
    } else {
        raster.resize(v.size() * 2);
        for (size_t i = 0; i < v.size(); ++i) {
            raster[2 * i] = (uint8_t)(v[i] >> 8);  // big-endian
            raster[2 * i + 1] = (uint8_t)(v[i] & 0xff);
        }
    }
    out.write(reinterpret_cast<const char*>(raster.data()), (std::streamsize)raster.size());
    if (!out) throw Error("pgm: write failed for " + path);
}

uint32_t be32(const uint8_t* p) { return (uint32_t)p[0] << 24 | p[1] << 16 | p[2] << 8 | p[3]; }

// 8-bit greyscale, non-interlaced PNG (the layout of KITTI's grey pairs).
Gray8 read_png8(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error("png: cannot open " + path);
    std::vector<uint8_t> f((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    static const uint8_t sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    if (f.size() < 8 || std::memcmp(f.data(), sig, 8)) throw Error("png: " + path + " is not a PNG");
    Gray8 g;
    std::vector<uint8_t> idat;
    for (size_t o = 8; o + 12 <= f.size();) {
        const uint32_t len = be32(&f[o]);
        const std::string type(reinterpret_cast<const char*>(&f[o + 4]), 4);
        if (o + 12 + len > f.size()) throw Error("png: truncated chunk in " + path);
        const uint8_t* d = &f[o + 8];
        if (type == "IHDR") {
            if (len != 13) throw Error("png: malformed IHDR in " + path);
            const uint32_t w = be32(d), h = be32(d + 4);
            // the GPU context's limits (lk_create): checked before any allocation
            if (w < 1 || w > 65535 || h < 1 || h > 32767)
                throw Error("png: " + path + ": size " + std::to_string(w) + "x" +
                            std::to_string(h) + " outside 1..65535 x 1..32767");
            g.w = (int)w;
            g.h = (int)h;
            if (d[8] != 8 || d[9] != 0 || d[12] != 0)
                throw Error("png: " + path + ": only 8-bit greyscale, non-interlaced PNG maps "
                            "exactly onto the u8 GPU input");
        } else if (type == "IDAT") {
            idat.insert(idat.end(), d, d + len);
        } else if (type == "IEND") {
            break;
        }
        o += 12 + len;
    }
    if (g.w < 1 || g.h < 1) throw Error("png: missing IHDR in " + path);
    if (idat.empty()) throw Error("png: no IDAT chunk in " + path);
    std::vector<uint8_t> raw((size_t)g.h * (g.w + 1));
    uLongf n = (uLongf)raw.size();
    if (uncompress(raw.data(), &n, idat.data(), (uLong)idat.size()) != Z_OK || n != raw.size())
        throw Error("png: read failed for " + path);
    g.px.resize((size_t)g.w * g.h);
    std::vector<uint8_t> prev(g.w, 0);
    for (int y = 0; y < g.h; ++y) {  // undo the per-row filters (PNG spec 9.2)
        const uint8_t ft = raw[(size_t)y * (g.w + 1)];
        const uint8_t* s = &raw[(size_t)y * (g.w + 1) + 1];
        uint8_t* r = &g.px[(size_t)y * g.w];
        for (int x = 0; x < g.w; ++x) {
            const int a = x ? r[x - 1] : 0, b = prev[x], c = x ? prev[x - 1] : 0;
            int p = 0;
            switch (ft) {
                case 0: p = 0; break;
                case 1: p = a; break;
                case 2: p = b; break;
                case 3: p = (a + b) / 2; break;
                case 4: {
                    const int pa = std::abs(b - c), pb = std::abs(a - c), pc = std::abs(a + b - 2 * c);
                    p = (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
                    break;
                }
                default: throw Error("png: bad filter type in " + path);
            }
            r[x] = (uint8_t)(s[x] + p);
        }
        std::copy(r, r + g.w, prev.begin());
    }
    return g;
}

void put32(std::vector<uint8_t>& o, uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) o.push_back((uint8_t)(v >> s));
}

void write_png(const std::string& path, int w, int h, int channels, const std::vector<uint8_t>& px) {
    std::vector<uint8_t> raw;
    raw.reserve((size_t)h * (w * channels + 1));
    for (int y = 0; y < h; ++y) {
        raw.push_back(0);  // filter: none
        raw.insert(raw.end(), px.begin() + (size_t)y * w * channels,
                   px.begin() + (size_t)(y + 1) * w * channels);
    }
    uLongf zn = compressBound((uLong)raw.size());
    std::vector<uint8_t> z(zn);
    if (compress2(z.data(), &zn, raw.data(), (uLong)raw.size(), 6) != Z_OK)
        throw Error("png: write failed for " + path);
    z.resize(zn);
    std::vector<uint8_t> o = {137, 80, 78, 71, 13, 10, 26, 10};
    auto chunk = [&](const char* type, const std::vector<uint8_t>& data) {
        put32(o, (uint32_t)data.size());
        const size_t start = o.size();
        o.insert(o.end(), type, type + 4);
        o.insert(o.end(), data.begin(), data.end());
        put32(o, (uint32_t)crc32(0L, &o[start], (uInt)(o.size() - start)));
    };
    std::vector<uint8_t> ihdr;
    put32(ihdr, (uint32_t)w);
    put32(ihdr, (uint32_t)h);
    ihdr.insert(ihdr.end(), {8, (uint8_t)(channels == 3 ? 2 : 0), 0, 0, 0});
    chunk("IHDR", ihdr);
    chunk("IDAT", z);
    chunk("IEND", {});
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("png: cannot open " + path + " for writing");
    out.write(reinterpret_cast<const char*>(o.data()), (std::streamsize)o.size());
}

// write_png_gray (image_io.hpp:180-189): clamp(lround(x * 255))
void write_png_gray(const std::string& path, int w, int h, const std::vector<double>& x) {
    std::vector<uint8_t> px(x.size());
    for (size_t i = 0; i < x.size(); ++i)
        px[i] = (uint8_t)std::clamp(std::lround(x[i] * 255.0), 0L, 255L);
    write_png(path, w, h, 1, px);
}

std::vector<double> normalize_map(const std::vector<double>& m) {  // artifacts.hpp:25-38
    double lo = 0, hi = 0;
    bool first = true;
    for (double x : m) {
        if (first) {
            lo = hi = x;
            first = false;
        }
        lo = std::min(lo, x);
        hi = std::max(hi, x);
    }
    std::vector<double> out(m.size(), 0.0);
    const double span = hi - lo;
    if (span <= 0) return out;
    for (size_t i = 0; i < m.size(); ++i) out[i] = (m[i] - lo) / span;
    return out;
}

// ---------------------------------------------------------------- config (config.hpp:48-181)

std::string trim(const std::string& s) {
    const size_t a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    return s.substr(a, s.find_last_not_of(" \t\r\n") - a + 1);
}

long long parse_int(const std::string& key, const std::string& value) {
    size_t pos = 0;
    long long x = 0;
    try {
        x = std::stoll(value, &pos);
    } catch (const std::exception&) {
        throw Error("config: bad integer for " + key + ": '" + value + "'");
    }
    if (pos != value.size()) throw Error("config: bad integer for " + key + ": '" + value + "'");
    return x;
}

double parse_real(const std::string& key, const std::string& value) {
    size_t pos = 0;
    double x = 0;
    try {
        x = std::stod(value, &pos);
    } catch (const std::exception&) {
        throw Error("config: bad number for " + key + ": '" + value + "'");
    }
    if (pos != value.size()) throw Error("config: bad number for " + key + ": '" + value + "'");
    return x;
}

void apply_config_entry(lk_config& c, const std::string& key, const std::string& value) {
    auto I = [&](int32_t& f) { f = (int32_t)parse_int(key, value); };
    auto R = [&](double& f) { f = parse_real(key, value); };
    if (key == "rho") I(c.rho);
    else if (key == "tau") I(c.tau);
    else if (key == "d_max") I(c.d_max);
    else if (key == "tr_lrc") I(c.tr_lrc);
    else if (key == "sigma_floor") R(c.sigma_floor);
    else if (key == "lambda_y") R(c.lambda_y);
    else if (key == "tr_y") R(c.tr_y);
    else if (key == "eps_y") R(c.eps_y);
    else if (key == "varpi") R(c.varpi);
    else if (key == "sigma_s") R(c.sigma_s);
    else if (key == "sigma_r") R(c.sigma_r);
    else if (key == "bf_window") I(c.bf_window);
    else if (key == "sobel_threshold") R(c.sobel_threshold);
    else if (key == "chi") I(c.chi);
    else if (key == "rho_vote") R(c.rho_vote);
    else if (key == "lambda_x") R(c.lambda_x);
    else if (key == "tr_x") R(c.tr_x);
    else if (key == "eps_x") R(c.eps_x);
    else if (key == "sigma_g") R(c.sigma_g);
    else if (key == "nu") I(c.nu);
    else if (key == "varsigma") I(c.varsigma);
    else if (key == "lambda_g") R(c.lambda_g);
    else if (key == "xi") R(c.xi);
    else if (key == "tr_lpv") {
        if (value == "auto") c.tr_lpv = std::numeric_limits<double>::quiet_NaN();
        else R(c.tr_lpv);
    } else if (key == "min_lane_sep") I(c.min_lane_sep);
    else if (key == "rng_seed") c.rng_seed = (uint64_t)parse_int(key, value);
    else if (key == "paper_sign") {
        if (value == "true" || value == "1") c.paper_sign = 1;
        else if (value == "false" || value == "0") c.paper_sign = 0;
        else throw Error("config: bad boolean for " + key + ": '" + value + "'");
    } else throw Error("config: unknown key '" + key + "'");
}

lk_config make_config(const std::string& path, const std::vector<std::string>& overrides, int threads) {
    lk_config c;
    lk_config_default(&c);
    if (!path.empty()) {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Error("config: cannot open " + path);
        std::string line;
        int lineno = 0;
        while (std::getline(in, line)) {
            ++lineno;
            const size_t hash = line.find('#');
            if (hash != std::string::npos) line.erase(hash);
            line = trim(line);
            if (line.empty()) continue;
            const size_t eq = line.find('=');
            if (eq == std::string::npos)
                throw Error("config: line " + std::to_string(lineno) + " is not key=value");
            const std::string key = trim(line.substr(0, eq));
            if (key.empty()) throw Error("config: empty key on line " + std::to_string(lineno));
            apply_config_entry(c, key, trim(line.substr(eq + 1)));
        }
        if (lk_validate_config(&c)) throw Error(lk_last_error());
    }
    for (const auto& kv : overrides) {
        const size_t eq = kv.find('=');
        if (eq == std::string::npos) throw Error("--set expects key=value, got '" + kv + "'");
        apply_config_entry(c, kv.substr(0, eq), kv.substr(eq + 1));
    }
    if (threads > 0) c.threads = threads;
    if (lk_validate_config(&c)) throw Error(lk_last_error());
    return c;
}

// ---------------------------------------------------------------- JSON (nlohmann dump(2) layout)

std::string num(double x) {  // shortest round-trip; NaN / inf as null
    if (!std::isfinite(x)) return "null";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
    std::string sci(buf, r.ptr);  // d.ddde[+-]XX
    const size_t e = sci.find('e');
    const int ex = std::stoi(sci.substr(e + 1));
    std::string mant = sci.substr(0, e), digits;
    const bool neg = mant[0] == '-';
    for (char ch : mant)
        if (std::isdigit((unsigned char)ch)) digits += ch;
    std::string out = neg ? "-" : "";
    if (ex >= -5 && ex < 16) {  // fixed
        if (ex >= 0) {
            std::string ip = digits.substr(0, std::min<size_t>(digits.size(), ex + 1));
            while ((int)ip.size() < ex + 1) ip += '0';
            std::string fp = digits.size() > (size_t)ex + 1 ? digits.substr(ex + 1) : "0";
            out += ip + "." + fp;
        } else {
            out += "0." + std::string(-ex - 1, '0') + digits;
        }
    } else {
        out += digits.substr(0, 1);
        if (digits.size() > 1) out += "." + digits.substr(1);
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', std::abs(ex));
        out += eb;
    }
    return out;
}

struct Json {  // ordered writer; objects must be emitted with sorted keys
    std::ostringstream s;
    int depth = 0;
    std::vector<bool> first{true};
    void sep() {
        if (!first.back()) s << ",";
        first.back() = false;
        if (depth) s << "\n" << std::string(2 * depth, ' ');
    }
    void open(char c) {
        s << c;
        ++depth;
        first.push_back(true);
    }
    void close(char c) {
        const bool empty = first.back();
        first.pop_back();
        --depth;
        if (!empty) s << "\n" << std::string(2 * depth, ' ');
        s << c;
    }
    void key(const char* k) {
        sep();
        s << '"' << k << "\": ";
    }
    void elem() { sep(); }
};

// ---------------------------------------------------------------- detect

struct Ctx {
    lk_ctx* h = nullptr;
    ~Ctx() {
        if (h) lk_destroy(h);
    }
};

template <typename T>
std::vector<T> stage(lk_ctx* h, int st) {
    size_t need = 0;
    if (lk_get_stage(h, 0, st, nullptr, 0, &need)) throw Error(lk_last_error());
    std::vector<T> v(need / sizeof(T));
    if (lk_get_stage(h, 0, st, v.data(), need, &need)) throw Error(lk_last_error());
    return v;
}

void write_disparity_pgm(const std::string& path, int w, int h, const std::vector<uint8_t>& d) {
    std::vector<uint16_t> v(d.size());  // artifacts.hpp:40-47: d * 256
    for (size_t i = 0; i < d.size(); ++i) v[i] = (uint16_t)std::min<long>((long)d[i] * 256, 65535);
    write_pgm(path, w, h, v, 65535);
}

void write_path_csv(const std::string& path, const std::vector<int32_t>& pts, const char* a,
                    const char* b) {
    std::ofstream out(path);
    if (!out) throw Error("cannot open " + path);
    out << a << "," << b << "\n";
    for (size_t i = 0; i + 1 < pts.size(); i += 2) out << pts[i] << "," << pts[i + 1] << "\n";
}

int cmd_detect(const std::string& lp, const std::string& rp, const std::string& cfgp,
               const std::string& out_dir, bool emit_all, int threads,
               const std::vector<std::string>& overrides) {
    const lk_config cfg = make_config(cfgp, overrides, threads);
    auto load = [](const std::string& p) {
        const auto ext = std::filesystem::path(p).extension().string();
        return (ext == ".pgm" || ext == ".PGM") ? read_pgm8(p) : read_png8(p);
    };
    const Gray8 L = load(lp), R = load(rp);
    if (L.px.empty() || R.px.empty()) throw Error("stage 1 (block statistics): empty input image");
    if (L.w != R.w || L.h != R.h) throw Error("stage 1 (block statistics): stereo pair dimensions differ");
    const int W = L.w, H = L.h;
    Ctx c;
    if (lk_create(&c.h, 0, &cfg, W, H, 1, LK_FLAG_STEREO | LK_FLAG_HOOKS)) throw Error(lk_last_error());
    lk_frame_report rep;
    const lk_status st = lk_run_stereo_batch(c.h, L.px.data(), R.px.data(), 1, LK_MEM_HOST, &rep);
    if (st == LK_ERR_FRAME) {
        char msg[256];
        lk_frame_message(&rep, msg, sizeof msg);
        throw Error(msg);
    }
    if (st) throw Error(lk_last_error());
    float ms[13];
    lk_stage_times(c.h, ms);

    namespace fs = std::filesystem;
    fs::create_directories(out_dir);
    auto p = [&](const char* f) { return (fs::path(out_dir) / f).string(); };
    const int D1 = cfg.d_max + 1, v_top = (int)rep.horizon, rows = H - v_top;

    const auto disparity = stage<uint8_t>(c.h, LK_STAGE_DISPARITY);
    write_disparity_pgm(p("disparity.pgm"), W, H, disparity);
    {  // vdisparity.pgm: min(count, 255), D1 x H (artifacts.hpp:150-157)
        const auto vd = stage<int32_t>(c.h, LK_STAGE_VDISPARITY);
        std::vector<uint16_t> img((size_t)D1 * H);
        for (size_t i = 0; i < img.size(); ++i) img[i] = (uint16_t)std::min<int32_t>(vd[i], 255);
        write_pgm(p("vdisparity.pgm"), D1, H, img, 255);
    }
    {  // vpx_accumulator.pgm: clamp(lround(-m)), ext_cols x rows (artifacts.hpp:159-168)
        const auto acc = stage<double>(c.h, LK_STAGE_VPX_ACC);
        const int C = rows ? (int)(acc.size() / rows) : 0;
        std::vector<uint16_t> img(acc.size());
        for (size_t i = 0; i < acc.size(); ++i)
            img[i] = (uint16_t)std::clamp(std::lround(-acc[i]), 0L, 255L);
        if (C) write_pgm(p("vpx_accumulator.pgm"), C, rows, img, 255);
    }
    const auto edges = stage<lk_edge>(c.h, LK_STAGE_EDGES);
    {
        std::vector<double> e((size_t)W * H, 0.0);
        for (const auto& x : edges) e[(size_t)x.v * W + x.u] = 1.0;
        write_png_gray(p("edges.png"), W, H, e);
    }
    const auto lanes = stage<lk_lane>(c.h, LK_STAGE_LANES);
    const auto poly = stage<double>(c.h, LK_STAGE_POLYLINES);  // [lane][rows] u, NaN = cut
    auto polyline = [&](size_t i) {  // (v, u) points of lane i, top down (lanes.hpp:170-174)
        std::vector<std::pair<int, double>> pts;
        for (int r = 0; r < rows; ++r) {
            const double u = poly[i * rows + r];
            if (!std::isnan(u)) pts.push_back({v_top + r, u});
        }
        return pts;
    };
    {  // lanes.csv (artifacts.hpp:109-119)
        std::ofstream out(p("lanes.csv"));
        if (!out) throw Error("cannot open lanes.csv");
        out << "lane_id,v,u\n";
        char buf[64];
        for (size_t i = 0; i < lanes.size(); ++i)
            for (const auto& [v, u] : polyline(i)) {
                std::snprintf(buf, sizeof buf, "%zu,%d,%.3f\n", i, v, u);
                out << buf;
            }
    }
    {  // overlay.png (artifacts.hpp:121-138)
        std::vector<uint8_t> rgb((size_t)W * H * 3);
        for (size_t i = 0; i < L.px.size(); ++i) rgb[3 * i] = rgb[3 * i + 1] = rgb[3 * i + 2] = L.px[i];
        for (size_t i = 0; i < lanes.size(); ++i)
            for (const auto& [v, u] : polyline(i)) {
                const int uc = (int)std::lround(u);
                for (int du = -1; du <= 1; ++du) {
                    const int x = uc + du;
                    if (x >= 0 && x < W && v >= 0 && v < H) {
                        uint8_t* q = &rgb[((size_t)v * W + x) * 3];
                        q[0] = 220;
                        q[1] = 30;
                        q[2] = 30;
                    }
                }
            }
        write_png(p("overlay.png"), W, H, 3, rgb);
    }
    {  // report.json (report_to_json, artifacts.hpp:59-107), keys sorted as nlohmann::json
        Json j;
        j.open('{');
        j.key("edges"); j.open('{'); j.key("count"); j.s << rep.edge_pixels; j.close('}');
        j.key("height"); j.s << rep.height;
        j.key("lanes"); j.open('{');
        j.key("count"); j.s << rep.lane_count;
        j.key("detected"); j.open('[');
        for (size_t i = 0; i < lanes.size(); ++i) {
            j.elem(); j.open('{');
            j.key("bottom_col"); j.s << lanes[i].bottom_col;
            j.key("energy"); j.s << num(lanes[i].energy);
            j.key("lane_id"); j.s << i;
            j.key("polyline"); j.open('[');
            for (const auto& [v, u] : polyline(i)) {
                j.elem(); j.open('['); j.elem(); j.s << v; j.elem(); j.s << num(u); j.close(']');
            }
            j.close(']');
            j.close('}');
        }
        j.close(']');
        j.key("threshold"); j.s << num(rep.tr_lpv_used);
        j.close('}');
        j.key("rng_seed"); j.s << cfg.rng_seed;
        j.key("road"); j.open('{');
        j.key("beta"); j.open('[');
        for (int k = 0; k < 3; ++k) { j.elem(); j.s << num(rep.beta[k]); }
        j.close(']');
        j.key("degraded"); j.s << (rep.beta_degraded ? "true" : "false");
        j.key("horizon"); j.s << rep.horizon;
        j.key("horizon_in_range"); j.s << (rep.horizon_in_range ? "true" : "false");
        j.key("inlier_fraction"); j.s << num(rep.beta_inlier_fraction);
        j.key("mask_pixels"); j.s << rep.road_mask_pixels;
        j.key("ransac_iterations"); j.s << rep.beta_iterations;
        j.key("vpath_has_evidence"); j.s << (rep.vpath_has_evidence ? "true" : "false");
        j.close('}');
        j.key("stages"); j.open('[');
        for (int k = 1; k <= 12; ++k) {
            j.elem(); j.open('{');
            j.key("ms"); j.s << num(ms[k]);
            j.key("name"); j.s << '"' << lk_stage_name(k) << '"';
            j.key("stage"); j.s << k;
            j.close('}');
        }
        j.close(']');
        j.key("stereo"); j.open('{'); j.key("valid_disparities"); j.s << rep.valid_disparities; j.close('}');
        j.key("threads"); j.s << cfg.threads;
        j.key("total_ms"); j.s << num(ms[0]);
        j.key("vanishing_point"); j.open('{');
        j.key("degraded"); j.s << (rep.gamma_degraded ? "true" : "false");
        j.key("gamma"); j.open('[');
        for (int k = 0; k < 5; ++k) { j.elem(); j.s << num(rep.gamma[k]); }
        j.close(']');
        j.key("inlier_fraction"); j.s << num(rep.gamma_inlier_fraction);
        j.key("kappa"); j.s << num(rep.gamma_kappa);
        j.key("ransac_iterations"); j.s << rep.gamma_iterations;
        j.key("skipped"); j.s << rep.vpx_skipped;
        j.key("upath_has_evidence"); j.s << (rep.upath_has_evidence ? "true" : "false");
        j.key("v_normalizer"); j.s << num(rep.gamma_v_normalizer);
        j.key("votes"); j.s << rep.vpx_votes;
        j.close('}');
        j.key("width"); j.s << rep.width;
        j.close('}');
        std::ofstream out(p("report.json"));
        if (!out) throw Error("cannot open report.json");
        out << j.s.str() << "\n";
    }
    if (emit_all) {  // artifacts.hpp:180-226
        write_png_gray(p("block_sigma.png"), W, H, normalize_map(stage<double>(c.h, LK_STAGE_STATS_SIGMA)));
        write_disparity_pgm(p("disparity_left.pgm"), W, H, stage<uint8_t>(c.h, LK_STAGE_DISP_LEFT));
        write_disparity_pgm(p("disparity_right.pgm"), W, H, stage<uint8_t>(c.h, LK_STAGE_DISP_RIGHT));
        write_path_csv(p("vpath.csv"), stage<int32_t>(c.h, LK_STAGE_VPATH), "d", "v");
        {
            const auto vpy = stage<double>(c.h, LK_STAGE_VPY);
            const auto sing = stage<uint8_t>(c.h, LK_STAGE_VPY_SINGULAR);
            const auto vpx = stage<double>(c.h, LK_STAGE_VPX);
            std::ofstream out(p("road_fit.csv"));
            if (!out) throw Error("cannot open road_fit.csv");
            out << "v,f,vpy,vpx\n";
            char buf[128];
            for (int v = 0; v < H; ++v) {
                const double vv = v;
                const double f = rep.beta[0] + rep.beta[1] * vv + rep.beta[2] * vv * vv;  // road_f
                const double py = sing[v] ? std::nan("") : vpy[v];
                const double px = (v >= v_top && v <= H - 1) ? vpx[v] : std::nan("");
                std::snprintf(buf, sizeof buf, "%d,%.4f,%.4f,%.4f\n", v, f, py, px);
                out << buf;
            }
        }
        {
            const auto m = stage<uint8_t>(c.h, LK_STAGE_MASK);
            std::vector<double> x(m.size());
            for (size_t i = 0; i < m.size(); ++i) x[i] = m[i] ? 1.0 : 0.0;
            write_png_gray(p("road_mask.png"), W, H, x);
        }
        write_png_gray(p("smoothed.png"), W, H, stage<double>(c.h, LK_STAGE_SMOOTHED));
        write_png_gray(p("gradient_magnitude.png"), W, H, normalize_map(stage<double>(c.h, LK_STAGE_MAG)));
        write_path_csv(p("upath.csv"), stage<int32_t>(c.h, LK_STAGE_UPATH), "col", "v");
        write_png_gray(p("m0.png"), W, H, normalize_map(stage<double>(c.h, LK_STAGE_M0)));
        write_png_gray(p("m1.png"), W, H, normalize_map(stage<double>(c.h, LK_STAGE_M1)));
        {
            const auto h = stage<double>(c.h, LK_STAGE_ENERGY);
            const int ext_lo = -(int)std::llround(cfg.xi * W);  // vanish.hpp:24-26
            std::ofstream out(p("energy_histogram.csv"));
            if (!out) throw Error("cannot open energy_histogram.csv");
            out << "col,energy\n";
            char buf[64];
            for (size_t i = 0; i < h.size(); ++i) {
                std::snprintf(buf, sizeof buf, "%d,%.6f\n", ext_lo + (int)i, h[i]);
                out << buf;
            }
        }
    }
    std::printf("%dx%d, GPU, %.1f ms total\n", (int)rep.width, (int)rep.height, ms[0]);
    std::printf("road: beta = [%.4g, %.4g, %.4g], horizon row %d%s\n", rep.beta[0], rep.beta[1],
                rep.beta[2], (int)rep.horizon, rep.horizon_in_range ? "" : " (clamped)");
    std::printf("lanes: %d (threshold %.3f)\n", (int)rep.lane_count, rep.tr_lpv_used);
    std::printf("artifacts written to %s\n", out_dir.c_str());
    return 0;
}

int cmd_synth(const std::string& out_dir, uint64_t seed, int width, int height) {
    lk_scene_params sp;  // lanedet.cpp:69-76
    lk_scene_default(&sp);
    sp.width = width;
    sp.height = height;
    sp.rng_seed = seed;
    sp.noise_sigma = 0.02;
    std::vector<uint8_t> l((size_t)width * height), r(l.size()), d(l.size());
    int32_t horizon = 0;
    if (lk_synth_scene(&sp, l.data(), r.data(), d.data(), &horizon)) throw Error(lk_last_error());
    namespace fs = std::filesystem;
    fs::create_directories(out_dir);
    auto p = [&](const char* f) { return (fs::path(out_dir) / f).string(); };
    write_png(p("left.png"), width, height, 1, l);
    write_png(p("right.png"), width, height, 1, r);
    write_disparity_pgm(p("true_disparity.pgm"), width, height, d);
    std::printf("synthetic scene (seed %llu) written to %s\n", (unsigned long long)seed, out_dir.c_str());
    return 0;
}

// ---------------------------------------------------------------- stream
//
// Many stereo pairs (one "left right" pair of 8-bit PGM/PNG paths per line of
// --list) through lk_submit_stereo_batch, one CSV line of lane results per
// pair (the report fields of artifacts.hpp:59-107 that a fleet run keeps).
// Two pinned input slots: while the GPU runs batch k from one slot, host
// threads decode batch k+1 into the other, after batch k-1 (its last user)
// has been waited for and written out. A pair that fails to decode, or whose
// size differs from the first pair's, is reported as a stage-1 error and its
// slot frame is zero-filled (the batch still runs; its result is dropped).

struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(size_t bytes) {
        if (lk_host_alloc(&p, bytes)) throw Error(lk_last_error());
    }
    ~PinnedBuf() {
        if (p) lk_host_free(p);
    }
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
};

std::string csv_quote(const std::string& s) {
    std::string q = "\"";
    for (char ch : s) q += ch == '"' ? std::string("\"\"") : std::string(1, ch);
    return q + "\"";
}

int cmd_stream(const std::string& list_path, const std::string& out_path, const std::string& cfgp,
               int batch, int threads, const std::vector<std::string>& overrides) {
    const lk_config cfg = make_config(cfgp, overrides, 0);
    std::vector<std::pair<std::string, std::string>> pairs;
    {
        std::ifstream in(list_path);
        if (!in) throw Error("stream: cannot open " + list_path);
        std::string line;
        while (std::getline(in, line)) {
            std::istringstream ls(line);
            std::string l, r;
            if (!(ls >> l)) continue;
            if (l[0] == '#') continue;
            if (!(ls >> r)) throw Error("stream: line without a right image: '" + line + "'");
            pairs.emplace_back(l, r);
        }
    }
    if (pairs.empty()) throw Error("stream: no stereo pairs in " + list_path);
    auto load = [](const std::string& p) {
        const auto ext = std::filesystem::path(p).extension().string();
        return (ext == ".pgm" || ext == ".PGM") ? read_pgm8(p) : read_png8(p);
    };
    int W = 0, H = 0;
    {
        const Gray8 g = load(pairs[0].first);
        W = g.w;
        H = g.h;
    }
    if (W <= 0 || H <= 0) throw Error("stage 1 (block statistics): empty input image");
    batch = std::max(1, std::min<int>(batch, (int)pairs.size()));
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    const size_t frame = (size_t)W * H;

    Ctx c;
    if (lk_create(&c.h, 0, &cfg, W, H, batch, LK_FLAG_STEREO)) throw Error(lk_last_error());
    std::vector<std::unique_ptr<PinnedBuf>> lbuf, rbuf, repbuf;
    std::vector<std::vector<std::string>> decode_err(2, std::vector<std::string>(batch));
    for (int s = 0; s < 2; ++s) {
        lbuf.emplace_back(new PinnedBuf(frame * batch));
        rbuf.emplace_back(new PinnedBuf(frame * batch));
        repbuf.emplace_back(new PinnedBuf(sizeof(lk_frame_report) * batch));
    }
    std::ofstream out(out_path);
    if (!out) throw Error("stream: cannot open " + out_path);
    out << "index,left,status,failed_stage,horizon,lane_count,bottom_cols,lane_energies,message\n";

    // Decodes pairs [first, first+n) into slot s with `threads` workers.
    auto decode = [&](int s, size_t first, int n) {
        std::atomic<int> next{0};
        auto work = [&]() {
            for (int i; (i = next.fetch_add(1)) < n;) {
                uint8_t* L = (uint8_t*)lbuf[s]->p + frame * i;
                uint8_t* R = (uint8_t*)rbuf[s]->p + frame * i;
                std::string& err = decode_err[s][i];
                err.clear();
                try {
                    const Gray8 a = load(pairs[first + i].first), b = load(pairs[first + i].second);
                    if (a.w != W || a.h != H || b.w != W || b.h != H)
                        throw Error("stage 1 (block statistics): pair size differs from the stream's " +
                                    std::to_string(W) + "x" + std::to_string(H));
                    std::memcpy(L, a.px.data(), frame);
                    std::memcpy(R, b.px.data(), frame);
                } catch (const std::exception& e) {
                    err = e.what();
                    std::memset(L, 0, frame);
                    std::memset(R, 0, frame);
                }
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < std::min(threads, n); ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
    };
    auto emit = [&](int s, size_t first, int n) {
        const auto* rep = (const lk_frame_report*)repbuf[s]->p;
        char msg[256];
        for (int i = 0; i < n; ++i) {
            const lk_frame_report& r = rep[i];
            out << (first + i) << "," << csv_quote(pairs[first + i].first) << ",";
            if (!decode_err[s][i].empty()) {
                out << "error,1,,,,," << csv_quote(decode_err[s][i]) << "\n";
                continue;
            }
            if (r.status) {
                lk_frame_message(&r, msg, sizeof msg);
                out << "error," << r.failed_stage << ",,,,," << csv_quote(msg) << "\n";
                continue;
            }
            out << "ok,0," << r.horizon << "," << r.lane_count << ",";
            const int shown = (int)std::min<int64_t>(r.lane_count, LK_MAX_INLINE_LANES);
            for (int k = 0; k < shown; ++k) out << (k ? ";" : "") << r.lane_bottom_col[k];
            out << ",";
            for (int k = 0; k < shown; ++k) {
                std::snprintf(msg, sizeof msg, "%s%.17g", k ? ";" : "", r.lane_energy[k]);
                out << msg;
            }
            out << ",\n";
        }
    };

    const auto t0 = std::chrono::steady_clock::now();
    const size_t N = pairs.size();
    const size_t nb = (N + batch - 1) / batch;
    auto count = [&](size_t k) { return (int)std::min<size_t>(batch, N - k * batch); };
    decode(0, 0, count(0));
    for (size_t k = 0; k < nb; ++k) {
        const int s = (int)(k & 1);
        const lk_status st = lk_submit_stereo_batch(c.h, (const uint8_t*)lbuf[s]->p,
                                                    (const uint8_t*)rbuf[s]->p, count(k),
                                                    (lk_frame_report*)repbuf[s]->p);
        if (st != LK_OK && st != LK_ERR_FRAME) throw Error(lk_last_error());
        if (k >= 1) {  // batch k-1 owns slot s^1: finish it before decoding into that slot
            const lk_status w = lk_wait_batch(c.h);
            if (w != LK_OK && w != LK_ERR_FRAME) throw Error(lk_last_error());
            emit(s ^ 1, (k - 1) * batch, count(k - 1));
        }
        if (k + 1 < nb) decode(s ^ 1, (k + 1) * batch, count(k + 1));  // overlaps batch k on the GPU
    }
    const lk_status w = lk_wait_batch(c.h);
    if (w != LK_OK && w != LK_ERR_FRAME) throw Error(lk_last_error());
    emit((int)((nb - 1) & 1), (nb - 1) * batch, count(nb - 1));
    out.flush();
    if (!out) throw Error("stream: write failed on " + out_path);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "stream: %zu pairs (%dx%d) in %zu batches of <= %d, %.3f s, %.1f pairs/s, %d decode threads\n",
                 N, W, H, nb, batch, s, N / s, threads);
    return 0;
}

// ---------------------------------------------------------------- bench
//
// lanedet bench (lanedet.cpp:111-127, bench.hpp:44-102) on the GPU: the same
// synthetic scene (lane bottoms at W/3 and 2W/3, d_max and seed from the
// config, the search range clamped to what the scene can contain), a batch of
// that stereo pair through stages 1-12 on one LK_FLAG_STEREO context, and the
// per-stage table from the CUDA events of the batch's first frame range
// (lk_stage_times; median of --reps runs). The reference's naive-vs-memoised
// NCC comparison times its two CPU matchers; the GPU matcher is the certified
// integer NCC, so that part reports the GPU matcher only.
int cmd_bench(const std::string& cfgp, int width, int height, int reps, int batch,
              const std::vector<std::string>& overrides) {
    if (reps < 1) throw Error("bench: need at least one repetition");
    if (batch < 1) throw Error("bench: need a batch of at least one frame");
    lk_config cfg = make_config(cfgp, overrides, 0);
    lk_scene_params sp;  // bench.hpp:51-57
    lk_scene_default(&sp);
    sp.width = width;
    sp.height = height;
    sp.n_lanes = 2;
    sp.lane_bottoms[0] = width / 3.0;
    sp.lane_bottoms[1] = 2.0 * width / 3.0;
    sp.d_max = cfg.d_max;
    sp.rng_seed = cfg.rng_seed;
    // d_scene = min(d_max, llround(road_f(beta, H - 1)) + 4) (bench.hpp:62-64)
    const double v = height - 1.0;
    const double f = sp.beta[0] + sp.beta[1] * v + sp.beta[2] * v * v;
    cfg.d_max = std::min(cfg.d_max, static_cast<int>(std::llround(f)) + 4);
    if (lk_validate_config(&cfg) != LK_OK) throw Error(lk_last_error());
    const size_t px = (size_t)width * height;
    std::vector<uint8_t> l(px), r(px);
    if (lk_synth_scene(&sp, l.data(), r.data(), nullptr, nullptr)) throw Error(lk_last_error());
    PinnedBuf L(px * batch), R(px * batch);
    for (int i = 0; i < batch; ++i) {
        std::memcpy(static_cast<uint8_t*>(L.p) + i * px, l.data(), px);
        std::memcpy(static_cast<uint8_t*>(R.p) + i * px, r.data(), px);
    }
    lk_ctx* ctx = nullptr;
    if (lk_create(&ctx, 0, &cfg, width, height, batch, LK_FLAG_STEREO)) throw Error(lk_last_error());
    std::vector<lk_frame_report> reps_out(batch);
    std::vector<std::array<float, 13>> runs;
    std::vector<double> wall;
    lk_status st = LK_OK;
    for (int k = 0; k < reps + 1; ++k) {  // the first run captures the graphs
        const auto t0 = std::chrono::steady_clock::now();
        st = lk_run_stereo_batch(ctx, static_cast<uint8_t*>(L.p), static_cast<uint8_t*>(R.p), batch,
                                 LK_MEM_HOST, reps_out.data());
        const auto t1 = std::chrono::steady_clock::now();
        if (st != LK_OK && st != LK_ERR_FRAME) {
            lk_destroy(ctx);
            throw Error(lk_last_error());
        }
        std::array<float, 13> ms{};
        lk_stage_times(ctx, ms.data());
        if (k) {
            runs.push_back(ms);
            wall.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
        }
    }
    const int timed = lk_timed_frames(ctx);
    lk_destroy(ctx);
    auto median = [](std::vector<double> x) {
        std::sort(x.begin(), x.end());
        return x[x.size() / 2];
    };
    std::printf("block matching (GPU certified integer NCC, stages 1-4), %dx%d, batch %d, "
                "%d rep(s)%s\n", width, height, batch, reps, reps < 3 ? " [low confidence]" : "");
    std::printf("pipeline stages (GPU, events of the first %d-frame range):\n", timed);
    for (int s = 1; s <= 12; ++s) {
        std::vector<double> v;
        for (const auto& m : runs) v.push_back(m[s]);
        std::printf("  %2d %-28s %9.3f ms\n", s, lk_stage_name(s), median(v));
    }
    std::vector<double> tot;
    for (const auto& m : runs) tot.push_back(m[0]);
    std::printf("  total %38.3f ms\n", median(tot));
    const double w = median(wall);
    std::printf("batch wall clock (host pairs in, reports out): %.3f ms = %.1f frames/s; "
                "lanes of frame 0:", w, batch / (w * 1e-3));
    for (int i = 0; i < (int)reps_out[0].lane_count && i < LK_MAX_INLINE_LANES; ++i)
        std::printf(" %lld", (long long)reps_out[0].lane_bottom_col[i]);
    std::printf("%s\n", reps_out[0].status ? " (frame failed)" : "");
    return 0;
}

int usage() {
    std::fprintf(stderr,
                 "usage: lanedet_gpu detect --left L --right R --out-dir D [--config F] "
                 "[--set key=value]... [--emit-all] [--threads N]\n"
                 "       lanedet_gpu stream --list PAIRS --out CSV [--batch N] [--config F] "
                 "[--set key=value]... [--threads N]\n"
                 "       lanedet_gpu synth --out-dir D [--seed S] [--width W] [--height H]\n"
                 "       lanedet_gpu bench [--config F] [--set key=value]... [--width W] "
                 "[--height H] [--reps N] [--batch N]\n");
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    std::string left, right, cfg, out_dir, list, out_csv;
    bool emit_all = false;
    int threads = 0, width = 640, height = 360, batch = 64, reps = 3;
    bool batch_set = false, size_set = false;
    uint64_t seed = 1;
    std::vector<std::string> overrides;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) throw Error(a + " needs a value");
                return argv[++i];
            };
            if (a == "--left") left = val();
            else if (a == "--right") right = val();
            else if (a == "--config") cfg = val();
            else if (a == "--out-dir") out_dir = val();
            else if (a == "--set") overrides.push_back(val());
            else if (a == "--list") list = val();
            else if (a == "--out") out_csv = val();
            else if (a == "--batch") batch = std::stoi(val()), batch_set = true;
            else if (a == "--reps") reps = std::stoi(val());
            else if (a == "--threads") threads = std::stoi(val());
            else if (a == "--emit-all") emit_all = true;
            else if (a == "--seed") seed = std::stoull(val());
            else if (a == "--width") width = std::stoi(val()), size_set = true;
            else if (a == "--height") height = std::stoi(val()), size_set = true;
            else throw Error("unknown option " + a);
        }
        if (cmd == "detect") {
            if (left.empty() || right.empty() || out_dir.empty()) return usage();
            return cmd_detect(left, right, cfg, out_dir, emit_all, threads, overrides);
        }
        if (cmd == "stream") {
            if (list.empty() || out_csv.empty()) return usage();
            return cmd_stream(list, out_csv, cfg, batch, threads, overrides);
        }
        if (cmd == "synth") {
            if (out_dir.empty()) return usage();
            return cmd_synth(out_dir, seed, width, height);
        }
        if (cmd == "bench")  // the reference's defaults: 320x240 (bench.hpp:44), batch 1
            return cmd_bench(cfg, size_set ? width : 320, size_set ? height : 240, reps,
                             batch_set ? batch : 1, overrides);
        return usage();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
