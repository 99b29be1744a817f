// wavelift_b200.hpp -- C++ drop-in for the reference transform API.
//
// Mirrors /root/reference/proj/include/wavelift/transform.hpp:14-95 (Image,
// QuadGrid, BoundaryMode, resolve_index, polyphase_split/merge, forward,
// inverse, PyramidLevel, Pyramid, multi_level_forward/inverse, worker_count),
// schemes.hpp:15-62 (SchemeKind, scheme_name, parse_scheme, Scheme,
// build_scheme, count_macs, count_barriers), wavelets.hpp:21-32 (WaveletSpec,
// get_wavelet) and subband_io.hpp:45-46 (boundary_name, parse_boundary), with
// the same value semantics (host float64 buffers) and the same exception
// classes. Scheme carries its step sequence (Step{matrix, needs_barrier,
// label}, schemes.hpp:34-45) and Convolution filters, read from the
// library's build_scheme tables; apply_step (transform.hpp:57-60) runs one
// StepMatrix on the GPU. Every transform runs on the GPU through the C-ABI of wl_dwt.h:
// samples are converted to float32, copied to device memory, transformed by
// the sm_100a kernels and copied back. There is no CPU fallback.
//
// Header-only; link with libwavelift_b200.so and libcudart.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstddef>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <vector>

#include "wl_dwt.h"

namespace wavelift {
inline namespace b200 {

struct Image {
    int width = 0;
    int height = 0;
    std::vector<double> samples;  // row-major, height*width
    Image() = default;
    Image(int w, int h) : width(w), height(h), samples(static_cast<std::size_t>(w) * h, 0.0) {}
    double& at(int r, int c) { return samples[static_cast<std::size_t>(r) * width + c]; }
    double at(int r, int c) const { return samples[static_cast<std::size_t>(r) * width + c]; }
};

enum Component : int { LL = 0, HL = 1, LH = 2, HH = 3 };

struct QuadGrid {
    int w = 0, h = 0;
    std::array<std::vector<double>, 4> planes;  // LL, HL, LH, HH
    QuadGrid() = default;
    QuadGrid(int w_, int h_) : w(w_), h(h_) {
        for (auto& p : planes) p.assign(static_cast<std::size_t>(w) * h, 0.0);
    }
    double& at(int comp, int r, int c) { return planes[comp][static_cast<std::size_t>(r) * w + c]; }
    double at(int comp, int r, int c) const {
        return planes[comp][static_cast<std::size_t>(r) * w + c];
    }
};

enum class BoundaryMode { periodic, symmetric };

enum class SchemeKind {
    Sweldens, Iwahashi, IwahashiStar, Explosive, ExplosiveStar,
    Monolithic, MonolithicStar, Polyphase, PolyphaseStar, Convolution,
};

struct WaveletSpec {
    std::string name;
    int id = 0;        // WL_CDF53 / WL_CDF97 / WL_DD137
    double zeta = 1.0;
};

// polyphase.hpp:24-38
enum class MatrixKind { T_H, T_V, S_H, S_V, T_I, R_I, S_I, T_E, R_E, S_E, T_MONO, S_MONO, N_FULL };

// laurent.hpp:75-115, reduced to what a step-walking caller reads: the terms
// c * z_m^km * z_n^kn of one matrix entry, keyed (k_m, k_n) in map order,
// coefficients as double (the reference's Coeff::to_double()).
struct LaurentPoly2 {
    using Exp = std::pair<int, int>;
    std::map<Exp, double> terms_;
    const std::map<Exp, double>& terms() const { return terms_; }
    bool is_zero() const { return terms_.empty(); }
    bool is_one() const {
        return terms_.size() == 1 && terms_.begin()->first == Exp{0, 0} &&
               terms_.begin()->second == 1.0;
    }
    double at(int km, int kn) const {
        const auto it = terms_.find({km, kn});
        return it == terms_.end() ? 0.0 : it->second;
    }
    void set_term(int km, int kn, double c) {
        if (c == 0.0) terms_.erase({km, kn});
        else terms_[{km, kn}] = c;
    }
    int tap_count() const { return static_cast<int>(terms_.size()); }
};

// polyphase.hpp:45-68
class StepMatrix {
public:
    explicit StepMatrix(MatrixKind kind = MatrixKind::N_FULL) : kind_(kind) {}
    static StepMatrix identity() {
        StepMatrix m;
        for (int k = 0; k < 4; ++k) m.m_[k * 4 + k].set_term(0, 0, 1.0);
        return m;
    }
    MatrixKind kind() const { return kind_; }
    void set_kind(MatrixKind k) { kind_ = k; }
    bool needs_barrier() const { return needs_barrier_; }
    void set_needs_barrier(bool b) { needs_barrier_ = b; }
    const LaurentPoly2& entry(int row, int col) const { return m_.at(row * 4 + col); }
    void set_entry(int row, int col, const LaurentPoly2& p) { m_.at(row * 4 + col) = p; }
    LaurentPoly2& mutable_entry(int row, int col) { return m_.at(row * 4 + col); }
    bool is_identity() const {
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c)
                if (r == c ? !entry(r, c).is_one() : !entry(r, c).is_zero()) return false;
        return true;
    }

private:
    std::array<LaurentPoly2, 16> m_;
    MatrixKind kind_;
    bool needs_barrier_ = true;
};

// schemes.hpp:34-38
struct Step {
    StepMatrix matrix;
    bool needs_barrier = true;
    std::string label;  // e.g. "T_H", "N(P1,U1)"
};

// wavelets.hpp:50-53
struct ConvFilters {
    LaurentPoly2 f_ll, f_hl, f_lh, f_hh;
};

// schemes.hpp:40-45
struct Scheme {
    SchemeKind kind = SchemeKind::Sweldens;
    WaveletSpec wavelet;
    std::vector<Step> steps;                  // empty for Convolution
    std::optional<ConvFilters> conv_filters;  // set only for Convolution
};

struct PyramidLevel {
    int w = 0, h = 0;
    std::vector<double> hl, lh, hh;
};

struct Pyramid {
    std::vector<PyramidLevel> details;  // finest level first
    int ll_w = 0, ll_h = 0;
    std::vector<double> ll;
};

namespace detail {

inline void check(int status) {
    if (status == WL_OK) return;
    const std::string msg = wl_last_error();
    if (status == WL_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer of floats.
struct DevBuf {
    float* p = nullptr;
    std::size_t n = 0;
    explicit DevBuf(std::size_t count) : n(count) {
        if (n) cuda(cudaMalloc(&p, n * sizeof(float)), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void upload(const double* src, std::size_t count, std::size_t offset = 0) {
        std::vector<float> f(src, src + count);
        cuda(cudaMemcpy(p + offset, f.data(), count * sizeof(float), cudaMemcpyHostToDevice),
             "cudaMemcpy H2D");
    }
    void download(double* dst, std::size_t count, std::size_t offset = 0) const {
        std::vector<float> f(count);
        cuda(cudaMemcpy(f.data(), p + offset, count * sizeof(float), cudaMemcpyDeviceToHost),
             "cudaMemcpy D2H");
        for (std::size_t i = 0; i < count; ++i) dst[i] = f[i];
    }
};

inline int boundary_id(BoundaryMode b) { return b == BoundaryMode::periodic ? WL_PERIODIC : WL_SYMMETRIC; }

}  // namespace detail

// wavelets.cpp:27-62
inline WaveletSpec get_wavelet(const std::string& name) {
    if (name == "cdf53") return {name, WL_CDF53, 1.4142135623730951};
    if (name == "cdf97") return {name, WL_CDF97, 1.149604398860241};
    if (name == "dd137") return {name, WL_DD137, 1.0};
    throw std::invalid_argument("unknown wavelet: " + name);
}

inline const std::vector<SchemeKind>& all_scheme_kinds() {
    static const std::vector<SchemeKind> k = {
        SchemeKind::Sweldens, SchemeKind::Iwahashi, SchemeKind::IwahashiStar,
        SchemeKind::Explosive, SchemeKind::ExplosiveStar, SchemeKind::Monolithic,
        SchemeKind::MonolithicStar, SchemeKind::Polyphase, SchemeKind::PolyphaseStar,
        SchemeKind::Convolution};
    return k;
}

// schemes.cpp:17-37
inline std::string scheme_name(SchemeKind kind) {
    static const char* n[] = {"sweldens",       "iwahashi",        "iwahashi_star",
                              "explosive",      "explosive_star",  "monolithic",
                              "monolithic_star", "polyphase",      "polyphase_star",
                              "convolution"};
    return n[static_cast<int>(kind)];
}
inline std::optional<SchemeKind> parse_scheme(const std::string& name) {
    for (SchemeKind k : all_scheme_kinds())
        if (scheme_name(k) == name) return k;
    return std::nullopt;
}

// subband_io.cpp:14-22
inline std::string boundary_name(BoundaryMode m) {
    return m == BoundaryMode::periodic ? "periodic" : "symmetric";
}
inline std::optional<BoundaryMode> parse_boundary(const std::string& s) {
    if (s == "periodic") return BoundaryMode::periodic;
    if (s == "symmetric") return BoundaryMode::symmetric;
    return std::nullopt;
}

// schemes.cpp:146-174: the step sequence as the library's tables hold it
// (generated from the same algebra, checked against the reference's dump).
inline Scheme build_scheme(SchemeKind kind, const WaveletSpec& w) {
    Scheme s;
    s.kind = kind;
    s.wavelet = w;
    const int ki = static_cast<int>(kind);
    const int n = wl_scheme_nsteps(w.id, ki);
    if (n < 0) detail::check(WL_EINVAL);
    for (int k = 0; k < n; ++k) {
        int mk = 0, nb = 0, nt = 0;
        char label[64];
        detail::check(wl_scheme_step(w.id, ki, k, &mk, &nb, &nt, label, sizeof label));
        std::vector<int> rows(nt), cols(nt), km(nt), kn(nt);
        std::vector<double> co(nt);
        wl_scheme_step_terms(w.id, ki, k, rows.data(), cols.data(), km.data(), kn.data(),
                             co.data(), nt);
        Step st;
        st.matrix.set_kind(static_cast<MatrixKind>(mk));
        st.matrix.set_needs_barrier(nb != 0);
        for (int t = 0; t < nt; ++t) st.matrix.mutable_entry(rows[t], cols[t]).set_term(km[t], kn[t], co[t]);
        st.needs_barrier = nb != 0;
        st.label = label;
        s.steps.push_back(std::move(st));
    }
    if (kind == SchemeKind::Convolution) {
        ConvFilters f;
        LaurentPoly2* dst[4] = {&f.f_ll, &f.f_hl, &f.f_lh, &f.f_hh};
        for (int which = 0; which < 4; ++which) {
            const int nt = wl_scheme_conv_filter(w.id, which, nullptr, nullptr, nullptr, 0);
            if (nt < 0) detail::check(WL_EINVAL);
            std::vector<int> km(nt), kn(nt);
            std::vector<double> co(nt);
            wl_scheme_conv_filter(w.id, which, km.data(), kn.data(), co.data(), nt);
            for (int t = 0; t < nt; ++t) dst[which]->set_term(km[t], kn[t], co[t]);
        }
        s.conv_filters = f;
    }
    return s;
}

// polyphase.cpp:301-340: the four 2-D filters reassembled into one 4x4
// polyphase matrix.
inline StepMatrix conv_polyphase_matrix(const ConvFilters& f) {
    StepMatrix m(MatrixKind::N_FULL);
    const LaurentPoly2* rows[4] = {&f.f_ll, &f.f_hl, &f.f_lh, &f.f_hh};
    for (int target = 0; target < 4; ++target) {
        const bool col_high = target == HL || target == HH, row_high = target == LH || target == HH;
        for (const auto& [e, c] : rows[target]->terms()) {
            const int km = e.first, kn = e.second;
            int a, b;
            bool codd, rodd;
            if (!col_high) { codd = km % 2 != 0; a = codd ? (km + 1) / 2 : km / 2; }
            else { codd = km % 2 == 0; a = codd ? km / 2 : (km - 1) / 2; }
            if (!row_high) { rodd = kn % 2 != 0; b = rodd ? (kn + 1) / 2 : kn / 2; }
            else { rodd = kn % 2 == 0; b = rodd ? kn / 2 : (kn - 1) / 2; }
            LaurentPoly2& en = m.mutable_entry(target, (rodd ? 2 : 0) + (codd ? 1 : 0));
            en.set_term(a, b, en.at(a, b) + c);
        }
    }
    return m;
}

// schemes.cpp:221-228
inline std::vector<StepMatrix> scheme_step_matrices(const Scheme& s) {
    if (s.kind == SchemeKind::Convolution) {
        if (!s.conv_filters) throw std::invalid_argument("convolution scheme without filters");
        return {conv_polyphase_matrix(*s.conv_filters)};
    }
    std::vector<StepMatrix> out;
    for (const Step& st : s.steps) out.push_back(st.matrix);
    return out;
}

inline long count_macs(const Scheme& s) {
    long macs = 0;
    detail::check(wl_scheme_info(s.wavelet.id, static_cast<int>(s.kind), WL_FORWARD, nullptr,
                                 &macs, nullptr, nullptr));
    return macs;
}
inline int count_barriers(const Scheme& s) {
    int b = 0;
    detail::check(wl_scheme_info(s.wavelet.id, static_cast<int>(s.kind), WL_FORWARD, &b,
                                 nullptr, nullptr, nullptr));
    return b;
}

inline int resolve_index(int i, int n, BoundaryMode b) {
    return wl_resolve_index(i, n, detail::boundary_id(b));
}

// One GPU does the work; kept for API parity with transform.cpp:11-29.
inline int worker_count() { return 1; }

// transform.cpp:74-98 (pure re-indexing; host side, exact).
inline QuadGrid polyphase_split(const Image& img) {
    if (img.width <= 0 || img.height <= 0 || img.width % 2 || img.height % 2)
        throw std::invalid_argument("polyphase_split requires even positive dimensions");
    QuadGrid q(img.width / 2, img.height / 2);
    for (int r = 0; r < q.h; ++r)
        for (int c = 0; c < q.w; ++c) {
            q.at(LL, r, c) = img.at(2 * r, 2 * c);
            q.at(HL, r, c) = img.at(2 * r, 2 * c + 1);
            q.at(LH, r, c) = img.at(2 * r + 1, 2 * c);
            q.at(HH, r, c) = img.at(2 * r + 1, 2 * c + 1);
        }
    return q;
}
inline Image polyphase_merge(const QuadGrid& q) {
    Image img(q.w * 2, q.h * 2);
    for (int r = 0; r < q.h; ++r)
        for (int c = 0; c < q.w; ++c) {
            img.at(2 * r, 2 * c) = q.at(LL, r, c);
            img.at(2 * r, 2 * c + 1) = q.at(HL, r, c);
            img.at(2 * r + 1, 2 * c) = q.at(LH, r, c);
            img.at(2 * r + 1, 2 * c + 1) = q.at(HH, r, c);
        }
    return img;
}

// transform.cpp:100-125: one step on the GPU (float32), out of place.
inline QuadGrid apply_step(const QuadGrid& q, const StepMatrix& step, BoundaryMode b) {
    const std::size_t n = static_cast<std::size_t>(q.w) * q.h;
    for (const auto& p : q.planes)
        if (p.size() != n) throw std::invalid_argument("quad grid plane size mismatch");
    std::vector<int> rows, cols, km, kn;
    std::vector<double> co;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c)
            for (const auto& [e, v] : step.entry(r, c).terms()) {
                rows.push_back(r);
                cols.push_back(c);
                km.push_back(e.first);
                kn.push_back(e.second);
                co.push_back(v);
            }
    detail::DevBuf in(4 * n), out(4 * n);
    for (int c = 0; c < 4; ++c) in.upload(q.planes[c].data(), n, c * n);
    detail::check(wl_apply_step(in.p, in.p + n, in.p + 2 * n, in.p + 3 * n, q.w, q.h, q.w,
                                static_cast<int>(co.size()), rows.data(), cols.data(), km.data(),
                                kn.data(), co.data(), detail::boundary_id(b), out.p, out.p + n,
                                out.p + 2 * n, out.p + 3 * n, q.w, nullptr));
    detail::cuda(cudaDeviceSynchronize(), "apply_step");
    QuadGrid o(q.w, q.h);
    for (int c = 0; c < 4; ++c) out.download(o.planes[c].data(), n, c * n);
    return o;
}

// transform.cpp:163-176. Host in / host out through wl_dwt2_forward_host
// (row-chunk pipeline: PCIe both ways overlaps the kernels).
inline QuadGrid forward(const Image& img, const Scheme& s, BoundaryMode b, bool apply_scaling) {
    if (img.width <= 0 || img.height <= 0 || img.width % 2 || img.height % 2)
        throw std::invalid_argument("forward requires even positive dimensions");
    const int qw = img.width / 2, qh = img.height / 2;
    const std::size_t n = static_cast<std::size_t>(qw) * qh;
    std::vector<float> in(img.samples.begin(), img.samples.end()), out(4 * n);
    detail::check(wl_dwt2_forward_host(in.data(), img.width, img.height, img.width, s.wavelet.id,
                                       static_cast<int>(s.kind), detail::boundary_id(b),
                                       apply_scaling ? 1 : 0, out.data(), out.data() + n,
                                       out.data() + 2 * n, out.data() + 3 * n, qw));
    QuadGrid q(qw, qh);
    for (int c = 0; c < 4; ++c)
        q.planes[c].assign(out.begin() + c * n, out.begin() + (c + 1) * n);
    return q;
}

// transform.cpp:178-196. The optional scheme selects that scheme's inverse
// kernel; the default is the reference's own (reversed negated Sweldens).
inline Image inverse(const QuadGrid& q, const WaveletSpec& w, BoundaryMode b, bool undo_scaling,
                     SchemeKind kind = SchemeKind::Sweldens) {
    const std::size_t n = static_cast<std::size_t>(q.w) * q.h;
    for (const auto& p : q.planes)
        if (p.size() != n) throw std::invalid_argument("quad grid plane size mismatch");
    std::vector<float> in(4 * n), out(4 * n);
    for (int c = 0; c < 4; ++c) std::copy(q.planes[c].begin(), q.planes[c].end(), in.begin() + c * n);
    detail::check(wl_dwt2_inverse_host(in.data(), in.data() + n, in.data() + 2 * n,
                                       in.data() + 3 * n, q.w, q.h, q.w, w.id,
                                       static_cast<int>(kind), detail::boundary_id(b),
                                       undo_scaling ? 1 : 0, out.data(), 2 * q.w));
    Image img(2 * q.w, 2 * q.h);
    img.samples.assign(out.begin(), out.end());
    return img;
}

// transform.cpp:198-227
inline Pyramid multi_level_forward(const Image& img, const Scheme& s, int levels, BoundaryMode b,
                                   bool apply_scaling) {
    if (levels < 1) throw std::invalid_argument("levels must be >= 1");
    if (levels > 30 || img.width % (1 << levels) || img.height % (1 << levels))
        throw std::invalid_argument("image dimensions must be divisible by 2^levels");
    const int W = img.width, H = img.height;
    detail::DevBuf in(img.samples.size()), pyr(wl_pyramid_elems(W, H, levels)),
        scratch(wl_pyramid_scratch_elems(W, H, levels));
    in.upload(img.samples.data(), img.samples.size());
    detail::check(wl_dwt2_pyramid_forward(in.p, W, H, levels, s.wavelet.id,
                                          static_cast<int>(s.kind), detail::boundary_id(b),
                                          apply_scaling ? 1 : 0, pyr.p, scratch.p, nullptr));
    detail::cuda(cudaDeviceSynchronize(), "multi_level_forward");
    Pyramid p;
    std::size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        PyramidLevel lev;
        lev.w = W >> (l + 1);
        lev.h = H >> (l + 1);
        const std::size_t n = static_cast<std::size_t>(lev.w) * lev.h;
        for (auto* v : {&lev.hl, &lev.lh, &lev.hh}) {
            v->resize(n);
            pyr.download(v->data(), n, off);
            off += n;
        }
        p.details.push_back(std::move(lev));
    }
    p.ll_w = W >> levels;
    p.ll_h = H >> levels;
    p.ll.resize(static_cast<std::size_t>(p.ll_w) * p.ll_h);
    pyr.download(p.ll.data(), p.ll.size(), off);
    return p;
}

// transform.cpp:229-256
inline Image multi_level_inverse(const Pyramid& p, const WaveletSpec& w, BoundaryMode b,
                                 bool undo_scaling, SchemeKind kind = SchemeKind::Sweldens) {
    if (p.details.empty()) throw std::invalid_argument("empty pyramid");
    if (p.ll.size() != static_cast<std::size_t>(p.ll_w) * p.ll_h)
        throw std::invalid_argument("approximation plane size does not match its dimensions");
    const int levels = static_cast<int>(p.details.size());
    const int W = p.details[0].w * 2, H = p.details[0].h * 2;
    for (int l = 0; l < levels; ++l) {
        const PyramidLevel& lev = p.details[l];
        if (lev.w != (W >> (l + 1)) || lev.h != (H >> (l + 1)))
            throw std::invalid_argument("pyramid level dimensions are inconsistent");
        const std::size_t n = static_cast<std::size_t>(lev.w) * lev.h;
        if (lev.hl.size() != n || lev.lh.size() != n || lev.hh.size() != n)
            throw std::invalid_argument("pyramid detail plane size does not match its level");
    }
    if (p.ll_w != (W >> levels) || p.ll_h != (H >> levels))
        throw std::invalid_argument("pyramid level dimensions are inconsistent");
    detail::DevBuf pyr(wl_pyramid_elems(W, H, levels)), out(static_cast<std::size_t>(W) * H),
        scratch(wl_pyramid_scratch_elems(W, H, levels));
    std::size_t off = 0;
    for (const PyramidLevel& lev : p.details)
        for (const auto* v : {&lev.hl, &lev.lh, &lev.hh}) {
            pyr.upload(v->data(), v->size(), off);
            off += v->size();
        }
    pyr.upload(p.ll.data(), p.ll.size(), off);
    detail::check(wl_dwt2_pyramid_inverse(pyr.p, W, H, levels, w.id, static_cast<int>(kind),
                                          detail::boundary_id(b), undo_scaling ? 1 : 0, out.p,
                                          scratch.p, nullptr));
    detail::cuda(cudaDeviceSynchronize(), "multi_level_inverse");
    Image img(W, H);
    out.download(img.samples.data(), img.samples.size());
    return img;
}

}  // namespace b200
}  // namespace wavelift
