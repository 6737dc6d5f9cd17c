// tagdsp_gpu.hpp -- header-only C++20 wrapper over the B200 C-ABI that
// restores the reference tagdsp detector API (/root/reference/proj/include/
// tagdsp/{types,dsp,detector}.hpp).  A reference caller switches with
//     namespace tagdsp = tagdsp_gpu;
// and its call sites -- e.g. proj/src/recording.cpp:271-285 (detect_recording)
// or proj/src/harness.cpp:42-45,60-61,87-90 (run_bench) -- compile unchanged:
//     auto demod = demodulate_window(blk, cfg, cache);
//     const TransformedCode& tc = prepare_code(code, shape, cache, codes);
//     auto dets = detect(demod.d, demod.u, transformed, det_cfg, rate, cache);
// Errors: TDG_EINVAL -> std::invalid_argument (the reference's precondition
// exceptions), anything else -> std::runtime_error.
//
// Differences a caller can observe: PlanCache owns a CUDA device + stream
// instead of FFTW plans; prepare_code is batched lazily (codes registered for
// one WindowShape are transformed on the GPU together at the next detect); and
// search() exposes the batched windows x lo_freq-bins x codes path.
#pragma once
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tagdsp_gpu.h"

namespace tagdsp_gpu {

namespace detail {
inline void check(int rc) {
    if (rc == TDG_OK) return;
    std::string msg = tdg_last_error();
    if (rc == TDG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("tagdsp_gpu: " + msg);
}
}  // namespace detail

// ---- types.hpp:16-57 -------------------------------------------------------
struct RawSampleBlock {
    std::vector<int16_t> samples;   // interleaved I,Q
    int64_t start_time = 0;
    double sample_rate = 8.0e6;
    size_t num_complex() const { return samples.size() / 2; }
};

struct ModulationParams {
    double sample_rate = 8.0e6;
    double bit_rate = 1.0e6;
    double freq_one = 250.0e3;
    double freq_zero = -250.0e3;
    size_t packet_bits = 8192;
    size_t samples_per_bit() const {
        double spb = sample_rate / bit_rate;
        auto n = static_cast<size_t>(spb + 0.5);
        if (n < 1 || std::abs(spb - double(n)) > 1e-9)
            throw std::invalid_argument("sample_rate / bit_rate must be a positive integer");
        return n;
    }
    size_t packet_samples() const { return packet_bits * samples_per_bit(); }
};

struct TagCode {
    std::string tag_id;
    std::vector<uint8_t> bits;
    ModulationParams mod;
};

// ---- dsp.hpp:25-36, 62-65 ---------------------------------------------------
struct DemodConfig {
    ModulationParams mod;
    double lo_freq = 0.0;
    double bandpass_center = 0.0;
    double bandpass_width = 1.5e6;
    size_t bandpass_taps = 200;
    float eps = 1e-12f;
    size_t composed_filter_len() const { return bandpass_taps + mod.samples_per_bit() - 1; }
    tdg_demod_config c() const {
        tdg_demod_config r{};
        r.mod = {mod.sample_rate, mod.bit_rate, mod.freq_one, mod.freq_zero, uint64_t(mod.packet_bits)};
        r.lo_freq = lo_freq;
        r.bandpass_center = bandpass_center;
        r.bandpass_width = bandpass_width;
        r.bandpass_taps = bandpass_taps;
        r.eps = eps;
        return r;
    }
};

struct DemodResult {
    std::vector<float> d;
    std::vector<float> u;
};

// ---- fft.hpp:17-56: the context a caller owns ------------------------------
class PlanCache {
public:
    explicit PlanCache(int device = 0) { detail::check(tdg_ctx_create(device, &ctx_)); }
    ~PlanCache() {
        for (auto& [k, w] : windows_) tdg_windows_destroy(w);
        tdg_ctx_destroy(ctx_);
    }
    PlanCache(const PlanCache&) = delete;
    PlanCache& operator=(const PlanCache&) = delete;
    tdg_ctx* handle() const { return ctx_; }
    // one reusable single-slot window set per window length
    tdg_windows* window(size_t len) {
        auto it = windows_.find(len);
        if (it != windows_.end()) return it->second;
        tdg_windows* w = nullptr;
        detail::check(tdg_windows_create(ctx_, len, 1, 1, &w));
        windows_[len] = w;
        return w;
    }

private:
    tdg_ctx* ctx_ = nullptr;
    std::map<size_t, tdg_windows*> windows_;
};

inline size_t pad_length(size_t n) {
    if (n < 1) throw std::invalid_argument("pad_length: n must be >= 1");
    return size_t(tdg_pad_length(n));
}

// demodulate_window (dsp.hpp:70-71)
inline DemodResult demodulate_window(const RawSampleBlock& block, const DemodConfig& cfg, PlanCache& cache) {
    if (block.samples.size() % 2 != 0) throw std::invalid_argument("convert: odd raw sample count");
    DemodResult r;
    const size_t n = block.num_complex();
    if (n == 0) return r;
    tdg_windows* w = cache.window(n);
    const tdg_demod_config c = cfg.c();
    const double lo = cfg.lo_freq;
    detail::check(tdg_demodulate(cache.handle(), w, &c, &lo, 1, block.samples.data(), n, block.start_time, n, 1));
    r.d.resize(n);
    r.u.resize(n);
    detail::check(tdg_windows_get_du(cache.handle(), w, 0, r.d.data(), r.u.data()));
    return r;
}

// ---- detector.hpp:13-106 ---------------------------------------------------
struct WindowShape {
    size_t window_len = 0;
    DemodConfig cfg;
    size_t corr_len() const {
        return pad_length(window_len + cfg.mod.packet_samples() + cfg.composed_filter_len());
    }
};

class CodeCache;

// Handle to one prepared code; the transformed data live on the GPU inside the
// CodeCache's per-shape code set.
struct TransformedCode {
    CodeCache* owner = nullptr;
    std::string tag_id;
    size_t window_len = 0;
    size_t nonzero_len = 0;     // filled once the shape's code set is built
    float energy = 0.0f;
    float abs_sum = 0.0f;
    size_t index = 0;           // position in the shape's code set
};

struct Detection {
    std::string tag_id;
    size_t peak_index = 0;
    float subsample_offset = 0.0f;
    double toa_seconds = 0.0;
    float peak_value = 0.0f;
    float w_c = 0.0f;
    float q = 0.0f;
    float p_c = 0.0f;
    float score = 0.0f;
    bool accepted = false;
    bool partial = false;
};

struct DetectionConfig {
    float threshold = 0.25f;
    int64_t window_start = 0;
};

struct DetectTimings {
    double correlation_s = 0.0;
    double peak_stats_s = 0.0;
};

// CodeCache (detector.hpp:37): (tag_id, window_len) -> TransformedCode, with
// the GPU code set per window shape rebuilt when codes were added.
class CodeCache {
public:
    ~CodeCache() {
        for (auto& [k, s] : shapes_)
            if (s.set) tdg_codeset_destroy(s.set);
    }
    struct Shape {
        DemodConfig cfg;
        std::vector<TagCode> codes;
        std::vector<TransformedCode*> handles;
        tdg_codeset* set = nullptr;
        bool dirty = true;
    };
    std::map<std::pair<std::string, size_t>, TransformedCode> entries;
    std::map<size_t, Shape> shapes_;

    tdg_codeset* build(PlanCache& cache, size_t window_len) {
        Shape& s = shapes_.at(window_len);
        if (!s.dirty) return s.set;
        if (s.set) tdg_codeset_destroy(s.set);
        s.set = nullptr;
        const size_t nb = s.cfg.mod.packet_bits;
        std::vector<uint8_t> bits(s.codes.size() * nb);
        for (size_t i = 0; i < s.codes.size(); ++i) {
            if (s.codes[i].bits.size() != nb) throw std::invalid_argument("prepare_code: bit count mismatch");
            std::copy(s.codes[i].bits.begin(), s.codes[i].bits.end(), bits.begin() + i * nb);
        }
        const tdg_demod_config c = s.cfg.c();
        detail::check(tdg_codeset_prepare(cache.handle(), &c, window_len, bits.data(), s.codes.size(), &s.set));
        for (size_t i = 0; i < s.handles.size(); ++i) {
            uint64_t n = 0, cl = 0;
            detail::check(tdg_codeset_info(s.set, i, &n, &s.handles[i]->energy, &s.handles[i]->abs_sum, &cl));
            s.handles[i]->nonzero_len = n;
        }
        s.dirty = false;
        return s.set;
    }
};

// prepare_code (detector.hpp:67-68): pure lookup the second time.
inline const TransformedCode& prepare_code(const TagCode& code, const WindowShape& shape, PlanCache& cache,
                                           CodeCache& codes) {
    auto key = std::make_pair(code.tag_id, shape.window_len);
    auto it = codes.entries.find(key);
    if (it != codes.entries.end()) return it->second;
    if (shape.window_len < shape.cfg.mod.packet_samples())
        throw std::invalid_argument("prepare_code: window shorter than a packet");
    auto& s = codes.shapes_[shape.window_len];
    if (s.codes.empty()) s.cfg = shape.cfg;
    TransformedCode tc;
    tc.owner = &codes;
    tc.tag_id = code.tag_id;
    tc.window_len = shape.window_len;
    tc.index = s.codes.size();
    auto [ins, ok] = codes.entries.emplace(key, tc);
    s.codes.push_back(code);
    s.handles.push_back(&ins->second);
    s.dirty = true;
    codes.build(cache, shape.window_len);   // keep reference semantics: fields valid on return
    return ins->second;
}

namespace detail {
inline Detection to_detection(const tdg_detection& r, const std::string& tag_id) {
    Detection d;
    d.tag_id = tag_id;
    d.peak_index = size_t(r.peak_index);
    d.subsample_offset = r.subsample_offset;
    d.toa_seconds = r.toa_seconds;
    d.peak_value = r.peak_value;
    d.w_c = r.w_c;
    d.q = r.q;
    d.p_c = r.p_c;
    d.score = r.score;
    d.accepted = r.accepted != 0;
    d.partial = r.partial != 0;
    return d;
}
}  // namespace detail

// detect (detector.hpp:103-106): one Detection per requested code, in order.
// All codes must come from one CodeCache shape (as the reference requires one
// window shape per batch, detector.cpp:108-112).
inline std::vector<Detection> detect(std::span<const float> d, std::span<const float> u,
                                     std::span<const TransformedCode* const> codes, const DetectionConfig& cfg,
                                     double sample_rate, PlanCache& cache, DetectTimings* timings = nullptr) {
    std::vector<Detection> out;
    if (codes.empty()) return out;
    CodeCache& code_cache = *codes.front()->owner;
    const size_t W = d.size();
    if (u.size() != W) throw std::invalid_argument("detect: d/u length mismatch");
    for (auto* tc : codes)
        if (tc->window_len != codes.front()->window_len || tc->owner != &code_cache)
            throw std::invalid_argument("batch_xcorr: mixed window shapes");
    if (codes.front()->window_len != W) throw std::invalid_argument("batch_xcorr: mixed window shapes");
    tdg_codeset* set = code_cache.build(cache, W);
    tdg_windows* w = cache.window(W);
    detail::check(tdg_windows_set_du(cache.handle(), w, 0, d.data(), u.data(), cfg.window_start));
    std::vector<tdg_detection> all(tdg_codeset_size(set));
    detail::check(tdg_detect(cache.handle(), w, set, cfg.threshold, sample_rate, all.data(), all.size()));
    out.reserve(codes.size());
    for (auto* tc : codes) out.push_back(detail::to_detection(all[tc->index], tc->tag_id));
    (void)timings;
    return out;
}

// Batched searching pass (detect_recording, recording.cpp:258-289, with a
// frequency-offset sweep): every window x bin x code of `shape`'s code set.
inline std::vector<tdg_detection> search(const RawSampleBlock& stream, const WindowShape& shape, size_t advance,
                                         const std::vector<double>& lo_bins, float threshold, PlanCache& cache,
                                         CodeCache& code_cache) {
    tdg_codeset* set = code_cache.build(cache, shape.window_len);
    const size_t n = stream.num_complex();
    const size_t nw = n >= shape.window_len ? (n - shape.window_len) / advance + 1 : 0;
    std::vector<tdg_detection> out(nw * lo_bins.size() * tdg_codeset_size(set));
    uint64_t n_out = 0;
    const tdg_demod_config c = shape.cfg.c();
    detail::check(tdg_search(cache.handle(), &c, lo_bins.data(), lo_bins.size(), stream.samples.data(), n,
                             stream.start_time, shape.window_len, advance, set, threshold, out.data(), out.size(),
                             &n_out));
    out.resize(n_out);
    return out;
}

// Batched tracking (the Tracking branch of simulate_recording,
// recording.cpp:360-378, for many scheduler Tasks at once): task i searches
// window [starts[i], starts[i] + shape.window_len) of `stream` for code
// codes[i] (prepared with prepare_code(code, shape, ...)).  One Detection per
// task, accepted or not, as detect() returns for a single code.
inline std::vector<Detection> track(const RawSampleBlock& stream, const WindowShape& shape,
                                    std::span<const int64_t> starts, std::span<const TransformedCode* const> codes,
                                    float threshold, PlanCache& cache) {
    std::vector<Detection> out;
    if (starts.size() != codes.size()) throw std::invalid_argument("track: one code per task");
    if (codes.empty()) return out;
    CodeCache& code_cache = *codes.front()->owner;
    for (auto* tc : codes)
        if (tc->window_len != shape.window_len || tc->owner != &code_cache)
            throw std::invalid_argument("batch_xcorr: mixed window shapes");
    tdg_codeset* set = code_cache.build(cache, shape.window_len);
    std::vector<tdg_track_task> tasks(codes.size());
    for (size_t i = 0; i < codes.size(); ++i) tasks[i] = {starts[i], codes[i]->index};
    std::vector<tdg_detection> recs(tasks.size());
    const tdg_demod_config c = shape.cfg.c();
    detail::check(tdg_track(cache.handle(), &c, stream.samples.data(), stream.num_complex(), stream.start_time,
                            tasks.data(), tasks.size(), set, threshold, recs.data()));
    out.reserve(recs.size());
    for (size_t i = 0; i < recs.size(); ++i) out.push_back(detail::to_detection(recs[i], codes[i]->tag_id));
    return out;
}

}  // namespace tagdsp_gpu
