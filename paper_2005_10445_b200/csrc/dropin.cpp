// libtagdsp_b200: the reference's fft / dsp / detector API (declared by
// include/tagdsp_b200/tagdsp/{fft,dsp,detector}.hpp, signatures of
// proj/include/tagdsp/{fft,dsp,detector}.hpp) implemented over the B200
// C-ABI (include/tagdsp_gpu.h).  Host C++ only: every transform, filter,
// correlation, peak search and statistic runs in libtagdsp_gpu.so's kernels;
// this file maps the reference's objects (PlanCache, CodeCache,
// TransformedCode, DemodResult) onto device contexts, code sets and window
// sets, and its preconditions onto the same exceptions.  Filter DESIGN
// (design_bandpass / matched_filters / compose: a few hundred taps, computed
// once) and interpolate_peak (three values) are host arithmetic, as in the
// product's own setup path.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numbers>
#include <set>
#include <stdexcept>
#include <string>

#include "tagdsp/detector.hpp"
#include "tagdsp_gpu.h"

namespace tagdsp {
namespace b200 {

void check(int rc) {
    if (rc == TDG_OK) return;
    std::string msg = tdg_last_error();
    if (rc == TDG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("tagdsp_b200: " + msg);
}

int default_device() {
    const char* e = std::getenv("TAGDSP_B200_DEVICE");
    return e ? std::atoi(e) : 0;
}

struct CodeSetHandle {
    tdg_codeset* cs = nullptr;
    explicit CodeSetHandle(tdg_codeset* c) : cs(c) {}
    ~CodeSetHandle() { tdg_codeset_destroy(cs); }
    CodeSetHandle(const CodeSetHandle&) = delete;
    CodeSetHandle& operator=(const CodeSetHandle&) = delete;
};

}  // namespace b200

namespace b200 {
struct CodeRef {
    std::shared_ptr<CodeSetHandle> set;
    size_t index = 0;
};

tdg_demod_config to_c(const DemodConfig& c) {
    tdg_demod_config r{};
    r.mod = {c.mod.sample_rate, c.mod.bit_rate, c.mod.freq_one, c.mod.freq_zero, uint64_t(c.mod.packet_bits)};
    r.lo_freq = c.lo_freq;
    r.bandpass_center = c.bandpass_center;
    r.bandpass_width = c.bandpass_width;
    r.bandpass_taps = c.bandpass_taps;
    r.eps = c.eps;
    return r;
}

// Per-PlanCache device state: the context, reusable single-slot window sets
// (one per window length), the prepare_code code sets (one per window shape),
// and which host d,u arrays are the device copy of the last demodulated
// window (detect() then skips their upload).
struct Device {
    tdg_ctx* ctx = nullptr;
    std::map<size_t, tdg_windows*> windows;
    std::map<std::vector<double>, std::shared_ptr<CodeSetHandle>> pools;
    std::set<size_t> fft_sizes;
    struct Resident {
        const float* d = nullptr;
        const float* u = nullptr;
        size_t n = 0;
        tdg_windows* w = nullptr;
        std::vector<float> probe;   // sampled values at demodulation time
    } last;

    explicit Device(int dev) { check(tdg_ctx_create(dev, &ctx)); }
    ~Device() {
        for (auto& [n, w] : windows) tdg_windows_destroy(w);
        tdg_ctx_destroy(ctx);
    }
    tdg_windows* window(size_t n, PlanCache::Stats& st) {
        auto it = windows.find(n);
        if (it != windows.end()) {
            ++st.buffer_hits;
            return it->second;
        }
        tdg_windows* w = nullptr;
        check(tdg_windows_create(ctx, n, 1, 1, &w));
        ++st.buffers_allocated;
        windows[n] = w;
        return w;
    }
    static std::vector<float> sample(const float* d, const float* u, size_t n) {
        std::vector<float> p;
        for (size_t k = 0; k < 64 && n; ++k) {
            const size_t i = (k * 7919 + k * k) % n;
            p.push_back(d[i]);
            p.push_back(u[i]);
        }
        return p;
    }
    // d,u of the window detect() runs on: the resident copy if the host
    // arrays are the ones demodulate_window returned (and unchanged at the
    // probed samples), else an upload
    tdg_windows* window_for(std::span<const float> d, std::span<const float> u, int64_t start,
                            PlanCache::Stats& st) {
        const size_t n = d.size();
        if (last.w && last.d == d.data() && last.u == u.data() && last.n == n && sample(d.data(), u.data(), n) == last.probe) {
            check(tdg_windows_set_start(ctx, last.w, 0, start));
            ++st.buffer_hits;
            return last.w;
        }
        tdg_windows* w = window(n, st);
        check(tdg_windows_set_du(ctx, w, 0, d.data(), u.data(), start));
        last = Resident{};
        return w;
    }
};

// the context of free functions without a PlanCache argument (find_peak,
// convert, mix, demodulate, statistics): one per process, created on first use
Device& free_device() {
    static std::mutex mu;
    static std::unique_ptr<Device> dev;
    std::lock_guard<std::mutex> lk(mu);
    if (!dev) dev = std::make_unique<Device>(default_device());
    return *dev;
}

const CodeRef& ref_of(const TransformedCode& tc) {
    if (!tc.device) throw std::invalid_argument("batch_xcorr: code has no device transform (not prepared by the B200 path)");
    return *tc.device;
}

}  // namespace b200

// ---- fft.hpp ---------------------------------------------------------------
PlanCache::PlanCache() : PlanCache(b200::default_device()) {}
PlanCache::PlanCache(int device) : dev_(std::make_unique<b200::Device>(device)) {}
PlanCache::~PlanCache() = default;

b200::Device& PlanCache::device() { return *dev_; }

namespace {
void run_fft(PlanCache& cache, b200::Device& dev, std::span<const cfloat> in, std::span<cfloat> out, bool inverse) {
    if (in.size() != out.size()) throw std::invalid_argument(inverse ? "inverse: size mismatch" : "forward: size mismatch");
    if (in.empty()) return;
    auto& st = cache.counters();
    if (dev.fft_sizes.insert(in.size()).second)
        ++st.plans_created;
    else
        ++st.plan_hits;
    b200::check(tdg_fft(dev.ctx, reinterpret_cast<const float*>(in.data()), reinterpret_cast<float*>(out.data()),
                        in.size(), inverse ? 1 : 0));
    if (inverse)
        ++st.inverse_execs;
    else
        ++st.forward_execs;
}
}  // namespace

void PlanCache::forward(std::span<const cfloat> in, std::span<cfloat> out) { run_fft(*this, *dev_, in, out, false); }
void PlanCache::inverse(std::span<const cfloat> in, std::span<cfloat> out) { run_fft(*this, *dev_, in, out, true); }

std::vector<cfloat>& PlanCache::work(const std::string& name, size_t n) {
    auto key = std::make_pair(name, n);
    auto it = work_.find(key);
    if (it != work_.end()) {
        ++stats_.buffer_hits;
        return it->second;
    }
    ++stats_.buffers_allocated;
    return work_.emplace(key, std::vector<cfloat>(n)).first->second;
}

std::vector<float>& PlanCache::work_real(const std::string& name, size_t n) {
    auto key = std::make_pair(name, n);
    auto it = work_real_.find(key);
    if (it != work_real_.end()) {
        ++stats_.buffer_hits;
        return it->second;
    }
    ++stats_.buffers_allocated;
    return work_real_.emplace(key, std::vector<float>(n)).first->second;
}

size_t pad_length(size_t n) {
    if (n < 1) throw std::invalid_argument("pad_length: n must be >= 1");
    return size_t(tdg_pad_length(n));
}

// ---- dsp.hpp ---------------------------------------------------------------
std::vector<cfloat> convert(const RawSampleBlock& block) {
    if (block.samples.size() % 2 != 0) throw std::invalid_argument("convert: odd raw sample count");
    std::vector<cfloat> out(block.samples.size() / 2);
    if (out.empty()) return out;
    b200::check(tdg_convert(b200::free_device().ctx, block.samples.data(), block.samples.size(),
                            reinterpret_cast<float*>(out.data())));
    return out;
}

void mix(std::span<cfloat> x, double lo_freq, int64_t start_index, double sample_rate) {
    if (lo_freq == 0.0 || x.empty()) return;
    b200::check(tdg_mix(b200::free_device().ctx, reinterpret_cast<float*>(x.data()), x.size(), lo_freq, start_index,
                        sample_rate));
}

// Filter design: the same formulas as the product's filter_spectra setup
// (tagdsp_gpu.cu, restating proj/src/dsp.cpp:37-73 with its float/double steps).
namespace {
void bandpass_taps(double center, double width, size_t taps, double fs, std::vector<cfloat>& out) {
    const double pi = std::numbers::pi;
    const double fc = width / 2.0, mid = double(taps - 1) / 2.0;
    std::vector<double> lp(taps);
    double sum = 0.0;
    for (size_t k = 0; k < taps; ++k) {
        const double t = double(k) - mid, x = 2.0 * fc * t / fs;
        const double sinc = (x == 0.0) ? 1.0 : std::sin(pi * x) / (pi * x);
        const double w = (taps == 1) ? 1.0 : 0.54 - 0.46 * std::cos(2.0 * pi * double(k) / double(taps - 1));
        lp[k] = sinc * w;
        sum += lp[k];
    }
    out.resize(taps);
    for (size_t k = 0; k < taps; ++k) {
        const double t = double(k) - mid, a = 2.0 * pi * center * t / fs, g = lp[k] / sum;
        out[k] = cfloat(float(g * std::cos(a)), float(g * std::sin(a)));
    }
}
void matched_taps(double freq, size_t spb, double fs, std::vector<cfloat>& out) {
    out.resize(spb);
    for (size_t k = 0; k < spb; ++k) {
        const double a = 2.0 * std::numbers::pi * freq * double(spb - 1 - k) / fs;
        out[k] = cfloat(float(std::cos(a)), float(-std::sin(a)));
    }
}
}  // namespace

FirFilter design_bandpass(double center, double width, size_t taps, double sample_rate) {
    if (taps < 1) throw std::invalid_argument("design_bandpass: taps must be >= 1");
    if (width <= 0.0) throw std::invalid_argument("design_bandpass: width must be positive");
    if (std::abs(center) + width / 2.0 > sample_rate / 2.0)
        throw std::invalid_argument("design_bandpass: band outside Nyquist");
    FirFilter f;
    bandpass_taps(center, width, taps, sample_rate, f.coeffs);
    return f;
}

std::pair<FirFilter, FirFilter> matched_filters(const ModulationParams& params) {
    const size_t spb = params.samples_per_bit();
    FirFilter h1, h0;
    matched_taps(params.freq_one, spb, params.sample_rate, h1.coeffs);
    matched_taps(params.freq_zero, spb, params.sample_rate, h0.coeffs);
    return {h1, h0};
}

FirFilter compose(const FirFilter& a, const FirFilter& b) {
    FirFilter f;
    if (a.coeffs.empty() || b.coeffs.empty()) return f;
    f.coeffs.assign(a.length() + b.length() - 1, cfloat{0.0f, 0.0f});
    for (size_t i = 0; i < a.length(); ++i)
        for (size_t j = 0; j < b.length(); ++j) f.coeffs[i + j] += a.coeffs[i] * b.coeffs[j];
    return f;
}

std::vector<cfloat> overlap_add_filter(std::span<const cfloat> x, const FirFilter& h, PlanCache& cache,
                                       ConvMode mode) {
    if (h.length() == 0) throw std::invalid_argument("overlap_add_filter: empty filter");
    if (x.empty()) return {};
    std::vector<cfloat> full(x.size() + h.length() - 1);
    b200::check(tdg_convolve(cache.device().ctx, reinterpret_cast<const float*>(x.data()), x.size(),
                             reinterpret_cast<const float*>(h.coeffs.data()), h.length(),
                             reinterpret_cast<float*>(full.data())));
    ++cache.counters().forward_execs;
    ++cache.counters().forward_execs;
    ++cache.counters().inverse_execs;
    if (mode == ConvMode::Same) full.resize(x.size());
    return full;
}

void demodulate(std::span<const cfloat> f1, std::span<const cfloat> f0, float eps, std::span<float> d,
                std::span<float> u) {
    if (f1.size() != f0.size() || d.size() != f1.size() || u.size() != f1.size())
        throw std::invalid_argument("demodulate: length mismatch");
    if (f1.empty()) return;
    b200::check(tdg_discriminate(b200::free_device().ctx, reinterpret_cast<const float*>(f1.data()),
                                 reinterpret_cast<const float*>(f0.data()), f1.size(), eps, d.data(), u.data()));
}

namespace {
DemodResult fetch_resident(PlanCache& cache, tdg_windows* w, size_t n) {
    auto& dev = cache.device();
    DemodResult r;
    r.d.resize(n);
    r.u.resize(n);
    b200::check(tdg_windows_get_du(dev.ctx, w, 0, r.d.data(), r.u.data()));
    dev.last = b200::Device::Resident{r.d.data(), r.u.data(), n, w, b200::Device::sample(r.d.data(), r.u.data(), n)};
    return r;
}
}  // namespace

DemodResult demodulate_window(const RawSampleBlock& block, const DemodConfig& cfg, PlanCache& cache) {
    if (block.samples.size() % 2 != 0) throw std::invalid_argument("convert: odd raw sample count");
    const size_t n = block.num_complex();
    if (n == 0) return {};
    auto& dev = cache.device();
    tdg_windows* w = dev.window(n, cache.counters());
    const tdg_demod_config c = b200::to_c(cfg);
    const double lo = cfg.lo_freq;
    b200::check(tdg_demodulate(dev.ctx, w, &c, &lo, 1, block.samples.data(), n, block.start_time, n, 1));
    return fetch_resident(cache, w, n);
}

DemodResult demodulate_signal(std::span<const cfloat> x, int64_t start_index, double lo_freq, const DemodConfig& cfg,
                              PlanCache& cache) {
    const size_t n = x.size();
    if (n == 0) return {};
    cfg.mod.samples_per_bit();
    auto& dev = cache.device();
    tdg_windows* w = dev.window(n, cache.counters());
    const tdg_demod_config c = b200::to_c(cfg);
    b200::check(tdg_demodulate_signal(dev.ctx, w, &c, lo_freq, reinterpret_cast<const float*>(x.data()), n,
                                      start_index));
    return fetch_resident(cache, w, n);
}

// ---- detector.hpp ----------------------------------------------------------
namespace {
void fill_from_set(TransformedCode& tc, std::shared_ptr<b200::CodeSetHandle> set, size_t index) {
    uint64_t nz = 0, cl = 0;
    b200::check(tdg_codeset_info(set->cs, index, &nz, &tc.energy, &tc.abs_sum, &cl));
    tc.nonzero_len = size_t(nz);
    tc.replica_d.resize(tc.nonzero_len);
    if (nz) b200::check(tdg_codeset_replica(set->cs, index, tc.replica_d.data()));
    auto ref = std::make_shared<b200::CodeRef>();
    ref->set = std::move(set);
    ref->index = index;
    tc.device = std::move(ref);
}
}  // namespace

TransformedCode make_transformed(std::string tag_id, std::span<const float> replica_d, std::span<const float> replica_u,
                                 size_t window_len, size_t corr_len, PlanCache& cache) {
    auto& dev = cache.device();
    const float* dp = replica_d.data();
    const float* up = replica_u.data();
    const uint64_t len = replica_d.size();
    tdg_codeset* cs = nullptr;
    b200::check(tdg_codeset_from_replicas(dev.ctx, window_len, corr_len, &dp, replica_u.empty() ? nullptr : &up, &len,
                                          1, &cs));
    TransformedCode tc;
    tc.tag_id = std::move(tag_id);
    tc.window_len = window_len;
    tc.corr_len = corr_len;
    fill_from_set(tc, std::make_shared<b200::CodeSetHandle>(cs), 0);
    tc.replica_u.assign(replica_u.begin(), replica_u.begin() + std::min(replica_u.size(), tc.nonzero_len));
    ++cache.counters().forward_execs;
    return tc;
}

const TransformedCode& prepare_code(const TagCode& code, const WindowShape& shape, PlanCache& cache, CodeCache& codes) {
    auto key = std::make_pair(code.tag_id, shape.window_len);
    auto it = codes.find(key);
    if (it != codes.end()) return it->second;   // pure lookup (detector.cpp:52-54)
    if (shape.window_len < shape.cfg.mod.packet_samples())
        throw std::invalid_argument("prepare_code: window shorter than a packet");
    if (code.bits.size() != shape.cfg.mod.packet_bits)
        throw std::invalid_argument("prepare_code: bit count does not match packet_bits");
    auto& dev = cache.device();
    const tdg_demod_config c = b200::to_c(shape.cfg);
    // the device code set of this shape: codes prepared for it are appended
    // (one transform per stored pair), so detect() over any of them is one batch
    std::vector<double> pk{double(shape.window_len), c.mod.sample_rate, c.mod.bit_rate, c.mod.freq_one,
                           c.mod.freq_zero, double(c.mod.packet_bits), c.bandpass_center, c.bandpass_width,
                           double(c.bandpass_taps), double(c.eps)};
    auto& pool = dev.pools[pk];
    size_t index = 0;
    if (!pool) {
        tdg_codeset* cs = nullptr;
        b200::check(tdg_codeset_prepare(dev.ctx, &c, shape.window_len, code.bits.data(), 1, &cs));
        pool = std::make_shared<b200::CodeSetHandle>(cs);
    } else {
        index = size_t(tdg_codeset_size(pool->cs));
        b200::check(tdg_codeset_append(dev.ctx, pool->cs, &c, code.bits.data(), 1));
    }
    TransformedCode tc;
    tc.tag_id = code.tag_id;
    tc.window_len = shape.window_len;
    tc.corr_len = shape.corr_len();
    fill_from_set(tc, pool, index);
    ++cache.counters().forward_execs;
    return codes.emplace(key, std::move(tc)).first->second;
}

namespace {
// group requested codes by device code set, preserving request order
struct Groups {
    std::vector<std::pair<tdg_codeset*, std::vector<size_t>>> sets;   // set, positions in the request
};
Groups group_codes(std::span<const TransformedCode* const> codes) {
    Groups g;
    for (size_t i = 0; i < codes.size(); ++i) {
        const auto& r = b200::ref_of(*codes[i]);
        auto it = std::find_if(g.sets.begin(), g.sets.end(), [&](auto& p) { return p.first == r.set->cs; });
        if (it == g.sets.end()) {
            g.sets.push_back({r.set->cs, {}});
            it = g.sets.end() - 1;
        }
        it->second.push_back(i);
    }
    return g;
}

void check_shapes(std::span<const float> d, std::span<const TransformedCode* const> codes, bool single) {
    const size_t corr_len = codes.front()->corr_len;
    for (const auto* tc : codes) {
        if (!single && tc->corr_len != corr_len) throw std::invalid_argument("batch_xcorr: mixed window shapes");
        if (d.size() + tc->nonzero_len > tc->corr_len + 1)
            throw std::invalid_argument(single ? "xcorr: window does not fit cached transform size"
                                               : "batch_xcorr: window does not fit transform size");
    }
}
}  // namespace

std::vector<std::vector<float>> batch_xcorr(std::span<const float> d, std::span<const TransformedCode* const> codes,
                                            PlanCache& cache) {
    std::vector<std::vector<float>> out;
    if (codes.empty()) return out;
    check_shapes(d, codes, false);
    auto& dev = cache.device();
    tdg_windows* w = dev.window(d.size(), cache.counters());
    b200::check(tdg_windows_set_du(dev.ctx, w, 0, d.data(), d.data(), 0));
    dev.last = b200::Device::Resident{};
    out.assign(codes.size(), std::vector<float>(d.size()));
    for (auto& [cs, pos] : group_codes(codes).sets) {
        std::vector<int64_t> idx;
        for (size_t p : pos) idx.push_back(int64_t(b200::ref_of(*codes[p]).index));
        std::vector<float> rows(pos.size() * d.size());
        b200::check(tdg_batch_xcorr(dev.ctx, w, 0, cs, idx.data(), idx.size(), rows.data()));
        for (size_t k = 0; k < pos.size(); ++k)
            std::copy(rows.begin() + std::ptrdiff_t(k * d.size()), rows.begin() + std::ptrdiff_t((k + 1) * d.size()),
                      out[pos[k]].begin());
    }
    ++cache.counters().forward_execs;   // one forward transform per batch (detector.cpp:115)
    cache.counters().inverse_execs += codes.size();
    return out;
}

std::vector<float> xcorr(std::span<const float> d, const TransformedCode& tc, PlanCache& cache) {
    const TransformedCode* one[1] = {&tc};
    check_shapes(d, std::span<const TransformedCode* const>(one, 1), true);
    return std::move(batch_xcorr(d, std::span<const TransformedCode* const>(one, 1), cache)[0]);
}

std::pair<size_t, float> find_peak(std::span<const float> xc) {
    if (xc.empty()) throw std::invalid_argument("find_peak: empty input");
    uint64_t j = 0;
    float v = 0.0f;
    b200::check(tdg_find_peak(b200::free_device().ctx, xc.data(), xc.size(), &j, &v));
    return {size_t(j), v};
}

float interpolate_peak(std::span<const float> xc, size_t j) {
    // three-point parabola on |xc| (detector.cpp:136-145), the same float
    // steps as the statistics kernel's epilogue
    if (j == 0 || j + 1 >= xc.size()) return 0.0f;
    const float a = std::abs(xc[j - 1]), b = std::abs(xc[j]), c = std::abs(xc[j + 1]);
    const float denom = a - 2.0f * b + c;
    if (denom >= 0.0f) return 0.0f;
    const float delta = 0.5f * (a - c) / denom;
    return std::clamp(delta, -0.5f, 0.5f);
}

Statistics statistics(std::span<const float> d, std::span<const float> u, const TransformedCode& tc, size_t j) {
    Statistics s;
    int partial = 0;
    b200::check(tdg_statistics(b200::free_device().ctx, d.data(), u.data(), d.size(), tc.replica_d.data(),
                               tc.replica_d.size(), j, &s.w_c, &s.q, &s.p_c, &partial));
    s.partial = partial != 0;
    return s;
}

std::vector<Detection> detect(std::span<const float> d, std::span<const float> u,
                              std::span<const TransformedCode* const> codes, const DetectionConfig& cfg,
                              double sample_rate, PlanCache& cache, DetectTimings* timings) {
    std::vector<Detection> out;
    if (codes.empty()) return out;
    if (u.size() != d.size()) throw std::invalid_argument("demodulate: length mismatch");
    check_shapes(d, codes, false);
    auto& dev = cache.device();
    tdg_windows* w = dev.window_for(d, u, cfg.window_start, cache.counters());
    if (timings) b200::check(tdg_set_option(dev.ctx, "detect_timings", 1));
    out.resize(codes.size());
    for (auto& [cs, pos] : group_codes(codes).sets) {
        std::vector<int64_t> idx;
        for (size_t p : pos) idx.push_back(int64_t(b200::ref_of(*codes[p]).index));
        std::vector<tdg_detection> recs(pos.size());
        b200::check(tdg_detect_codes(dev.ctx, w, cs, idx.data(), idx.size(), cfg.threshold, sample_rate, recs.data(),
                                     recs.size()));
        if (timings) {
            double a = 0, b = 0;
            b200::check(tdg_detect_timings(dev.ctx, &a, &b));
            timings->correlation_s += a;
            timings->peak_stats_s += b;
        }
        for (size_t k = 0; k < pos.size(); ++k) {
            const tdg_detection& r = recs[k];
            Detection& o = out[pos[k]];
            o.tag_id = codes[pos[k]]->tag_id;
            o.peak_index = size_t(r.peak_index);
            o.subsample_offset = r.subsample_offset;
            o.toa_seconds = r.toa_seconds;
            o.peak_value = r.peak_value;
            o.w_c = r.w_c;
            o.q = r.q;
            o.p_c = r.p_c;
            o.score = r.score;
            o.accepted = r.accepted != 0;
            o.partial = r.partial != 0;
        }
    }
    if (timings) b200::check(tdg_set_option(dev.ctx, "detect_timings", 0));
    ++cache.counters().forward_execs;   // one forward transform of d per batch
    cache.counters().inverse_execs += codes.size();
    return out;
}

}  // namespace tagdsp
