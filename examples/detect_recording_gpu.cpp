// Example drop-in caller: the reference's detect_recording loop
// (proj/src/recording.cpp:258-289) written against the reference API, compiled
// against the B200 wrapper by aliasing the namespace.  Build:
//   g++ -std=c++20 -Iinclude examples/detect_recording_gpu.cpp \
//       -Lpaper_2005_10445_b200 -ltagdsp_gpu -Wl,-rpath,$PWD/paper_2005_10445_b200
#include <cstdio>

#include "tagdsp_gpu.hpp"

namespace tagdsp = tagdsp_gpu;
using namespace tagdsp;

std::vector<Detection> detect_recording(const RawSampleBlock& rec, const std::vector<TagCode>& roster,
                                        const DemodConfig& demod_cfg, float threshold, size_t window,
                                        size_t advance) {
    PlanCache cache;
    CodeCache code_cache;
    WindowShape shape{window, demod_cfg};
    std::vector<const TransformedCode*> transformed;
    for (const auto& code : roster) transformed.push_back(&prepare_code(code, shape, cache, code_cache));
    std::vector<Detection> all;
    size_t total = rec.num_complex();
    for (size_t start = 0; start + window <= total; start += advance) {
        RawSampleBlock blk;
        blk.sample_rate = rec.sample_rate;
        blk.start_time = rec.start_time + int64_t(start);
        blk.samples.assign(rec.samples.begin() + std::ptrdiff_t(2 * start),
                           rec.samples.begin() + std::ptrdiff_t(2 * (start + window)));
        auto demod = demodulate_window(blk, demod_cfg, cache);
        DetectionConfig det_cfg{threshold, blk.start_time};
        auto dets = detect(demod.d, demod.u, transformed, det_cfg, rec.sample_rate, cache);
        all.insert(all.end(), dets.begin(), dets.end());
    }
    return all;
}

int main(int argc, char** argv) {
    std::printf("pad_length(865743) = %zu\n", pad_length(865743));
    if (argc < 2) return 0;   // "run" needs a GPU
    DemodConfig cfg;
    std::vector<TagCode> roster(2);
    for (size_t i = 0; i < roster.size(); ++i) {
        roster[i].tag_id = "t" + std::to_string(i);
        roster[i].bits.assign(cfg.mod.packet_bits, uint8_t(i & 1));
        roster[i].mod = cfg.mod;
    }
    RawSampleBlock rec;
    rec.samples.assign(2 * 1600000, 0);
    auto dets = detect_recording(rec, roster, cfg, 0.25f, 800000, 720000);
    std::printf("%zu detections\n", dets.size());
    return 0;
}
