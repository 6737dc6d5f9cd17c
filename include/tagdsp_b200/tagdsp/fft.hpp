// B200 drop-in for the reference's tagdsp/fft.hpp (proj/include/tagdsp/fft.hpp).
//
// Put include/tagdsp_b200 BEFORE the reference's include directory and link
// libtagdsp_b200.so instead of the reference's fft.cpp / dsp.cpp /
// detector.cpp: the reference's own callers (recording.cpp, harness.cpp,
// scheduler.cpp, codegen.cpp and its test suites) then compile unchanged and
// run the detector path on the GPU.  types.hpp, codegen.hpp, scheduler.hpp,
// harness.hpp and recording.hpp stay the reference's.
//
// PlanCache: the caller-owned context of the reference, here one CUDA device
// context (stream, transform tables, device scratch) plus the reference's
// named host work arrays and its Stats counters.  forward/inverse run the
// GPU's {2,3,5,7}-smooth Stockham transform (tdg_fft).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "tagdsp/types.hpp"

namespace tagdsp {

namespace b200 {
struct Device;   // per-PlanCache device state (dropin.cpp)
}

class PlanCache {
public:
    // Same counters as the reference (fft.hpp:19-26): plans = device transform
    // tables built, buffers = device allocations, execs = transforms run (the
    // batched detect path counts one forward per window and one inverse per
    // code, as the reference does), hits = reuses.
    struct Stats {
        uint64_t plans_created = 0;
        uint64_t buffers_allocated = 0;
        uint64_t forward_execs = 0;
        uint64_t inverse_execs = 0;
        uint64_t plan_hits = 0;
        uint64_t buffer_hits = 0;
    };

    PlanCache();                       // CUDA device 0 (or TAGDSP_B200_DEVICE)
    explicit PlanCache(int device);
    ~PlanCache();
    PlanCache(const PlanCache&) = delete;
    PlanCache& operator=(const PlanCache&) = delete;

    // out = DFT(in); in.size() == out.size() == transform size.
    void forward(std::span<const cfloat> in, std::span<cfloat> out);
    // out = IDFT(in) / n.
    void inverse(std::span<const cfloat> in, std::span<cfloat> out);

    std::vector<cfloat>& work(const std::string& name, size_t n);
    std::vector<float>& work_real(const std::string& name, size_t n);

    const Stats& stats() const { return stats_; }

    // B200 extension: the device state behind this cache
    b200::Device& device();
    Stats& counters() { return stats_; }

private:
    std::unique_ptr<b200::Device> dev_;
    std::map<std::pair<std::string, size_t>, std::vector<cfloat>> work_;
    std::map<std::pair<std::string, size_t>, std::vector<float>> work_real_;
    Stats stats_;
};

size_t pad_length(size_t n);

}  // namespace tagdsp
