// Detection records as the reference's JSON lines (detection_json_line,
// proj/src/recording.cpp:228-242): the same nlohmann::json object and dump(),
// so number formatting (Grisu2 shortest round-trip, "e+XX" exponents) and
// string escaping are byte-identical to the reference's output.  Host code of
// libtagdsp_gpu.so; no device work.
#include <cstdio>
#include <string>

#include <nlohmann/json.hpp>

#include "tagdsp_gpu.h"

extern "C" int tdg_detection_json_line(const tdg_detection* r, const char* tag_id, char* out, uint64_t cap,
                                       uint64_t* len) {
    try {
        // Detection stores size_t / float / double / bool (detector.hpp:39-51)
        nlohmann::json j = {
            {"tag_id", std::string(tag_id)},
            {"toa_seconds", r->toa_seconds},
            {"peak_index", static_cast<size_t>(r->peak_index)},
            {"subsample_offset", r->subsample_offset},
            {"w_c", r->w_c},
            {"q", r->q},
            {"p_c", r->p_c},
            {"score", r->score},
            {"accepted", r->accepted != 0},
            {"partial", r->partial != 0},
        };
        const std::string s = j.dump();
        if (len) *len = s.size();
        if (s.size() + 1 > cap) return TDG_EINVAL;
        std::snprintf(out, cap, "%s", s.c_str());
        return TDG_OK;
    } catch (...) {
        return TDG_EINTERNAL;
    }
}
