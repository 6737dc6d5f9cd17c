// tagdsp_b200_run: the reference's application layer (recording.cpp,
// harness.cpp, scheduler.cpp, codegen.cpp -- compiled UNMODIFIED from the
// reference tree) running on the B200 detector path through the drop-in
// headers include/tagdsp_b200 + libtagdsp_b200.so (integration/Makefile).
//
//   detect    <rec.iq> <config.json> <out.jsonl>      detect_recording (recording.cpp:258-289)
//   simulate  <rec.iq> <config.json> <events.jsonl> <compute_ratio>
//                                                     simulate_recording (recording.cpp:291-389)
//   simulate-batched  (same arguments)                the same scheduler run, with the
//             searching and tracking windows read from a device-resident
//             CircularBuffer (tdg_ring, fed with the blocks Scheduler::push_samples
//             sees) and every tracking task that is due computed in ONE batched
//             tdg_track_ring call; the reference Scheduler still issues and
//             completes the tasks one at a time in its own order, so the event
//             log must be byte-identical to `simulate`'s
//   bench     <window_len> <repeats> <windows> <pattern counts...>
//                                                     run_bench (harness.cpp:28-104) incl. its
//                                                     correctness gate; bench_summary_json out
// Exit codes as the reference CLI (tools/tagdsp_cli.cpp:171-177):
// std::invalid_argument -> 2, other errors -> 1.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "tagdsp/codegen.hpp"
#include "tagdsp/recording.hpp"
#include "tagdsp_gpu.h"

using namespace tagdsp;

namespace {

void ck(int rc) {
    if (rc == TDG_OK) return;
    std::string m = tdg_last_error();
    if (rc == TDG_EINVAL) throw std::invalid_argument(m);
    throw std::runtime_error(m);
}

int cmd_detect(const std::string& rec_path, const std::string& cfg_path, const std::string& out_path) {
    auto rec = read_recording(rec_path);
    auto cfg = load_run_config(cfg_path);
    auto t0 = std::chrono::steady_clock::now();
    auto dets = detect_recording(rec, cfg);
    auto t1 = std::chrono::steady_clock::now();
    std::ofstream out(out_path);
    size_t acc = 0;
    for (const auto& d : dets) {
        out << detection_json_line(d) << "\n";
        acc += d.accepted;
    }
    std::cerr << "detect: " << dets.size() << " detections (" << acc << " accepted) in "
              << std::chrono::duration<double>(t1 - t0).count() << " s\n";
    return 0;
}

void write_events(const std::string& path, const std::vector<SchedulerEvent>& ev) {
    std::ofstream out(path);
    for (const auto& e : ev) out << event_json_line(e) << "\n";
}

int cmd_simulate(const std::string& rec_path, const std::string& cfg_path, const std::string& out_path, double ratio) {
    auto rec = read_recording(rec_path);
    auto cfg = load_run_config(cfg_path);
    auto res = simulate_recording(rec, cfg, ratio);
    write_events(out_path, res.events);
    std::printf("{\"detections\": %zu, \"misses\": %zu, \"events\": %zu, \"searched_fraction_pct\": %.6f}\n",
                res.detections, res.misses, res.events.size(), res.searched_fraction_pct);
    return 0;
}

// The simulate_recording loop (recording.cpp:291-389) with the detector work
// batched on the device: same feed, same Scheduler calls in the same order.
int cmd_simulate_batched(const std::string& rec_path, const std::string& cfg_path, const std::string& out_path,
                         double ratio) {
    auto rec = read_recording(rec_path);
    auto cfg = load_run_config(cfg_path);
    const double rate = rec.block.sample_rate;
    const size_t total = rec.block.num_complex();
    Scheduler sched(cfg.sched);
    DemodConfig demod_cfg = cfg.demod;
    demod_cfg.mod.sample_rate = rate;
    const auto search_window = size_t(cfg.sched.window_s * rate + 0.5);
    const auto track_window = size_t((cfg.sched.track_pre_s + cfg.sched.track_post_s) * rate + 0.5);
    const int64_t pre = int64_t(cfg.sched.track_pre_s * rate + 0.5);
    const int64_t post = int64_t(cfg.sched.track_post_s * rate + 0.5);

    std::map<std::string, size_t> code_index;
    std::vector<uint8_t> bits;
    for (const auto& t : cfg.tags) {
        auto code = gen_code(t.seed, demod_cfg.mod, t.id);
        code_index[t.id] = code_index.size();
        bits.insert(bits.end(), code.bits.begin(), code.bits.end());
        sched.add_tag(code, t.period_s);
    }
    const size_t n_codes = cfg.tags.size();
    tdg_demod_config c{};
    c.mod = {demod_cfg.mod.sample_rate, demod_cfg.mod.bit_rate, demod_cfg.mod.freq_one, demod_cfg.mod.freq_zero,
             uint64_t(demod_cfg.mod.packet_bits)};
    c.lo_freq = demod_cfg.lo_freq;
    c.bandpass_center = demod_cfg.bandpass_center;
    c.bandpass_width = demod_cfg.bandpass_width;
    c.bandpass_taps = demod_cfg.bandpass_taps;
    c.eps = demod_cfg.eps;

    tdg_ctx* ctx = nullptr;
    ck(tdg_ctx_create(0, &ctx));
    tdg_codeset *cs_search = nullptr, *cs_track = nullptr;
    ck(tdg_codeset_prepare(ctx, &c, search_window, bits.data(), n_codes, &cs_search));
    ck(tdg_codeset_prepare(ctx, &c, track_window, bits.data(), n_codes, &cs_track));
    // device mirror of the scheduler's CircularBuffer (same capacity)
    tdg_ring* ring = nullptr;
    ck(tdg_ring_create(ctx, sched.buffer().capacity(), &ring));

    SimulationResult result;
    int64_t produced = 0;
    double clock_s = 0.0;
    auto feed = [&](int64_t upto) {
        upto = std::min(upto, int64_t(total));
        if (upto <= produced) return;
        RawSampleBlock blk;
        blk.sample_rate = rate;
        blk.start_time = produced;
        blk.samples.assign(rec.block.samples.begin() + std::ptrdiff_t(2 * produced),
                           rec.block.samples.begin() + std::ptrdiff_t(2 * upto));
        sched.push_samples(blk);
        ck(tdg_ring_push(ring, blk.samples.data(), blk.num_complex(), blk.start_time, nullptr));
        produced = upto;
    };
    auto readable = [&](int64_t s, int64_t e) { return s >= sched.buffer().head() && e <= sched.buffer().tail(); };
    auto to_det = [&](const tdg_detection& r, const std::string& id) {
        Detection d;
        d.tag_id = id;
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
    };
    // results of tracking tasks computed ahead, keyed by (tag index, start):
    // a task's detection depends only on its samples and code
    std::map<std::pair<size_t, int64_t>, std::optional<Detection>> track_cache;
    size_t batches = 0, batched_tasks = 0;
    const double lo = demod_cfg.lo_freq;
    std::vector<tdg_detection> recs(n_codes);

    while (true) {
        feed(int64_t(clock_s * rate));
        auto task = sched.next_task();
        if (!task) {
            if (produced >= int64_t(total)) break;
            clock_s += 0.001;
            continue;
        }
        const double elapsed = ratio * double(task->end - task->start) / rate;
        if (task->kind == TaskKind::Searching) {
            std::vector<Detection> dets;
            if (readable(task->start, task->end)) {
                ck(tdg_search_ring(ctx, ring, &c, &lo, 1, task->start, search_window, search_window, 1, cs_search,
                                   cfg.threshold, recs.data(), recs.size(), 1));
                for (auto idx : task->tag_indices) {
                    const auto& id = sched.tags()[idx].code.tag_id;
                    dets.push_back(to_det(recs[code_index.at(id)], id));
                }
            }
            sched.complete_search(*task, dets, elapsed);
            for (const auto& d : dets)
                if (d.accepted) ++result.detections;
        } else {
            const size_t tag = task->tag_indices[0];
            auto key = std::make_pair(tag, task->start);
            if (!track_cache.count(key)) {
                // every tracking task due now (make_track_task's windows,
                // scheduler.cpp:89-113), in one batch
                std::vector<tdg_track_task> tasks;
                std::vector<std::pair<size_t, int64_t>> keys;
                const auto& tags = sched.tags();
                for (size_t i = 0; i < tags.size(); ++i) {
                    if (tags[i].mode != TagMode::Tracking) continue;
                    const int64_t s = int64_t(tags[i].next_predicted_toa) - pre;
                    const int64_t e = int64_t(tags[i].next_predicted_toa) + post;
                    if (e > sched.buffer().tail() || track_cache.count({i, s})) continue;
                    if (!readable(s, e)) {
                        track_cache[{i, s}] = std::nullopt;   // evicted: a miss, as read() fails
                        continue;
                    }
                    tasks.push_back({s, uint64_t(code_index.at(tags[i].code.tag_id))});
                    keys.push_back({i, s});
                }
                if (!tasks.empty()) {
                    std::vector<tdg_detection> tr(tasks.size());
                    ck(tdg_track_ring(ctx, ring, &c, tasks.data(), tasks.size(), cs_track, cfg.threshold, tr.data(), 1));
                    ++batches;
                    batched_tasks += tasks.size();
                    for (size_t k = 0; k < tasks.size(); ++k) {
                        auto d = to_det(tr[k], tags[keys[k].first].code.tag_id);
                        track_cache[keys[k]] = d.accepted ? std::optional<Detection>(d) : std::nullopt;
                    }
                }
                if (!track_cache.count(key)) track_cache[key] = std::nullopt;
            }
            std::optional<Detection> best = track_cache[key];
            track_cache.erase(key);
            // the reference reads the window now: evicted since the batch ran -> a miss
            if (!readable(task->start, task->end)) best = std::nullopt;
            if (best)
                ++result.detections;
            else
                ++result.misses;
            sched.complete_track(*task, best, elapsed);
        }
        clock_s += elapsed;
    }
    write_events(out_path, sched.events());
    int64_t covered = sched.frontier();
    const double frac = covered > 0 ? 100.0 * double(sched.searched_samples()) / double(covered) : 0.0;
    std::printf("{\"detections\": %zu, \"misses\": %zu, \"events\": %zu, \"searched_fraction_pct\": %.6f, "
                "\"track_batches\": %zu, \"batched_track_tasks\": %zu}\n",
                result.detections, result.misses, sched.events().size(), frac, batches, batched_tasks);
    tdg_ring_destroy(ring);
    tdg_codeset_destroy(cs_search);
    tdg_codeset_destroy(cs_track);
    tdg_ctx_destroy(ctx);
    return 0;
}

int cmd_bench(size_t window_len, size_t repeats, size_t windows, const std::vector<size_t>& counts) {
    BenchScenario sc;
    sc.window_len = window_len;
    sc.repeats = repeats;
    sc.windows = windows;
    sc.pattern_counts = counts;
    auto res = run_bench(sc);   // throws if the correctness gate fails
    std::printf("%s\n", bench_summary_json(res, 0.5).c_str());
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw std::invalid_argument("usage: tagdsp_b200_run detect|simulate|simulate-batched|bench ...");
        const std::string cmd = argv[1];
        if (cmd == "detect" && argc == 5) return cmd_detect(argv[2], argv[3], argv[4]);
        if (cmd == "simulate" && argc == 6) return cmd_simulate(argv[2], argv[3], argv[4], std::stod(argv[5]));
        if (cmd == "simulate-batched" && argc == 6)
            return cmd_simulate_batched(argv[2], argv[3], argv[4], std::stod(argv[5]));
        if (cmd == "bench" && argc >= 6) {
            std::vector<size_t> counts;
            for (int i = 5; i < argc; ++i) counts.push_back(size_t(std::stoul(argv[i])));
            return cmd_bench(std::stoul(argv[2]), std::stoul(argv[3]), std::stoul(argv[4]), counts);
        }
        throw std::invalid_argument("bad arguments for " + cmd);
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
