// Per-cell output writers: experiment.cpp:94-183 (metrics_to_json, write_turns_csv,
// event_to_json, write_events_jsonl) and the cell loop :424-440, paths relative to
// /root/reference/proj. See cs_output.hpp.
#include "cs_output.hpp"

#include <cstdio>
#include <fstream>
#include <stdexcept>

#include "json.hpp"

namespace csb {
namespace {

using json = nlohmann::ordered_json;  // the reference's alias (json_alias.hpp:8): insertion-ordered keys

double ms(double us) { return us / 1000.0; }  // experiment.cpp:72

std::string to_hex(uint64_t v) {  // hashing.cpp:8-12
    char buf[19];
    std::snprintf(buf, sizeof(buf), "0x%016llx", (unsigned long long)v);
    return buf;
}

std::string format_double(double v) {  // experiment.cpp:132-136
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

json policy_config_json(const CellOut& c) {  // experiment.cpp:74-92
    if (c.policy == "ttl") return json{{"pin_horizon_ms", ms(c.ttl_pin_horizon_us)}};
    if (c.policy == "cachesage") {
        return json{{"skip", c.skip},
                    {"take", c.take},
                    {"tau", c.tau},
                    {"e_max", c.e_max},
                    {"w_pred", c.w_pred},
                    {"window", c.window},
                    {"gate",
                     {{"min_confidence", c.min_confidence},
                      {"min_row_count", c.min_row_count},
                      {"budget_per_step", c.budget_per_step}}}};
    }
    return json(nullptr);
}

const char* kind_name(uint8_t k) {  // hashing.cpp:14-24
    switch (k) {
        case EventRec::kBlockTouch: return "block_touch";
        case EventRec::kRequestArrival: return "request_arrival";
        case EventRec::kAgentDispatch: return "agent_dispatch";
        case EventRec::kTurnComplete: return "turn_complete";
    }
    return "tool_return";
}

}  // namespace

void write_cell(const CellOut& c, const std::string& dir) {
    // aggregate_metrics (metrics.cpp:5-26) over the turns in turn_id order + finalize (engine.cpp:394-413)
    long prompt = 0, cached = 0;
    double ttft_sum = 0.0, lat_sum = 0.0;
    for (const TurnRec& t : c.turns) {
        prompt += t.prompt_tokens;
        cached += t.cached_tokens;
        ttft_sum += t.ttft_us;
        lat_sum += t.latency_us;
    }
    const double hit = prompt > 0 ? (double)cached / (double)prompt : 0.0;
    const double n = (double)c.turns.size();
    const double mean_ttft = c.turns.empty() ? 0.0 : ttft_sum / n;
    const double mean_lat = c.turns.empty() ? 0.0 : lat_sum / n;
    const double thr = c.sim_duration_us > 0.0 ? n / (c.sim_duration_us / 1e6) : 0.0;
    const uint64_t n_turns = c.turns.size();

    const json metrics{
        {"schema", "cachesage-metrics/v1"},
        {"workload", c.workload},
        {"policy", c.policy},
        {"seed", c.seed},
        {"engine",
         {{"budget_blocks", c.budget_blocks},
          {"block_size", c.block_size},
          {"concurrency", c.concurrency},
          {"prefetch", c.prefetch},
          {"cost_model",
           {{"prefill_per_token_us", c.prefill_per_token_us},
            {"prefill_base_us", c.prefill_base_us},
            {"decode_per_token_us", c.decode_per_token_us}}}}},
        {"hit_rate", hit},
        {"mean_ttft_ms", ms(mean_ttft)},
        {"mean_latency_ms", ms(mean_lat)},
        {"throughput_turns_per_s", thr},
        {"sim_duration_ms", ms(c.sim_duration_us)},
        {"turns", n_turns},
        {"total_prompt_tokens", prompt},
        {"total_cached_tokens", cached},
        {"evictions", c.evictions},
        {"truncated_admissions", c.truncated},
        {"warmup",
         {{"executed", c.warmups_executed},
          {"dropped", c.warmups_dropped},
          {"prompt_tokens", c.warmup_prompt_tokens},
          {"uncached_tokens", c.warmup_uncached_tokens},
          {"time_ms", ms(c.warmup_time_us)}}},
        {"policy_config", policy_config_json(c)}};
    {
        std::ofstream out(dir + "/metrics.json");
        if (!out) throw std::runtime_error("cannot write " + dir + "/metrics.json");
        out << metrics.dump(2) << '\n';
    }
    {
        std::ofstream out(dir + "/turns.csv");
        if (!out) throw std::runtime_error("cannot write " + dir + "/turns.csv");
        out << "turn_id,session,turn,agent,label,prompt_tokens,cached_tokens,"
               "ttft_ms,latency_ms,arrival_ms,start_ms,end_ms\n";
        for (const TurnRec& t : c.turns) {
            const std::string& label = t.label >= 0 && t.label < (int)c.labels.size() ? c.labels[t.label] : "";
            out << t.turn_id << ',' << t.session << ',' << t.turn_index << ',' << to_hex(t.agent) << ',' << label
                << ',' << t.prompt_tokens << ',' << t.cached_tokens << ',' << format_double(ms(t.ttft_us)) << ','
                << format_double(ms(t.latency_us)) << ',' << format_double(ms(t.arrival_us)) << ','
                << format_double(ms(t.start_us)) << ',' << format_double(ms(t.end_us)) << '\n';
        }
    }
    if (c.events) {
        std::ofstream out(dir + "/events.jsonl");
        if (!out) throw std::runtime_error("cannot write " + dir + "/events.jsonl");
        out << json{{"schema", "cachesage-events/v1"}}.dump() << '\n';
        for (const EventRec& e : *c.events) {
            json j{{"tick", e.tick}, {"kind", kind_name(e.kind)}};
            switch (e.kind) {
                case EventRec::kBlockTouch:
                    j["key"] = to_hex(e.a);
                    j["agent"] = e.has_b ? json(to_hex(e.b)) : json(nullptr);
                    break;
                case EventRec::kRequestArrival:
                    j["request"] = e.a;
                    j["agent"] = to_hex(e.b);
                    break;
                case EventRec::kAgentDispatch:
                    j["prev"] = e.has_a ? json(to_hex(e.a)) : json(nullptr);
                    j["next"] = to_hex(e.b);
                    break;
                default:
                    j["request"] = e.a;
                    break;
            }
            out << j.dump() << '\n';
        }
    }
}

}  // namespace csb
