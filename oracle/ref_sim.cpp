// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Runs the reference's discrete-event schedule model (flashlab
// core/include/flashlab/pipeline_sim.hpp: parse_resource_model, simulate,
// validate_trace, work_model) on one shape with a resource-model file, and
// prints the result as one JSON object. Built by oracle/Makefile from the
// reference sources where they lie into oracle/_ref/flashlab_sim.
//
//   flashlab_sim MODEL_FILE N D BLOCK_ROWS BLOCK_COLS BACKWARD FP8 SCHEDULE
//   SCHEDULE: serial | warpspec | warpspec+pingpong | pingpong+2stage |
//             pingpong+3stage | overlap-only
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>

#include "flashlab/pipeline_sim.hpp"

using namespace flashlab;

int main(int argc, char** argv) {
  if (argc != 9) {
    std::fprintf(stderr, "usage: %s MODEL N D BR BC BACKWARD FP8 SCHEDULE\n", argv[0]);
    return 2;
  }
  try {
    std::ifstream f(argv[1]);
    if (!f) throw std::invalid_argument(std::string("cannot open ") + argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    const ResourceModel model = parse_resource_model(ss.str());
    const std::map<std::string, ScheduleKind> kinds = {
        {"serial", ScheduleKind::serial()},
        {"warpspec", ScheduleKind::warpspec()},
        {"warpspec+pingpong", ScheduleKind::warpspec_pingpong()},
        {"pingpong+2stage", ScheduleKind::pingpong_2stage()},
        {"pingpong+3stage", ScheduleKind::pingpong_3stage()},
        {"overlap-only", ScheduleKind::overlap_only()}};
    auto it = kinds.find(argv[8]);
    if (it == kinds.end()) throw std::invalid_argument("unknown schedule");
    ScheduleKind kind = it->second;
    kind.fp8 = std::atoi(argv[7]) != 0;
    SimShape shape;
    shape.n = std::strtoull(argv[2], nullptr, 10);
    shape.d = std::strtoull(argv[3], nullptr, 10);
    shape.block_rows = std::strtoull(argv[4], nullptr, 10);
    shape.block_cols = std::strtoull(argv[5], nullptr, 10);
    shape.backward = std::atoi(argv[6]) != 0;
    const SimReport r = simulate(shape, model, kind);
    const bool trace_ok = validate_trace(r).empty();
    const WorkModel wm = work_model(shape.n, shape.d,
                                    kind.fp8 ? FloatFormatId::fp8e4m3 : FloatFormatId::fp16, model);
    std::printf("{\"schedule\": \"%s\", \"makespan_cycles\": %.17g, \"events\": %zu, \"trace_valid\": %s, "
                "\"matmul_flops_per_exp\": %.17g, \"softmax_cycle_fraction\": %.17g",
                kind_name(r.kind).c_str(), r.makespan, r.trace.size(), trace_ok ? "true" : "false",
                wm.matmul_flops_per_exp, wm.softmax_cycle_fraction);
    for (const auto& [k, v] : r.busy) std::printf(", \"busy_%s\": %.17g", k.c_str(), v);
    for (const auto& [k, v] : r.utilization) std::printf(", \"util_%s\": %.17g", k.c_str(), v);
    std::printf(", \"model_text\": \"");
    for (char c : resource_model_text(model)) std::printf(c == '\n' ? "\\n" : "%c", c);
    std::printf("\"}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  return 0;
}
