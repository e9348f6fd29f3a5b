// ref_bench_main.cpp -- TEST INFRASTRUCTURE: the reference's own bench harness (src/bench.cpp
// run_scenario + report writers, compiled unmodified by `make -C oracle ref`) behind a minimal
// argv front end, because the reference CLI needs CLI11 (absent here). Same options and defaults
// as `voxline bench` (tools/voxline_cli.cpp:125-134, 143-183); used only to time the reference's
// CPU path beside `voxgpu bench` (profiles/), never by the product.
//   ref_bench SCENARIO [--seed N] [--reps R] [--warmup W] [--scale S] [--workers N]
//             [--group-size G] [--report CSV]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <thread>

#include "voxline/bench.hpp"

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_bench single|fixed-batch|arbitrary [options]\n");
        return 2;
    }
    const std::string sc = argv[1];
    voxline::ScenarioKind kind;
    if (sc == "single") kind = voxline::ScenarioKind::single_segment;
    else if (sc == "fixed-batch") kind = voxline::ScenarioKind::fixed_batch;
    else if (sc == "arbitrary") kind = voxline::ScenarioKind::arbitrary_batch;
    else {
        std::fprintf(stderr, "error: unknown scenario: %s\n", sc.c_str());
        return 2;
    }
    unsigned long long seed = 1;
    int reps = 5, warmup = 2, group = 64;
    int workers = (int)std::max(1u, std::thread::hardware_concurrency());
    double scale = 1.0;
    std::string report;
    for (int i = 2; i + 1 < argc; i += 2) {
        const std::string a = argv[i];
        const char* v = argv[i + 1];
        if (a == "--seed") seed = std::strtoull(v, nullptr, 10);
        else if (a == "--reps") reps = std::atoi(v);
        else if (a == "--warmup") warmup = std::atoi(v);
        else if (a == "--scale") scale = std::atof(v);
        else if (a == "--workers") workers = std::atoi(v);
        else if (a == "--group-size") group = std::atoi(v);
        else if (a == "--report") report = v;
        else {
            std::fprintf(stderr, "unknown option %s\n", a.c_str());
            return 2;
        }
    }
    try {
        const voxline::Scenario s = voxline::default_scenario(kind, seed, reps, warmup, scale);
        const voxline::PartitionConfig cfg{group, workers};
        const auto records = voxline::run_scenario(s, cfg);
        voxline::print_report_table(std::cout, records);
        if (!report.empty()) {
            std::ofstream out(report);
            voxline::write_report_csv(out, records);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    }
    return 0;
}
