// voxgpu_cli.cpp -- `voxgpu`, the reference CLI's hot-path subcommands on the B200 path.
//
// Mirrors tools/voxline_cli.cpp (reference, /root/reference/proj):
//   voxgpu batch --input segs.csv --out out.vox3 [--format xyz|vox3] [--workers N]
//                [--group-size G]                                    (cmd_batch, :101-129)
//   voxgpu voxelize --start x,y,z --end x,y,z --out path [--format xyz|vox3]   (cmd_voxelize,
//                :86-91; parametric only: the walk method is out of scope)
//   voxgpu bench --scenario single|fixed-batch|arbitrary [--seed N] [--reps R] [--warmup W]
//                [--scale S] [--report CSV] [--report-json JSON] [--workers N] [--group-size G]
//                (cmd_bench, :143-183 over src/bench.cpp:148-313: the paper's Table 2-4 shapes,
//                same parameter points, sub-seeds, CSV columns, JSON layout and stdout table)
// Same defaults (format xyz), same stderr summary line, same exit codes (:237-253): 0 ok,
// 2 bad input (invalid_argument / range_error / usage), 3 I/O failure or internal error.
// Every voxel comes from the CUDA kernels through include/voxgpu.h; --workers/--group-size
// are validated (>= 1) like the reference but cannot change the output.
#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/voxgpu.h"

namespace {

constexpr int kExitOk = 0, kExitBadInput = 2, kExitIoFailure = 3;

int usage(const char* msg) {
    std::fprintf(stderr,
                 "%s\nusage: voxgpu batch --input FILE.csv --out PATH [--format xyz|vox3] "
                 "[--workers N] [--group-size G]\n"
                 "       voxgpu voxelize --start x,y,z --end x,y,z --out PATH "
                 "[--format xyz|vox3]\n"
                 "       voxgpu bench --scenario single|fixed-batch|arbitrary [--seed N] [--reps R] "
                 "[--warmup W] [--scale S] [--report CSV] [--report-json JSON] [--workers N] "
                 "[--group-size G]\n",
                 msg);
    return kExitBadInput;
}

bool parse_int(const char* s, int& out) {
    char* e = nullptr;
    errno = 0;
    const long v = std::strtol(s, &e, 10);
    if (!*s || *e || errno || v < 1 || v > 1 << 30) return false;
    out = (int)v;
    return true;
}

bool parse_point(const char* s, double p[3]) {
    int n = 0;
    const char* c = s;
    while (n < 3) {
        char* e = nullptr;
        p[n] = std::strtod(c, &e);
        if (e == c) return false;
        ++n;
        if (n < 3) {
            if (*e != ',') return false;
            c = e + 1;
        } else if (*e) {
            return false;
        }
    }
    return true;
}

// Map a failed call onto the reference CLI's error lines and exit codes.
int fail(vxg_context* ctx, vxg_status s, const std::string& what) {
    const char* msg = ctx ? vxg_last_error(ctx) : "";
    if (s == VXG_INVALID_ARGUMENT || s == VXG_RANGE_ERROR) {
        std::fprintf(stderr, "error: %s\n", (msg && *msg) ? msg : what.c_str());
        return kExitBadInput;
    }
    if (s == VXG_IO_ERROR) {
        std::fprintf(stderr, "error: %s\n", what.c_str());
        return kExitIoFailure;
    }
    std::fprintf(stderr, "internal error: %s%s%s\n", what.c_str(), (msg && *msg) ? ": " : "",
                 msg ? msg : "");
    return kExitIoFailure;
}

double ms_since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

int run_segments(const std::vector<vxg_segment>& segs, const std::string& out,
                 const std::string& format, bool summary) {
    vxg_context* ctx = nullptr;
    vxg_status s = vxg_create(0, &ctx);
    if (s) return fail(nullptr, s, "no usable CUDA device for libvoxgpu (there is no CPU fallback)");
    const auto t0 = std::chrono::steady_clock::now();
    vxg_batch* b = nullptr;
    s = vxg_batch_create(ctx, segs.data(), (int64_t)segs.size(), VXG_MEM_HOST, &b);
    if (s) {
        const int rc = fail(ctx, s, "batch_preprocess");
        vxg_destroy(ctx);
        return rc;
    }
    const double pre_ms = ms_since(t0);
    int64_t n = 0, nmax = 0, cap = 0, total = 0;
    vxg_batch_info(b, &n, &nmax, &cap);
    vxg_voxel* vox = static_cast<vxg_voxel*>(vxg_host_alloc(sizeof(vxg_voxel) * (size_t)std::max<int64_t>(cap, 1)));
    int64_t* off = static_cast<int64_t*>(vxg_host_alloc(sizeof(int64_t) * (size_t)(n + 1)));
    int rc = kExitOk;
    const auto t1 = std::chrono::steady_clock::now();
    s = (vox && off) ? vxg_batch_emit_list(b, vox, cap, off, &total, VXG_MEM_HOST) : VXG_OUT_OF_MEMORY;
    const double kernel_ms = ms_since(t1);
    if (s) rc = fail(ctx, s, "batch_voxelize");
    if (!rc) {
        s = vxg_write_chains(out.c_str(), format == "vox3" ? 0 : 1, vox, off, n);
        if (s) rc = fail(ctx, s, "cannot write output file: " + out);
    }
    if (!rc && summary)
        std::fprintf(stderr,
                     "batch: %lld segments, %lld voxels | preprocess %.3f ms, kernel %.3f ms, "
                     "assemble %.3f ms\n",
                     (long long)n, (long long)total, pre_ms, kernel_ms, 0.0);
    vxg_host_free(vox);
    vxg_host_free(off);
    vxg_batch_destroy(b);
    vxg_destroy(ctx);
    return rc;
}

// ------------------------------------------------------------------------------- bench
// src/bench.cpp's harness on the GPU path. Workloads are bit-identical to the reference's (the
// SplitMix64 sub-seed per parameter point, gen_segment_of_length / gen_arbitrary_batch on the
// GPU generator); every time is a median of `reps` on a monotonic clock after `warmup` runs.
// Methods (one record each per parameter point):
//   sequential    one vxg_voxelize_parametric call per segment (the reference's per-segment map,
//                 here one GPU round trip each: the latency regime)
//   batch         vxg_run_batch: host segments in, host chains out (run_batch's contract, H2D
//                 and D2H inside the timed call)
//   batch-device  segments resident in HBM, list + chain offsets emitted into device buffers
//                 (kernel-side throughput; not in the reference, which has no device)
struct SplitMix {
    uint64_t state;
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
};

struct BenchRecord {
    std::string scenario;
    long long parameter;
    std::string method;
    int workers, group_size;
    double median_ms;
    long long total_voxels;
    double mvps;
};

double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

// nlohmann::json's number output: shortest round-trip digits, integral values keep ".0".
std::string json_double(double v) {
    char b[40];
    for (int p = 1; p <= 17; ++p) {
        std::snprintf(b, sizeof b, "%.*g", p, v);
        if (std::strtod(b, nullptr) == v) break;
    }
    std::string s = b;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

std::string json_str(const std::string& s) { return "\"" + s + "\""; }

struct BenchFail {
    int code;
    std::string msg;
};

[[noreturn]] void bench_fail(vxg_context* ctx, vxg_status s, const std::string& what) {
    const char* m = ctx ? vxg_last_error(ctx) : "";
    throw BenchFail{s == VXG_INVALID_ARGUMENT || s == VXG_RANGE_ERROR ? kExitBadInput : kExitIoFailure,
                    what + ((m && *m) ? ": " + std::string(m) : std::string())};
}

int cmd_bench(const std::string& scenario, uint64_t seed, int reps, int warmup, double scale,
              const std::string& report_csv, const std::string& report_json, int workers,
              int group) {
    int kind;  // 0 single, 1 fixed-batch, 2 arbitrary (src/bench.cpp kind_label)
    if (scenario == "single") kind = 0;
    else if (scenario == "fixed-batch") kind = 1;
    else if (scenario == "arbitrary") kind = 2;
    else {
        std::fprintf(stderr, "error: unknown scenario: %s\n", scenario.c_str());
        return kExitBadInput;
    }
    if (reps < 1) {
        std::fprintf(stderr, "error: run_scenario: repetitions must be >= 1\n");
        return kExitBadInput;
    }
    // default_scenario (src/bench.cpp:288-313)
    auto scaled = [scale](long long v) { return std::max<long long>(1, std::llround((double)v * scale)); };
    std::vector<long long> params;
    long long count = 1;
    if (kind == 0) params = {scaled(1000), scaled(10000), scaled(100000), scaled(1000000)};
    if (kind == 1) params = {scaled(20), scaled(200), scaled(2000), scaled(20000)}, count = 1024;
    if (kind == 2) count = 1024, params = {std::max<long long>(count, scaled(10000000))};

    vxg_context* ctx = nullptr;
    vxg_status st = vxg_create(0, &ctx);
    if (st) return fail(nullptr, st, "no usable CUDA device for libvoxgpu (there is no CPU fallback)");
    std::vector<BenchRecord> records;
    SplitMix seeder{seed};
    using Clock = std::chrono::steady_clock;
    auto timed = [&](auto&& body) {
        for (int w = 0; w < warmup; ++w) body();
        std::vector<double> t;
        for (int r = 0; r < reps; ++r) {
            const auto t0 = Clock::now();
            body();
            t.push_back(ms_since(t0));
        }
        return std::max(median(t), 1e-6);
    };
    const char* label = kind == 0 ? "single" : kind == 1 ? "fixed-batch" : "arbitrary";
    try {
        for (const long long parameter : params) {
            const uint64_t point_seed = seeder.next();
            std::vector<vxg_segment> segs((size_t)count);
            if (kind == 2) {
                if ((st = vxg_gen_arbitrary_batch(ctx, parameter, count, point_seed, segs.data())))
                    bench_fail(ctx, st, "gen_arbitrary_batch");
            } else {
                std::vector<int64_t> lens((size_t)count, parameter);
                std::vector<uint64_t> seeds((size_t)count);
                if (kind == 0) {
                    seeds[0] = point_seed;
                } else {
                    SplitMix rng{point_seed};
                    for (auto& x : seeds) x = rng.next();
                }
                if ((st = vxg_gen_segments(ctx, count, lens.data(), seeds.data(), 0, 0, 0, 0,
                                           segs.data(), VXG_MEM_HOST)))
                    bench_fail(ctx, st, "gen_segment_of_length");
            }
            // capacity (sum N_i + 1) sizes every buffer
            vxg_batch* b = nullptr;
            if ((st = vxg_batch_create(ctx, segs.data(), count, VXG_MEM_HOST, &b)))
                bench_fail(ctx, st, "batch_preprocess");
            int64_t n = 0, nmax = 0, cap = 0;
            vxg_batch_info(b, &n, &nmax, &cap);
            vxg_batch_destroy(b);
            std::vector<vxg_voxel> chain((size_t)nmax + 2);

            long long total = 0;
            double med = timed([&] {
                total = 0;
                for (const vxg_segment& sg : segs) {
                    int64_t c = 0;
                    if ((st = vxg_voxelize_parametric(ctx, &sg, chain.data(), (int64_t)chain.size(), &c)))
                        bench_fail(ctx, st, "voxelize_parametric");
                    total += c;
                }
            });
            records.push_back({label, parameter, "sequential", 1, 1, med, total, total / (med / 1e3) / 1e6});

            vxg_voxel* vox = static_cast<vxg_voxel*>(vxg_host_alloc(sizeof(vxg_voxel) * (size_t)cap));
            int64_t* off = static_cast<int64_t*>(vxg_host_alloc(sizeof(int64_t) * (size_t)(count + 1)));
            if (!vox || !off) bench_fail(ctx, VXG_OUT_OF_MEMORY, "pinned host buffers");
            med = timed([&] {
                int64_t t = 0;
                if ((st = vxg_run_batch(ctx, segs.data(), count, vox, cap, off, &t, nullptr)))
                    bench_fail(ctx, st, "run_batch");
                total = t;
            });
            vxg_host_free(vox);
            vxg_host_free(off);
            records.push_back({label, parameter, "batch", workers, group, med, total, total / (med / 1e3) / 1e6});

            void *d_segs = nullptr, *d_out = nullptr, *d_off = nullptr;
            if (cudaMalloc(&d_segs, sizeof(vxg_segment) * (size_t)count) ||
                cudaMalloc(&d_out, sizeof(vxg_voxel) * (size_t)cap) ||
                cudaMalloc(&d_off, sizeof(int64_t) * (size_t)(count + 1)))
                bench_fail(ctx, VXG_OUT_OF_MEMORY, "device buffers");
            cudaMemcpy(d_segs, segs.data(), sizeof(vxg_segment) * (size_t)count, cudaMemcpyHostToDevice);
            med = timed([&] {
                vxg_batch* bd = nullptr;
                if ((st = vxg_batch_create(ctx, static_cast<const vxg_segment*>(d_segs), count,
                                           VXG_MEM_DEVICE, &bd)))
                    bench_fail(ctx, st, "batch_preprocess (device)");
                int64_t t = 0;
                st = vxg_batch_emit_list(bd, static_cast<vxg_voxel*>(d_out), cap,
                                         static_cast<int64_t*>(d_off), &t, VXG_MEM_DEVICE);
                vxg_batch_destroy(bd);
                if (st) bench_fail(ctx, st, "batch_voxelize (device)");
                total = t;
            });
            cudaFree(d_segs);
            cudaFree(d_out);
            cudaFree(d_off);
            records.push_back({label, parameter, "batch-device", workers, group, med, total,
                               total / (med / 1e3) / 1e6});
        }
    } catch (const BenchFail& f) {
        std::fprintf(stderr, "error: %s\n", f.msg.c_str());
        vxg_destroy(ctx);
        return f.code;
    }
    vxg_destroy(ctx);

    // print_report_table (src/bench.cpp:272-286)
    std::printf("%-12s %12s %-10s %7s %6s %12s %14s %10s\n", "scenario", "parameter", "method",
                "workers", "group", "median_ms", "total_voxels", "MVps");
    for (const BenchRecord& r : records)
        std::printf("%-12s %12lld %-10s %7d %6d %12.3f %14lld %10.2f\n", r.scenario.c_str(),
                    r.parameter, r.method.c_str(), r.workers, r.group_size, r.median_ms,
                    r.total_voxels, r.mvps);
    std::fflush(stdout);
    if (!report_csv.empty()) {  // write_report_csv (:226-239)
        FILE* f = std::fopen(report_csv.c_str(), "w");
        if (!f) {
            std::fprintf(stderr, "error: cannot open report file: %s\n", report_csv.c_str());
            return kExitIoFailure;
        }
        bool ok = std::fprintf(f, "scenario,parameter,method,workers,group_size,median_ms,total_voxels,mvps\n") > 0;
        for (const BenchRecord& r : records)
            ok = ok && std::fprintf(f, "%s,%lld,%s,%d,%d,%.9g,%lld,%.9g\n", r.scenario.c_str(),
                                    r.parameter, r.method.c_str(), r.workers, r.group_size,
                                    r.median_ms, r.total_voxels, r.mvps) > 0;
        if (std::fclose(f) != 0 || !ok) {
            std::fprintf(stderr, "error: write failed: %s\n", report_csv.c_str());
            return kExitIoFailure;
        }
    }
    if (!report_json.empty()) {  // write_report_json (:241-270): nlohmann dump(2), sorted keys
        FILE* f = std::fopen(report_json.c_str(), "w");
        if (!f) {
            std::fprintf(stderr, "error: cannot open report file: %s\n", report_json.c_str());
            return kExitIoFailure;
        }
        std::string j = "{\n  \"metadata\": {\n    \"group_size\": " + std::to_string(group) + ",\n";
        if (kind == 2) j += "    \"length_distribution\": \"log-uniform [1, 2*mean]\",\n";
        j += "    \"repetitions\": " + std::to_string(reps) + ",\n    \"scale\": " + json_double(scale) +
             ",\n    \"scenario\": " + json_str(label) + ",\n    \"seed\": " + std::to_string(seed) +
             ",\n    \"segment_count\": " + std::to_string(kind == 0 ? 1 : count) +
             ",\n    \"warmup\": " + std::to_string(warmup) + ",\n    \"workers\": " +
             std::to_string(workers) + "\n  },\n  \"records\": [";
        for (size_t i = 0; i < records.size(); ++i) {
            const BenchRecord& r = records[i];
            j += std::string(i ? "," : "") + "\n    {\n      \"group_size\": " + std::to_string(r.group_size) +
                 ",\n      \"median_ms\": " + json_double(r.median_ms) + ",\n      \"method\": " +
                 json_str(r.method) + ",\n      \"mvps\": " + json_double(r.mvps) +
                 ",\n      \"parameter\": " + std::to_string(r.parameter) + ",\n      \"scenario\": " +
                 json_str(r.scenario) + ",\n      \"total_voxels\": " + std::to_string(r.total_voxels) +
                 ",\n      \"workers\": " + std::to_string(r.workers) + "\n    }";
        }
        j += records.empty() ? "]\n}\n" : "\n  ]\n}\n";
        const bool ok = std::fwrite(j.data(), 1, j.size(), f) == j.size();
        if (std::fclose(f) != 0 || !ok) {
            std::fprintf(stderr, "error: write failed: %s\n", report_json.c_str());
            return kExitIoFailure;
        }
    }
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage("a subcommand is required (batch | voxelize | bench)");
    const std::string cmd = argv[1];
    std::string input, out, format = "xyz";
    bool have_start = false, have_end = false;
    double start[3], end[3];
    int workers = (int)std::max(1u, std::thread::hardware_concurrency()), group = 64;
    // bench options (tools/voxline_cli.cpp:125-134, 211-226)
    std::string scenario, report_csv, report_json;
    unsigned long long seed = 1;
    int reps = 5, warmup = 2;
    double scale = 1.0;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (i + 1 >= argc) return usage(("missing value for " + a).c_str());
        const char* v = argv[++i];
        if (a == "--input" && cmd == "batch") input = v;
        else if (a == "--out") out = v;
        else if (a == "--format") {
            format = v;
            if (format != "xyz" && format != "vox3") return usage("--format: xyz or vox3");
        } else if (a == "--workers" && (cmd == "batch" || cmd == "bench")) {
            if (!parse_int(v, workers)) return usage("--workers: a positive number");
        } else if (a == "--group-size" && (cmd == "batch" || cmd == "bench")) {
            if (!parse_int(v, group)) return usage("--group-size: a positive number");
        } else if (a == "--start" && cmd == "voxelize") {
            if (!(have_start = parse_point(v, start))) return usage("--start: x,y,z");
        } else if (a == "--end" && cmd == "voxelize") {
            if (!(have_end = parse_point(v, end))) return usage("--end: x,y,z");
        } else if (a == "--scenario" && cmd == "bench") {
            scenario = v;
        } else if (a == "--seed" && cmd == "bench") {
            char* e = nullptr;
            errno = 0;
            seed = std::strtoull(v, &e, 10);
            if (!*v || *e || errno || *v == '-') return usage("--seed: a non-negative integer");
        } else if (a == "--reps" && cmd == "bench") {
            if (!parse_int(v, reps)) return usage("--reps: a positive number");
        } else if (a == "--warmup" && cmd == "bench") {
            char* e = nullptr;
            const long w = std::strtol(v, &e, 10);
            if (!*v || *e || w < 0 || w > 1 << 20) return usage("--warmup: a non-negative number");
            warmup = (int)w;
        } else if (a == "--scale" && cmd == "bench") {
            char* e = nullptr;
            scale = std::strtod(v, &e);
            if (!*v || *e || !(scale > 0) || !std::isfinite(scale)) return usage("--scale: a positive number");
        } else if (a == "--report" && cmd == "bench") {
            report_csv = v;
        } else if (a == "--report-json" && cmd == "bench") {
            report_json = v;
        } else if (a == "--method" && cmd == "voxelize") {
            if (std::strcmp(v, "parametric") != 0)
                return usage("--method: only parametric is on the GPU path");
        } else {
            return usage(("unknown option " + a).c_str());
        }
    }
    if (cmd == "bench") {
        if (scenario.empty()) return usage("--scenario is required");
        return cmd_bench(scenario, seed, reps, warmup, scale, report_csv, report_json, workers, group);
    }
    if (out.empty()) return usage("--out is required");
    if (cmd == "batch") {
        if (input.empty()) return usage("--input is required");
        vxg_segment* segs = nullptr;
        int64_t n = 0, bad = -1;
        const vxg_status s = vxg_read_segments_csv(input.c_str(), &segs, &n, &bad);
        if (s == VXG_IO_ERROR) {  // the reference reports an unreadable input as bad input
            std::fprintf(stderr, "error: cannot read input file: %s\n", input.c_str());
            return kExitBadInput;
        }
        if (s == VXG_INVALID_ARGUMENT) {
            std::fprintf(stderr,
                         "error: segments csv: line %lld: expected 6 finite decimal fields "
                         "(sx,sy,sz,ex,ey,ez)\n",
                         (long long)bad);
            return kExitBadInput;
        }
        if (s) return fail(nullptr, s, "read_segments_csv");
        std::vector<vxg_segment> v(segs, segs + n);
        vxg_free(segs);
        if (v.empty()) {
            std::fprintf(stderr, "error: input contains no segments: %s\n", input.c_str());
            return kExitBadInput;
        }
        return run_segments(v, out, format, true);
    }
    if (cmd == "voxelize") {
        if (!have_start || !have_end) return usage("--start and --end are required");
        for (int a = 0; a < 3; ++a)
            if (!std::isfinite(start[a]) || !std::isfinite(end[a])) {
                std::fprintf(stderr, "error: coordinates must be finite\n");
                return kExitBadInput;
            }
        vxg_segment s{start[0], start[1], start[2], end[0], end[1], end[2]};
        // a single chain: the reference writes the plain (multi = false) forms
        vxg_context* ctx = nullptr;
        vxg_status st = vxg_create(0, &ctx);
        if (st) return fail(nullptr, st, "no usable CUDA device for libvoxgpu (there is no CPU fallback)");
        std::vector<vxg_voxel> chain(4096);
        int64_t count = 0;
        for (;;) {
            st = vxg_voxelize_parametric(ctx, &s, chain.data(), (int64_t)chain.size(), &count);
            if (st == VXG_LOGIC_ERROR && count > (int64_t)chain.size()) {
                chain.resize((size_t)count);
                continue;
            }
            break;
        }
        int rc = st ? fail(ctx, st, "voxelize_parametric") : kExitOk;
        if (!rc) {
            FILE* f = std::fopen(out.c_str(), "wb");
            if (!f) {
                rc = fail(ctx, VXG_IO_ERROR, "cannot open output file: " + out);
            } else {
                bool ok = true;
                if (format == "vox3") {  // VOX3 version 1 (src/formats.cpp:170-173)
                    unsigned char h[16] = {'V', 'O', 'X', '3', 1, 0, 0, 0};
                    for (int i = 0; i < 8; ++i) h[8 + i] = (unsigned char)((uint64_t)count >> (8 * i));
                    ok = std::fwrite(h, 1, 16, f) == 16 &&
                         (count == 0 || std::fwrite(chain.data(), 12, (size_t)count, f) == (size_t)count);
                } else {
                    for (int64_t k = 0; ok && k < count; ++k)
                        ok = std::fprintf(f, "%d %d %d\n", chain[k].x, chain[k].y, chain[k].z) > 0;
                }
                if (std::fclose(f) != 0 || !ok) rc = fail(ctx, VXG_IO_ERROR, "write failed: " + out);
            }
        }
        vxg_destroy(ctx);
        return rc;
    }
    return usage(("unknown subcommand " + cmd).c_str());
}
