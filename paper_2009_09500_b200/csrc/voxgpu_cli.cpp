// voxgpu_cli.cpp -- `voxgpu`, the reference CLI's hot-path subcommands on the B200 path.
//
// Mirrors tools/voxline_cli.cpp (reference, /root/reference/proj):
//   voxgpu batch --input segs.csv --out out.vox3 [--format xyz|vox3] [--workers N]
//                [--group-size G]                                    (cmd_batch, :101-129)
//   voxgpu voxelize --start x,y,z --end x,y,z --out path [--format xyz|vox3]   (cmd_voxelize,
//                :86-91; parametric only: the walk method is out of scope)
// Same defaults (format xyz), same stderr summary line, same exit codes (:237-253): 0 ok,
// 2 bad input (invalid_argument / range_error / usage), 3 I/O failure or internal error.
// Every voxel comes from the CUDA kernels through include/voxgpu.h; --workers/--group-size
// are validated (>= 1) like the reference but cannot change the output.
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/voxgpu.h"

namespace {

constexpr int kExitOk = 0, kExitBadInput = 2, kExitIoFailure = 3;

int usage(const char* msg) {
    std::fprintf(stderr,
                 "%s\nusage: voxgpu batch --input FILE.csv --out PATH [--format xyz|vox3] "
                 "[--workers N] [--group-size G]\n"
                 "       voxgpu voxelize --start x,y,z --end x,y,z --out PATH "
                 "[--format xyz|vox3]\n",
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

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage("a subcommand is required (batch | voxelize)");
    const std::string cmd = argv[1];
    std::string input, out, format = "xyz";
    bool have_start = false, have_end = false;
    double start[3], end[3];
    int workers = 1, group = 64;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (i + 1 >= argc) return usage(("missing value for " + a).c_str());
        const char* v = argv[++i];
        if (a == "--input" && cmd == "batch") input = v;
        else if (a == "--out") out = v;
        else if (a == "--format") {
            format = v;
            if (format != "xyz" && format != "vox3") return usage("--format: xyz or vox3");
        } else if (a == "--workers" && cmd == "batch") {
            if (!parse_int(v, workers)) return usage("--workers: a positive number");
        } else if (a == "--group-size" && cmd == "batch") {
            if (!parse_int(v, group)) return usage("--group-size: a positive number");
        } else if (a == "--start" && cmd == "voxelize") {
            if (!(have_start = parse_point(v, start))) return usage("--start: x,y,z");
        } else if (a == "--end" && cmd == "voxelize") {
            if (!(have_end = parse_point(v, end))) return usage("--end: x,y,z");
        } else if (a == "--method" && cmd == "voxelize") {
            if (std::strcmp(v, "parametric") != 0)
                return usage("--method: only parametric is on the GPU path");
        } else {
            return usage(("unknown option " + a).c_str());
        }
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
