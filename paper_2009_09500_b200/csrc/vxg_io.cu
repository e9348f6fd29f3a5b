// vxg_io.cu -- host-side formats around the hot path, native C++:
//
//   vxg_read_segments_csv    read_segments_csv (src/formats.cpp:92-132): same grammar (six
//                            strtod fields, trailing blanks allowed, finite), same skipped lines
//                            ('#' first, all-blank) and the same error message naming the first
//                            bad line -- parsed by all host threads over newline-aligned chunks
//   vxg_write_chains         write_vox3_multi / write_xyz_multi (src/formats.cpp:140-185) of a
//                            batch's chains, straight from the GPU list: the VOX3 v2 body IS the
//                            flat 12-B record list, the segment table is the chain-offset diff
//
// No voxel is computed here: the chains come from vxg_batch_emit_list (the CUDA kernels).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/voxgpu.h"

namespace {

struct Line {
    const char* b;
    const char* e;
};

bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// One CSV line -> 6 doubles, following read_segments_csv: cells split on ',' (std::getline
// semantics: a trailing ',' ends the line without an extra empty cell), each cell parsed by
// strtod (what std::stod calls) with only whitespace allowed after the number, every value
// finite, exactly six cells.
bool parse_line(const char* b, const char* e, double out[6]) {
    std::string cell;
    int n = 0;
    const char* p = b;
    while (p < e) {
        const char* q = p;
        while (q < e && *q != ',') ++q;
        if (n >= 6) return false;
        cell.assign(p, q);
        const char* c = cell.c_str();
        char* end = nullptr;
        errno = 0;
        const double v = std::strtod(c, &end);
        if (end == c) return false;     // std::stod: invalid_argument
        if (errno == ERANGE) return false;  // std::stod: out_of_range (overflow or underflow)
        while (*end && is_space(*end)) ++end;
        if (*end || !std::isfinite(v)) return false;
        out[n++] = v;
        p = q < e ? q + 1 : q;
    }
    return n == 6;
}

bool skipped(const char* b, const char* e) {
    if (b < e && *b == '#') return true;
    for (const char* p = b; p < e; ++p)
        if (!is_space(*p)) return false;
    return true;
}

}  // namespace

extern "C" {

VXG_API vxg_status vxg_read_segments_csv(const char* path, vxg_segment** out, int64_t* n,
                                         int64_t* bad_line) {
    if (!path || !out || !n) return VXG_INVALID_ARGUMENT;
    *out = nullptr;
    *n = 0;
    if (bad_line) *bad_line = -1;
    FILE* f = std::fopen(path, "rb");
    if (!f) return VXG_IO_ERROR;
    std::vector<char> buf;
    {
        std::fseek(f, 0, SEEK_END);
        const long sz = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        if (sz < 0) {
            std::fclose(f);
            return VXG_IO_ERROR;
        }
        buf.resize((size_t)sz);
        if (sz > 0 && std::fread(buf.data(), 1, (size_t)sz, f) != (size_t)sz) {
            std::fclose(f);
            return VXG_IO_ERROR;
        }
        std::fclose(f);
    }
    // lines (std::getline: split on '\n'; a final unterminated line counts)
    std::vector<Line> lines;
    {
        const char* p = buf.data();
        const char* end = p + buf.size();
        while (p < end) {
            const char* q = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
            if (!q) q = end;
            lines.push_back({p, q});
            p = q + (q < end ? 1 : 0);
        }
    }
    const int64_t L = (int64_t)lines.size();
    // per line: -1 skipped, 0 ok, 1 bad; parse in parallel into a line-indexed scratch
    std::vector<double> vals((size_t)L * 6);
    std::vector<signed char> state((size_t)L, -1);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, L / 4096));
    std::vector<std::thread> pool;
    for (int64_t t = 0; t < nt; ++t) {
        pool.emplace_back([&, t] {
            const int64_t a = L * t / nt, b = L * (t + 1) / nt;
            for (int64_t i = a; i < b; ++i) {
                if (skipped(lines[(size_t)i].b, lines[(size_t)i].e)) continue;
                state[(size_t)i] = parse_line(lines[(size_t)i].b, lines[(size_t)i].e,
                                              vals.data() + 6 * i) ? 0 : 1;
            }
        });
    }
    for (auto& th : pool) th.join();
    int64_t count = 0;
    for (int64_t i = 0; i < L; ++i) {
        if (state[(size_t)i] == 1) {
            if (bad_line) *bad_line = i + 1;  // the first malformed line, 1-based
            return VXG_INVALID_ARGUMENT;
        }
        if (state[(size_t)i] == 0) ++count;
    }
    vxg_segment* segs =
        static_cast<vxg_segment*>(std::malloc(sizeof(vxg_segment) * (size_t)std::max<int64_t>(count, 1)));
    if (!segs) return VXG_OUT_OF_MEMORY;
    int64_t j = 0;
    for (int64_t i = 0; i < L; ++i)
        if (state[(size_t)i] == 0) std::memcpy(&segs[j++], vals.data() + 6 * i, sizeof(vxg_segment));
    *out = segs;
    *n = count;
    return VXG_OK;
}

VXG_API void vxg_free(void* p) { std::free(p); }

}  // extern "C"

// ------------------------------------------------------------------------------- writers
namespace {

bool put_le64(FILE* f, uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
    return std::fwrite(b, 1, 8, f) == 8;
}

// "x y z\n" with std::ostream's integer formatting (plain decimal, '-' for negatives).
char* put_int(char* p, int32_t v) {
    char tmp[12];
    int n = 0;
    uint32_t u = v < 0 ? 0u - (uint32_t)v : (uint32_t)v;
    do {
        tmp[n++] = (char)('0' + u % 10);
        u /= 10;
    } while (u);
    if (v < 0) *p++ = '-';
    while (n) *p++ = tmp[--n];
    return p;
}

}  // namespace

extern "C" {

VXG_API vxg_status vxg_write_chains(const char* path, int format, const vxg_voxel* voxels,
                                    const int64_t* chain_off, int64_t n) {
    if (!path || !chain_off || n < 0 || (format != 0 && format != 1)) return VXG_INVALID_ARGUMENT;
    FILE* f = std::fopen(path, "wb");
    if (!f) return VXG_IO_ERROR;
    std::vector<char> io(1 << 22);
    std::setvbuf(f, io.data(), _IOFBF, io.size());
    const uint64_t total = (uint64_t)(chain_off[n] - chain_off[0]);
    bool ok = true;
    if (format == 0) {  // VOX3 v2: magic, u32 version, u64 total, u64 n, u64 per chain, records
        ok = std::fwrite("VOX3", 1, 4, f) == 4;
        const unsigned char ver[4] = {2, 0, 0, 0};
        ok = ok && std::fwrite(ver, 1, 4, f) == 4 && put_le64(f, total) && put_le64(f, (uint64_t)n);
        for (int64_t i = 0; ok && i < n; ++i) ok = put_le64(f, (uint64_t)(chain_off[i + 1] - chain_off[i]));
        // the records: 12-B little-endian (x, y, z) == the flat list's bytes (x86 is LE)
        if (ok && total) ok = std::fwrite(voxels + chain_off[0], 12, total, f) == total;
    } else {  // xyz: "# segment i" before each chain, one "x y z" line per voxel
        std::vector<char> line(1 << 20);
        for (int64_t i = 0; ok && i < n; ++i) {
            char* p = line.data();
            p += std::snprintf(p, 32, "# segment %lld\n", (long long)i);
            for (int64_t k = chain_off[i]; k < chain_off[i + 1]; ++k) {
                if (p - line.data() > (long)line.size() - 64) {
                    ok = std::fwrite(line.data(), 1, (size_t)(p - line.data()), f) ==
                         (size_t)(p - line.data());
                    p = line.data();
                    if (!ok) break;
                }
                p = put_int(p, voxels[k].x);
                *p++ = ' ';
                p = put_int(p, voxels[k].y);
                *p++ = ' ';
                p = put_int(p, voxels[k].z);
                *p++ = '\n';
            }
            if (ok) ok = std::fwrite(line.data(), 1, (size_t)(p - line.data()), f) ==
                         (size_t)(p - line.data());
        }
    }
    if (std::fclose(f) != 0) ok = false;
    return ok ? VXG_OK : VXG_IO_ERROR;
}

}  // extern "C"
