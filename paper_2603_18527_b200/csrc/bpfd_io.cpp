// bpfd_io.cpp -- native implementation of include/bornsweep_io.h (host side of the I/O row,
// SURVEY.md 8(f) #4).  Plain stdio: one header write + one payload write per field, so
// multi-GB fields stream at disk speed; the layout is the reference's (proj/src/field.cpp).
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>

#include "bornsweep_io.h"

namespace {

thread_local std::string g_err;
constexpr char kMagic[4] = {'B', 'P', 'F', 'D'};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

size_t payload_doubles(int32_t nx, int32_t ny, int32_t dtype) {
    return (size_t)nx * (size_t)ny * (dtype == BP_BPFD_COMPLEX128 ? 2 : 1);
}

bool valid_dtype(int32_t d) { return d == BP_BPFD_REAL64 || d == BP_BPFD_COMPLEX128; }

// "%.17g": std::ostream with precision(17) and the default float field (the reference's CSV
// writers, field.cpp:143,153 and iterate.cpp:158)
void put(FILE* f, double v) { std::fprintf(f, "%.17g", v); }

}  // namespace

extern "C" {

const char* bp_io_last_error(void) { return g_err.c_str(); }

int bp_bpfd_save(const char* path, int32_t nx, int32_t ny, int32_t dtype, const double* data) {
    if (!path || (!data && nx * ny > 0)) return fail(1, "null argument");
    if (nx < 0 || ny < 0 || !valid_dtype(dtype)) return fail(1, "bad field shape or dtype");
    File out;
    out.f = std::fopen(path, "wb");
    if (!out.f) return fail(2, std::string("cannot open for writing: ") + path);
    const uint32_t hdr[3] = {(uint32_t)nx, (uint32_t)ny, (uint32_t)dtype};
    const size_t n = payload_doubles(nx, ny, dtype);
    if (std::fwrite(kMagic, 1, 4, out.f) != 4 || std::fwrite(hdr, 4, 3, out.f) != 3 ||
        std::fwrite(data, sizeof(double), n, out.f) != n)
        return fail(2, std::string("write failed: ") + path);
    if (std::fclose(out.f) != 0) {
        out.f = nullptr;
        return fail(2, std::string("write failed: ") + path);
    }
    out.f = nullptr;
    return 0;
}

static int read_header(FILE* f, uint32_t* hdr) {
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        return fail(2, "field file: bad magic");
    if (std::fread(hdr, 4, 3, f) != 3) return fail(2, "field file: truncated header");
    return 0;
}

int bp_bpfd_info(const char* path, int32_t* nx, int32_t* ny, int32_t* dtype) {
    if (!path) return fail(1, "null argument");
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) return fail(2, std::string("cannot open for reading: ") + path);
    uint32_t hdr[3];
    if (int rc = read_header(in.f, hdr)) return rc;
    if (nx) *nx = (int32_t)hdr[0];
    if (ny) *ny = (int32_t)hdr[1];
    if (dtype) *dtype = (int32_t)hdr[2];
    return 0;
}

int bp_bpfd_load(const char* path, int32_t nx, int32_t ny, int32_t dtype, double* out) {
    if (!path || !out) return fail(1, "null argument");
    if (!valid_dtype(dtype)) return fail(1, "bad dtype");
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) return fail(2, std::string("cannot open for reading: ") + path);
    uint32_t hdr[3];
    if (int rc = read_header(in.f, hdr)) return rc;
    if ((int32_t)hdr[2] != dtype)
        return fail(2, dtype == BP_BPFD_REAL64 ? "field file: expected real64" : "field file: expected complex128");
    if ((int32_t)hdr[0] != nx || (int32_t)hdr[1] != ny) return fail(1, "field file: shape mismatch");
    const size_t n = payload_doubles(nx, ny, dtype);
    if (std::fread(out, sizeof(double), n, in.f) != n) return fail(2, "field file: truncated payload");
    return 0;
}

int bp_csv_export(const char* path, int32_t nx, int32_t ny, int32_t dtype, const double* data) {
    if (!path || !data || !valid_dtype(dtype)) return fail(1, "null argument or bad dtype");
    File out;
    out.f = std::fopen(path, "w");
    if (!out.f) return fail(2, std::string("cannot open for writing: ") + path);
    const bool cx = dtype == BP_BPFD_COMPLEX128;
    std::fputs(cx ? "ix,iy,re,im\n" : "ix,iy,value\n", out.f);
    for (int32_t i = 0; i < nx; ++i)
        for (int32_t j = 0; j < ny; ++j) {
            const size_t k = (size_t)i * ny + j;
            std::fprintf(out.f, "%d,%d,", i, j);
            if (cx) {
                put(out.f, data[2 * k]);
                std::fputc(',', out.f);
                put(out.f, data[2 * k + 1]);
            } else {
                put(out.f, data[k]);
            }
            std::fputc('\n', out.f);
        }
    return 0;
}

int bp_trace_csv_write(const char* path, int32_t n, const double* res_l2, const double* res_reta) {
    if (!path || n < 0 || (n > 0 && (!res_l2 || !res_reta))) return fail(1, "null argument");
    File out;
    out.f = std::fopen(path, "w");
    if (!out.f) return fail(2, std::string("cannot open for writing: ") + path);
    std::fputs("step,res_l2_rel,res_Reta_rel\n", out.f);
    for (int32_t i = 0; i < n; ++i) {
        std::fprintf(out.f, "%d,", i);
        put(out.f, res_l2[i]);
        std::fputc(',', out.f);
        put(out.f, res_reta[i]);
        std::fputc('\n', out.f);
    }
    return 0;
}

}  // extern "C"
