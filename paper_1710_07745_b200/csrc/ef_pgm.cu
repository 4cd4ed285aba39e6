// ef_pgm.cu -- PGM ingest and egress for the drop-in (image.py:87-135 and the
// CLI's detect path, cli.py:82-90 + bench.py:129-133).
//
// Ingest: the header is parsed on the host (the reference's grammar: tokens
// separated by whitespace, '#' comments to end of line, P5 binary or P2 ASCII,
// maxval 1..255, exactly one whitespace byte before a P5 payload) and the
// pixels are decoded straight to u8 -- into a pinned buffer when the caller
// passes one -- instead of the reference's float64 array, so they can go to the
// GPU at 1 byte per pixel.  Errors carry the reference's message and byte
// offset (PgmFormatError(message, offset)).
// Egress: the traced edge map becomes the P5 payload (0 / 255 per pixel) on the
// device, next to the edge map; only the payload crosses PCIe.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "edgeforge_b200.h"
#include "ef_internal.h"
#include "ef_launch.cuh"

namespace {

thread_local std::string g_pgm_err;

bool is_space(uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c; }

// Python's repr() of a bytes token: b'...' (or b"..." when it holds a quote and
// no double quote), \t \n \r \\ escaped, other non-printables as \xhh.
std::string py_bytes_repr(const uint8_t* p, size_t n) {
    bool has_sq = false, has_dq = false;
    for (size_t i = 0; i < n; ++i) {
        has_sq |= p[i] == '\'';
        has_dq |= p[i] == '"';
    }
    const char q = (has_sq && !has_dq) ? '"' : '\'';
    std::string s = "b";
    s += q;
    for (size_t i = 0; i < n; ++i) {
        const uint8_t c = p[i];
        if (c == '\\') s += "\\\\";
        else if (c == (uint8_t)q) { s += '\\'; s += (char)c; }
        else if (c == '\t') s += "\\t";
        else if (c == '\n') s += "\\n";
        else if (c == '\r') s += "\\r";
        else if (c < 0x20 || c >= 0x7f) {
            char b[8];
            std::snprintf(b, sizeof b, "\\x%02x", c);
            s += b;
        } else s += (char)c;
    }
    s += q;
    return s;
}

struct Cursor {
    const uint8_t* d;
    size_t n;
    size_t pos = 0;
};

struct PgmError {
    std::string msg;
    int64_t offset;
};

// next token: skip whitespace and comments; false + error at end of data
bool next_token(Cursor& c, size_t& start, size_t& len, PgmError& e) {
    while (c.pos < c.n) {
        if (c.d[c.pos] == '#') {
            while (c.pos < c.n && c.d[c.pos] != '\n') ++c.pos;
        } else if (is_space(c.d[c.pos])) {
            ++c.pos;
        } else {
            break;
        }
    }
    if (c.pos >= c.n) {
        e = {"unexpected end of header", (int64_t)c.pos};
        return false;
    }
    start = c.pos;
    while (c.pos < c.n && !is_space(c.d[c.pos]) && c.d[c.pos] != '#') ++c.pos;
    len = c.pos - start;
    return true;
}

typedef unsigned __int128 u128;

std::string u128_str(u128 v) {
    if (v == 0) return "0";
    std::string s;
    while (v) {
        s.insert(s.begin(), (char)('0' + (int)(v % 10)));
        v /= 10;
    }
    return s;
}

// a decimal token (bytes.isdigit semantics); values beyond 2^64-1 saturate
// (`huge` set) -- they can only fail later checks
bool int_token(Cursor& c, const char* what, unsigned long long& v, bool& huge, PgmError& e) {
    size_t start, len;
    if (!next_token(c, start, len, e)) return false;
    for (size_t i = 0; i < len; ++i)
        if (c.d[start + i] < '0' || c.d[start + i] > '9') {
            e = {std::string("non-numeric ") + what + " token " + py_bytes_repr(c.d + start, len), (int64_t)start};
            return false;
        }
    u128 acc = 0;
    huge = false;
    for (size_t i = 0; i < len; ++i) {
        acc = acc * 10 + (unsigned)(c.d[start + i] - '0');
        if (acc > (u128)~0ull) {
            huge = true;
            acc = (u128)~0ull;
        }
    }
    v = (unsigned long long)acc;
    return true;
}

int fail_pgm(const PgmError& e, int64_t* err_offset) {
    g_pgm_err = e.msg;
    if (err_offset) *err_offset = e.offset;
    return EF_EINVAL;
}

}  // namespace

namespace ef {
__global__ void pgm_edges_kernel(const uint8_t* __restrict__ fin, long long n, uint8_t* __restrict__ out) {
    const long long nv = (((reinterpret_cast<uintptr_t>(fin) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) ? n / 16 : 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 v = reinterpret_cast<const uint4*>(fin)[i];
        // byte != 0 -> 0xff: (b | b >> 1 | ... ) & 1 per byte, times 255
        auto expand = [](unsigned w) {
            unsigned t = w | (w >> 4);
            t |= t >> 2;
            t |= t >> 1;
            return (t & 0x01010101u) * 0xffu;
        };
        reinterpret_cast<uint4*>(out)[i] = make_uint4(expand(v.x), expand(v.y), expand(v.z), expand(v.w));
    }
    for (long long i = nv * 16 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = fin[i] ? 255 : 0;
}
}  // namespace ef

extern "C" {

const char* ef_pgm_last_error(void) { return g_pgm_err.c_str(); }

int ef_pgm_parse(const uint8_t* data, size_t n, ef_pgm_info* info, int64_t* err_offset) {
    if (!data && n) return EF_EINVAL;
    if (!info) return EF_EINVAL;
    Cursor c{data, n};
    PgmError e;
    size_t ms, ml;
    if (!next_token(c, ms, ml, e)) return fail_pgm(e, err_offset);
    const bool p5 = ml == 2 && data[ms] == 'P' && data[ms + 1] == '5';
    const bool p2 = ml == 2 && data[ms] == 'P' && data[ms + 1] == '2';
    if (!p5 && !p2)
        return fail_pgm({"bad magic number " + py_bytes_repr(data + ms, ml) + ", expected P5 or P2", (int64_t)ms},
                        err_offset);
    unsigned long long w, h, mv;
    bool hw, hh, hm;
    if (!int_token(c, "width", w, hw, e) || !int_token(c, "height", h, hh, e) || !int_token(c, "maxval", mv, hm, e))
        return fail_pgm(e, err_offset);
    auto num = [](unsigned long long v, bool huge) { return huge ? std::string("(>18446744073709551615)") : std::to_string(v); };
    if (w < 1 || h < 1)
        return fail_pgm({"bad dimensions " + num(w, hw) + "x" + num(h, hh), (int64_t)c.pos}, err_offset);
    if (mv < 1 || mv > 255)
        return fail_pgm({"maxval " + num(mv, hm) + " out of supported range 1..255", (int64_t)c.pos}, err_offset);
    const u128 count = (u128)w * (u128)h;
    info->binary = p5 ? 1 : 0;
    info->maxval = (int32_t)mv;
    info->payload_offset = (int64_t)c.pos;
    if (p5) {
        if (c.pos >= n || !is_space(data[c.pos]))
            return fail_pgm({"missing whitespace after maxval", (int64_t)c.pos}, err_offset);
        const size_t at = c.pos + 1;
        const size_t avail = n - at;
        if ((u128)avail < count || hw || hh)
            return fail_pgm({"truncated payload: expected " + (hw || hh ? std::string("(overflow)") : u128_str(count)) +
                                 " bytes, got " + std::to_string(avail < count ? avail : (size_t)count),
                             (int64_t)n},
                            err_offset);
        info->payload_offset = (int64_t)at;
    }
    if (w > (unsigned long long)INT32_MAX || h > (unsigned long long)INT32_MAX)
        return fail_pgm({"image dimensions above 2^31-1 are not supported", (int64_t)c.pos}, err_offset);
    info->width = (int32_t)w;
    info->height = (int32_t)h;
    return EF_OK;
}

int ef_pgm_decode_u8(const uint8_t* data, size_t n, const ef_pgm_info* info, uint8_t* h_dst, int64_t* err_offset) {
    if (!data || !info || !h_dst) return EF_EINVAL;
    const int64_t count = (int64_t)info->width * info->height;
    int64_t pos;
    int maxv = 0;
    if (info->binary) {
        const uint8_t* p = data + info->payload_offset;
        // copy + running maximum in one pass (the payload may go to pinned memory)
        for (int64_t i = 0; i < count; ++i) {
            const uint8_t v = p[i];
            h_dst[i] = v;
            maxv = v > maxv ? v : maxv;
        }
        pos = info->payload_offset;  // the reference reports the offset of the payload start
    } else {
        Cursor c{data, n, (size_t)info->payload_offset};
        PgmError e;
        for (int64_t i = 0; i < count; ++i) {
            unsigned long long v;
            bool huge;
            if (!int_token(c, "pixel", v, huge, e))
                return fail_pgm({"truncated payload: pixel " + std::to_string(i) + " of " + std::to_string(count) +
                                     " missing",
                                 e.offset},
                                err_offset);
            const int vi = v > 255 ? 256 : (int)v;  // > maxval either way
            h_dst[i] = (uint8_t)(vi > 255 ? 255 : vi);
            maxv = vi > maxv ? vi : maxv;
        }
        pos = (int64_t)c.pos;
    }
    if (maxv > info->maxval)
        return fail_pgm({"pixel value exceeds maxval " + std::to_string(info->maxval), pos}, err_offset);
    return EF_OK;
}

int ef_pgm_header(int32_t width, int32_t height, char* h_out, size_t cap) {
    if (width < 1 || height < 1 || !h_out) return EF_EINVAL;
    const int len = std::snprintf(h_out, cap, "P5\n%d %d\n255\n", width, height);
    if (len < 0 || (size_t)len >= cap) return EF_EINVAL;
    return len;
}

int ef_pgm_encode_edges(const uint8_t* d_final, int64_t n, uint8_t* d_payload, void* stream) {
    if (n < 0 || (n && (!d_final || !d_payload))) return EF_EINVAL;
    if (!n) return EF_OK;
    const long long blocks = std::min<long long>((n / 16 + 255) / 256 + 1, 4096);
    ef::pgm_edges_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_final, n, d_payload);
    return cudaGetLastError() == cudaSuccess ? EF_OK : EF_ECUDA;
}

}  // extern "C"
