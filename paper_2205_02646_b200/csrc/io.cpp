// io.cpp -- the reference's file formats, host side:
// binary PGM (P5, 8/16-bit), TQSP pattern text files and TQSM float64 containers
// (frames and full-precision image dumps), behind the C ABI in tqsb.h so that the
// CLI (tools/tqsb_cli.cpp), the C++ face (include/tqsb/io.hpp) and the Python
// tests share one implementation.
//
// Format and error behaviour follow include/tqs/io.hpp:1-35 and src/io.cpp:1-271 of
// the reference: files written here are byte-identical to the reference's, the
// readers accept exactly what the reference accepts, and failures carry the
// reference's "<path>: <what>" messages (runtime_error -> TQSB_EIO,
// invalid_argument -> TQSB_EINVAL).
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tqsb/tqsb.h"

int tqsb_internal_set_error(int code, const std::string& msg);  // plan.cpp

namespace {

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

[[noreturn]] void io_fail(const std::string& path, const std::string& what) {
    throw IoError(path + ": " + what);
}

// whole-file read; the parsers below work on the byte vector
std::vector<unsigned char> slurp(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) io_fail(path, "cannot open for reading");
    std::vector<unsigned char> buf;
    unsigned char chunk[1 << 16];
    size_t n;
    while ((n = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + n);
    std::fclose(f);
    return buf;
}

void spit(const std::string& path, const std::vector<unsigned char>& bytes) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) io_fail(path, "cannot open for writing");
    const bool ok = bytes.empty() || std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
    if (std::fclose(f) != 0 || !ok) io_fail(path, "write failed");
}

void put_u32(std::vector<unsigned char>& o, uint32_t v) {
    for (int i = 0; i < 4; ++i) o.push_back(static_cast<unsigned char>(v >> (8 * i)));
}
void put_u64(std::vector<unsigned char>& o, uint64_t v) {
    for (int i = 0; i < 8; ++i) o.push_back(static_cast<unsigned char>(v >> (8 * i)));
}
uint64_t get_le(const unsigned char* p, int n) {
    uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= uint64_t(p[i]) << (8 * i);
    return v;
}

// ---------------------------------------------------------------- PGM (P5)
// Header tokens: whitespace-separated, '#' starts a comment to end of line when it
// opens a token; the whitespace byte ending the maxval token is consumed and the
// samples follow it (the reference's pnm_token, io.cpp:33-50).
struct Cursor {
    const std::vector<unsigned char>& b;
    size_t i = 0;
    int get() { return i < b.size() ? b[i++] : EOF; }
};

std::string header_token(Cursor& c) {
    std::string tok;
    int ch;
    while ((ch = c.get()) != EOF) {
        if (ch == '#') {
            while ((ch = c.get()) != EOF && ch != '\n') {
            }
            continue;
        }
        if (!std::isspace(ch)) {
            tok.push_back(char(ch));
            break;
        }
    }
    while ((ch = c.get()) != EOF && !std::isspace(ch)) tok.push_back(char(ch));
    return tok;
}

long header_long(const std::string& path, const std::string& tok, const char* field) {
    try {
        size_t used = 0;
        const long v = std::stol(tok, &used);
        if (used == tok.size()) return v;
    } catch (const std::exception&) {
    }
    io_fail(path, std::string("malformed ") + field + " field");
}

void read_pgm(const std::string& path, int* rows, int* cols, double* out) {
    const std::vector<unsigned char> b = slurp(path);
    Cursor c{b};
    if (header_token(c) != "P5") io_fail(path, "not a binary PGM (P5) file");
    const long w = header_long(path, header_token(c), "width");
    const long h = header_long(path, header_token(c), "height");
    const long maxval = header_long(path, header_token(c), "maxval");
    if (w <= 0 || h <= 0) io_fail(path, "non-positive dimensions");
    if (maxval <= 0 || maxval > 65535) io_fail(path, "unsupported maxval");
    const size_t n = size_t(w) * size_t(h), bps = maxval < 256 ? 1 : 2;
    if (b.size() - c.i < n * bps) io_fail(path, "truncated pixel data");
    *rows = int(h);
    *cols = int(w);
    if (!out) return;
    const double step = 1.0 / double(maxval);
    const unsigned char* s = b.data() + c.i;
    for (size_t k = 0; k < n; ++k)  // 16-bit samples are big-endian
        out[k] = (bps == 1 ? unsigned(s[k]) : (unsigned(s[2 * k]) << 8 | s[2 * k + 1])) * step;
}

void write_pgm(const std::string& path, const double* img, int rows, int cols, int bits) {
    if (bits != 8 && bits != 16) throw std::invalid_argument("write_pgm: bit depth must be 8 or 16");
    if (rows <= 0 || cols <= 0) throw std::invalid_argument("write_pgm: empty image");
    const unsigned top = bits == 8 ? 255u : 65535u;
    const std::string head = "P5\n" + std::to_string(cols) + " " + std::to_string(rows) + "\n" +
                             std::to_string(top) + "\n";
    std::vector<unsigned char> o(head.begin(), head.end());
    const size_t n = size_t(rows) * cols;
    o.reserve(o.size() + n * (bits / 8));
    for (size_t k = 0; k < n; ++k) {
        const double x = img[k] < 0.0 ? 0.0 : (img[k] > 1.0 ? 1.0 : img[k]);
        const unsigned q = static_cast<unsigned>(std::lround(x * top));
        if (bits == 16) o.push_back(static_cast<unsigned char>(q >> 8));
        o.push_back(static_cast<unsigned char>(q & 0xff));
    }
    spit(path, o);
}

// ---------------------------------------------------------------- TQSM
// "TQSM", u32 rows, u32 cols (little-endian), rows*cols float64 row-major
void read_tqsm(const std::string& path, int* rows, int* cols, double* out) {
    const std::vector<unsigned char> b = slurp(path);
    if (b.size() < 4 || std::memcmp(b.data(), "TQSM", 4) != 0) io_fail(path, "not a TQSM file");
    if (b.size() < 12) io_fail(path, "implausible dimensions");
    const uint64_t r = get_le(b.data() + 4, 4), c = get_le(b.data() + 8, 4);
    if (r == 0 || c == 0 || r > (1u << 20) || c > (1u << 20)) io_fail(path, "implausible dimensions");
    if (b.size() - 12 < r * c * 8) io_fail(path, "truncated payload");
    *rows = int(r);
    *cols = int(c);
    if (!out) return;
    for (size_t k = 0; k < r * c; ++k) {
        const uint64_t bits = get_le(b.data() + 12 + 8 * k, 8);
        std::memcpy(out + k, &bits, 8);
    }
}

void write_tqsm(const std::string& path, const double* v, int rows, int cols) {
    std::vector<unsigned char> o = {'T', 'Q', 'S', 'M'};
    put_u32(o, uint32_t(rows));
    put_u32(o, uint32_t(cols));
    const size_t n = size_t(rows) * size_t(cols);
    o.reserve(o.size() + 8 * n);
    for (size_t k = 0; k < n; ++k) {
        uint64_t bits;
        std::memcpy(&bits, v + k, 8);
        put_u64(o, bits);
    }
    spit(path, o);
}

// ---------------------------------------------------------------- TQSP
// "TQSP v1 period=<P> seed=<S> rng=<name>", then P/2 rows of P/2 quadrant digits
struct PatternText {
    int period = 0;
    unsigned long long seed = 0;
    std::string rng;
    std::vector<uint8_t> opaque;
};

PatternText read_tqsp(const std::string& path) {
    const std::vector<unsigned char> b = slurp(path);
    std::istringstream in(std::string(b.begin(), b.end()));
    std::string line;
    if (!std::getline(in, line)) io_fail(path, "empty pattern file");
    std::istringstream head(line);
    std::string magic, version, field;
    head >> magic >> version;
    if (magic != "TQSP" || version != "v1") io_fail(path, "not a TQSP v1 pattern file");
    PatternText p;
    bool have_period = false, have_seed = false;
    while (head >> field) {
        const size_t eq = field.find('=');
        if (eq == std::string::npos) io_fail(path, "malformed header field '" + field + "'");
        const std::string key = field.substr(0, eq), val = field.substr(eq + 1);
        if (key == "period") {
            p.period = int(header_long(path, val, "period"));
            have_period = true;
        } else if (key == "seed") {
            try {
                p.seed = std::stoull(val);
            } catch (const std::exception&) {
                io_fail(path, "malformed seed field");
            }
            have_seed = true;
        } else if (key == "rng") {
            p.rng = val;
        } else {
            io_fail(path, "unknown header field '" + key + "'");
        }
    }
    if (!have_period || !have_seed) io_fail(path, "header missing period or seed");
    if (p.period < 4 || p.period % 2 != 0) io_fail(path, "invalid period");
    const int pc = p.period / 2;
    for (int r = 0; r < pc; ++r) {
        if (!std::getline(in, line)) io_fail(path, "truncated pattern grid");
        std::istringstream row(line);
        for (int c = 0; c < pc; ++c) {
            int q;
            if (!(row >> q) || q < 0 || q > 3) io_fail(path, "invalid quadrant digit in pattern grid");
            p.opaque.push_back(uint8_t(q));
        }
        int extra;
        if (row >> extra) io_fail(path, "excess values in pattern row");
    }
    return p;
}

void write_tqsp(const std::string& path, int period, unsigned long long seed, const std::string& rng,
                const uint8_t* opaque) {
    std::string s = "TQSP v1 period=" + std::to_string(period) + " seed=" + std::to_string(seed) +
                    " rng=" + rng + "\n";
    const int pc = period / 2;
    for (int r = 0; r < pc; ++r) {
        for (int c = 0; c < pc; ++c) {
            if (c) s.push_back(' ');
            s += std::to_string(int(opaque[size_t(r) * pc + c]));
        }
        s.push_back('\n');
    }
    spit(path, std::vector<unsigned char>(s.begin(), s.end()));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return TQSB_OK;
    } catch (const std::invalid_argument& e) {
        return tqsb_internal_set_error(TQSB_EINVAL, e.what());
    } catch (const std::exception& e) {
        return tqsb_internal_set_error(TQSB_EIO, e.what());
    }
}

}  // namespace

extern "C" {

int tqsb_io_read(const char* path, int kind, int* rows, int* cols, double* out) {
    return guarded([&] {
        if (!path || !rows || !cols) throw std::invalid_argument("tqsb_io_read: null argument");
        const std::string p(path);
        switch (kind) {
            case TQSB_IO_PGM: read_pgm(p, rows, cols, out); break;
            case TQSB_IO_TQSM: read_tqsm(p, rows, cols, out); break;
            case TQSB_IO_ANY: {  // sniff the leading magic (read_image_any, io.cpp:261-269)
                std::FILE* f = std::fopen(path, "rb");
                if (!f) io_fail(p, "cannot open for reading");
                char magic[4] = {0, 0, 0, 0};
                const size_t got = std::fread(magic, 1, 4, f);
                std::fclose(f);
                if (got == 4 && std::memcmp(magic, "TQSM", 4) == 0)
                    read_tqsm(p, rows, cols, out);
                else
                    read_pgm(p, rows, cols, out);
                break;
            }
            default: throw std::invalid_argument("tqsb_io_read: unknown kind");
        }
    });
}

int tqsb_io_write_pgm(const char* path, const double* image, int rows, int cols, int bits) {
    return guarded([&] {
        if (!path || (!image && rows > 0 && cols > 0))
            throw std::invalid_argument("tqsb_io_write_pgm: null argument");
        write_pgm(path, image, rows, cols, bits);
    });
}

int tqsb_io_write_tqsm(const char* path, const double* values, int rows, int cols) {
    return guarded([&] {
        if (!path || !values || rows < 0 || cols < 0)
            throw std::invalid_argument("tqsb_io_write_tqsm: invalid argument");
        write_tqsm(path, values, rows, cols);
    });
}

int tqsb_io_read_pattern(const char* path, int* period, uint64_t* seed, char* rng, size_t rng_cap,
                         uint8_t* opaque) {
    return guarded([&] {
        if (!path || !period) throw std::invalid_argument("tqsb_io_read_pattern: null argument");
        const PatternText p = read_tqsp(path);
        *period = p.period;
        if (seed) *seed = p.seed;
        if (rng && rng_cap > 0) {
            const size_t n = std::min(rng_cap - 1, p.rng.size());
            std::memcpy(rng, p.rng.data(), n);
            rng[n] = '\0';
        }
        if (opaque) std::memcpy(opaque, p.opaque.data(), p.opaque.size());
    });
}

int tqsb_io_write_pattern(const char* path, int period, uint64_t seed, const char* rng,
                          const uint8_t* opaque) {
    return guarded([&] {
        if (!path || !opaque || period < 4 || period % 2 != 0)
            throw std::invalid_argument("tqsb_io_write_pattern: invalid argument");
        write_tqsp(path, period, seed, rng ? rng : "", opaque);
    });
}

}  // extern "C"
