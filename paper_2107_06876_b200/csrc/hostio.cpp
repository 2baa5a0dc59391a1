// Data formats and problem generators on either side of the path (SURVEY.md
// §8(f) row 3): LCNPTS1 / text point files (io.cpp) and the seeded
// uniform-ball / clustered generators (generators.cpp) the reference runner
// feeds into the solver (runner.cpp:180-204). Host code: files and RNG draws
// live on the host; the points then go to the device through the operator
// entry points. The generators draw from the same libstdc++ mt19937_64 and
// distributions as the reference, so the points are bit-identical.
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "lcn_b200.h"

namespace {

thread_local std::string g_io_error;

struct IoError {
    int code;
    std::string msg;
};

constexpr char kMagic[7] = {'L', 'C', 'N', 'P', 'T', 'S', '1'};

template <class F>
int io_guard(F&& f) {
    try {
        f();
        return LCN_OK;
    } catch (const IoError& e) {
        g_io_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_io_error = "out of host memory";
        return LCN_E_INVALID_ARGUMENT;
    }
}

[[noreturn]] void invalid(const std::string& m) { throw IoError{LCN_E_INVALID_ARGUMENT, m}; }

uint64_t read_u64_le(std::istream& in) {  // io.cpp:16-22
    std::array<unsigned char, 8> b{};
    in.read(reinterpret_cast<char*>(b.data()), 8);
    uint64_t v = 0;
    for (int k = 7; k >= 0; --k) v = (v << 8) | b[static_cast<size_t>(k)];
    return v;
}

void write_u64_le(std::ostream& out, uint64_t v) {
    std::array<unsigned char, 8> b{};
    for (int k = 0; k < 8; ++k) b[static_cast<size_t>(k)] = static_cast<unsigned char>(v >> (8 * k));
    out.write(reinterpret_cast<const char*>(b.data()), 8);
}

// PointSet::validate (geometry.cpp:10-18)
void validate(const std::vector<double>& x, uint64_t n, uint64_t d, const std::string& id) {
    if (n == 0 || d == 0) invalid("point set '" + id + "' is empty");
    for (double v : x)
        if (!std::isfinite(v)) invalid("point set '" + id + "' has non-finite coordinates");
}

// read_points_text (io.cpp:33-63): `n d`, then n rows of d values; blank
// lines and lines starting with '#' are skipped
void read_text(std::istream& in, const std::string& id, std::vector<double>& x, uint64_t& n, uint64_t& d) {
    std::string line;
    auto next = [&](std::string& out) {
        while (std::getline(in, out)) {
            const size_t pos = out.find_first_not_of(" \t\r");
            if (pos == std::string::npos || out[pos] == '#') continue;
            return true;
        }
        return false;
    };
    if (!next(line)) invalid("point file is empty");
    std::istringstream header(line);
    size_t hn = 0, hd = 0;
    if (!(header >> hn >> hd) || hn == 0 || hd == 0) invalid("point file header must be `n d` with n, d >= 1");
    n = hn;
    d = hd;
    x.assign(n * d, 0.0);
    for (size_t i = 0; i < n; ++i) {
        if (!next(line)) invalid("point file truncated at row " + std::to_string(i));
        std::istringstream row(line);
        for (size_t k = 0; k < d; ++k)
            if (!(row >> x[i * d + k])) invalid("point file row " + std::to_string(i) + " has fewer than d values");
    }
    validate(x, n, d, id);
}

// read_points_binary (io.cpp:77-95): magic, u64-LE n, u64-LE d, n*d f64-LE
void read_binary(std::istream& in, const std::string& id, std::vector<double>& x, uint64_t& n, uint64_t& d) {
    char magic[7];
    in.read(magic, 7);
    if (!in || std::memcmp(magic, kMagic, 7) != 0) invalid("bad point file magic");
    n = read_u64_le(in);
    d = read_u64_le(in);
    if (!in || n == 0 || d == 0) invalid("bad point file header");
    x.assign(n * d, 0.0);
    in.read(reinterpret_cast<char*>(x.data()), static_cast<std::streamsize>(x.size() * sizeof(double)));
    if (!in) invalid("point file truncated");
    validate(x, n, d, id);
}

// read_points_file (io.cpp:105-116): sniff the magic, else text
void read_file(const char* path, std::vector<double>& x, uint64_t& n, uint64_t& d) {
    if (!path) invalid("null path");
    std::ifstream in(path, std::ios::binary);
    if (!in) invalid(std::string("cannot open point file '") + path + "'");
    char magic[7];
    in.read(magic, 7);
    const bool binary = in && std::memcmp(magic, kMagic, 7) == 0;
    in.clear();
    in.seekg(0);
    if (binary) read_binary(in, path, x, n, d);
    else read_text(in, path, x, n, d);
}

// gaussian_direction (generators.cpp:10-22)
void gaussian_direction(std::mt19937_64& rng, double* out, size_t d) {
    std::normal_distribution<double> gauss(0.0, 1.0);
    double norm2 = 0.0;
    do {
        norm2 = 0.0;
        for (size_t k = 0; k < d; ++k) {
            out[k] = gauss(rng);
            norm2 += out[k] * out[k];
        }
    } while (norm2 == 0.0);
    const double inv = 1.0 / std::sqrt(norm2);
    for (size_t k = 0; k < d; ++k) out[k] *= inv;
}

}  // namespace

extern "C" {

const char* lcn_io_last_error(void) { return g_io_error.c_str(); }

int lcn_points_read(const char* path, double* out, size_t* n, size_t* d) {
    return io_guard([&] {
        if (!n || !d) invalid("null size pointers");
        std::vector<double> x;
        uint64_t rn = 0, rd = 0;
        read_file(path, x, rn, rd);
        if (out) {
            if (*n != rn || *d != rd) invalid("lcn_points_read: buffer shape differs from the file (query first)");
            std::memcpy(out, x.data(), x.size() * sizeof(double));
        }
        *n = rn;
        *d = rd;
    });
}

int lcn_points_write(const char* path, const double* pts, size_t n, size_t d, int binary) {
    return io_guard([&] {
        if (!path || (!pts && n * d)) invalid("null argument");
        std::ofstream out(path, binary ? std::ios::binary : std::ios::out);
        if (!out) invalid(std::string("cannot open '") + path + "' for writing");
        if (binary) {  // write_points_binary (io.cpp:97-103)
            out.write(kMagic, 7);
            write_u64_le(out, n);
            write_u64_le(out, d);
            out.write(reinterpret_cast<const char*>(pts), static_cast<std::streamsize>(n * d * sizeof(double)));
        } else {  // write_points_text (io.cpp:65-75): precision 17, default float format
            out << n << ' ' << d << '\n';
            out.precision(17);
            for (size_t i = 0; i < n; ++i) {
                for (size_t k = 0; k < d; ++k) {
                    if (k) out << ' ';
                    out << pts[i * d + k];
                }
                out << '\n';
            }
        }
        if (!out) invalid(std::string("write to '") + path + "' failed");
    });
}

// sample_uniform_ball (generators.cpp:26-40)
int lcn_sample_uniform_ball(size_t n, size_t d, uint64_t seed, double* out) {
    return io_guard([&] {
        if (n == 0 || d == 0) invalid("sample_uniform_ball: n and d must be positive");
        if (!out) invalid("null output");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unif(0.0, 1.0);
        for (size_t i = 0; i < n; ++i) {
            double* x = out + i * d;
            gaussian_direction(rng, x, d);
            const double radius = std::pow(unif(rng), 1.0 / static_cast<double>(d));
            for (size_t k = 0; k < d; ++k) x[k] *= radius;
        }
    });
}

// sample_clustered (generators.cpp:42-106): c centres >= D apart in a box of
// side 2 D ceil(c^(1/d)); both sides draw n points, each from a uniformly
// chosen centre plus a uniform-ball offset of radius r.
int lcn_sample_clustered(size_t n, size_t d, size_t c, double D, double r, uint64_t seed, double* p_out,
                         double* q_out, double* centers_out) {
    return io_guard([&] {
        if (n == 0 || d == 0 || c == 0) invalid("sample_clustered: sizes must be positive");
        if (!(D > 0.0) || !(r >= 0.0)) invalid("sample_clustered: D must be positive and r nonnegative");
        if (!p_out || !q_out) invalid("null output");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unif(0.0, 1.0);
        const double side = 2.0 * D * std::ceil(std::pow(static_cast<double>(c), 1.0 / static_cast<double>(d)));
        std::vector<double> ctr(c * d);
        for (size_t ci = 0; ci < c; ++ci) {
            int attempts = 0;
            while (true) {
                if (++attempts > 1000)
                    invalid("sample_clustered: cannot place centers >= D apart (D too large for box)");
                for (size_t k = 0; k < d; ++k) ctr[ci * d + k] = unif(rng) * side;
                bool ok = true;
                for (size_t cj = 0; cj < ci && ok; ++cj) {
                    double dist2 = 0.0;
                    for (size_t k = 0; k < d; ++k) {
                        const double diff = ctr[ci * d + k] - ctr[cj * d + k];
                        dist2 += diff * diff;
                    }
                    if (dist2 < D * D) ok = false;
                }
                if (ok) break;
            }
        }
        std::uniform_int_distribution<size_t> pick(0, c - 1);
        std::vector<double> dir(d);
        for (double* side_out : {p_out, q_out}) {
            for (size_t i = 0; i < n; ++i) {
                const size_t ci = pick(rng);
                gaussian_direction(rng, dir.data(), d);
                const double radius = r * std::pow(unif(rng), 1.0 / static_cast<double>(d));
                for (size_t k = 0; k < d; ++k) side_out[i * d + k] = ctr[ci * d + k] + radius * dir[k];
            }
        }
        if (centers_out) std::memcpy(centers_out, ctr.data(), ctr.size() * sizeof(double));
    });
}

}  // extern "C"
