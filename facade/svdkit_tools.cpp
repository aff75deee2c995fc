// svdkit_tools.cpp — the reference's experiment tooling on the B200 engine:
// cost model (cost_model.hpp), CSV matrices (csv_io.hpp), IDX images
// (idx_io.hpp) and the benchmark grid (bench.hpp).
//
// The cost model and the IDX header check go through the C-ABI
// (svdk_cost_model, svdk_idx_parse); images_to_matrix expands the pixels on
// the GPU (svdk_idx_to_matrix); run_grid times compute_svd and residual_delta,
// both GPU calls. Text formats are produced here so files and reports are
// byte-compatible with the reference's (checked in tests/test_host_tools.py
// and tests/test_gpu_facade.py).
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <map>
#include <sstream>
#include <string_view>
#include <system_error>

#include "svdk.h"
#include "svdkit/svdkit.hpp"

namespace svdkit {

namespace detail {
svdk_ctx* engine_ctx();
void engine_check(int code, std::size_t offset);
}  // namespace detail

namespace {

void check(int code, std::size_t offset = 0) { detail::engine_check(code, offset); }

CostEstimate cost(int model, std::size_t m, std::size_t n, std::size_t l, std::size_t i) {
    CostEstimate c;
    check(svdk_cost_model(model, m, n, l, i, &c.flops, &c.space_entries, &c.space_bytes));
    return c;
}

}  // namespace

// ---------------------------------------------------------------- cost model
CostEstimate truncated_cost(std::size_t m, std::size_t n) {
    return cost(SVDK_COST_TRUNCATED, m, n, 0, 0);
}
CostEstimate randomized_cost(std::size_t m, std::size_t n, std::size_t l, std::size_t i) {
    return cost(SVDK_COST_RANDOMIZED, m, n, l, i);
}
CostEstimate randomized_cost_practical(std::size_t m, std::size_t n) {
    return cost(SVDK_COST_RANDOMIZED_PRACTICAL, m, n, 0, 0);
}
CostEstimate krylov_cost(std::size_t m, std::size_t n, std::size_t l, std::size_t i) {
    return cost(SVDK_COST_KRYLOV, m, n, l, i);
}
CostEstimate krylov_cost_practical(std::size_t m, std::size_t n) {
    return cost(SVDK_COST_KRYLOV_PRACTICAL, m, n, 0, 0);
}
CostEstimate krylov_cost_per_step(std::size_t m, std::size_t n, std::size_t l, std::size_t i) {
    return cost(SVDK_COST_KRYLOV_PER_STEP, m, n, l, i);
}

// ---------------------------------------------------------------- CSV
std::string format_double(double value) {
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof buf, value);  // shortest round trip
    return std::string(buf, r.ptr);
}

namespace {

constexpr std::string_view kBlank = " \t\r";

std::string_view strip(std::string_view s) {
    const std::size_t a = s.find_first_not_of(kBlank);
    if (a == std::string_view::npos) return {};
    return s.substr(a, s.find_last_not_of(kBlank) - a + 1);
}

double number(std::string_view raw, std::size_t line) {
    const std::string_view t = strip(raw);
    double v = 0.0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (t.empty() || r.ec != std::errc{} || r.ptr != t.data() + t.size() || !std::isfinite(v))
        throw FormatError("csv: line " + std::to_string(line) + ": bad number '" + std::string(raw) + "'",
                          line);
    return v;
}

}  // namespace

DenseMatrix read_matrix_csv(std::istream& in) {
    std::vector<double> rowmajor;
    std::size_t width = 0, rows = 0, line_no = 0;
    std::string line;
    while (std::getline(in, line)) {
        ++line_no;
        if (strip(line).empty()) continue;
        std::size_t fields = 0;
        std::string_view rest(line);
        for (;;) {
            const std::size_t comma = rest.find(',');
            rowmajor.push_back(number(rest.substr(0, comma), line_no));
            ++fields;
            if (comma == std::string_view::npos) break;
            rest.remove_prefix(comma + 1);
        }
        if (rows > 0 && fields != width)
            throw FormatError("csv: line " + std::to_string(line_no) + " has " + std::to_string(fields) +
                                  " fields, expected " + std::to_string(width),
                              line_no);
        width = fields;
        ++rows;
    }
    if (rows == 0) throw FormatError("csv: no data rows", 0);
    DenseMatrix a(rows, width);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < width; ++j) a(i, j) = rowmajor[i * width + j];
    return a;
}

DenseMatrix read_matrix_csv_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open " + path);
    return read_matrix_csv(in);
}

void write_matrix_csv(const DenseMatrix& a, std::ostream& out) {
    for (std::size_t i = 0; i < a.rows(); ++i) {
        for (std::size_t j = 0; j < a.cols(); ++j) {
            if (j) out << ',';
            out << format_double(a(i, j));
        }
        out << '\n';
    }
}

namespace {

template <class F>
void write_file(const std::string& path, std::ios::openmode mode, F&& body) {
    std::ofstream out(path, mode);
    if (!out) throw IoError("cannot open " + path + " for writing");
    body(out);
    if (!out) throw IoError("write failed: " + path);
}

}  // namespace

void write_matrix_csv_file(const DenseMatrix& a, const std::string& path) {
    write_file(path, std::ios::out, [&](std::ostream& o) { write_matrix_csv(a, o); });
}

void write_vector_csv_file(const std::vector<double>& values, const std::string& path) {
    write_file(path, std::ios::out, [&](std::ostream& o) {
        for (double v : values) o << format_double(v) << '\n';
    });
}

// ---------------------------------------------------------------- IDX
IdxImageSet parse_idx_images(std::span<const std::uint8_t> bytes) {
    uint64_t dims[3] = {0, 0, 0}, offset = 0;
    const int code = svdk_idx_parse(bytes.data(), bytes.size(), dims, &offset);
    check(code, offset);
    IdxImageSet s;
    s.count = dims[0];
    s.height = dims[1];
    s.width = dims[2];
    s.pixels.assign(bytes.begin() + 16, bytes.end());
    return s;
}

IdxImageSet load_idx_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    const std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(in)),
                                          std::istreambuf_iterator<char>());
    return parse_idx_images(bytes);
}

DenseMatrix images_to_matrix(const IdxImageSet& set) {
    const std::size_t p = set.height * set.width;
    if (set.pixels.size() != set.count * p)
        throw ParamError("images_to_matrix: pixel buffer does not match the dimensions");
    std::vector<double> out(set.count * p);
    if (!out.empty())
        check(svdk_idx_to_matrix(detail::engine_ctx(), set.pixels.data(),
                                 static_cast<int64_t>(set.count), static_cast<int64_t>(p),
                                 out.data()));
    return DenseMatrix(set.count, p, std::move(out));
}

DenseMatrix image_as_matrix(const IdxImageSet& set, std::size_t index) {
    if (index >= set.count)
        throw ParamError("image index " + std::to_string(index) + " out of range, have " +
                         std::to_string(set.count) + " images");
    DenseMatrix img(set.height, set.width);
    const std::uint8_t* px = set.pixels.data() + index * set.height * set.width;
    for (std::size_t r = 0; r < set.height; ++r)
        for (std::size_t c = 0; c < set.width; ++c)
            img(r, c) = static_cast<double>(px[r * set.width + c]) / 255.0;
    return img;
}

// ---------------------------------------------------------------- bench grid
namespace {

// sketch-method seed stream offset (bench.cpp:22-24)
constexpr std::uint64_t kMethodSeedOffset = 0x9e3779b97f4a7c15ULL;

bool by_name(SvdMethod a, SvdMethod b) {
    return std::string_view(method_name(a)) < std::string_view(method_name(b));
}

}  // namespace

std::vector<std::pair<std::size_t, std::size_t>> expand_grid(const BenchConfig& cfg) {
    if (cfg.row_sizes.empty() || cfg.col_sizes.empty()) throw ParamError("bench: empty grid");
    if (cfg.methods.empty()) throw ParamError("bench: no methods selected");
    if (cfg.repeats < 1) throw ParamError("bench: repeats must be >= 1");
    if (!(cfg.l_fraction > 0.0 && cfg.l_fraction <= 1.0))
        throw ParamError("bench: l_fraction must be in (0, 1]");
    std::vector<std::size_t> rows = cfg.row_sizes, cols = cfg.col_sizes;
    std::sort(rows.begin(), rows.end());
    std::sort(cols.begin(), cols.end());
    if (rows.front() < cols.back()) {
        // report the first offending cell in input order, like the reference
        for (std::size_t m : cfg.row_sizes)
            for (std::size_t n : cfg.col_sizes)
                if (m < n)
                    throw ParamError("bench: grid cell " + std::to_string(m) + "x" + std::to_string(n) +
                                     " violates m >= n");
    }
    std::vector<std::pair<std::size_t, std::size_t>> cells;
    cells.reserve(rows.size() * cols.size());
    for (std::size_t m : rows)
        for (std::size_t n : cols) cells.emplace_back(m, n);
    return cells;
}

std::size_t sketch_width_for(const BenchConfig& cfg, std::size_t n) {
    const auto l = static_cast<std::size_t>(std::ceil(cfg.l_fraction * static_cast<double>(n)));
    return std::clamp<std::size_t>(l, 1, n);
}

GridResult run_grid(const BenchConfig& cfg) {
    const auto cells = expand_grid(cfg);
    std::vector<SvdMethod> methods = cfg.methods;
    std::sort(methods.begin(), methods.end(), by_name);
    methods.erase(std::unique(methods.begin(), methods.end()), methods.end());
    GridResult out;
    for (const auto& [m, n] : cells) {
        const double bytes = 8.0 * static_cast<double>(m) * static_cast<double>(n);
        const std::size_t l = sketch_width_for(cfg, n);
        for (SvdMethod method : methods) {
            if (bytes > cfg.memory_cap_bytes) {
                out.skipped.push_back({method, m, n,
                                       "matrix needs " + std::to_string(bytes) + " bytes, cap is " +
                                           std::to_string(cfg.memory_cap_bytes)});
                continue;
            }
            const std::size_t width = (cfg.iterations + 1) * l;
            if (method == SvdMethod::Krylov && width > m) {
                out.skipped.push_back({method, m, n,
                                       "krylov block width " + std::to_string(width) +
                                           " exceeds m = " + std::to_string(m)});
                continue;
            }
            CostEstimate model;
            switch (method) {
                case SvdMethod::Truncated: model = truncated_cost(m, n); break;
                case SvdMethod::Randomized: model = randomized_cost(m, n, l, cfg.iterations); break;
                case SvdMethod::Krylov: model = krylov_cost(m, n, l, cfg.iterations); break;
                default: throw ParamError("bench: no published cost model for lanczos");
            }
            std::vector<double> secs;
            double delta = 0.0;
            for (std::size_t trial = 0; trial < cfg.repeats; ++trial) {
                const DenseMatrix a = gaussian_matrix(m, n, RngSeed{cfg.seed.value + trial});
                const MethodParams params{l, cfg.iterations,
                                          RngSeed{cfg.seed.value + kMethodSeedOffset + trial}};
                const auto t0 = std::chrono::steady_clock::now();
                const SvdResult s = compute_svd(a, method, params);
                const auto t1 = std::chrono::steady_clock::now();
                secs.push_back(std::chrono::duration<double>(t1 - t0).count());
                delta += residual_delta(a, s);
            }
            const double reps = static_cast<double>(cfg.repeats);
            double mean = 0.0;
            for (double t : secs) mean += t;
            mean /= reps;
            double var = 0.0;
            if (cfg.repeats > 1) {
                for (double t : secs) var += (t - mean) * (t - mean);
                var /= reps - 1.0;
            }
            out.records.push_back({method, m, n, cfg.repeats, mean, std::sqrt(var), delta / reps,
                                   model.flops, model.space_bytes});
        }
    }
    return out;
}

std::string to_csv(const std::vector<BenchRecord>& records) {
    std::string s = "method,m,n,repeats,mean_seconds,std_seconds,delta,model_flops,model_space_bytes\n";
    for (const BenchRecord& r : records) {
        s += method_name(r.method);
        for (std::size_t v : {r.m, r.n, r.repeats}) s += "," + std::to_string(v);
        for (double v : {r.mean_seconds, r.std_seconds, r.delta, r.model_flops, r.model_space_bytes})
            s += "," + format_double(v);
        s += '\n';
    }
    return s;
}

void write_csv_file(const std::vector<BenchRecord>& records, const std::string& path) {
    write_file(path, std::ios::binary, [&](std::ostream& o) { o << to_csv(records); });
}

OrderingReport summarize_ordering(const std::vector<BenchRecord>& records) {
    std::map<std::pair<std::size_t, std::size_t>, std::vector<const BenchRecord*>> cells;
    for (const BenchRecord& r : records) cells[{r.m, r.n}].push_back(&r);
    OrderingReport rep;
    std::size_t agree = 0;
    for (const auto& [shape, recs] : cells) {
        auto order = [&](double BenchRecord::*key) {
            std::vector<const BenchRecord*> v = recs;
            std::sort(v.begin(), v.end(), [&](const BenchRecord* a, const BenchRecord* b) {
                if (a->*key != b->*key) return a->*key < b->*key;
                return by_name(a->method, b->method);
            });
            std::vector<SvdMethod> o;
            for (const BenchRecord* r : v) o.push_back(r->method);
            return o;
        };
        OrderingCell c;
        c.m = shape.first;
        c.n = shape.second;
        c.by_seconds = order(&BenchRecord::mean_seconds);
        c.by_flops = order(&BenchRecord::model_flops);
        c.agree = c.by_seconds == c.by_flops;
        agree += c.agree;
        rep.cells.push_back(std::move(c));
    }
    rep.agreement = rep.cells.empty() ? 0.0
                                      : static_cast<double>(agree) / static_cast<double>(rep.cells.size());
    return rep;
}

std::string format_report(const OrderingReport& report) {
    auto chain = [](const std::vector<SvdMethod>& v) {
        std::string s;
        for (std::size_t i = 0; i < v.size(); ++i) s += (i ? " < " : "") + std::string(method_name(v[i]));
        return s;
    };
    std::string s =
        "cell            measured (fast->slow)              modeled (cheap->costly)            agree\n";
    char line[160];
    for (const OrderingCell& c : report.cells) {
        std::snprintf(line, sizeof line, "%6zux%-6zu  %-34s %-34s %s\n", c.m, c.n, chain(c.by_seconds).c_str(),
                      chain(c.by_flops).c_str(), c.agree ? "yes" : "NO");
        s += line;
    }
    std::snprintf(line, 64, "ranking agreement: %.2f\n", report.agreement);
    return s + line;
}

}  // namespace svdkit
