// tools_test.cpp — a reference-style caller of the experiment tooling
// (svdkit/{cost_model,csv_io,idx_io,bench}.hpp) linked to libsvdkit.so.
//
//   tools_test host   prints cost-model values, number formatting, CSV / IDX
//                     error offsets and the bench CSV / ordering report for
//                     fixed inputs; tests/test_host_tools.py recomputes every
//                     line with the reference (oracle/_ref) and compares.
//                     Touches no GPU.
//   tools_test gpu    images_to_matrix and a tiny run_grid on the GPU
//                     (tests/test_gpu_facade.py).
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "svdkit/bench.hpp"
#include "svdkit/cost_model.hpp"
#include "svdkit/csv_io.hpp"
#include "svdkit/idx_io.hpp"

using namespace svdkit;

namespace {

std::vector<std::uint8_t> idx(std::uint32_t magic, std::uint32_t c, std::uint32_t h, std::uint32_t w,
                              std::size_t payload, std::size_t extra = 0) {
    std::vector<std::uint8_t> b;
    for (std::uint32_t v : {magic, c, h, w})
        for (int s = 24; s >= 0; s -= 8) b.push_back(static_cast<std::uint8_t>(v >> s));
    for (std::size_t k = 0; k < payload + extra; ++k) b.push_back(static_cast<std::uint8_t>((k * 7 + 3) & 255));
    return b;
}

std::vector<BenchRecord> records() {
    // the same table as tests/test_host_tools.py::TOOL_RECORDS
    return {
        {SvdMethod::Truncated, 1000, 100, 3, 0.012, 0.0005, 1e-15, 2.0e7, 8.0e5},
        {SvdMethod::Randomized, 1000, 100, 3, 0.004, 0.0001, 3.5e-3, 1.1e7, 6.4e5},
        {SvdMethod::Krylov, 1000, 100, 3, 0.007, 0.0, 2.5e-4, 9.9e10, 1.2e6},
        {SvdMethod::Truncated, 4000, 300, 1, 0.25, 0.0, 0.0, 7.2e8, 2.0e7},
        {SvdMethod::Randomized, 4000, 300, 1, 0.25, 0.0, 0.5, 3.3e8, 1.5e7},
    };
}

int host() {
    const std::size_t shapes[][4] = {{10, 4, 2, 1}, {60000, 784, 392, 1}, {200000, 1024, 1024, 2},
                                     {3, 4, 1, 1},  {10, 4, 5, 1},        {10, 4, 2, 0}};
    for (const auto& s : shapes) {
        for (int model = 0; model < 6; ++model) {
            std::printf("cost %d %zu %zu %zu %zu ", model, s[0], s[1], s[2], s[3]);
            try {
                CostEstimate c;
                switch (model) {
                    case 0: c = truncated_cost(s[0], s[1]); break;
                    case 1: c = randomized_cost(s[0], s[1], s[2], s[3]); break;
                    case 2: c = randomized_cost_practical(s[0], s[1]); break;
                    case 3: c = krylov_cost(s[0], s[1], s[2], s[3]); break;
                    case 4: c = krylov_cost_practical(s[0], s[1]); break;
                    default: c = krylov_cost_per_step(s[0], s[1], s[2], s[3]); break;
                }
                std::printf("%a %a %a\n", c.flops, c.space_entries, c.space_bytes);
            } catch (const ParamError&) {
                std::printf("ParamError\n");
            }
        }
    }
    for (double v : {0.0, -0.0, 0.1, 1e-4, 1e-5, 123.0, 1e16, 1e21, 123456789012345680.0, 5e-324,
                     1.7976931348623157e308, -2.5e-7, 299792458.0, 0.30000000000000004})
        std::printf("fmt %a %s\n", v, format_double(v).c_str());
    for (const char* text : {"1,2\n3\n", "1,x\n", "", "1,2\n\n3,nan\n"}) {
        std::istringstream in(text);
        try {
            read_matrix_csv(in);
            std::printf("csv ok\n");
        } catch (const FormatError& e) {
            std::printf("csv FormatError %zu\n", e.offset());
        }
    }
    {
        std::istringstream in("1.5, -2e-3\n\n 7,8\r\n");
        const DenseMatrix a = read_matrix_csv(in);
        std::ostringstream out;
        write_matrix_csv(a, out);
        std::printf("csvrt %zu %zu %s", a.rows(), a.cols(), out.str().c_str());
    }
    const std::vector<std::vector<std::uint8_t>> cases = {
        idx(0x803, 3, 4, 5, 60),      idx(0x803, 1, 1, 1, 1),      std::vector<std::uint8_t>(7, 0),
        idx(0x801, 3, 4, 5, 60),      idx(0x803, 0, 4, 5, 0),      idx(0x803, 3, 4, 5, 59),
        idx(0x803, 3, 4, 5, 60, 2),
    };
    for (std::size_t k = 0; k < cases.size(); ++k) {
        try {
            const IdxImageSet s = parse_idx_images(cases[k]);
            const DenseMatrix img = image_as_matrix(s, s.count - 1);
            std::printf("idx %zu %zu %zu %zu %a\n", k, s.count, s.height, s.width, img(img.rows() - 1, 0));
        } catch (const FormatError& e) {
            std::printf("idx %zu FormatError %zu\n", k, e.offset());
        }
    }
    const BenchConfig cfg{{4000, 1000}, {300, 100}, {SvdMethod::Truncated}};
    for (const auto& [m, n] : expand_grid(cfg)) std::printf("cell %zu %zu\n", m, n);
    for (std::size_t n : {1, 3, 784, 1001}) std::printf("width %zu %zu\n", n, sketch_width_for(cfg, n));
    std::printf("--csv--\n%s--report--\n%s--end--\n", to_csv(records()).c_str(),
                format_report(summarize_ordering(records())).c_str());
    return 0;
}

int gpu() {
    const auto bytes = idx(0x803, 70, 9, 11, 70 * 99);
    const IdxImageSet s = parse_idx_images(bytes);
    const DenseMatrix a = images_to_matrix(s);
    int bad = 0;
    for (std::size_t i = 0; i < s.count; ++i)
        for (std::size_t p = 0; p < 99; ++p)
            bad += a(i, p) != static_cast<double>(s.pixels[i * 99 + p]) / 255.0;
    BenchConfig cfg{{300}, {40}, {SvdMethod::Krylov, SvdMethod::Randomized, SvdMethod::Truncated}};
    cfg.repeats = 2;
    const GridResult g = run_grid(cfg);
    for (const BenchRecord& r : g.records) bad += !(r.mean_seconds > 0.0 && r.delta >= 0.0 && r.delta < 1.0);
    bad += g.records.size() != 3 || g.records[2].delta > 1e-12;
    std::printf("%s%s", to_csv(g.records).c_str(), format_report(summarize_ordering(g.records)).c_str());
    std::printf(bad ? "tools_test gpu: FAIL %d\n" : "tools_test gpu: ok\n", bad);
    return bad ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "host";
    return mode == "gpu" ? gpu() : host();
}
