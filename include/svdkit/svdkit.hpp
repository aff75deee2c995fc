// svdkit.hpp — C++ drop-in facade of the B200 engine (libsvdkit.so).
//
// Declares the public API of the reference library svdkit (reference
// proj/include/svdkit/{dense_matrix,errors,kernels,svd_methods,pca}.hpp) with
// identical names, signatures and exception behaviour, so existing callers
// recompile unchanged against this header set and link libsvdkit.so instead.
// Every compute call is forwarded to the C-ABI in svdk.h (GPU); the
// per-file headers next to this one just include it.
//
// Additions over the reference: SvdMethod::Lanczos, and EngineError for
// CUDA / NCCL / allocation failures that have no reference counterpart.
#ifndef SVDKIT_B200_SVDKIT_HPP
#define SVDKIT_B200_SVDKIT_HPP

#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <iosfwd>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace svdkit {

// ---------------------------------------------------------------- errors
// (reference errors.hpp:11-55)
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class DimensionError : public Error {
public:
    using Error::Error;
};
class ParamError : public Error {
public:
    using Error::Error;
};
class NumericalError : public Error {
public:
    NumericalError(const std::string& what, double residual) : Error(what), residual_(residual) {}
    double residual() const { return residual_; }

private:
    double residual_ = 0.0;
};
class FormatError : public Error {
public:
    FormatError(const std::string& what, std::size_t offset) : Error(what), offset_(offset) {}
    std::size_t offset() const { return offset_; }

private:
    std::size_t offset_ = 0;
};
class IoError : public Error {
public:
    using Error::Error;
};
/// Engine-side failure (CUDA, NCCL, device allocation); no reference analogue.
class EngineError : public Error {
public:
    using Error::Error;
};

// ---------------------------------------------------------------- DenseMatrix
// Column-major fp64 owner (reference dense_matrix.hpp:19-60); entry (i, j) is
// data()[i + j * rows()].
class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(std::size_t rows, std::size_t cols);
    DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data);
    static DenseMatrix identity(std::size_t n);
    static DenseMatrix from_rows(std::initializer_list<std::initializer_list<double>> rows);

    std::size_t rows() const { return nr_; }
    std::size_t cols() const { return nc_; }
    std::size_t size() const { return v_.size(); }
    bool empty() const { return v_.empty(); }
    double operator()(std::size_t i, std::size_t j) const { return v_[i + j * nr_]; }
    double& operator()(std::size_t i, std::size_t j) { return v_[i + j * nr_]; }
    double* col(std::size_t j) { return v_.data() + j * nr_; }
    const double* col(std::size_t j) const { return v_.data() + j * nr_; }
    const std::vector<double>& data() const { return v_; }
    bool operator==(const DenseMatrix& other) const = default;

private:
    std::size_t nr_ = 0;
    std::size_t nc_ = 0;
    std::vector<double> v_;
};

std::string shape_string(const DenseMatrix& a);

// ---------------------------------------------------------------- kernels
// (reference kernels.hpp:12-72)
struct RngSeed {
    std::uint64_t value = 0;
};
DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b);
DenseMatrix matmul_transposed_left(const DenseMatrix& a, const DenseMatrix& b);
DenseMatrix transpose(const DenseMatrix& a);
DenseMatrix gram(const DenseMatrix& a);
double frobenius_norm_sq(const DenseMatrix& a);
double frobenius_norm(const DenseMatrix& a);

struct QrResult {
    DenseMatrix q;
    DenseMatrix r;
    std::size_t rank;
};
QrResult qr_thin(const DenseMatrix& h);

struct EigResult {
    std::vector<double> eigenvalues;
    DenseMatrix eigenvectors;
};
EigResult eig_sym(const DenseMatrix& s);
EigResult eig_sym(const DenseMatrix& s, int max_sweeps);

DenseMatrix gaussian_matrix(std::size_t rows, std::size_t cols, RngSeed seed);

// ---------------------------------------------------------------- methods
// (reference svd_methods.hpp:13-65)
enum class SvdMethod { Truncated, Randomized, Krylov, Lanczos };
const char* method_name(SvdMethod method);
std::optional<SvdMethod> method_from_name(std::string_view name);

struct MethodParams {
    std::size_t sketch_width = 1;      ///< l (Lanczos: number of steps, 0 = n)
    std::size_t power_iterations = 1;  ///< q / Krylov depth
    RngSeed seed{0};
    static MethodParams defaults_for(std::size_t n, RngSeed seed = RngSeed{0});
};

struct SvdResult {
    DenseMatrix u;
    std::vector<double> sigma;
    DenseMatrix v;
    std::size_t rank = 0;
    SvdMethod method = SvdMethod::Truncated;
};

SvdResult truncated_svd(const DenseMatrix& a);
SvdResult randomized_pca(const DenseMatrix& a, const MethodParams& p);
SvdResult krylov_svd(const DenseMatrix& a, const MethodParams& p);
SvdResult lanczos_svd(const DenseMatrix& a, const MethodParams& p);
SvdResult truncate_rank(const SvdResult& s, std::size_t k);
SvdResult compute_svd(const DenseMatrix& a, SvdMethod method, const MethodParams& p);
SvdResult compute_svd_any(const DenseMatrix& a, SvdMethod method, const MethodParams& p);

// ---------------------------------------------------------------- PCA
// (reference pca.hpp:14-58)
enum class Orientation { ColumnsAreExamples, RowsAreExamples };

struct CenterResult {
    DenseMatrix centered;
    std::vector<double> mean;
};
CenterResult center(const DenseMatrix& a, Orientation orientation);
double total_variance(const DenseMatrix& centered);
std::optional<std::size_t> select_components(const std::vector<double>& eigenvalues, double total,
                                             double threshold);

struct PcaModel {
    DenseMatrix basis;
    std::vector<double> eigenvalues;
    double total_variance = 0.0;
    Orientation orientation = Orientation::RowsAreExamples;
    std::vector<double> mean;
};
PcaModel fit_pca(const DenseMatrix& data, Orientation orientation, SvdMethod method,
                 const MethodParams& params, bool center_data = true);
DenseMatrix transform(const PcaModel& model, const DenseMatrix& a);
double residual_delta(const DenseMatrix& a, const SvdResult& s);

// ---------------------------------------------------------------- cost model
// (reference cost_model.hpp:9-49; closed forms evaluated by svdk_cost_model)
struct CostEstimate {
    double flops = 0.0;
    double space_entries = 0.0;
    double space_bytes = 0.0;  ///< always exactly 8 * space_entries
};
CostEstimate krylov_cost(std::size_t m, std::size_t n, std::size_t l, std::size_t i);
CostEstimate krylov_cost_practical(std::size_t m, std::size_t n);
CostEstimate krylov_cost_per_step(std::size_t m, std::size_t n, std::size_t l, std::size_t i);
CostEstimate randomized_cost(std::size_t m, std::size_t n, std::size_t l, std::size_t i);
CostEstimate randomized_cost_practical(std::size_t m, std::size_t n);
CostEstimate truncated_cost(std::size_t m, std::size_t n);

// ---------------------------------------------------------------- CSV
// (reference csv_io.hpp:12-27)
std::string format_double(double value);
DenseMatrix read_matrix_csv(std::istream& in);
DenseMatrix read_matrix_csv_file(const std::string& path);
void write_matrix_csv(const DenseMatrix& a, std::ostream& out);
void write_matrix_csv_file(const DenseMatrix& a, const std::string& path);
void write_vector_csv_file(const std::vector<double>& values, const std::string& path);

// ---------------------------------------------------------------- IDX
// (reference idx_io.hpp:12-36); images_to_matrix expands on the GPU
struct IdxImageSet {
    std::size_t count = 0;
    std::size_t height = 0;
    std::size_t width = 0;
    std::vector<std::uint8_t> pixels;  ///< count*height*width bytes, row-major per image
};
IdxImageSet parse_idx_images(std::span<const std::uint8_t> bytes);
IdxImageSet load_idx_file(const std::string& path);
DenseMatrix images_to_matrix(const IdxImageSet& set);
DenseMatrix image_as_matrix(const IdxImageSet& set, std::size_t index);

// ---------------------------------------------------------------- bench grid
// (reference bench.hpp:13-88); factorisations and delta run on the GPU
struct BenchConfig {
    std::vector<std::size_t> row_sizes;
    std::vector<std::size_t> col_sizes;
    std::vector<SvdMethod> methods;
    std::size_t repeats = 10;
    RngSeed seed{42};
    double l_fraction = 0.5;
    std::size_t iterations = 1;
    double memory_cap_bytes = 2.0 * 1024 * 1024 * 1024;
};
struct BenchRecord {
    SvdMethod method = SvdMethod::Truncated;
    std::size_t m = 0;
    std::size_t n = 0;
    std::size_t repeats = 0;
    double mean_seconds = 0.0;
    double std_seconds = 0.0;
    double delta = 0.0;
    double model_flops = 0.0;
    double model_space_bytes = 0.0;
};
struct SkippedCell {
    SvdMethod method = SvdMethod::Truncated;
    std::size_t m = 0;
    std::size_t n = 0;
    std::string reason;
};
struct GridResult {
    std::vector<BenchRecord> records;
    std::vector<SkippedCell> skipped;
};
std::vector<std::pair<std::size_t, std::size_t>> expand_grid(const BenchConfig& cfg);
std::size_t sketch_width_for(const BenchConfig& cfg, std::size_t n);
GridResult run_grid(const BenchConfig& cfg);
std::string to_csv(const std::vector<BenchRecord>& records);
void write_csv_file(const std::vector<BenchRecord>& records, const std::string& path);
struct OrderingCell {
    std::size_t m = 0;
    std::size_t n = 0;
    std::vector<SvdMethod> by_seconds;
    std::vector<SvdMethod> by_flops;
    bool agree = false;
};
struct OrderingReport {
    std::vector<OrderingCell> cells;
    double agreement = 0.0;
};
OrderingReport summarize_ordering(const std::vector<BenchRecord>& records);
std::string format_report(const OrderingReport& report);

}  // namespace svdkit

#endif
