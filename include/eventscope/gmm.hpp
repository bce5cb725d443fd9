// eventscope/gmm.hpp — gmm-core drop-in on the B200 backend.
//
// The reference ships no gmm header (proj/include holds only errors.hpp); the
// signatures below are the SPEC op signatures SPEC.md:261,271,281,291,301 with
// the types of SPEC.md:247-258.  Every op runs on the GPU through the C-ABI in
// eventscope_b200.h — there is no CPU fallback.  Failures throw
// eventscope::Error with the SPEC's stable names.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "eventscope/errors.hpp"

namespace eventscope {

/// N x d event feature matrix; data is row-major (row i = x_i).
/// A strided view of an external buffer (e.g. a column-major Eigen matrix)
/// can be described with MatrixView instead, avoiding a copy.
struct FeatureMatrix {
    std::int64_t rows = 0;
    int dim = 0;
    std::vector<double> data;                 // rows * dim, row-major
    std::vector<std::string> feature_names;   // dim entries (optional)
    using Standardization = std::vector<std::pair<double, double>>;
    Standardization standardization;          // per column (mean, stddev), optional
    std::vector<std::int64_t> event_index;    // back-references (optional)
};

struct MatrixView {
    const double* data = nullptr;
    std::int64_t rows = 0;
    int dim = 0;
    std::int64_t row_stride = 0;  // element (i,j) at data[i*row_stride + j*col_stride]
    std::int64_t col_stride = 1;
    static MatrixView of(const FeatureMatrix& X) { return {X.data.data(), X.rows, X.dim, X.dim, 1}; }
};

enum class Init { Random, KMeansPP };
/// Diagonal covariances are an extension (the reference has none).
enum class CovarianceType { Full, Diagonal };

struct FitOptions {
    Init init = Init::KMeansPP;
    double tol = 1e-6;
    int max_iter = 200;
    std::optional<double> reg;        // default 1e-6 * tr(S)/d; 0 disables
    std::uint64_t seed = 0;
    CovarianceType covariance_type = CovarianceType::Full;
};

struct FitReport {
    int iterations = 0;
    double final_log_likelihood = 0.0;
    std::vector<double> per_iteration_log_likelihoods;
    bool converged = false;
    std::uint64_t seed = 0;
};

struct GmmModel {
    int K = 0;
    int d = 0;
    std::vector<double> weights;      // K
    std::vector<double> means;        // K * d
    std::vector<double> covariances;  // K * d * d (row-major per component)
    FitReport fit_report;
};

struct Responsibilities {
    std::int64_t rows = 0;
    int K = 0;
    std::vector<double> gamma;        // rows * K
};

double component_log_density(const GmmModel& model, std::span<const double> x, int k);
double mixture_density(const GmmModel& model, std::span<const double> x);
Responsibilities responsibilities(const GmmModel& model, const FeatureMatrix& X);
GmmModel fit_em(const FeatureMatrix& X, int K, const FitOptions& opts = {});
std::pair<int, std::vector<double>> select_k_bic(const FeatureMatrix& X, std::span<const int> k_range,
                                                 const FitOptions& opts = {});

// Batched forms of the same math (score_samples / predict of the north star).
std::vector<double> score_samples(const GmmModel& model, const FeatureMatrix& X);  // log p(x_i)
std::vector<int> predict(const GmmModel& model, const FeatureMatrix& X);           // argmax_k gamma_ik

// Model serialization: {k, weights, means, covariances, fit_report}.
std::string to_json(const GmmModel& model);
GmmModel model_from_json(const std::string& json);

namespace b200 {
/// Device selection for the free functions above (default: $ES_DEVICE or 0).
void set_device(int device);
}  // namespace b200

}  // namespace eventscope
