// eventscope/detect.hpp — anomaly-detect drop-in on the
// B200 backend: Def. 1 / Alg. 2 best-component density
// thresholding, the mixture-density ablation, and quantile
// calibration of delta.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "eventscope/gmm.hpp"

namespace eventscope {

enum class DetectMode { Component, Mixture };

struct DetectorConfig {
    std::optional<double> delta;
    std::optional<double> quantile_q = 0.01;
    int K = 2;
    double train_window = 0.5;
    DetectMode mode = DetectMode::Component;
};

struct DetectionReport {
    std::vector<std::uint8_t> flags;
    std::vector<std::int64_t> anomaly_indices;
    std::vector<int> best_component;
    std::vector<double> log_density;
    GmmModel model;
    double delta = 0.0;
    double log_delta = 0.0;           // the single shared log(delta) every comparison used
};

/// flag_i iff log p(x_i | theta_k*) < log delta, k* = argmax_k p(x_i | theta_k)
/// (ties -> lowest k).  delta > 0.
DetectionReport detect(const GmmModel& model, const FeatureMatrix& X, double delta,
                       DetectMode mode = DetectMode::Component);
/// Same, with delta given by its logarithm (no exp/log round trip).
DetectionReport detect_log(const GmmModel& model, const FeatureMatrix& X, double log_delta,
                           DetectMode mode = DetectMode::Component);
/// q-quantile (h = (n-1) q, linear interpolation) of the training densities.
double calibrate_threshold(const GmmModel& model, const FeatureMatrix& X_train, double q,
                           DetectMode mode = DetectMode::Component);
/// Calibration returning (delta, log delta).
std::pair<double, double> calibrate_threshold_log(const GmmModel& model, const FeatureMatrix& X_train, double q,
                                                  DetectMode mode = DetectMode::Component);

struct PipelineResult {               // run_pipeline outputs (EvalSummary: eval-bench, not built)
    DetectionReport report;           // over ALL events; report.model is in standardized space
    FeatureMatrix::Standardization standardization;  // per column (mean, stddev) of the train split
    std::int64_t n_train = 0;
};

/// run_pipeline over a time-ordered feature matrix: the first
/// floor(train_window * N) rows are the training split; columns are z-scored with its
/// mean and population stddev (zero-variance columns centred only) when `standardize`;
/// a cfg.K-component GMM is fitted there; delta = cfg.quantile_q-quantile of the training
/// densities (or cfg.delta); every event is scored per detect.  Errors: InsufficientTraining
/// (training split < 10 K), plus the component ops' errors.
PipelineResult run_pipeline(const FeatureMatrix& X, const DetectorConfig& cfg, const FitOptions& opts = {},
                            bool standardize = true);

}  // namespace eventscope
