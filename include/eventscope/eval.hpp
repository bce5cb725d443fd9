// eventscope/eval.hpp — eval-bench drop-in on the B200 backend:
// confusion counts and metrics, the KMeans baseline (k-means++ + Lloyd on the device),
// and the K x q sensitivity sweep over run_pipeline.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "eventscope/detect.hpp"

namespace eventscope {

struct ConfusionMatrix {              // SPEC.md:420-422 (anomaly = positive class)
    std::int64_t tp = 0, fp = 0, tn = 0, fn = 0;
};

struct EvalSummary {
    double accuracy = 0.0, precision = 0.0, recall = 0.0, f1 = 0.0;
    ConfusionMatrix cm;
    std::string method = "gmm";
    int K = 0;
    double q = 0.0;
};

/// SPEC.md:431-437; throws Data/LengthMismatch.  Counted on the device.
ConfusionMatrix confusion(const std::vector<std::uint8_t>& labels, const std::vector<std::uint8_t>& flags);
/// SPEC.md:439-446; zero-division conventions 0; throws Data/EmptyMatrix.
EvalSummary metrics(const ConfusionMatrix& cm);

struct KMeansBaseline {
    std::vector<double> centroids;    // K x d, row-major
    double threshold = 0.0;
    std::vector<std::uint8_t> flags;
    std::vector<double> scores;       // distance to the nearest centroid
    std::int64_t n_flagged = 0;
    int iterations = 0;
};
/// k-means++ seeding and Lloyd's algorithm on the first train_window fraction of X;
/// flag iff the nearest-centroid distance exceeds the (1-q)-quantile of the train
/// distances.  Throws Data/TooFewPoints when the train split has fewer than K rows.
KMeansBaseline kmeans_baseline(const FeatureMatrix& X, int K, double q, std::uint64_t seed,
                               double train_window = 0.5, int max_iter = 100);

struct SweepCell {                    // one CSV row
    std::string layer;
    int K = 0;
    double q = 0.0;
    int seed_count = 0;
    double accuracy = 0.0, precision = 0.0, recall = 0.0, f1 = 0.0;
    std::string status = "ok";
};
/// full K x q grid of run_pipeline cells averaged over seeds; a failing
/// cell records its error name in `status` instead of aborting the sweep.
std::vector<SweepCell> sensitivity_sweep(const FeatureMatrix& X, const std::vector<std::uint8_t>& labels,
                                         const std::vector<int>& K_range, const std::vector<double>& q_range,
                                         const std::vector<std::uint64_t>& seeds, const std::string& layer = "all",
                                         double train_window = 0.5);
/// The grid as CSV: layer,K,q,seed_count,accuracy,precision,recall,f1,status.
std::string sweep_csv(const std::vector<SweepCell>& grid);

}  // namespace eventscope
