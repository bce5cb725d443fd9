// Drop-in usage of the eventscope C++ API (include/eventscope/*.hpp) on the
// B200 backend: fit -> calibrate -> detect -> JSON round trip, plus the
// error conventions of errors.hpp.  Built and run by tests/test_gpu_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "eventscope/detect.hpp"
#include "eventscope/eval.hpp"
#include "eventscope/events.hpp"
#include "eventscope/gmm.hpp"

int main() {
    using namespace eventscope;
    // 0.5 N(-5,1) + 0.5 N(5,1), K=2 -> means within 0.2, weights within 0.05
    std::mt19937_64 rng(7);
    std::normal_distribution<double> n01(0.0, 1.0);
    FeatureMatrix X;
    X.rows = 2000;
    X.dim = 1;
    for (int i = 0; i < 2000; ++i) X.data.push_back((i < 1000 ? -5.0 : 5.0) + n01(rng));
    FitOptions opts;
    opts.seed = 3;
    GmmModel m = fit_em(X, 2, opts);
    const int lo = m.means[0] < m.means[1] ? 0 : 1;
    bool ok = std::fabs(m.means[lo] + 5) < 0.2 && std::fabs(m.means[1 - lo] - 5) < 0.2 &&
              std::fabs(m.weights[0] - 0.5) < 0.05;
    // SPEC.md:267 closed form
    GmmModel unit{1, 1, {1.0}, {0.0}, {1.0}, {}};
    const double v = component_log_density(unit, std::vector<double>{0.0}, 0);
    ok = ok && std::fabs(v + 0.9189385332046727) < 1e-9;
    // x=0 normal, x=4 flagged, x=3 (density == delta) normal
    FeatureMatrix P{3, 1, {0.0, 4.0, 3.0}, {}, {}, {}};
    const double ld3 = component_log_density(unit, std::vector<double>{3.0}, 0);
    DetectionReport r = detect_log(unit, P, ld3);
    ok = ok && r.flags[0] == 0 && r.flags[1] == 1 && r.flags[2] == 0 && r.anomaly_indices.size() == 1;
    // calibrate + detect on the fitted model
    const double delta = calibrate_threshold(m, X, 0.01);
    DetectionReport r2 = detect(m, X, delta);
    ok = ok && r2.anomaly_indices.size() <= 20;
    // run_pipeline: standardize on the train window, fit, calibrate on it, detect all rows
    FeatureMatrix Xi;  // interleave the two clusters so the train window holds both
    Xi.rows = X.rows;
    Xi.dim = 1;
    for (int i = 0; i < 1000; ++i) Xi.data.insert(Xi.data.end(), {X.data[i], X.data[1000 + i]});
    PipelineResult pr = run_pipeline(Xi, DetectorConfig{std::nullopt, 0.01, 2, 0.5, DetectMode::Component}, FitOptions{});
    ok = ok && pr.report.flags.size() == (size_t)X.rows && pr.standardization.size() == (size_t)X.dim &&
         pr.n_train == X.rows / 2 && pr.report.delta > 0.0 && pr.report.model.K == 2;
    // eval-bench: k-means baseline on the interleaved clusters, confusion / metrics
    KMeansBaseline kb = kmeans_baseline(Xi, 2, 0.01, 5);
    const int lo2 = kb.centroids[0] < kb.centroids[1] ? 0 : 1;
    ok = ok && std::fabs(kb.centroids[lo2] + 5) < 0.2 && std::fabs(kb.centroids[1 - lo2] - 5) < 0.2 &&
         kb.flags.size() == (size_t)Xi.rows && kb.iterations >= 1;
    const ConfusionMatrix cm = confusion({1, 1, 0, 0}, {1, 0, 1, 0});
    const EvalSummary es = metrics(cm);
    ok = ok && cm.tp == 1 && cm.fp == 1 && cm.tn == 1 && cm.fn == 1 && std::fabs(es.f1 - 0.5) < 1e-15;
    const std::vector<SweepCell> grid =
        sensitivity_sweep(Xi, std::vector<std::uint8_t>(Xi.rows, 0), {2}, {0.01}, {0, 1});
    ok = ok && grid.size() == 1 && grid[0].status == "ok" && grid[0].seed_count == 2 &&
         sweep_csv(grid).rfind("layer,K,q,", 0) == 0;
    // extract_features on the device: Nccl duration 999, 9 bytes -> [3, 1]
    EventColumns ec;
    ec.layer = {3, 0};
    ec.ts_start = {10, 20};
    ec.duration_ns = {999, 99};
    ec.message_bytes = {9.0, NAN};
    const FeatureMatrix F = extract_features(ec, Layer::Nccl);
    ok = ok && F.rows == 1 && F.dim == 2 && F.data[0] == 3.0 && F.data[1] == 1.0 && F.event_index[0] == 0;
    // JSON round trip (within 1e-15 per entry)
    GmmModel back = model_from_json(to_json(m));
    for (size_t i = 0; i < m.covariances.size(); ++i) ok = ok && back.covariances[i] == m.covariances[i];
    ok = ok && back.fit_report.per_iteration_log_likelihoods == m.fit_report.per_iteration_log_likelihoods;
    // error conventions (errors.hpp)
    try {
        FeatureMatrix tiny{2, 1, {0.0, 0.0}, {}, {}, {}};
        fit_em(tiny, 3);
        ok = false;
    } catch (const Error& e) {
        ok = ok && e.kind() == ErrorKind::Data && e.name() == "TooFewPoints";
    }
    std::printf("%s means=(%.4f, %.4f) weights=(%.4f, %.4f) iters=%d flagged=%zu\n", ok ? "OK" : "FAIL", m.means[0],
                m.means[1], m.weights[0], m.weights[1], m.fit_report.iterations, r2.anomaly_indices.size());
    return ok ? 0 : 1;
}
