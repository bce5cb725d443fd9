// eventscope_api.cpp — the C++ drop-in (include/eventscope/{gmm,detect}.hpp)
// implemented over the C-ABI.  Each free function uploads its matrix to a
// per-thread default context, runs the B200 kernels, and converts status
// codes into eventscope::Error with the C-ABI's stable names.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>

#include "eventscope/detect.hpp"
#include "eventscope/eval.hpp"
#include "eventscope/events.hpp"
#include "eventscope/gmm.hpp"
#include "eventscope_b200.h"

namespace eventscope {
namespace {

int g_device = -1;

[[noreturn]] void rethrow(int status) {
    const std::string name = es_last_error_name();
    const std::string msg = es_last_error_message();
    switch (status) {
        case ES_ERR_DATA: throw Error::data(name, msg);
        case ES_ERR_NUMERIC: throw Error::numeric(name, msg);
        default: throw Error(ErrorKind::Io, name, msg);
    }
}

void check(int status) {
    if (status != ES_OK) rethrow(status);
}

struct Ctx {
    es_ctx* c = nullptr;
    int device = -1;
    ~Ctx() {
        if (c) es_ctx_destroy(c);
    }
};

es_ctx* ctx() {
    thread_local Ctx t;
    int dev = g_device;
    if (dev < 0) {
        const char* e = std::getenv("ES_DEVICE");
        dev = e ? std::atoi(e) : 0;
    }
    if (!t.c || t.device != dev) {
        if (t.c) es_ctx_destroy(t.c);
        t.c = nullptr;
        check(es_ctx_create(dev, &t.c));
        t.device = dev;
    }
    return t.c;
}

struct Dataset {
    es_dataset* ds = nullptr;
    ~Dataset() {
        if (ds) es_dataset_destroy(ds);
    }
};

void upload(const FeatureMatrix& X, Dataset& out) {
    if (X.rows < 0 || X.dim < 1 || (int64_t)X.data.size() != X.rows * X.dim)
        throw Error::data("DimensionMismatch", "FeatureMatrix data size does not match rows * dim");
    check(es_dataset_create(ctx(), X.data.data(), X.rows, X.dim, X.dim, 1, &out.ds));
}

es_gmm_params view(const GmmModel& m) {
    if (m.K < 1 || (int)m.weights.size() != m.K || (int)m.means.size() != m.K * m.d ||
        (int)m.covariances.size() != m.K * m.d * m.d)
        throw Error::data("InvalidModel", "GmmModel arrays do not match K and d");
    return es_gmm_params{m.K, m.d, const_cast<double*>(m.weights.data()), const_cast<double*>(m.means.data()),
                         const_cast<double*>(m.covariances.data())};
}

void need_dim(const GmmModel& m, int d) {
    if (m.d != d) throw Error::data("DimensionMismatch", "model dimension does not match the input");
}

es_fit_opts c_opts(const FitOptions& o) {
    es_fit_opts r{};
    r.init = o.init == Init::Random ? ES_INIT_RANDOM : ES_INIT_KMEANSPP;
    r.tol = o.tol;
    r.max_iter = o.max_iter;
    r.reg = o.reg ? *o.reg : -1.0;
    r.seed = o.seed;
    r.covariance_type = o.covariance_type == CovarianceType::Diagonal ? ES_COV_DIAG : ES_COV_FULL;
    return r;
}

}  // namespace

namespace b200 {
void set_device(int device) { g_device = device; }
}  // namespace b200

double component_log_density(const GmmModel& model, std::span<const double> x, int k) {
    need_dim(model, (int)x.size());
    es_gmm_params p = view(model);
    double out = 0.0;
    check(es_gmm_component_log_density(ctx(), &p, x.data(), k, &out));
    return out;
}

double mixture_density(const GmmModel& model, std::span<const double> x) {
    need_dim(model, (int)x.size());
    es_gmm_params p = view(model);
    double ll = 0.0;
    check(es_gmm_mixture_log_density(ctx(), &p, x.data(), &ll));
    return std::exp(ll);
}

Responsibilities responsibilities(const GmmModel& model, const FeatureMatrix& X) {
    need_dim(model, X.dim);
    Dataset ds;
    upload(X, ds);
    es_gmm_params p = view(model);
    Responsibilities r;
    r.rows = X.rows;
    r.K = model.K;
    r.gamma.resize((size_t)X.rows * model.K);
    check(es_gmm_responsibilities(ctx(), ds.ds, &p, r.gamma.data()));
    return r;
}

static GmmModel fit_on(es_dataset* ds, int K, int d, const FitOptions& opts) {
    es_fit_opts o = c_opts(opts);
    GmmModel m;
    m.K = K;
    m.d = d;
    m.weights.resize(std::max(K, 0));
    m.means.resize((size_t)std::max(K, 0) * d);
    m.covariances.resize((size_t)std::max(K, 0) * d * d);
    es_gmm_params out{K, d, m.weights.data(), m.means.data(), m.covariances.data()};
    es_fit_report rep{};
    std::vector<double> per((size_t)std::max(o.max_iter, 0) + 1);
    check(es_gmm_fit(ctx(), ds, K, &o, nullptr, &out, &rep, per.data()));
    per.resize(rep.n_per_iter);
    m.fit_report = FitReport{rep.iterations, rep.final_log_likelihood, std::move(per), rep.converged != 0, rep.seed};
    return m;
}

GmmModel fit_em(const FeatureMatrix& X, int K, const FitOptions& opts) {
    Dataset ds;
    upload(X, ds);
    return fit_on(ds.ds, K, X.dim, opts);
}

std::pair<int, std::vector<double>> select_k_bic(const FeatureMatrix& X, std::span<const int> k_range,
                                                 const FitOptions& opts) {
    Dataset ds;
    upload(X, ds);
    es_fit_opts o = c_opts(opts);
    std::vector<int32_t> kr(k_range.begin(), k_range.end());
    std::vector<double> bic(kr.size());
    int32_t best = 0;
    check(es_gmm_select_k_bic(ctx(), ds.ds, kr.data(), (int32_t)kr.size(), &o, &best, bic.data()));
    return {best, bic};
}

std::vector<double> score_samples(const GmmModel& model, const FeatureMatrix& X) {
    need_dim(model, X.dim);
    Dataset ds;
    upload(X, ds);
    es_gmm_params p = view(model);
    std::vector<double> ll(X.rows);
    check(es_gmm_score(ctx(), ds.ds, &p, ll.data(), nullptr, nullptr, nullptr, nullptr));
    return ll;
}

std::vector<int> predict(const GmmModel& model, const FeatureMatrix& X) {
    need_dim(model, X.dim);
    Dataset ds;
    upload(X, ds);
    es_gmm_params p = view(model);
    std::vector<int32_t> pr(X.rows);
    check(es_gmm_score(ctx(), ds.ds, &p, nullptr, pr.data(), nullptr, nullptr, nullptr));
    return std::vector<int>(pr.begin(), pr.end());
}

DetectionReport detect_log(const GmmModel& model, const FeatureMatrix& X, double log_delta, DetectMode mode) {
    need_dim(model, X.dim);
    Dataset ds;
    upload(X, ds);
    es_gmm_params p = view(model);
    DetectionReport r;
    r.flags.resize(X.rows);
    r.best_component.resize(X.rows);
    r.log_density.resize(X.rows);
    std::vector<int32_t> bk(X.rows);
    std::vector<int64_t> idx(X.rows);
    int64_t nloc = 0, ng = 0;
    check(es_gmm_detect(ctx(), ds.ds, &p, log_delta, mode == DetectMode::Mixture ? ES_DETECT_MIXTURE : ES_DETECT_COMPONENT,
                        r.flags.data(), bk.data(), r.log_density.data(), idx.data(), &nloc, &ng));
    idx.resize(nloc);
    r.anomaly_indices = std::move(idx);
    r.best_component.assign(bk.begin(), bk.end());
    r.model = model;
    r.log_delta = log_delta;
    r.delta = std::exp(log_delta);
    return r;
}

DetectionReport detect(const GmmModel& model, const FeatureMatrix& X, double delta, DetectMode mode) {
    if (!(delta > 0.0)) throw Error::data("RangeViolation", "delta must be > 0");
    DetectionReport r = detect_log(model, X, std::log(delta), mode);  // comparison in log space
    r.delta = delta;
    return r;
}

std::pair<double, double> calibrate_threshold_log(const GmmModel& model, const FeatureMatrix& X_train, double q,
                                                  DetectMode mode) {
    if (X_train.rows < 1) throw Error::data("EmptyTraining", "training split is empty");
    need_dim(model, X_train.dim);
    Dataset ds;
    upload(X_train, ds);
    es_gmm_params p = view(model);
    double delta = 0.0, log_delta = 0.0;
    check(es_gmm_calibrate(ctx(), ds.ds, &p, X_train.rows, q,
                           mode == DetectMode::Mixture ? ES_DETECT_MIXTURE : ES_DETECT_COMPONENT, &delta, &log_delta));
    return {delta, log_delta};
}

double calibrate_threshold(const GmmModel& model, const FeatureMatrix& X_train, double q, DetectMode mode) {
    return calibrate_threshold_log(model, X_train, q, mode).first;
}

namespace {
PipelineResult run_pipeline_on(Dataset& ds, const FeatureMatrix& X, const DetectorConfig& cfg, const FitOptions& opts,
                               bool standardize) {
    const int d = X.dim, K = cfg.K;
    es_pipeline_cfg c{};
    c.K = K;
    c.train_window = cfg.train_window;
    c.quantile_q = cfg.delta ? 0.0 : cfg.quantile_q.value_or(0.0);
    c.delta = cfg.delta.value_or(0.0);
    c.standardize = standardize ? 1 : 0;
    c.mode = cfg.mode == DetectMode::Mixture ? ES_DETECT_MIXTURE : ES_DETECT_COMPONENT;
    c.fit = c_opts(opts);
    PipelineResult r;
    GmmModel& m = r.report.model;
    m.K = K;
    m.d = d;
    m.weights.resize(std::max(K, 0));
    m.means.resize((size_t)std::max(K, 0) * d);
    m.covariances.resize((size_t)std::max(K, 0) * d * d);
    es_gmm_params out{K, d, m.weights.data(), m.means.data(), m.covariances.data()};
    es_fit_report rep{};
    std::vector<double> mean(d), scale(d);
    std::vector<int32_t> bk(X.rows);
    std::vector<int64_t> idx(std::max<int64_t>(X.rows, 1));
    r.report.flags.resize(X.rows);
    r.report.log_density.resize(X.rows);
    int64_t nloc = 0, ng = 0;
    check(es_run_pipeline(ctx(), ds.ds, &c, &out, &rep, mean.data(), scale.data(), &r.report.delta,
                          &r.report.log_delta, r.report.flags.data(), bk.data(), r.report.log_density.data(),
                          idx.data(), &nloc, &ng));
    m.fit_report = FitReport{rep.iterations, rep.final_log_likelihood, {}, rep.converged != 0, rep.seed};
    idx.resize(nloc);
    r.report.anomaly_indices = std::move(idx);
    r.report.best_component.assign(bk.begin(), bk.end());
    for (int j = 0; j < d; ++j) r.standardization.emplace_back(mean[j], scale[j]);
    r.n_train = (std::int64_t)std::floor(cfg.train_window * (double)X.rows);
    return r;
}
}  // namespace

PipelineResult run_pipeline(const FeatureMatrix& X, const DetectorConfig& cfg, const FitOptions& opts,
                            bool standardize) {
    Dataset ds;
    upload(X, ds);
    return run_pipeline_on(ds, X, cfg, opts, standardize);
}

// ------------------------------------------------------------------ event features
FeatureMatrix extract_features(const EventColumns& e, Layer layer) {
    const int64_t n = (int64_t)e.layer.size();
    if ((int64_t)e.ts_start.size() != n || (int64_t)e.duration_ns.size() != n)
        throw Error::data("LengthMismatch", "event columns differ in length");
    auto opt = [&](const std::vector<double>& v) -> const double* {
        if (v.empty()) return nullptr;
        if ((int64_t)v.size() != n) throw Error::data("LengthMismatch", "event columns differ in length");
        return v.data();
    };
    es_event_columns c{e.layer.data(), e.ts_start.data(), e.duration_ns.data(), opt(e.message_bytes),
                       opt(e.util_pct), opt(e.mem_used_mb), opt(e.temp_c)};
    Dataset ds;
    std::vector<int64_t> idx(std::max<int64_t>(n, 1));
    int64_t bad = -1;
    check(es_events_extract(ctx(), &c, n, (int32_t)layer, &ds.ds, idx.data(), &bad));
    int64_t nl = 0, ng = 0, off = 0;
    int32_t D = 0;
    check(es_dataset_info(ds.ds, &nl, &ng, &off, &D));
    FeatureMatrix X;
    X.rows = nl;
    X.dim = D;
    X.data.resize((size_t)nl * D);
    check(es_dataset_read_rows(ds.ds, 0, nl, X.data.data()));
    idx.resize(nl);
    X.event_index = std::move(idx);
    if (layer == Layer::GpuSample)
        X.feature_names = {"util_pct", "mem_used_mb", "temp_c"};
    else if (layer == Layer::Nccl)
        X.feature_names = {"log10_duration_ns", "log10_message_bytes"};
    else
        X.feature_names = {"log10_duration_ns"};
    return X;
}

// ------------------------------------------------------------------ eval-bench
ConfusionMatrix confusion(const std::vector<std::uint8_t>& labels, const std::vector<std::uint8_t>& flags) {
    if (labels.size() != flags.size()) throw Error::data("LengthMismatch", "labels and flags differ in length");
    int64_t out[4] = {0, 0, 0, 0};
    check(es_confusion(ctx(), labels.data(), flags.data(), (int64_t)labels.size(), out));
    return ConfusionMatrix{out[0], out[1], out[2], out[3]};
}

EvalSummary metrics(const ConfusionMatrix& cm) {
    const double n = (double)(cm.tp + cm.fp + cm.tn + cm.fn);
    if (!(n > 0)) throw Error::data("EmptyMatrix", "confusion matrix has no events");
    EvalSummary e;
    e.cm = cm;
    e.accuracy = (double)(cm.tp + cm.tn) / n;
    e.precision = cm.tp + cm.fp ? (double)cm.tp / (double)(cm.tp + cm.fp) : 0.0;
    e.recall = cm.tp + cm.fn ? (double)cm.tp / (double)(cm.tp + cm.fn) : 0.0;
    e.f1 = e.precision + e.recall > 0.0 ? 2.0 * e.precision * e.recall / (e.precision + e.recall) : 0.0;
    return e;
}

KMeansBaseline kmeans_baseline(const FeatureMatrix& X, int K, double q, std::uint64_t seed, double train_window,
                               int max_iter) {
    Dataset ds;
    upload(X, ds);
    KMeansBaseline r;
    r.centroids.resize((size_t)std::max(K, 0) * X.dim);
    r.flags.resize(X.rows);
    r.scores.resize(X.rows);
    int32_t it = 0;
    check(es_kmeans_baseline(ctx(), ds.ds, K, q, train_window, seed, max_iter, r.centroids.data(), &r.threshold,
                             r.flags.data(), r.scores.data(), &r.n_flagged, &it));
    r.iterations = it;
    return r;
}

std::vector<SweepCell> sensitivity_sweep(const FeatureMatrix& X, const std::vector<std::uint8_t>& labels,
                                         const std::vector<int>& K_range, const std::vector<double>& q_range,
                                         const std::vector<std::uint64_t>& seeds, const std::string& layer,
                                         double train_window) {
    if (K_range.empty() || q_range.empty() || seeds.empty())
        throw Error::data("EmptyRange", "K_range, q_range and seeds must be nonempty");
    if ((int64_t)labels.size() != X.rows) throw Error::data("LengthMismatch", "labels do not match the events");
    Dataset ds;
    upload(X, ds);  // one upload shared by every cell
    std::vector<SweepCell> grid;
    for (int K : K_range)
        for (double q : q_range) {
            SweepCell c;
            c.layer = layer;
            c.K = K;
            c.q = q;
            double acc[4] = {0, 0, 0, 0};
            for (std::uint64_t sd : seeds) {
                try {
                    DetectorConfig cfg;
                    cfg.K = K;
                    cfg.quantile_q = q;
                    cfg.train_window = train_window;
                    FitOptions fo;
                    fo.seed = sd;
                    const PipelineResult pr = run_pipeline_on(ds, X, cfg, fo, true);
                    const EvalSummary e = metrics(confusion(labels, pr.report.flags));
                    acc[0] += e.accuracy;
                    acc[1] += e.precision;
                    acc[2] += e.recall;
                    acc[3] += e.f1;
                    ++c.seed_count;
                } catch (const Error& e) {
                    c.status = e.name();
                }
            }
            if (c.seed_count) {
                c.accuracy = acc[0] / c.seed_count;
                c.precision = acc[1] / c.seed_count;
                c.recall = acc[2] / c.seed_count;
                c.f1 = acc[3] / c.seed_count;
            } else {
                c.accuracy = c.precision = c.recall = c.f1 = NAN;
            }
            grid.push_back(c);
        }
    return grid;
}

std::string sweep_csv(const std::vector<SweepCell>& grid) {
    std::ostringstream o;
    o.precision(17);
    o << "layer,K,q,seed_count,accuracy,precision,recall,f1,status\n";
    for (const SweepCell& c : grid)
        o << c.layer << ',' << c.K << ',' << c.q << ',' << c.seed_count << ',' << c.accuracy << ',' << c.precision
          << ',' << c.recall << ',' << c.f1 << ',' << c.status << '\n';
    return o.str();
}

// ------------------------------------------------------------------ JSON
namespace {

void put_array(std::ostringstream& o, const std::vector<double>& v) {
    o << '[';
    char buf[40];
    for (size_t i = 0; i < v.size(); ++i) {
        std::snprintf(buf, sizeof buf, "%.17g", v[i]);
        o << (i ? "," : "") << buf;
    }
    o << ']';
}

struct Parser {
    const std::string& s;
    size_t i = 0;
    void ws() {
        while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
    }
    [[noreturn]] void bad(const char* what) { throw Error::data("ParseError", std::string("model JSON: ") + what); }
    void expect(char c) {
        ws();
        if (i >= s.size() || s[i] != c) bad("unexpected character");
        ++i;
    }
    bool peek(char c) {
        ws();
        return i < s.size() && s[i] == c;
    }
    std::string str() {
        expect('"');
        size_t j = s.find('"', i);
        if (j == std::string::npos) bad("unterminated string");
        std::string r = s.substr(i, j - i);
        i = j + 1;
        return r;
    }
    double num() {
        ws();
        char* end = nullptr;
        double v = std::strtod(s.c_str() + i, &end);
        if (end == s.c_str() + i) {
            if (s.compare(i, 4, "true") == 0) { i += 4; return 1.0; }
            if (s.compare(i, 5, "false") == 0) { i += 5; return 0.0; }
            bad("number expected");
        }
        i = end - s.c_str();
        return v;
    }
    void flat(std::vector<double>& out) {  // nested arrays flattened in order
        if (peek('[')) {
            expect('[');
            if (peek(']')) { expect(']'); return; }
            while (true) {
                flat(out);
                if (peek(',')) { expect(','); continue; }
                expect(']');
                return;
            }
        }
        out.push_back(num());
    }
};

}  // namespace

std::string to_json(const GmmModel& m) {
    std::ostringstream o;
    char buf[40];
    o << "{\"k\":" << m.K << ",\"d\":" << m.d << ",\"weights\":";
    put_array(o, m.weights);
    o << ",\"means\":";
    put_array(o, m.means);
    o << ",\"covariances\":";
    put_array(o, m.covariances);
    const FitReport& r = m.fit_report;
    std::snprintf(buf, sizeof buf, "%.17g", r.final_log_likelihood);
    o << ",\"fit_report\":{\"iterations\":" << r.iterations << ",\"final_log_likelihood\":" << buf
      << ",\"per_iteration_log_likelihoods\":";
    put_array(o, r.per_iteration_log_likelihoods);
    o << ",\"converged\":" << (r.converged ? "true" : "false") << ",\"seed\":" << r.seed << "}}";
    return o.str();
}

GmmModel model_from_json(const std::string& json) {
    Parser p{json};
    GmmModel m;
    p.expect('{');
    auto object = [&](auto&& self, GmmModel& mm, bool report) -> void {
        if (p.peek('}')) { p.expect('}'); return; }
        while (true) {
            const std::string key = p.str();
            p.expect(':');
            if (!report && key == "fit_report") {
                p.expect('{');
                self(self, mm, true);
            } else {
                std::vector<double> v;
                p.flat(v);
                if (report) {
                    FitReport& r = mm.fit_report;
                    if (key == "iterations") r.iterations = (int)v.at(0);
                    else if (key == "final_log_likelihood") r.final_log_likelihood = v.at(0);
                    else if (key == "per_iteration_log_likelihoods") r.per_iteration_log_likelihoods = v;
                    else if (key == "converged") r.converged = v.at(0) != 0.0;
                    else if (key == "seed") r.seed = (std::uint64_t)v.at(0);
                } else {
                    if (key == "k") mm.K = (int)v.at(0);
                    else if (key == "d") mm.d = (int)v.at(0);
                    else if (key == "weights") mm.weights = v;
                    else if (key == "means") mm.means = v;
                    else if (key == "covariances") mm.covariances = v;
                }
            }
            if (p.peek(',')) { p.expect(','); continue; }
            p.expect('}');
            return;
        }
    };
    object(object, m, false);
    if (m.d == 0 && m.K > 0) m.d = (int)(m.means.size() / m.K);
    view(m);  // validates array sizes
    return m;
}

}  // namespace eventscope
