// Benchmark records, emitters and the `bench` CLI over the device path
// (include/bcad/bench.hpp; the reference's proj/src/bench.cpp behaviour:
// run_cell_once 112-128, the equivalence gate 131-148, run_hmlstm_for
// 163-214, run_arity_for 216-307, emit/parse 347-415, bench_main 417-520).
// Built into libbcad_host.so; the `bcad_bench` executable is bench_main.cpp.
#include "bcad/bench.hpp"

#include <algorithm>
#include <array>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <limits>
#include <sstream>
#include <tuple>
#include <utility>

#include "bcad/bcad.hpp"

namespace bcad::bench {

std::string device_impl_name(const std::string& impl) {
    return impl.rfind(kDevicePrefix, 0) == 0 ? impl : std::string(kDevicePrefix) + impl;
}

namespace {

std::uint64_t now_ns() {
    return static_cast<std::uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
            .count());
}

struct Stats {
    std::uint64_t min_ns = 0, median_ns = 0, mean_ns = 0;
};

// min, median (mean of the middle pair, rounded), mean (rounded).
Stats summarize(std::vector<std::uint64_t> t) {
    std::sort(t.begin(), t.end());
    Stats s;
    s.min_ns = t.front();
    const std::size_t n = t.size();
    s.median_ns = n % 2 ? t[n / 2]
                        : static_cast<std::uint64_t>(
                              std::llround((static_cast<double>(t[n / 2 - 1]) + static_cast<double>(t[n / 2])) / 2.0));
    double sum = 0;
    for (std::uint64_t v : t) sum += static_cast<double>(v);
    s.mean_ns = static_cast<std::uint64_t>(std::llround(sum / static_cast<double>(n)));
    return s;
}

// "cuda-mixed-cache" and "mixed-cache" both select mixed-cache.
std::string base_impl(const std::string& name) {
    const std::string p = kDevicePrefix;
    return name.rfind(p, 0) == 0 ? name.substr(p.size()) : name;
}

bool known_impl(const std::string& name) {
    const std::string b = base_impl(name);
    return b == kImplMixedCache || b == kImplMixedRecompute || b == kImplReverseUnfused || b == kImplForwardOnly;
}

void validate_common(const BenchConfig& cfg) {
    if (cfg.repetitions < 1) throw ConfigError("repetitions must be >= 1");
    if (cfg.warmup < 0) throw ConfigError("warmup must be >= 0");
    if (cfg.sizes.empty()) throw ConfigError("at least one size is required");
    for (std::int64_t n : cfg.sizes)
        if (n < 1) throw ConfigError("matrix side must be >= 1, got " + std::to_string(n));
    if (cfg.threads < 0) throw ConfigError("threads must be >= 0");
}

void sync() { check(bcad_cu_stream_synchronize(current_stream())); }

template <class Real>
struct CellRun {
    CellGradients<Real> grads;
    std::uint64_t tape_nodes = 0;
    std::uint64_t peak_cached_bytes = 0;
};

// One gradient computation of the n x n cell (reference run_cell_once).
template <class Real>
CellRun<Real> run_cell_once(const std::string& impl, const CellInputs<Real>& in, const Tensor<Real>& seed) {
    CellRun<Real> r;
    if (impl == kImplForwardOnly) {
        // forward-mode diagonals, then the seed-weighted products w * D_j
        const BroadcastKernel<Real> kernel = cell_update_kernel<Real>();
        ForwardBroadcastResult<Real> fwd = broadcast_diag_jacobian<Real>(kernel, true, in.c_prev, in.f, in.i, in.g,
                                                                         in.z1, in.z2);
        const BroadcastKernel<Real> mul(2, 1, "mul");
        auto vjp = [&](int j) { return std::move(broadcast_apply<Real>(mul, seed, fwd.jacobian.entry(0, j))[0]); };
        r.grads = CellGradients<Real>{vjp(0), vjp(1), vjp(2), vjp(3)};
        const auto vol = static_cast<std::uint64_t>(fwd.jacobian.out_shape.volume());
        r.peak_cached_bytes = (1 + static_cast<std::uint64_t>(fwd.jacobian.inputs)) * vol * sizeof(Real);
        return r;
    }
    Tape<Real> tape;
    CellGraph<Real> graph;
    if (impl == kImplMixedCache) graph = cell_update_fused(tape, in, MixedPolicy::CacheForward);
    else if (impl == kImplMixedRecompute) graph = cell_update_fused(tape, in, MixedPolicy::RecomputeReverse);
    else if (impl == kImplReverseUnfused) graph = cell_update_unfused(tape, in);
    else throw ConfigError("unknown implementation: " + impl);
    const Gradients<Real> g = tape.backward(graph.out, seed);
    r.grads = CellGradients<Real>{g.at(graph.c_prev), g.at(graph.f), g.at(graph.i), g.at(graph.g)};
    r.tape_nodes = tape.size();
    r.peak_cached_bytes = static_cast<std::uint64_t>(tape.peak_cached_bytes());
    return r;
}

template <class Real>
bool close_tensors(const Tensor<Real>& a, const Tensor<Real>& b, double rtol, double atol) {
    if (!(a.shape() == b.shape())) return false;
    const std::vector<Real> x = a.to_host(), y = b.to_host();
    for (std::size_t e = 0; e < x.size(); ++e) {
        const double u = static_cast<double>(x[e]), v = static_cast<double>(y[e]);
        if (std::fabs(u - v) > atol + rtol * std::max(std::fabs(u), std::fabs(v))) return false;
    }
    return true;
}

template <class Real>
void check_equivalence(const std::vector<std::string>& impls, const std::vector<CellRun<Real>>& runs, std::int64_t n) {
    const double tol = std::is_same_v<Real, double> ? 1e-5 : 1e-4;
    for (std::size_t k = 1; k < runs.size(); ++k) {
        const auto pair = [&](const Tensor<Real>& a, const Tensor<Real>& b, const char* which) {
            if (!close_tensors(a, b, tol, tol))
                throw EquivalenceFailure("gradient mismatch between " + device_impl_name(impls[0]) + " and " +
                                         device_impl_name(impls[k]) + " on d/d" + which + " at n=" + std::to_string(n));
        };
        pair(runs[0].grads.c_prev, runs[k].grads.c_prev, "c_prev");
        pair(runs[0].grads.f, runs[k].grads.f, "f");
        pair(runs[0].grads.i, runs[k].grads.i, "i");
        pair(runs[0].grads.g, runs[k].grads.g, "g");
    }
}

template <class Real>
void dump_gradients(std::ostream& os, const std::string& impl, std::int64_t n, const CellGradients<Real>& g) {
    const std::pair<const char*, const Tensor<Real>*> items[] = {
        {"dc_prev", &g.c_prev}, {"df", &g.f}, {"di", &g.i}, {"dg", &g.g}};
    for (const auto& [name, t] : items) {
        os << "# impl=" << impl << " n=" << n << " grad=" << name << "\n";
        t->write_csv(os);
    }
}

template <class Real>
std::vector<BenchRecord> run_hmlstm_for(const BenchConfig& cfg) {
    std::vector<std::string> impls;
    for (const std::string& s : cfg.impls) impls.push_back(base_impl(s));
    std::ofstream dump;
    if (!cfg.dump_grads_path.empty()) {
        dump.open(cfg.dump_grads_path);
        if (!dump) throw IoError("cannot open " + cfg.dump_grads_path + " for writing");
    }
    std::vector<BenchRecord> records;
    for (std::int64_t n : cfg.sizes) {
        Rng rng(mix_seed(cfg.rng_seed, static_cast<std::uint64_t>(n)));
        const CellInputs<Real> inputs = random_cell_inputs<Real>(n, rng);
        const Tensor<Real> seed(Shape{n, n}, Real(1));
        // gate: nothing is timed unless every implementation agrees
        std::vector<CellRun<Real>> gate;
        std::vector<std::uint64_t> evals;  // measured: the device census around each gate run
        for (const std::string& impl : impls) {
            const std::uint64_t before = counter_totals().transcendental_evals;
            gate.push_back(run_cell_once(impl, inputs, seed));
            evals.push_back(counter_totals().transcendental_evals - before);
        }
        check_equivalence(impls, gate, n);
        if (dump.is_open()) dump_gradients(dump, impls.front(), n, gate.front().grads);
        for (std::size_t k = 0; k < impls.size(); ++k) {
            for (int w = 0; w < cfg.warmup; ++w) (void)run_cell_once(impls[k], inputs, seed);
            sync();
            std::vector<std::uint64_t> samples;
            for (int rep = 0; rep < cfg.repetitions; ++rep) {
                const std::uint64_t t0 = now_ns();
                (void)run_cell_once(impls[k], inputs, seed);
                sync();
                samples.push_back(now_ns() - t0);
            }
            const Stats st = summarize(std::move(samples));
            BenchRecord rec;
            rec.workload = "hmlstm";
            rec.impl = impls[k];
            rec.n = n;
            rec.arity = 0;
            rec.reps = cfg.repetitions;
            rec.min_ns = st.min_ns;
            rec.median_ns = st.median_ns;
            rec.mean_ns = st.mean_ns;
            rec.tape_nodes = gate[k].tape_nodes;
            rec.peak_cached_bytes = gate[k].peak_cached_bytes;
            rec.transcendental_evals = evals[k];
            rec.rng_seed = cfg.rng_seed;
            records.push_back(std::move(rec));
        }
    }
    return records;
}

constexpr int kArities[] = {1, 2, 3, 4, 5, 8, 16, 18, 32};  // registered tanh_product_<A> bodies

template <class Real>
std::vector<BenchRecord> run_arity_for(const BenchConfig& cfg) {
    std::vector<BenchRecord> records;
    const std::int64_t n = cfg.sizes.front();
    // finite-difference rule of the reference's FdConfig (oracle.hpp:18-28)
    const double step_scale = std::cbrt(static_cast<double>(std::numeric_limits<Real>::epsilon()));
    const double rel_tol = std::is_same_v<Real, double> ? 1e-5 : 1e-2;
    auto step_at = [&](double x) { return step_scale * std::max(1.0, std::fabs(x)); };
    for (int arity : cfg.arities) {
        Rng rng(mix_seed(cfg.rng_seed, static_cast<std::uint64_t>(arity) * 131071u + static_cast<std::uint64_t>(n)));
        const BroadcastKernel<Real> kernel(arity, 1, "tanh_product_" + std::to_string(arity));
        std::vector<Tensor<Real>> inputs;
        for (int j = 0; j < arity; ++j) inputs.push_back(random_pm1<Real>(Shape{n, n}, rng));
        std::vector<const Tensor<Real>*> ptrs;
        for (const Tensor<Real>& t : inputs) ptrs.push_back(&t);
        const std::uint64_t evals_before = counter_totals().transcendental_evals;
        ForwardBroadcastResult<Real> fwd = broadcast_diag_jacobian<Real>(kernel, ptrs, true);
        const std::uint64_t evals = counter_totals().transcendental_evals - evals_before;  // measured
        if (fwd.jacobian.inputs != arity) throw Error("partial-vector width does not match the kernel arity");

        // spot checks against central differences of the device body at one
        // point, away from the reflect_below_half boundary (x = 0.5)
        std::vector<std::vector<Real>> host_in;
        for (const Tensor<Real>& t : inputs) host_in.push_back(t.to_host());
        auto body_at = [&](const std::vector<Real>& point) -> Real {
            std::vector<Tensor<Real>> cell;
            for (Real v : point) cell.push_back(Tensor<Real>::from(Shape{1}, std::vector<Real>{v}));
            std::vector<const Tensor<Real>*> cp;
            for (const Tensor<Real>& t : cell) cp.push_back(&t);
            return broadcast_apply<Real>(kernel, std::span<const Tensor<Real>* const>(cp))[0][0];
        };
        const std::int64_t vol = fwd.jacobian.out_shape.volume();
        for (int check_no = 0; check_no < 8; ++check_no) {
            std::size_t j = 0;
            std::int64_t e = 0;
            bool found = false;
            for (int attempt = 0; attempt < 64 && !found; ++attempt) {
                j = static_cast<std::size_t>(rng.below(static_cast<std::uint64_t>(arity)));
                e = static_cast<std::int64_t>(rng.below(static_cast<std::uint64_t>(vol)));
                const double x = static_cast<double>(host_in[j][static_cast<std::size_t>(e)]);
                found = std::fabs(x - 0.5) > 4.0 * step_at(x);
            }
            if (!found) continue;
            std::vector<Real> point;
            for (int a = 0; a < arity; ++a) point.push_back(host_in[static_cast<std::size_t>(a)][static_cast<std::size_t>(e)]);
            const Real x = point[j];
            const Real h = static_cast<Real>(step_at(static_cast<double>(x)));
            point[j] = x + h;
            const Real up = body_at(point);
            point[j] = x - h;
            const Real down = body_at(point);
            if (!std::isfinite(static_cast<double>(up)) || !std::isfinite(static_cast<double>(down)))
                throw NonFiniteValue("finite-difference probe produced a non-finite value");
            const Real fd = (up - down) / (Real(2) * h);
            const Real ad = fwd.jacobian.entry(0, static_cast<int>(j))[e];
            const double scale = std::max({1.0, std::fabs(static_cast<double>(fd)), std::fabs(static_cast<double>(ad))});
            if (std::fabs(static_cast<double>(fd - ad)) > rel_tol * scale)
                throw EquivalenceFailure("arity " + std::to_string(arity) +
                                         ": derivative disagrees with finite differences at cell " + std::to_string(e));
        }
        for (int w = 0; w < cfg.warmup; ++w) (void)broadcast_diag_jacobian<Real>(kernel, ptrs, true);
        sync();
        std::vector<std::uint64_t> samples;
        for (int rep = 0; rep < cfg.repetitions; ++rep) {
            const std::uint64_t t0 = now_ns();
            (void)broadcast_diag_jacobian<Real>(kernel, ptrs, true);
            sync();
            samples.push_back(now_ns() - t0);
        }
        const Stats st = summarize(std::move(samples));
        BenchRecord rec;
        rec.workload = "arity";
        rec.impl = kImplForwardOnly;
        rec.n = n;
        rec.arity = arity;
        rec.reps = cfg.repetitions;
        rec.min_ns = st.min_ns;
        rec.median_ns = st.median_ns;
        rec.mean_ns = st.mean_ns;
        rec.tape_nodes = 0;
        rec.peak_cached_bytes = (1 + static_cast<std::uint64_t>(arity)) * static_cast<std::uint64_t>(vol) * sizeof(Real);
        rec.transcendental_evals = evals;
        rec.rng_seed = cfg.rng_seed;
        records.push_back(std::move(rec));
    }
    return records;
}

std::vector<BenchRecord> sorted(std::span<const BenchRecord> records) {
    std::vector<BenchRecord> out(records.begin(), records.end());
    std::sort(out.begin(), out.end(), [](const BenchRecord& a, const BenchRecord& b) {
        return std::tie(a.workload, a.impl, a.n, a.arity) < std::tie(b.workload, b.impl, b.n, b.arity);
    });
    return out;
}

std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (unsigned char c : s) {
        if (c == '"' || c == '\\') {
            o += '\\';
            o += static_cast<char>(c);
        } else if (c < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", c);
            o += buf;
        } else {
            o += static_cast<char>(c);
        }
    }
    return o + "\"";
}

// ---- a small JSON reader: arrays of flat objects with string / integer
// members are all the record format needs; numbers keep their literal text so
// 64-bit integers round-trip exactly.
struct JValue {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    std::string text;  // String contents or Number literal
    std::vector<JValue> items;
    std::vector<std::pair<std::string, JValue>> members;
};

class JReader {
public:
    explicit JReader(std::string s) : s_(std::move(s)) {}
    JValue document() {
        JValue v = value();
        ws();
        if (p_ != s_.size()) fail("trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const std::string& what) const {
        throw IoError("invalid benchmark JSON: " + what + " at offset " + std::to_string(p_));
    }
    void ws() {
        while (p_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[p_]))) ++p_;
    }
    bool eat(char c) {
        ws();
        if (p_ < s_.size() && s_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail(std::string("expected '") + c + "'");
    }
    std::string str() {
        expect('"');
        std::string o;
        while (true) {
            if (p_ >= s_.size()) fail("unterminated string");
            const char c = s_[p_++];
            if (c == '"') break;
            if (c != '\\') {
                o += c;
                continue;
            }
            if (p_ >= s_.size()) fail("bad escape");
            const char e = s_[p_++];
            switch (e) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    if (p_ + 4 > s_.size()) fail("bad \\u escape");
                    const unsigned cp = static_cast<unsigned>(std::stoul(s_.substr(p_, 4), nullptr, 16));
                    p_ += 4;
                    if (cp < 0x80) o += static_cast<char>(cp);
                    else fail("non-ASCII \\u escape");
                    break;
                }
                default: fail("bad escape");
            }
        }
        return o;
    }
    JValue value() {
        ws();
        if (p_ >= s_.size()) fail("unexpected end");
        JValue v;
        const char c = s_[p_];
        if (c == '{') {
            ++p_;
            v.kind = JValue::Object;
            if (eat('}')) return v;
            do {
                ws();
                std::string key = str();
                expect(':');
                v.members.emplace_back(std::move(key), value());
            } while (eat(','));
            expect('}');
        } else if (c == '[') {
            ++p_;
            v.kind = JValue::Array;
            if (eat(']')) return v;
            do v.items.push_back(value());
            while (eat(','));
            expect(']');
        } else if (c == '"') {
            v.kind = JValue::String;
            v.text = str();
        } else if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
            const std::size_t b = p_;
            ++p_;
            while (p_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[p_])) || s_[p_] == '.' ||
                                      s_[p_] == 'e' || s_[p_] == 'E' || s_[p_] == '+' || s_[p_] == '-'))
                ++p_;
            v.kind = JValue::Number;
            v.text = s_.substr(b, p_ - b);
        } else if (s_.compare(p_, 4, "true") == 0 || s_.compare(p_, 5, "false") == 0) {
            v.kind = JValue::Bool;
            p_ += s_[p_] == 't' ? 4 : 5;
        } else if (s_.compare(p_, 4, "null") == 0) {
            p_ += 4;
        } else {
            fail("unexpected character");
        }
        return v;
    }

    std::string s_;
    std::size_t p_ = 0;
};

const JValue& member(const JValue& obj, const char* key) {
    for (const auto& [k, v] : obj.members)
        if (k == key) return v;
    throw IoError(std::string("malformed benchmark record: missing \"") + key + "\"");
}
std::string as_string(const JValue& v, const char* key) {
    if (v.kind != JValue::String) throw IoError(std::string("malformed benchmark record: \"") + key + "\" is not a string");
    return v.text;
}
template <class I>
I as_int(const JValue& v, const char* key) {
    const bool neg = !v.text.empty() && v.text[0] == '-';
    if (v.kind != JValue::Number || v.text.find_first_of(".eE") != std::string::npos || (neg && std::is_unsigned_v<I>))
        throw IoError(std::string("malformed benchmark record: \"") + key + "\" is not an integer");
    try {
        if constexpr (std::is_unsigned_v<I>) return static_cast<I>(std::stoull(v.text));
        else return static_cast<I>(std::stoll(v.text));
    } catch (const std::exception&) {
        throw IoError(std::string("malformed benchmark record: \"") + key + "\" out of range");
    }
}

// ---- CLI (the reference uses CLI11; same subcommands, options and codes)
const char* kUsage =
    "Gradient benchmarks for broadcast automatic differentiation (device)\n"
    "usage: bench <hmlstm|arity> [options]\n"
    "  hmlstm: --n N[,N...] (default 64,128,256)  --dump-grads PATH\n"
    "  arity:  --n N (default 256)  --arities A[,A...]  --max-arity A\n"
    "  common: --impl LIST  --reps R  --warmup W  --seed S  --precision f32|f64\n"
    "          --format csv|json  --out PATH  --threads T (ignored on the device)\n";

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::vector<std::string> split_commas(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    std::istringstream is(s);
    while (std::getline(is, cur, ','))
        if (!cur.empty()) out.push_back(cur);
    return out;
}

template <class I>
I parse_int(const std::string& opt, const std::string& v) {
    try {
        std::size_t used = 0;
        const long long x = std::stoll(v, &used);
        if (used != v.size()) throw std::invalid_argument(v);
        if (x < static_cast<long long>(std::numeric_limits<I>::min()) ||
            static_cast<unsigned long long>(x) > static_cast<unsigned long long>(std::numeric_limits<I>::max()))
            throw std::out_of_range(v);
        return static_cast<I>(x);
    } catch (const std::exception&) {
        throw ParseError(opt + ": '" + v + "' is not a valid integer");
    }
}

}  // namespace

std::vector<BenchRecord> run_hmlstm_bench(const BenchConfig& cfg) {
    validate_common(cfg);
    if (cfg.impls.empty()) throw ConfigError("at least one implementation is required");
    for (const std::string& impl : cfg.impls)
        if (!known_impl(impl)) throw ConfigError("unknown implementation: " + impl);
    return cfg.precision == Precision::F64 ? run_hmlstm_for<double>(cfg) : run_hmlstm_for<float>(cfg);
}

std::vector<BenchRecord> run_arity_bench(const BenchConfig& cfg) {
    validate_common(cfg);
    if (cfg.sizes.size() != 1) throw ConfigError("the arity workload takes exactly one matrix side");
    if (cfg.arities.empty()) throw ConfigError("at least one arity is required");
    for (int a : cfg.arities) {
        if (a < 1 || a > kMaxPartials)
            throw ConfigError("arity " + std::to_string(a) + " outside [1, " + std::to_string(kMaxPartials) + "]");
        if (std::find(std::begin(kArities), std::end(kArities), a) == std::end(kArities))
            throw ConfigError("arity " + std::to_string(a) +
                              " has no registered device body (registered: 1, 2, 3, 4, 5, 8, 16, 18, 32)");
    }
    return cfg.precision == Precision::F64 ? run_arity_for<double>(cfg) : run_arity_for<float>(cfg);
}

void emit(std::span<const BenchRecord> records, OutputFormat format, std::ostream& os) {
    const std::vector<BenchRecord> rows = sorted(records);
    if (format == OutputFormat::Csv) {
        os << kCsvHeader << "\n";
        for (const BenchRecord& r : rows)
            os << r.workload << ',' << r.impl << ',' << r.n << ',' << r.arity << ',' << r.reps << ',' << r.min_ns << ','
               << r.median_ns << ',' << r.mean_ns << ',' << r.tape_nodes << ',' << r.peak_cached_bytes << ','
               << r.transcendental_evals << ',' << r.rng_seed << "\n";
        return;
    }
    // two-space indented array of objects, members in header order
    if (rows.empty()) {
        os << "[]\n";
        return;
    }
    os << "[\n";
    for (std::size_t k = 0; k < rows.size(); ++k) {
        const BenchRecord& r = rows[k];
        os << "  {\n"
           << "    \"workload\": " << json_string(r.workload) << ",\n"
           << "    \"impl\": " << json_string(r.impl) << ",\n"
           << "    \"n\": " << r.n << ",\n"
           << "    \"arity\": " << r.arity << ",\n"
           << "    \"reps\": " << r.reps << ",\n"
           << "    \"min_ns\": " << r.min_ns << ",\n"
           << "    \"median_ns\": " << r.median_ns << ",\n"
           << "    \"mean_ns\": " << r.mean_ns << ",\n"
           << "    \"tape_nodes\": " << r.tape_nodes << ",\n"
           << "    \"peak_cached_bytes\": " << r.peak_cached_bytes << ",\n"
           << "    \"transcendental_evals\": " << r.transcendental_evals << ",\n"
           << "    \"rng_seed\": " << r.rng_seed << "\n"
           << "  }" << (k + 1 < rows.size() ? ",\n" : "\n");
    }
    os << "]\n";
}

void emit_to_path(std::span<const BenchRecord> records, OutputFormat format, const std::string& path) {
    std::ofstream os(path);
    if (!os) throw IoError("cannot open " + path + " for writing");
    emit(records, format, os);
    if (!os) throw IoError("failed writing " + path);
}

std::vector<BenchRecord> parse_json_records(std::istream& is) {
    std::ostringstream buf;
    buf << is.rdbuf();
    const JValue doc = JReader(buf.str()).document();
    if (doc.kind != JValue::Array) throw IoError("benchmark JSON must be an array of records");
    std::vector<BenchRecord> out;
    for (const JValue& item : doc.items) {
        if (item.kind != JValue::Object) throw IoError("malformed benchmark record: not an object");
        BenchRecord r;
        r.workload = as_string(member(item, "workload"), "workload");
        r.impl = as_string(member(item, "impl"), "impl");
        r.n = as_int<std::int64_t>(member(item, "n"), "n");
        r.arity = as_int<int>(member(item, "arity"), "arity");
        r.reps = as_int<int>(member(item, "reps"), "reps");
        r.min_ns = as_int<std::uint64_t>(member(item, "min_ns"), "min_ns");
        r.median_ns = as_int<std::uint64_t>(member(item, "median_ns"), "median_ns");
        r.mean_ns = as_int<std::uint64_t>(member(item, "mean_ns"), "mean_ns");
        r.tape_nodes = as_int<std::uint64_t>(member(item, "tape_nodes"), "tape_nodes");
        r.peak_cached_bytes = as_int<std::uint64_t>(member(item, "peak_cached_bytes"), "peak_cached_bytes");
        r.transcendental_evals = as_int<std::uint64_t>(member(item, "transcendental_evals"), "transcendental_evals");
        r.rng_seed = as_int<std::uint64_t>(member(item, "rng_seed"), "rng_seed");
        out.push_back(std::move(r));
    }
    return out;
}

int bench_main(int argc, const char* const* argv) {
    BenchConfig cfg;
    std::string precision = "f64", format = "csv", sub;
    int max_arity = 0;
    bool sizes_given = false, arities_given = false;
    try {
        std::vector<std::string> args(argv + 1, argv + argc);
        for (const std::string& a : args)
            if (a == "--help" || a == "-h") {
                std::cout << kUsage;
                return 0;
            }
        if (args.empty()) throw ParseError("a subcommand is required: hmlstm or arity");
        sub = args[0];
        if (sub != "hmlstm" && sub != "arity") throw ParseError("unknown subcommand '" + sub + "'");
        for (std::size_t k = 1; k < args.size(); ++k) {
            std::string opt = args[k], val;
            const std::size_t eq = opt.find('=');
            if (opt.rfind("--", 0) != 0) throw ParseError("unexpected argument '" + opt + "'");
            if (eq != std::string::npos) {
                val = opt.substr(eq + 1);
                opt = opt.substr(0, eq);
            } else {
                if (k + 1 >= args.size()) throw ParseError(opt + " needs a value");
                val = args[++k];
            }
            if (opt == "--impl") {
                cfg.impls = split_commas(val);
            } else if (opt == "--reps") {
                cfg.repetitions = parse_int<int>(opt, val);
            } else if (opt == "--warmup") {
                cfg.warmup = parse_int<int>(opt, val);
            } else if (opt == "--seed") {
                cfg.rng_seed = static_cast<std::uint64_t>(parse_int<long long>(opt, val));
            } else if (opt == "--precision") {
                if (val != "f32" && val != "f64") throw ParseError("--precision must be f32 or f64");
                precision = val;
            } else if (opt == "--format") {
                if (val != "csv" && val != "json") throw ParseError("--format must be csv or json");
                format = val;
            } else if (opt == "--out") {
                cfg.out_path = val;
            } else if (opt == "--threads") {
                cfg.threads = parse_int<int>(opt, val);
            } else if (opt == "--n") {
                if (!sizes_given) cfg.sizes.clear();
                for (const std::string& s : split_commas(val)) cfg.sizes.push_back(parse_int<std::int64_t>(opt, s));
                sizes_given = true;
            } else if (opt == "--dump-grads" && sub == "hmlstm") {
                cfg.dump_grads_path = val;
            } else if (opt == "--arities" && sub == "arity") {
                if (!arities_given) cfg.arities.clear();
                for (const std::string& s : split_commas(val)) cfg.arities.push_back(parse_int<int>(opt, s));
                arities_given = true;
            } else if (opt == "--max-arity" && sub == "arity") {
                max_arity = parse_int<int>(opt, val);
            } else {
                throw ParseError("unknown option " + opt + " for " + sub);
            }
        }
    } catch (const ParseError& e) {
        std::cerr << e.what() << "\n" << kUsage;
        return 1;
    }

    try {
        cfg.precision = precision == "f64" ? Precision::F64 : Precision::F32;
        cfg.format = format == "csv" ? OutputFormat::Csv : OutputFormat::Json;
        if (const char* env = std::getenv("BCAD_THREADS")) {
            try {
                cfg.threads = std::stoi(env);
            } catch (const std::exception&) {
                throw ConfigError("BCAD_THREADS must be an integer, got '" + std::string(env) + "'");
            }
        }
        std::vector<BenchRecord> records;
        if (sub == "hmlstm") {
            cfg.workload = Workload::HmLstm;
            if (!sizes_given) cfg.sizes = {64, 128, 256};
            records = run_hmlstm_bench(cfg);
        } else {
            cfg.workload = Workload::Arity;
            if (!sizes_given) cfg.sizes = {256};
            if (max_arity > 0 && !arities_given) {
                cfg.arities.clear();
                for (int a = 1; a < max_arity; a *= 2) cfg.arities.push_back(a);
                cfg.arities.push_back(max_arity);
            }
            records = run_arity_bench(cfg);
        }
        std::cerr << "bench: " << records.size() << " record(s), device=cuda, precision=" << precision
                  << ", seed=" << cfg.rng_seed << "\n";
        if (cfg.out_path.empty()) emit(records, cfg.format, std::cout);
        else emit_to_path(records, cfg.format, cfg.out_path);
        return 0;
    } catch (const EquivalenceFailure& e) {
        std::cerr << "equivalence failure: " << e.what() << "\n";
        return 2;
    } catch (const ConfigError& e) {
        std::cerr << "config error: " << e.what() << "\n";
        return 1;
    } catch (const IoError& e) {
        std::cerr << "io error: " << e.what() << "\n";
        return 1;
    } catch (const Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}

}  // namespace bcad::bench
