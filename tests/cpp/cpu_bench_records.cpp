// Bench record formats and CLI error paths of the drop-in bench API
// (include/bcad/bench.hpp) — the host-only claims of the reference's
// proj/tests/test_bench.cpp (csv ordering 154-185, json 187-216, cli
// 218-234). Needs no GPU: nothing here launches device work.
#include <sstream>
#include <string>
#include <vector>

#include "bcad/bench.hpp"
#include "bcad/errors.hpp"
#include "mini_test.hpp"

using namespace bcad;
using namespace bcad::bench;

namespace {

BenchRecord sample(const char* impl, std::uint64_t nodes) {
    BenchRecord r;
    r.workload = "hmlstm";
    r.impl = impl;
    r.n = 64;
    r.arity = 0;
    r.reps = 10;
    r.min_ns = 1111;
    r.median_ns = 2222;
    r.mean_ns = 3333;
    r.tape_nodes = nodes;
    r.peak_cached_bytes = 999;
    r.transcendental_evals = 12288;
    r.rng_seed = 42;
    return r;
}

}  // namespace

TEST_CASE("csv emission is bit-stable and exactly ordered") {
    std::vector<BenchRecord> records;
    std::ostringstream empty;
    emit(records, OutputFormat::Csv, empty);
    CHECK(empty.str() == std::string(kCsvHeader) + "\n");
    records = {sample("cuda-reverse-unfused", 14), sample("cuda-mixed-cache", 7)};
    std::ostringstream os;
    emit(records, OutputFormat::Csv, os);
    CHECK(os.str() == std::string(kCsvHeader) + "\n" +
                          "hmlstm,cuda-mixed-cache,64,0,10,1111,2222,3333,7,999,12288,42\n" +
                          "hmlstm,cuda-reverse-unfused,64,0,10,1111,2222,3333,14,999,12288,42\n");
}

TEST_CASE("json round-trips records exactly, including 64-bit fields") {
    std::vector<BenchRecord> records = {sample("cuda-mixed-recompute", 7), sample("mixed-cache", 7)};
    records[0].rng_seed = 18446744073709551615ull;
    records[1].workload = "arity";
    records[1].arity = 18;
    records[1].impl = "weird \"quoted\" \\ name";
    std::stringstream buf;
    emit(records, OutputFormat::Json, buf);
    const auto parsed = parse_json_records(buf);
    REQUIRE(parsed.size() == 2);
    std::ostringstream a, b;
    emit(records, OutputFormat::Json, a);
    emit(parsed, OutputFormat::Json, b);
    CHECK(a.str() == b.str());
    bool found = false;
    for (const BenchRecord& r : parsed) found = found || r.rng_seed == 18446744073709551615ull;
    CHECK(found);
    std::ostringstream none;
    emit(std::vector<BenchRecord>{}, OutputFormat::Json, none);
    std::istringstream back(none.str());
    CHECK(parse_json_records(back).empty());
}

TEST_CASE("emit_to_path surfaces io errors") {
    const std::vector<BenchRecord> records;
    CHECK_THROWS_AS(emit_to_path(records, OutputFormat::Csv, "/nonexistent-dir/out.csv"), IoError);
}

TEST_CASE("malformed json is rejected") {
    std::istringstream garbage("{not json");
    CHECK_THROWS_AS((void)parse_json_records(garbage), IoError);
    std::istringstream wrong_shape("{\"a\": 1}");
    CHECK_THROWS_AS((void)parse_json_records(wrong_shape), IoError);
    std::istringstream missing_fields("[{\"workload\": \"hmlstm\"}]");
    CHECK_THROWS_AS((void)parse_json_records(missing_fields), IoError);
    std::istringstream wrong_type(
        "[{\"workload\": \"hmlstm\", \"impl\": \"x\", \"n\": \"64\", \"arity\": 0, \"reps\": 1, \"min_ns\": 1, "
        "\"median_ns\": 1, \"mean_ns\": 1, \"tape_nodes\": 1, \"peak_cached_bytes\": 1, \"transcendental_evals\": 1, "
        "\"rng_seed\": 1}]");
    CHECK_THROWS_AS((void)parse_json_records(wrong_type), IoError);
}

TEST_CASE("device implementation names") {
    CHECK(device_impl_name(kImplMixedCache) == "cuda-mixed-cache");
    CHECK(device_impl_name("cuda-forward-only") == "cuda-forward-only");
}

TEST_CASE("config validation happens before any device work") {
    BenchConfig cfg;
    cfg.sizes = {0};
    CHECK_THROWS_AS((void)run_hmlstm_bench(cfg), ConfigError);
    cfg = BenchConfig{};
    cfg.repetitions = 0;
    CHECK_THROWS_AS((void)run_hmlstm_bench(cfg), ConfigError);
    cfg = BenchConfig{};
    cfg.impls = {"warp-speed"};
    CHECK_THROWS_AS((void)run_hmlstm_bench(cfg), ConfigError);
    cfg = BenchConfig{};
    cfg.impls.clear();
    CHECK_THROWS_AS((void)run_hmlstm_bench(cfg), ConfigError);
    BenchConfig ar;
    ar.workload = Workload::Arity;
    ar.sizes = {16};
    ar.arities = {0};
    CHECK_THROWS_AS((void)run_arity_bench(ar), ConfigError);
    ar.arities = {33};
    CHECK_THROWS_AS((void)run_arity_bench(ar), ConfigError);
    ar.arities = {6};  // in range, but no registered device body
    CHECK_THROWS_AS((void)run_arity_bench(ar), ConfigError);
    ar.arities = {1, 2};
    ar.sizes = {16, 32};
    CHECK_THROWS_AS((void)run_arity_bench(ar), ConfigError);
}

TEST_CASE("cli: config errors exit 1, help exits 0") {
    const char* bad[] = {"bench", "hmlstm", "--n", "0"};
    CHECK(bench_main(4, bad) == 1);
    const char* unknown[] = {"bench", "hmlstm", "--impl", "alien"};
    CHECK(bench_main(4, unknown) == 1);
    const char* no_sub[] = {"bench"};
    CHECK(bench_main(1, no_sub) == 1);
    const char* bad_opt[] = {"bench", "arity", "--dump-grads", "x"};
    CHECK(bench_main(4, bad_opt) == 1);
    const char* bad_int[] = {"bench", "hmlstm", "--reps", "many"};
    CHECK(bench_main(4, bad_int) == 1);
    const char* help[] = {"bench", "--help"};
    CHECK(bench_main(2, help) == 0);
}

MINI_MAIN
