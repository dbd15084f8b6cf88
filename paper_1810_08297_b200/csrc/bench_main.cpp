// `bcad_bench`: the reference's `bench` executable (proj/src/bench.cpp
// bench_main) over the device path: bcad_bench hmlstm|arity [options].
#include "bcad/bench.hpp"

int main(int argc, char** argv) { return bcad::bench::bench_main(argc, argv); }
