// hsolve_bench: the reference's command-line tool (proj/tools/hsolve_bench.cpp
// -> hsolve::bench::cli_main) linked against the B200 libraries.
#include "hsolve/bench.hpp"

int main(int argc, char** argv) { return hsolve::bench::cli_main(argc, argv); }
