// bse_main.cpp — the `bse` executable (proj/src/main.cpp's role): forwards to bse::cli::run.
#include "bse/cli.hpp"

int main(int argc, char** argv) { return bse::cli::run(argc, argv); }
