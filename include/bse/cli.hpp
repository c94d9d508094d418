#pragma once
// `bse` command-line tool: drop-in for /root/reference/proj/include/bse/cli.hpp (subcommands
// generate / solve / verify / bench, same options, exit codes and `error: <Kind>: <detail>`
// line on standard error).

namespace bse::cli {

// Process exit code: 0 success, 2 usage error, 3-14 one per domain error class (--help).
int run(int argc, char** argv);

}  // namespace bse::cli
