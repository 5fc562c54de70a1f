/* traceopt_bench: the reference CLI (cli.hpp:116-200) on the B200 path. */
#include "bae_b200.h"

int main(int argc, char** argv) { return bae_cli_main(argc, (const char* const*)argv); }
