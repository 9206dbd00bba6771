#!/bin/bash
# Golden output of the reference's own acceptance gate (proj/tests/acceptance_main.cpp),
# built UNCHANGED against the reference library compiled by oracle/Makefile (oracle/_ref).
# Criterion 7 drives the reference CLI, which is out of scope for both builds; its path is a
# stand-in that always fails.  Run here (needs /root/reference); the GPU test compares the
# drop-in's run of the same program with this file (timings stripped).
set -e
cd "$(dirname "$0")/../.."
make -C oracle ref >/dev/null
g++ -std=gnu++20 -O3 -DNDEBUG -I oracle/shim -I /root/reference/proj/include -I /root/reference/proj/tests \
    -I tests/cpp '-DCHEBPR_CLI_PATH="/bin/false"' -o /tmp/ref_acceptance /root/reference/proj/tests/acceptance_main.cpp \
    -L oracle/_ref -lchebpr_ref -Wl,-rpath,"$PWD/oracle/_ref" -pthread
/tmp/ref_acceptance > tests/golden/acceptance_reference.txt || true
