#!/bin/bash
# ASan + UBSan run of the C oracle (CPU): builds tools/oracle_asan.c with the oracle and runs it;
# the log goes to profiles/sanitizer/r02_oracle_asan_ubsan.log.
set -e
cd "$(dirname "$0")/.."
gcc -std=c99 -O1 -g -fsanitize=address,undefined -fno-sanitize-recover=all -fno-omit-frame-pointer \
    -ffp-contract=off tools/oracle_asan.c oracle/fz_oracle.c -lm -o /tmp/oracle_asan
{ echo "# gcc $(gcc -dumpversion) -fsanitize=address,undefined -fno-sanitize-recover=all"; \
  ASAN_OPTIONS=detect_leaks=1:abort_on_error=0 UBSAN_OPTIONS=print_stacktrace=1 /tmp/oracle_asan 2>&1; \
  echo "exit status $?"; } | tee profiles/sanitizer/r02_oracle_asan_ubsan.log
