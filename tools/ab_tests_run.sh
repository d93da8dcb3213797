#!/bin/bash
# usage: bash tools/ab_tests_run.sh "TEST FILES" ROUNDS SPEC... (GPU tests, then tools/ab_run.sh)
mkdir -p gpurun_out
tests=$1; shift
if [ -n "$tests" ]; then
  python -m pytest $tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
  echo "tests_rc=$?"; tail -3 gpurun_out/ab_tests.log
fi
bash tools/ab_run.sh "$@" 2>&1
