#!/bin/bash
# The GPU test suite against the bounds-checked build (make checked; run under gpurun):
# every LDPC_CHECK that fails prints its condition and traps, failing the test.
LIB=$PWD/build/checked/libldpc.so
mkdir -p gpurun_out
{
  echo "library: build/checked/libldpc.so sha256 $(sha256sum $LIB | cut -c1-64)"
  echo "trap sites in the checked SASS: $(cuobjdump -sass $LIB | grep -c 'BPT.TRAP')"
  LDPC_LIBRARY=$LIB python -c "import paper_cs_0609090_b200 as P; print('binding loads', P.LIB_PATH.replace('$PWD/', ''))"
  LDPC_LIBRARY=$LIB timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6
} > gpurun_out/checked_build_tests.log 2>&1
tail -3 gpurun_out/checked_build_tests.log
