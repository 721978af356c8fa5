#!/bin/bash
# The bounds-checked build (-DSCL_CHECKED: every computed global-write index checked on the device, a
# violation traps with its line) through the GPU parity tests and fixed-seed fuzz cases -- the stand-in
# for compute-sanitizer, which this GPU pool does not allow.  Run on the GPU box:
#   bash tools/checked.sh [N_FUZZ] > gpurun_out/checked.txt 2>&1
N=${1:-200}
python -c "import sys; sys.path.insert(0, 'paper_2212_07597_b200'); import _build; _build.build(force=True, lib=_build.HERE + '/libscl_checked.so', extra=('-DSCL_CHECKED',))" || exit 1
export SCL_LIB=paper_2212_07597_b200/libscl_checked.so
echo "== checked build: GPU parity tests"
timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py 2>&1 | tail -3
echo "== checked build: tools/fuzz.py $N cases, seeds 1 and 2"
timeout 1200 python tools/fuzz.py $N 1 2>&1 | tail -2
timeout 1200 python tools/fuzz.py $N 2 2>&1 | tail -2
echo "== checked build: tools/fuzz.py $N cases with the chain split forced, seed 3"
FUZZ_CHAIN=2 timeout 1200 python tools/fuzz.py $N 3 2>&1 | tail -2
echo "== checked build: tools/sanitize.py"
timeout 900 python tools/sanitize.py 2>&1 | tail -4
