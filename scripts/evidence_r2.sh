# Evidence run of the current build on one B200: GPU suite, smoke, the C++
# drop-in (single device), then the bench/launch-list/ncu pass of prof_round2.sh.
# Usage: bash scripts/evidence_r2.sh <tag> [prof]    (outputs under gpurun_out/)
tag=${1:-r2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_$tag.txt 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.txt 2>&1; echo smoke rc=$?
timeout 300 oracle/_ref/dropin_test > gpurun_out/dropin_$tag.txt 2>&1; echo dropin rc=$?
timeout 400 python bench.py --impl reference > gpurun_out/ref_$tag.json 2> gpurun_out/ref_$tag.err; echo ref rc=$?
if [ "$2" = "prof" ]; then bash scripts/prof_round2.sh $tag; fi
