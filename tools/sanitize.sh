#!/bin/bash
# compute-sanitizer over the device parity suite (small configs: C1, C2,
# adversarial and fallback streams, engine knobs, the sharded protocol, the
# walk known answers). One log per tool under gpurun_out/; the summaries are
# copied to profiles/ by hand. Usage: gpurun -- bash tools/sanitize.sh [TOOLS...]
mkdir -p gpurun_out
TOOLS=${@:-memcheck racecheck synccheck initcheck}
SEL="tests/test_gpu_replay.py tests/test_gpu_walks.py tests/test_gpu_shard.py tests/test_gpu_engines.py tests/test_gpu_decisions.py"
for t in $TOOLS; do
  extra=""
  [ "$t" = "memcheck" ] && extra="--leak-check no"
  timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $t $extra --target-processes all --print-limit 50 \
    --log-file gpurun_out/san_$t.%p.log \
    python -m pytest -q -m gpu $SEL -k "not c3 and not slow" -p no:cacheprovider \
    > gpurun_out/san_${t}_pytest.log 2>&1
  echo "$t exit $?"
  grep -h "ERROR SUMMARY" gpurun_out/san_$t.*.log | sort | uniq -c | head
  tail -2 gpurun_out/san_${t}_pytest.log
done
