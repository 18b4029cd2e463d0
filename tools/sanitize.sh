#!/bin/bash
# compute-sanitizer over the device parity suite (small configs: C1, C2,
# adversarial and fallback streams, engine knobs, the sharded protocol, the
# walk known answers). One log per tool under gpurun_out/; the summaries are
# copied to profiles/ by hand. Usage: gpurun -- bash tools/sanitize.sh [TOOLS...]
mkdir -p gpurun_out
TOOLS=${@:-memcheck racecheck synccheck initcheck}
SEL="tests/test_gpu_replay.py tests/test_gpu_walks.py tests/test_gpu_shard.py tests/test_gpu_engines.py tests/test_gpu_decisions.py tests/test_gpu_stream_gen.py tests/test_gpu_checkpoint.py"
for t in $TOOLS; do
  extra=""
  [ "$t" = "memcheck" ] && extra="--leak-check no"
  timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $t $extra --target-processes all --print-limit ${SAN_PRINT_LIMIT:-20000} \
    --log-file gpurun_out/san_$t.%p.log \
    python -m pytest -q -m gpu $SEL -k "not c3 and not slow" -p no:cacheprovider \
    > gpurun_out/san_${t}_pytest.log 2>&1
  echo "$t exit $?"
  python tools/san_summary.py gpurun_out/san_$t.*.log > gpurun_out/san_${t}_summary.txt
  head -40 gpurun_out/san_${t}_summary.txt
  # keep the raw logs small enough to travel back
  for f in gpurun_out/san_$t.*.log; do head -3000 "$f" > "$f.head" && mv "$f.head" "$f"; done
  tail -2 gpurun_out/san_${t}_pytest.log
done
