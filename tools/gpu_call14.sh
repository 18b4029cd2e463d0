mkdir -p gpurun_out
(cd _ab/h64 && timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_c4.py -m gpu -x -q > /root/repo/gpurun_out/pytest_h64.log 2>&1; echo "pytest h64 exit $?"; tail -n 2 /root/repo/gpurun_out/pytest_h64.log)
for v in base h64; do
  if [ $v = base ]; then d=.; else d=_ab/$v; fi
  (cd $d && timeout 600 python bench.py --config C4 --no-cpu-baseline > /root/repo/gpurun_out/ab_h64c4_$v.json 2>/dev/null); echo "c4 $v $?"
  (cd $d && timeout 600 python bench.py --no-cpu-baseline > /root/repo/gpurun_out/ab_h64c5_$v.json 2>/dev/null); echo "c5 $v $?"
done
python tools/ab_table.py gpurun_out/ab_h64*.json
