mkdir -p gpurun_out
bash tools/ab_run.sh split 1 split06 split07 split09
for v in base split06 split07 split09; do
  if [ $v = base ]; then d=.; else d=_ab/$v; fi
  (cd $d && timeout 600 python bench.py --config C4 --no-cpu-baseline > /root/repo/gpurun_out/ab_splitc4_$v.json 2>/dev/null); echo "c4 $v $?"
done
python tools/ab_table.py gpurun_out/ab_splitc4_*.json
