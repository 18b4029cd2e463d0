mkdir -p gpurun_out
for i in 1 2; do
(cd _ab/pre_image && timeout 600 python bench.py --no-cpu-baseline > ../../gpurun_out/ab_pre_$i.json 2>/dev/null); echo "pre $?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_head_$i.json 2>/dev/null; echo "head $?"
done
