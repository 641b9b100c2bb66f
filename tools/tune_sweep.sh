# Build-variant sweep on the GPU box: launch bounds x sampler unroll.
# usage: bash tools/tune_sweep.sh "256,4,2 256,3,2 ..."   (threads,minblocks,unroll)
for v in $1; do
  IFS=, read t b u <<< "$v"
  make -C paper_2108_13976_b200/csrc clean > /dev/null
  make -C paper_2108_13976_b200/csrc -j16 EXTRA="-DWDG_MAX_THREADS=$t -DWDG_MIN_BLOCKS=$b -DWDG_SAMPLE_UNROLL=$u" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  spill=$(grep -A1 'Function properties for .*tag_env_kernelILb0ELb1ELb1ELi5ELb1E' paper_2108_13976_b200/lib/obj/ptxas.log | tail -1 | sed 's/ *//')
  r=$(timeout 300 python bench.py --steps 1000 --warmup 20 --e2e-steps 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" 2>&1)
  echo "variant t=$t b=$b u=$u -> $r | $spill"
done
make -C paper_2108_13976_b200/csrc clean > /dev/null; make -C paper_2108_13976_b200/csrc -j16 > /dev/null 2>&1
