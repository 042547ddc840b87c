# ncu --set full of one kernel of a bench step: bash tools/ncu_kernel.sh TAG REGEX [SKIP]
TAG=$1; RE=$2; SKIP=${3:-3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$RE" -s $SKIP -c 1 \
  -o $OUT/full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-variants > $OUT/ncu.log 2>&1
ls -la $OUT
