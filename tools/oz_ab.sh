mkdir -p gpurun_out
run() { OZ_BLOCK=$1 OZ_INTERLEAVE=$2 OZ_STAGES=$3 timeout 120 ./tools/ozaki_test time $4 $5 2 $6; }
(for cfg in "1000 0 4" "1000 0 0" "1000 1 0" "12 0 0" "12 1 0" "6 0 0" "24 0 0"; do
  set -- $cfg
  run $1 $2 $3 100000 8010 4
  run $1 $2 $3 50000 1010 5
  run $1 $2 $3 500000 8292 16
done) > gpurun_out/ab.log 2>&1
