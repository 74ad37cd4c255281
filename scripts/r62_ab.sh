OLD=paper_2602_11456_b200/libsparsedelta_r60.so; NEW=paper_2602_11456_b200/libsparsedelta.so
mkdir -p gpurun_out/r62
bash scripts/gpu_run.sh r62 tests
bash scripts/ab.sh r62 $OLD $NEW 3 > gpurun_out/r62/ab_m3.txt 2>&1
for P in "0.5 uniform" "0.5 rowblock" "0.1 uniform" "0.1 rowblock" "0.01 rowblock"; do
  set -- $P
  bash scripts/ab.sh r62 $OLD $NEW 1 --config M5 --rho $1 --pattern $2 --steps 10 >> gpurun_out/r62/ab_dense.txt 2>&1
done
bash scripts/gpu_run.sh r62 fullsize
cat gpurun_out/r62/ab_m3.txt gpurun_out/r62/ab_dense.txt
