# validation of the working tree: GPU tests, A/B vs the r60 build, full-size parity, bench,
# sweep, ncu launch list and per-launch DRAM traffic (every ncu run after plain runs exit 0)
T=${TAG:-r65}
OLD=paper_2602_11456_b200/libsparsedelta_r60.so; NEW=paper_2602_11456_b200/libsparsedelta.so
mkdir -p gpurun_out/$T
bash scripts/gpu_run.sh $T smoke tests
bash scripts/ab.sh $T $OLD $NEW 2 > gpurun_out/$T/ab_m3.txt 2>&1
for P in "0.5 uniform" "0.5 rowblock" "0.1 uniform" "0.1 rowblock"; do
  set -- $P
  bash scripts/ab.sh $T $OLD $NEW 1 --config M5 --rho $1 --pattern $2 --steps 10 >> gpurun_out/$T/ab_dense.txt 2>&1
done
cat gpurun_out/$T/ab_m3.txt gpurun_out/$T/ab_dense.txt
bash scripts/gpu_run.sh $T fullsize bench sweep launches traffic
