# A4 occupancy A/B: launch bounds (256, 6) (tree) vs (256, 5), interleaved on one box
T=r66; mkdir -p gpurun_out/$T
NEW=paper_2602_11456_b200/libsparsedelta.so; MB5=paper_2602_11456_b200/libsparsedelta_mb5.so
bash scripts/ab.sh $T $NEW $MB5 3 > gpurun_out/$T/ab_m3.txt 2>&1
bash scripts/ab.sh $T $NEW $MB5 1 --config M5 --rho 0.5 --pattern uniform --steps 10 >> gpurun_out/$T/ab_dense.txt 2>&1
bash scripts/ab.sh $T $NEW $MB5 1 --config M5 --rho 0.1 --pattern uniform --steps 10 >> gpurun_out/$T/ab_dense.txt 2>&1
cat gpurun_out/$T/ab_m3.txt gpurun_out/$T/ab_dense.txt
