# final-tree validation (one GPU): smoke, GPU tests, full-size parity, bench + reference arm,
# sweep, ncu launch list + per-launch DRAM traffic, K1 dense-tile threshold at 10 % uniform
T=${TAG:-r67}
bash scripts/gpu_run.sh $T smoke tests
bash scripts/gpu_run.sh $T bench
EXTRA="--config M5 --rho 0.1 --pattern uniform --steps 10" bash scripts/tune.sh $T env:DELTA_K1_DENSE_TILE 1024 2048 4096
bash scripts/gpu_run.sh $T fullsize sweep launches traffic
