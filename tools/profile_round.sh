#!/bin/bash
# Round evidence on one GPU: the default bench line, then (only after it exits
# 0) the ncu launch list of the same command and one --set full capture of the
# iteration and integrate kernels. Outputs go to gpurun_out/; summaries are
# copied into profiles/ by tools/ncu_summary.py.
set -e
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
bash tools/all_configs.sh > gpurun_out/${TAG}_all_configs.txt 2>&1 || true
bash tools/contact_windows.sh > gpurun_out/${TAG}_contact_windows.txt 2>&1 || true
bash tools/whole_runs.sh > gpurun_out/${TAG}_whole_runs.txt 2>&1 || true
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_iteration -s 40 -c 1 -f \
    -o gpurun_out/${TAG}_iteration python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_ncu_iter.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_integrate|k_neighbours|k_onesweep|k_body_partners" -s 8 -c 4 -f \
    -o gpurun_out/${TAG}_prologue python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_ncu_prologue.log 2>&1
# The cluster kernel for bodies above one CTA (16^3 boxes touching in rows).
ncu --set full --import-source on --clock-control none -k regex:k_iteration_big -s 20 -c 1 -f \
    -o gpurun_out/${TAG}_iteration_big python tools/big_body_bench.py --sizes 16 --case pile --frames 1 \
    > gpurun_out/${TAG}_ncu_big.log 2>&1 || true
echo done
