#!/bin/bash
# Round evidence on one GPU (run under gpurun): the default bench line (C5,
# tail window), the pile configs' whole runs with clocks, then -- only after
# the unprofiled commands exited 0 -- the ncu launch list of one landed C5
# frame and --set full captures of the iteration / neighbour-search /
# prologue kernels in the same state. Outputs go to gpurun_out/; summaries
# are copied into profiles/ by tools/ncu_summary.py.
#   bash tools/profile_round.sh r02_v2 [tests]
TAG=${1:-r02}
mkdir -p gpurun_out
if [ "$2" = "tests" ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.txt 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_gputests.txt
fi
python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err || exit 1
python bench.py --impl reference --steps 5 --warmup 3 >> gpurun_out/${TAG}_bench.jsonl 2>> gpurun_out/${TAG}_bench.err
bash tools/whole_runs.sh 3 4 > gpurun_out/${TAG}_whole_runs.txt 2>&1
bash tools/all_configs.sh > gpurun_out/${TAG}_all_configs.txt 2>&1
# ncu: one landed C5 frame (frame 90), profiler window only.
python tools/ncu_window.py --config 5 --preroll 90 --frames 1 > gpurun_out/${TAG}_window.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c5_frame90.csv \
    python tools/ncu_window.py --config 5 --preroll 90 --frames 1 > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_iteration -s 4 -c 1 -f \
    -o gpurun_out/${TAG}_iteration_c5_frame90 python tools/ncu_window.py --config 5 --preroll 90 --substeps 1 \
    > gpurun_out/${TAG}_ncu_iter.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_integrate|k_neighbours|k_onesweep|k_cell_ranges|k_near" -c 8 -f \
    -o gpurun_out/${TAG}_prologue_c5_frame90 python tools/ncu_window.py --config 5 --preroll 90 --substeps 1 \
    > gpurun_out/${TAG}_ncu_prologue.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_iteration -s 4 -c 1 -f \
    -o gpurun_out/${TAG}_iteration_c3_frame400 python tools/ncu_window.py --config 3 --preroll 400 --substeps 1 \
    > gpurun_out/${TAG}_ncu_iter_c3.log 2>&1
echo done
