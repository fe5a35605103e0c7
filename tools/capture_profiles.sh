#!/bin/bash
# Round-end evidence on one B200 (run through gpurun): bench lines, smoke,
# the executor bench, launch lists and ncu --set full captures.  Every ncu
# pass runs only after the same command has exited 0 without ncu.  Outputs
# land in gpurun_out/cap/.
cd "$(dirname "$0")/.."
O=gpurun_out/cap
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
lscpu > $O/lscpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1 || echo "smoke failed"
timeout 1200 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err || echo "bench failed"
timeout 900 python bench.py --impl reference > $O/bench_reference.jsonl 2> $O/bench_reference.err
timeout 600 ./tests/cpp/test_host --bench-f1 4 > $O/f1_host_executor.txt 2>&1
timeout 300 ./oracle/_ref/ref_integration > $O/ref_integration.txt 2>&1
# launch list of the bench command (serialised, cold-cache: shares, not absolutes);
# the first 160 launches are the setup synthesis of the 80 resident tiles
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-configs > $O/bench_small.jsonl 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 160 -c 400 --csv \
    --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-configs \
    > $O/ncu_bench.log 2>&1
# one tile, every launch with DRAM / L2 / instruction / atomic counters
timeout 300 python tools/prof_tile.py --tiles 1 --passes 1 > $O/prof_tile1.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,lts__t_bytes.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum \
    --clock-control none --csv --log-file $O/stage_launches.csv \
    python tools/prof_tile.py --tiles 1 --passes 1 > $O/ncu_stage.log 2>&1
# the same counters without ncu's cache flush (second of two tiles: the L2
# keeps producers' outputs for their consumers as in the pipeline)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,lts__t_bytes.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum \
    --clock-control none --cache-control none --csv --log-file $O/stage_launches_warm_l2.csv \
    python tools/prof_tile.py --tiles 2 --passes 1 > $O/ncu_stage_warm.log 2>&1
# full captures: the streaming kernel and the dominant stage's kernels
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:k_colordeconv_tma|k_ws_arrows|k_ws_basins|k_ws_separate|k_ws_union|k_ws_plateau" -c 6 \
  -o $O/full python tools/prof_tile.py --tiles 1 --passes 1 > $O/ncu_full.log 2>&1
python tools/prof_tile.py --tiles 4 --passes 3 > $O/prof_tile.log 2>&1
python tools/prof_texture.py > $O/prof_texture.log 2>&1
ls -la $O
