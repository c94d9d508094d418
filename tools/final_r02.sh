#!/bin/bash
# Round-2 evidence pass on one B200 (run through gpurun): GPU tests, the default bench line,
# the reference arm, a CHOL+SVD bench line, config 4 / config 5 full checks, the ncu launch
# list of the bench command and full captures of the three dominant kernels.
O=gpurun_out/r02
mkdir -p $O
make -s -C paper_2008_08825_b200 >/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > $O/gputests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_chol.json 2> $O/bench_chol.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --method chol-svd --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cholsvd.json 2> $O/bench_cholsvd.err; echo "cholsvd rc=$?"
timeout 900 python tools/big_check.py 16384 both > $O/config4_n16384.log 2>&1; echo "config4 rc=$?"
timeout 900 python tools/batch64_check.py 4096 chol > $O/config5_batch64.log 2>&1; echo "config5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-chol-svd > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hetrd_panel_kernel -s 4 -c 1 -o $O/hetrd python tools/run_once.py chol 4096 > $O/ncu_hetrd.log 2>&1; echo "ncu hetrd rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gebrd_panel_kernel -s 4 -c 1 -o $O/gebrd python tools/run_once.py chol-svd 4096 > $O/ncu_gebrd.log 2>&1; echo "ncu gebrd rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zgemm_dmma_kernel -c 1 -o $O/zgemm python tools/gemm_probe.py 4096 > $O/ncu_zgemm.log 2>&1; echo "ncu zgemm rc=$?"
