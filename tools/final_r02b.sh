#!/bin/bash
# Round-2 evidence pass (second session) on one B200 (run through gpurun): GPU tests, the default bench line,
# the reference arm, a CHOL+SVD bench line, config 4 / config 5 full checks, the ncu launch
# list of the bench command and full captures of the three dominant kernels.
O=gpurun_out/r02b
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
BSE_SOLO_PANEL_CTAS=37 timeout 900 ncu --set full --import-source on --clock-control none -k regex:hetrd_panel_kernel -s 4 -c 1 -o $O/hetrd37 python tools/run_once.py chol 4096 > $O/ncu_hetrd37.log 2>&1; echo "ncu hetrd37 rc=$?"
BSE_SOLO_PANEL_CTAS=37 timeout 300 python tools/trace_hetrd.py 4096 > $O/hetrd_trace_37.txt 2>&1; echo "t37 rc=$?"
timeout 300 python tools/trace_hetrd.py 4096 > $O/hetrd_trace_148.txt 2>&1; echo "t148 rc=$?"
BSE_SOLO_PANEL_CTAS=37 timeout 300 python tools/trace_gebrd.py 4096 > $O/gebrd_trace_37.txt 2>&1; echo "g37 rc=$?"
timeout 300 python tools/trace_gebrd.py 4096 > $O/gebrd_trace_148.txt 2>&1; echo "g148 rc=$?"
