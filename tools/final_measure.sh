make -s -C paper_2008_08825_b200 >/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/g_smi.txt
timeout 900 python bench.py > gpurun_out/g_bench_chol.log 2>&1; echo "chol rc=$?"
timeout 900 python bench.py --method chol-svd > gpurun_out/g_bench_cholsvd.log 2>&1; echo "cholsvd rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_chol.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --lanes 1 > gpurun_out/g_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hetrd_panel_kernel -s 4 -c 1 -o gpurun_out/g_hetrd python tools/run_once.py chol 4096 > gpurun_out/g_ncu_hetrd.log 2>&1; echo "ncu hetrd rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zgemm_dmma_kernel -c 1 -o gpurun_out/g_zgemm python tools/gemm_probe.py 4096 > gpurun_out/g_ncu_zgemm.log 2>&1; echo "ncu zgemm rc=$?"
tail -1 gpurun_out/g_bench_chol.log | cut -c1-400
tail -1 gpurun_out/g_bench_cholsvd.log | cut -c1-300
tail -1 gpurun_out/g_bench_ref.log | cut -c1-300
