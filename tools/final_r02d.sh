#!/bin/bash
# Round-2 evidence, final pass (streaming V download, small-sigma SVD vectors, alignment checks): GPU tests and the bench lines.
O=gpurun_out/r02d
mkdir -p $O
make -s -C paper_2008_08825_b200 >/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > $O/gputests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_chol.json 2> $O/bench_chol.err; echo "bench rc=$?"
timeout 900 python bench.py --method chol-svd --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cholsvd.json 2> $O/bench_cholsvd.err; echo "cholsvd rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/batch64_check.py 4096 chol > $O/config5_batch64.log 2>&1; echo "config5 rc=$?"
