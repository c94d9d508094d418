# developer iteration script (gpurun): GPU tests, hetrd traces, bench
O=gpurun_out/${ITER:-it}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "tests rc=$?"
BSE_SOLO_PANEL_CTAS=37 timeout 300 python tools/trace_hetrd.py 4096 > $O/trace37.txt 2>&1; echo "t37 rc=$?"
timeout 300 python tools/trace_hetrd.py 4096 > $O/trace148.txt 2>&1; echo "t148 rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
