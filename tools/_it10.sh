O=gpurun_out/${ITER}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputests.log 2>&1; echo "tests rc=$?"
BSE_SOLO_PANEL_CTAS=37 timeout 300 python tools/trace_hetrd.py 4096 > $O/trace37.txt 2>&1; echo "t37 rc=$?"
timeout 300 python tools/trace_hetrd.py 4096 > $O/trace148.txt 2>&1; echo "t148 rc=$?"
BSE_SOLO_PANEL_CTAS=37 timeout 900 ncu --set full --import-source on --clock-control none -k regex:hetrd_panel_kernel -s 4 -c 1 -o $O/hetrd37 python tools/run_once.py chol 4096 > $O/ncu.log 2>&1; echo "ncu rc=$?"
