make -s -C paper_2008_08825_b200 >/dev/null
for cfg in "4 0" "4 24" "4 30" "4 48" "5 24" "6 20" "6 24"; do
  set -- $cfg
  BSE_PANEL_CTAS=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --lanes $1 > gpurun_out/sw_$1_$2.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2.log').read().strip().splitlines()[-1]); print('lanes=$1 cap=$2', round(d['value'],2), round(d['s_per_solve']*1e3,1), d['clocks'])"
done
