# Batch-lane / panel-CTA-cap sweep of the CHOL bench line (developer tool, run through gpurun;
# CFGS="lanes:cap ..." tokens, cap 0 = the default 148/lanes)
make -s -C paper_2008_08825_b200 >/dev/null
for cfg in ${CFGS:-4:0 4:24 4:30 4:48 5:0 5:24 3:0}; do
  set -- ${cfg/:/ }
  BSE_PANEL_CTAS=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-chol-svd --steps ${STEPS:-6} --warmup 3 --lanes $1 > gpurun_out/sw_$1_$2.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2.log').read().strip().splitlines()[-1]); print('lanes=$1 cap=$2', round(d['value'],2), round(d['s_per_solve']*1e3,1), d['clocks']['sm_mhz'], 'panel in-lane', round(d['roofline_panel']['frac'],3), 'gemm in-lane', round(d['roofline_gemm']['frac'],3))"
done
