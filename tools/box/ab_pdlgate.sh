#!/bin/bash
# PDL gated by vector size (HEAD): every config, vs TSK_NO_PDL=1
mkdir -p gpurun_out
for i in 1 2; do for c in c1 c4 c2 c3 c3full; do for pdl in 1 0; do
  echo -n "$c nopdl=$pdl: " >> gpurun_out/ab_pdlgate.txt
  TSK_NO_PDL=$pdl timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-embed-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step'],4), round(d['value'],2), d['clocks']['reasons'])" >> gpurun_out/ab_pdlgate.txt
done; done; done
timeout 2400 python -m pytest tests -m gpu -q -x -rf > gpurun_out/ab_pdlgate_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_pdlgate_pytest.log
