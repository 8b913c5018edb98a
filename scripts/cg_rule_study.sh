#!/bin/bash
# CG stopping-rule study (SSNAL_CG_RULE 0: true Newton residual, 1: the reference's reduced
# residual): config 3 at 1/10 scale, config 2 and config 3 at full size
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cgr_build.log 2>&1
for rule in 0 1; do
  echo "rule=$rule config3/10:" $(SSNAL_CG_RULE=$rule python scripts/cg_study.py run 400000 100000 | tail -1)
done
for rule in 0 1; do
  echo "rule=$rule config2:" $(SSNAL_CG_RULE=$rule python scripts/run_config.py 2 1.0 2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); d.pop('trace'); print(json.dumps(d))")
done
echo "rule=1 config3:" $(SSNAL_CG_RULE=1 python scripts/run_config.py 3 1.0 1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); d.pop('trace'); print(json.dumps(d))")
