# Same-box sweep of the long-row level kernel (fsb_dpg_level_q): threshold FSB_DPG_Q, shape FSB_DPG_QCFG
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 200 python bench.py --op $OP --steps ${STEPS:-100} --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(\"$OP $*\", d[\"ms_per_step\"], d.get(\"checked\"))"; }
for OP in ${OPS:-decode repair update}; do
  for cfg in ${RUNS:-"FSB_DPG_Q=0" "FSB_DPG_Q=12"}; do run ${cfg//,/ }; done
done
