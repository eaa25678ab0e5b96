python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/sanitize.sh gpurun_out
for r in "64,512" "512,2048"; do
  for m in tool_cache prefix vanilla; do
    timeout 900 python bench.py --steps 400 --warmup 20 --no-cpu --engine-mode $m --reason $r > gpurun_out/r2t_mode_${m}_${r/,/-}.log 2>/dev/null
    echo "$m reason=$r rc=$?"; tail -1 gpurun_out/r2t_mode_${m}_${r/,/-}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['tool_resume_ms']['p50'], d['tool_resume_ms']['p90'], d['step_mix']['mixed_steps'], d['step_mix']['mixed_tokens_avg'], d['clocks']['sm_mhz'])"
  done
done
