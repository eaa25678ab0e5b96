#!/bin/bash
# Engine-side tool cache (in-place ingest) vs evict-to-prefix vs vanilla re-prefill on the same
# B200, across reasoning lengths per turn (what prefix mode re-prefills at every call) and tool
# output lengths (what every mode ingests). One JSON line per run -> $OUT/mode_sweep.jsonl
OUT=${1:-gpurun_out}
mkdir -p $OUT
for trace in "--reason 64,512" "--reason 512,2048" "--reason 64,512 --output 1024,4096"; do
  for mode in tool_cache prefix vanilla; do
    timeout 400 python bench.py --steps 300 --warmup 20 --no-cpu --engine-mode $mode $trace 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'mode': '$mode', 'trace': '$trace', 'value': d['value'], 'e2e': d['e2e']['value'], 'tool_resume_ms': d['tool_resume_ms'], 'step_mix': {k: d['step_mix'][k] for k in ('decode_steps', 'mixed_steps', 'mixed_tokens_avg', 'decode_ms_avg', 'mixed_ms_avg')}, 'fates': d['fates'], 'evictions': d['evictions'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $OUT/mode_sweep.jsonl
  done
done
cat $OUT/mode_sweep.jsonl
