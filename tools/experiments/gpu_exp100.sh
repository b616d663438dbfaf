# chunk size for cfg4 (the backward is single-buffered: smaller chunks start the next slice's loads earlier)
B="python bench.py --steps 30 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
run() { echo "$1 :: $(env $2 timeout 300 $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])')"; }
run default "X=1"
run "chunk 784" "IABN_FUSED_CHUNK=784"
run "chunk 392" "IABN_FUSED_CHUNK=392"
run "chunk 1568" "IABN_FUSED_CHUNK=1568"
run default2 "X=1"
