for cfg in C4 C3; do
for v in 0 1 2; do
echo "== $cfg lean $v"
python tools/apply_bw.py --tune sweep_lean=$v $cfg 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['solve_ms'], d['kkt_ms'], d['prec_ms'])"
done; done
