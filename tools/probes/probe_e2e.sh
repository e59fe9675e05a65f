OUT=gpurun_out/e2e
mkdir -p $OUT
for ns in 1 2 4 6; do
B2C_E2E_STREAMS=$ns timeout 600 python bench.py --no-cpu --steps 3 > $OUT/b$ns.json 2>/dev/null
python -c "import json;d=json.loads(open('$OUT/b$ns.json').read().strip().splitlines()[-1]);print($ns, d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"
done
