for v in 0 1 2 4; do
for cfg in data grid function; do
    PFW_LIB=build/libpfw_pf$v.so timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf$v $cfg', d['value'], d['ms_per_step'])"
done
done
