for v in sg8 sg4 sg4mb4; do
for cfg in adversarial data; do
    PFW_LIB=build/libpfw_$v.so timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $cfg', d['value'], d['ms_per_step'], d['roofline'].get('blocks_read_per_packet'))"
done
done
