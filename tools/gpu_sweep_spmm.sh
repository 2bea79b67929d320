for cfg in "2048 256" "4096 256" "4096 512" "8192 512" "8192 1024" "2048 128" "4096 1024"; do
  set -- $cfg
  timeout 300 python bench.py --tb $1 --warp $2 --steps 10 --warmup 3 --no-cpu --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['ms_per_step'], d['roofline']['frac'])"
done
