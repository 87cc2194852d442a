# same-box A/B of two kernel builds on the GLOBAL-variant configs 5 and 3, two rounds
CS=paper_1702_07409_b200/csrc
b() { python bench.py --config $1 --no-cpu --e2e-steps 0 --steps 400 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2; }
for round in 1 2; do
  for v in A B; do
    cp tools/gpu/ab/${v}_fsb_kernels.cu $CS/fsb_kernels.cu; python -c "from paper_1702_07409_b200 import build; build.build(force=True)" >/dev/null 2>&1
    echo "$v: c5 $(b 5) c3 $(b 3) c5cols $(python bench.py --config 5 --no-cpu --e2e-steps 0 --steps 400 --variant global | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2)"
  done
done
