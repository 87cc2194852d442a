# same-box A/B of two kernel builds (tools/gpu/ab/{A,B}_fsb_kernels.cu) on configs 7 and 4 and
# config 4's per-rank shares (tools/gpu/stripe_share.py), two rounds
CS=paper_1702_07409_b200/csrc
b() { python bench.py --config $1 --no-cpu --e2e-steps 0 --steps 400 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2; }
for round in 1 2; do
  for v in A B; do
    cp tools/gpu/ab/${v}_fsb_kernels.cu $CS/fsb_kernels.cu; python -c "from paper_1702_07409_b200 import build; build.build(force=True)" >/dev/null 2>&1
    echo "$v: c7 $(b 7) c4 $(b 4) c2 $(b 2) shares $(python tools/gpu/stripe_share.py 300 | python -c 'import json,sys; print([x["ms"] for x in json.loads(sys.stdin.read())["per_rank_share"]])')"
  done
done
