#!/usr/bin/env bash
# Re-run every measurement DESIGN.md quotes (one B200; ~10 min).
#   bash tools/reproduce.sh [outdir]
set -euo pipefail
out=${1:-gpurun_out/reproduce}
mkdir -p "$out"
python -m paper_2408_06506_b200.build
python -m pytest tests -q -m gpu | tail -1
for c in 1 2 3 4 5; do python bench.py --config "$c" > "$out/bench_c$c.json"; done
python bench.py --impl reference > "$out/bench_ref.json"
for e in 512 1024 2048; do python bench.py --envs "$e" --no-cpu-baseline --no-e2e > "$out/shard_e$e.json"; done
python tools/pcie_bw.py > "$out/pcie.json"
python tools/bench_depth.py > "$out/depth.json"
python tools/bench_augment.py > "$out/augment.txt"
python tools/bench_pyramid.py 2048 > "$out/pyramid.txt"
python tools/bench_pyramid_fused.py 8192 > "$out/pyramid_fused.txt"
python tools/dropin_breakdown.py 1024 > "$out/dropin.txt"
for d in 2 3 4; do python tools/bench_binned.py 8192 "$d"; done > "$out/binned.txt"
python tools/bench_env.py 4096 > "$out/env.txt"
python tools/k1_drift.py 40 > "$out/k1_drift.txt"
bash tools/ff_quad_ab.sh > "$out/ff_quad_ab.txt"
python - "$out" <<'PY'
import json, sys, pathlib
out = pathlib.Path(sys.argv[1])
for f in sorted(out.glob("bench_c*.json")) + [out / "bench_ref.json"]:
    d = json.loads(f.read_text().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(f.name, round(d["value"]), d.get("ms_per_step"), r.get("frac"), (d.get("e2e") or {}).get("value"))
PY
# two ranks sharing the one GPU (gloo collectives): a functional check of the
# sharding and the validation gather -- the digest must equal bench_c3.json's
TACSL_DIST_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 10 --no-cpu-baseline --no-e2e --also "" --sustain-s 0 \
  > "$out/bench_c3_2ranks_gloo_1gpu.json"
