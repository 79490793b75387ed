# A/B: cooperative vs plain launch of the staged kernels at small sizes (latency, graph replay).
set -u
mkdir -p gpurun_out/r02d/coop
for pass in 1 2; do
for nc in 0 1; do
TM_NONCOOP=$nc timeout 600 python tools/latency.py --k 2,8 --P 2048,32768,131072,524288 --flavours default,oneshot,reg,tma > gpurun_out/r02d/coop/nc${nc}_p${pass}.jsonl 2>gpurun_out/r02d/coop/nc${nc}_p${pass}.err
echo "noncoop=$nc pass $pass rc=$?"
done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(dict)
for nc in (0, 1):
    for p in (1, 2):
        for line in open(f"gpurun_out/r02d/coop/nc{nc}_p{p}.jsonl"):
            r = json.loads(line)
            key = (r["P"], r["k"], r["path"], r.get("flavour"))
            d[key].setdefault(nc, []).append(r["us"])
for key, v in sorted(d.items(), key=lambda kv: (kv[0][0], kv[0][1], str(kv[0][3]))):
    print(key, "coop", [round(x, 2) for x in v.get(0, [])], "plain", [round(x, 2) for x in v.get(1, [])])
PY
