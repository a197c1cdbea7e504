# same-box A/B: previous libgnna (round-2 start) vs the working tree (+ experiment variants)
rm -f gpurun_out/prev_ab.jsonl
for i in 1 2; do
GNNA_LIB=paper_2006_06608_b200/variants/libgnna_prev.so timeout 300 python scripts/k3p_ab.py prev >> gpurun_out/prev_ab.jsonl 2>&1
timeout 300 python scripts/k3p_ab.py cur >> gpurun_out/prev_ab.jsonl 2>&1
for v in $VARIANTS; do GNNA_LIB=paper_2006_06608_b200/variants/libgnna_$v.so timeout 300 python scripts/k3p_ab.py $v >> gpurun_out/prev_ab.jsonl 2>&1; done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/prev_ab.jsonl"):
    try:
        r = json.loads(l)
    except Exception:
        continue
    d[(r["case"], r["tag"])].append((r["ms"], r["ok"]))
for (c, t), v in sorted(d.items()):
    print(c, t, [round(x * 1000, 1) for x, _ in v], all(o for _, o in v))
PY
