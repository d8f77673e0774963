"""Per-class DRAM traffic vs algorithmic bytes of the weight GEMMs from the
committed ncu --set full captures (profiles/<round>_full_raw.csv: one launch of each
class in layer order QKV, attention, O, gate/up, down, QKV; <round>_head_raw.csv: the
head GEMM), 7B configs[1] shapes.  Writes profiles/<round>_ncu_traffic.json, which
bench.py reads for roofline.traffic."""
import csv, json, os, sys
PREFIX = sys.argv[1] if len(sys.argv) > 1 else "r2"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d, H, ffn, V, np_ = 4096, 32, 11008, 32000, 16
alg = {"qkv": 3 * H * 128 * d * 2 + 2 * np_ * d * 2, "o": d * H * 128 * 2 + 2 * np_ * H * 128 * 2,
       "gate_up": 2 * ffn * d * 2 + 2 * np_ * d * 2, "down": d * ffn * 2 + 2 * np_ * ffn * 2,
       "head": V * d * 2 + 2 * np_ * d * 2}
per_tick = {"qkv": 32, "o": 32, "gate_up": 32, "down": 32, "head": 1}


def rows(path):
    r = list(csv.reader(open(path)))
    h = r[0]
    ix = [h.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum")]
    return [(x[ix[0]], float(x[ix[1]]) * 1e6, float(x[ix[2]]) * 1e6) for x in r[2:]]


main = [x for x in rows(os.path.join(ROOT, "profiles", PREFIX + "_full_raw.csv")) if "gemm" in x[0]]
head = rows(os.path.join(ROOT, "profiles", PREFIX + "_head_raw.csv"))
names = ["qkv", "o", "gate_up", "down"]
classes = []
for name, (k, rd, wr) in zip(names, main[:4]):
    classes.append(dict(cls=name, kernel=k.split("(")[0], dram_bytes=rd + wr, algorithmic_bytes=alg[name]))
k, rd, wr = head[0]
classes.append(dict(cls="head", kernel=k.split("(")[0], dram_bytes=rd + wr, algorithmic_bytes=alg["head"]))
tot_d = sum(c["dram_bytes"] * per_tick[c["cls"]] for c in classes)
tot_a = sum(c["algorithmic_bytes"] * per_tick[c["cls"]] for c in classes)
out = dict(source="ncu --set full --clock-control none, one launch per GEMM class (tools/evidence_r2.sh)",
           classes=classes, ratio_weighted_per_tick=tot_d / tot_a)
json.dump(out, open(os.path.join(ROOT, "profiles", PREFIX + "_ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
