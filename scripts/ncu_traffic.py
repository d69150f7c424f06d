"""DRAM traffic per launch of the bench's kernel classes, from an ncu metrics CSV of one solo
decode pass (and optionally one ViT pass):

  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
      --csv --log-file gpurun_out/traffic_dec.csv python scripts/pass_profile.py --stage dec --profile
  python scripts/ncu_traffic.py gpurun_out/traffic_dec.csv [gpurun_out/traffic_vit.csv] --out profiles/ncu_traffic.json \
      [--model qwen2vl-2b]   (entries are kept per model name)

Writes {class: mean (read + write) bytes per launch} for the classes bench.py reports
(dec_gemv = decode linears except lm_head; lm_head; dec_attn; vit_gemm; vit_attn).
"""
import csv
import json
import sys
from collections import defaultdict


def classify(name, stage):
    if stage == "dec":
        if "decode_attn" in name:
            return "dec_attn"
        if "gemv" in name:
            # lm_head = the EPI_F32_ARGMAX (7) instantiation: gemv_umma_kernel<7, 1, RING>, gemv_tma <..7..>
            return "lm_head" if ("_kernel<7," in name or "7, 1>" in name or "1, 1, 7" in name or "ARGMAX" in name) \
                else "dec_gemv"
    if stage == "vit":
        if "gemm_tc" in name:
            return "vit_gemm"
        if "fmha" in name or "flash" in name:
            return "vit_attn"
    return None


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else "profiles/ncu_traffic.json"
    model = sys.argv[sys.argv.index("--model") + 1] if "--model" in sys.argv else "qwen2vl-7b"
    args = [a for a in args if a not in (out, model)]
    per = defaultdict(lambda: defaultdict(float))   # (launch id) -> metric
    names = {}
    res = defaultdict(list)
    for path in args:
        stage = "vit" if "vit" in path else "dec"
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
        hdr = rows[0]
        iid, ik, im, iv, iu = (hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"),
                               hdr.index("Metric Value"), hdr.index("Metric Unit"))
        per.clear()
        for r in rows[1:]:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(r[iu], 1)
            try:
                v = float(r[iv].replace(",", ""))
            except ValueError:
                continue
            per[r[iid]][r[im]] = v * (scale if "bytes" in r[im] else 1)
            names[r[iid]] = r[ik]
        for lid, m in per.items():
            cls = classify(names[lid], stage)
            if cls:
                res[cls].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
    summary = {k: round(sum(v) / len(v)) for k, v in res.items() if v}
    summary["_launches"] = {k: len(v) for k, v in res.items()}
    summary["_how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one solo pass "
                       "(scripts/pass_profile.py --profile); mean bytes per launch per class")
    try:
        allm = json.load(open(out))
        if "dec_gemv" in allm:          # older flat file: the 7B numbers
            allm = {"qwen2vl-7b": allm}
    except Exception:
        allm = {}
    allm[model] = summary
    json.dump(allm, open(out, "w"), indent=1)
    print(json.dumps(allm))


if __name__ == "__main__":
    main()
