"""Summarise ncu outputs into profiles/ (committed evidence).

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
  python tools/ncu_summary.py full gpurun_out/prof_full.ncu-rep profiles/r01_ncu_full.md \
      [--traffic profiles/traffic.json --key similarity --match sim_wide]

--traffic merges dram read+write bytes of the first kernel whose name contains
--match into the json under --key (bench.py reads it as roofline.traffic).
"""
import re
import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]


def launches(src, dst):
    rows = [r for r in csv.reader(l for l in open(src) if not l.startswith("=="))]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("hsd::<unnamed>::", "").replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1e3)
    # one-time setup kernels (synthetic data, the bf16 filter copy) are not part of the step
    setup = lambda k: k.startswith(("gen_", "at::")) or k.endswith("to_bf16_kernel")
    total_step = sum(sum(v) for k, v in agg.items() if not setup(k))
    with open(dst, "w") as f:
        f.write(f"# ncu launch list — `{' '.join(sys.argv[1:3])}`\n\n")
        f.write("Per-launch device time (ncu `gpu__time_duration.sum --clock-control none`, serialised and "
                "cold-cache: compare shares, not absolutes).\n\n")
        f.write("| kernel | launches | mean us | total us | share of hot-path time |\n|---|---:|---:|---:|---:|\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            share = f"{100 * sum(v) / total_step:.1f}%" if not setup(k) else "-"
            f.write(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {share} |\n")
    print(open(dst).read())


def full(src, dst, traffic=None, key="similarity", match="sim_wide"):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = ["# ncu --set full summary — `%s`\n" % src,
           "| kernel | " + " | ".join(n for _, n in FULL_METRICS) + " |",
           "|---|" + "---:|" * len(FULL_METRICS)]
    tr = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("hsd::<unnamed>::", "").replace("void ", "")
        vals = []
        for m, _ in FULL_METRICS:
            v = d.get(m, "")
            u = units[h.index(m)] if m in h else ""
            vals.append(f"{v} {u}".strip())
        out.append(f"| `{name}` | " + " | ".join(vals) + " |")
        if re.search(match, name) and key not in tr and "dram__bytes_read.sum" in d:
            def to_bytes(m):
                v = float(d[m].replace(",", ""))
                u = units[h.index(m)]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            tr[key] = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    with open(dst, "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))
    if traffic and tr:
        try:
            with open(traffic) as f:
                old = json.load(f)
        except Exception:
            old = {}
        old.update(tr)
        with open(traffic, "w") as f:
            json.dump(old, f, indent=1)
        print(traffic, old)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        opt = {sys.argv[i]: sys.argv[i + 1] for i in range(4, len(sys.argv) - 1, 2)}
        full(sys.argv[2], sys.argv[3], opt.get("--traffic"), opt.get("--key", "similarity"),
             opt.get("--match", "sim_wide"))
