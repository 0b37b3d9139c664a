"""Summarise attn_cycles_ab.sh output: per lib and shape, mean kernel cycles
(sm__cycles_elapsed.max), tensor-pipe % and instructions, relative to the
first lib.    python profiles/cycles_summary.py FILE.csv"""
import collections
import csv
import sys

rows = collections.defaultdict(lambda: collections.defaultdict(list))
order = []
for r in csv.reader(open(sys.argv[1])):
    if len(r) < 5:
        continue
    lib, shape, metric, value = r[0], r[1], r[-4] if False else r[-3], r[-1]
    key = (lib.split("/")[-1], shape)
    if key not in order:
        order.append(key)
    try:
        rows[key][metric].append(float(value.replace(",", "")))
    except ValueError:
        pass
base = {}
for lib, shape in order:
    d = rows[(lib, shape)]
    cyc = sum(d["sm__cycles_elapsed.max"]) / max(1, len(d["sm__cycles_elapsed.max"]))
    ten = sum(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]) / max(
        1, len(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]))
    ins = sum(d["smsp__inst_executed.sum"]) / max(1, len(d["smsp__inst_executed.sum"]))
    base.setdefault(shape, cyc)
    print(f"{lib:32s} {shape:12s} cycles {cyc/1e6:8.3f} M ({cyc / base[shape]:.3f}x)  tensor {ten:5.1f} %  inst {ins/1e6:7.1f} M")
