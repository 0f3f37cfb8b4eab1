"""Per-round kernel breakdown from an ncu launch list (--metrics gpu__time_duration.sum --csv).

Rounds are delimited by the k_l2_flush launch bench.py issues before every timed step.
    python profiles/launch_summary.py gpurun_out/launches_c2.csv [top_n]
"""
import csv, collections, sys, statistics
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
i_name = hdr.index('Kernel Name'); i_val = hdr.index('Metric Value')
data = [(r[i_name], float(r[i_val].replace(',', ''))) for r in rows[1:]]
flush = [i for i, (n, _) in enumerate(data) if 'k_l2_flush' in n]
rounds = []
for a, b in zip(flush, flush[1:] + [len(data)]):
    seg = data[a + 1:b]
    ends = [i for i, (n, _) in enumerate(seg) if 'k_batch_keys' in n]
    if len(ends) > 1:
        seg = seg[:ends[1]]
    # a segment that holds bench.py's final verify() (full inference) is not a round
    if any('k_first_mismatch' in n or 'k_node_work' in n for n, _ in seg):
        continue
    rounds.append(seg)
print('timed rounds', len(rounds))
per = collections.defaultdict(list)
tot = []
for seg in rounds:
    agg = collections.defaultdict(float)
    for n, v in seg:
        agg[n.split('(')[0].replace('void ', '')[:70]] += v / 1e3
    for k, v in agg.items():
        per[k].append(v)
    tot.append(sum(v for _, v in seg) / 1e3)
print('sum of kernel us per round: mean %.1f median %.1f min %.1f max %.1f' % (statistics.mean(tot), statistics.median(tot), min(tot), max(tot)))
for k, v in sorted(per.items(), key=lambda x: -statistics.mean(x[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f'{statistics.mean(v):8.1f} mean {statistics.median(v):8.1f} med {max(v):8.1f} max  {k}')
