"""Per-call DRAM traffic from an ncu launch list of a per-call bench run:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file L.csv \
        python bench.py --per-call --steps 1 --warmup 1 --no-e2e --no-cpu --workload W
    python tools/traffic.py L.csv W [profiles/traffic.json]

Groups the repo's kernels into calls (k_range_w opens a compress call: its
encode call is every kernel from k_geometry's successor to k_copy_payloads;
k_decode_plan opens a decode call) and assigns jobs in the bench's order.
The second occurrence of each job (the timed step) is recorded under the
workload in traffic.json: encode_call_dram_bytes, decode_call_dram_bytes,
range_dram_bytes, and the serialized ncu durations."""
import collections
import csv
import json
import os
import sys

JOBS = {"hacc280m": ["pos", "vel"], "snapshot2b": ["pos", "vel"], "lidar500m": ["lidar"],
        "decomp1b": ["eb0.01", "eb0.001", "eb0.0001"]}


def launches(path):
    hdr = None
    cur = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if 'Kernel Name' in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        x = dict(zip(hdr, r))
        key = x['ID']
        d = cur.setdefault(key, {"name": x['Kernel Name'].split('(')[0].replace('void ', '').strip()})
        v = float(x['Metric Value'].replace(',', ''))
        unit = x.get('Metric Unit', '')
        if x['Metric Name'].startswith('dram__bytes'):
            mul = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}.get(unit, 1)
            d['dram'] = d.get('dram', 0.0) + v * mul
        elif x['Metric Name'] == 'gpu__time_duration.sum':
            mul = {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0, 'ns': 1e-6, 'us': 1e-3, 'ms': 1.0}.get(unit, 1e-6)
            d['ms'] = v * mul
    return list(cur.values())


def main(path, workload, out="profiles/traffic.json"):
    jobs = JOBS[workload]
    calls = {"enc": [], "dec": [], "rng": []}
    state = None
    for k in launches(path):
        n = k["name"]
        if "gpzb::" not in n:
            continue
        if "k_range_w" in n:
            calls["rng"].append(k)
            calls["enc"].append([])
            state = "geom"
            continue
        if "k_geometry" in n:
            state = "enc"
            continue
        if "k_decode_plan" in n:
            calls["dec"].append([k])
            state = "dec"
            continue
        if state == "enc" and calls["enc"]:
            calls["enc"][-1].append(k)
        elif state == "dec" and calls["dec"]:
            calls["dec"][-1].append(k)
    res = {}
    nj = len(jobs)
    for kind, key in (("enc", "encode_call"), ("dec", "decode_call")):
        seq = calls[kind]
        for i, job in enumerate(jobs):
            idx = nj + i if len(seq) >= 2 * nj else i  # the timed step's call
            if idx >= len(seq):
                continue
            ks = seq[idx]
            r = res.setdefault(job, {})
            r[f"{key}_dram_bytes"] = sum(k.get("dram", 0.0) for k in ks)
            r[f"{key}_ncu_ms"] = sum(k.get("ms", 0.0) for k in ks)
            r[f"{key}_kernels"] = {k["name"].split("::")[-1]: [k.get("dram", 0.0), k.get("ms", 0.0)] for k in ks}
    for i, job in enumerate(jobs):
        idx = nj + i if len(calls["rng"]) >= 2 * nj else i
        if idx < len(calls["rng"]):
            res.setdefault(job, {})["range_dram_bytes"] = calls["rng"][idx].get("dram", 0.0)
    db = {}
    if os.path.exists(out):
        db = json.load(open(out))
    db[workload] = res
    json.dump(db, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
