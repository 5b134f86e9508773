"""Key metrics of an ncu --page details --csv dump (one line per metric)."""
import csv
import sys

SECTIONS = ('GPU Speed Of Light Throughput', 'Launch Statistics', 'Occupancy', 'Warp State Statistics',
            'Compute Workload Analysis', 'Memory Workload Analysis', 'Instruction Statistics', 'Scheduler Statistics')
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get('Section Name') in SECTIONS and d['Metric Name']:
        print(f"{d['Kernel Name'][:28]:28s} {d['Metric Name'][:48]:48s} {d['Metric Value']} {d['Metric Unit']}")
