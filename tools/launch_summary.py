"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d['Metric Name'] == 'gpu__time_duration.sum' and 'k_red_probe' not in d['Kernel Name']:
                nm = d['Kernel Name'].split('(')[0].replace('gvom::<unnamed>::', '')
                v = float(d['Metric Value'].replace(',', ''))
                if d['Metric Unit'] == 'usecond':
                    v *= 1000
                agg[nm[-48:]].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':48s} {'n':>4s} {'mean us':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:48s} {len(v):4d} {sum(v)/len(v)/1000:9.2f} {sum(v)/tot:6.3f}")


if __name__ == '__main__':
    main(sys.argv[1])
