"""Tabulate scripts/gemm_trace.py output: python scripts/gtrace_table.py <file.jsonl>..."""
import json
import sys

for f in sys.argv[1:]:
    L = [json.loads(l) for l in open(f) if l.startswith("{")]
    print(f, L[0])
    print("%5s %5s %5s %4s %3s | %6s %6s %6s %6s %6s %6s %6s %6s %6s %6s" % (
        "M", "N", "K", "cta", "sp", "fstart", "wait", "full", "accum", "ready", "stored", "pushed", "recvd", "reduced", "end"))
    for r in L[1:]:
        g = lambda k: ("%6.2f" % r[k]) if r.get(k) is not None else "     -"
        print("%5d %5d %5d %4d %3d | %s %s %s %s %s %s %s %s %s %s" % (
            r['M'], r['N'], r['K'], r['ctas'], r['splits'], g('first_start'), g('wait_max'), g('full_max'),
            g('accum_max'), g('epi_ready_max'), g('stored_max'), g('parked_max'), g('csync1_max'), g('reduced_max'),
            g('end_max')))
