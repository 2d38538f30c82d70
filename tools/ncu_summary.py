"""Summarise ncu reports: key metrics + opcode mix + top stall reasons.
usage: python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep [...]"""
import csv, collections, io, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'lts__t_bytes.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']


def run(args):
    return subprocess.run(['ncu', '-i'] + args, capture_output=True, text=True).stdout


def summary(rep):
    out = []
    rows = list(csv.reader(io.StringIO(run([rep, '--page', 'raw', '--csv']))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else '?'
    out.append(f"== {rep}\nkernel: {name[:110]}")
    for k in KEYS:
        for i, h in enumerate(hdr):
            if h == k:
                out.append(f"  {k:70s} {vals[i]:>16} {units[i]}")
    # stall reasons (smsp__pcsamp_warps_issue_stalled_*)
    st = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled_')
          and not h.endswith('_not_issued')]
    st = sorted(((h.replace('smsp__pcsamp_warps_issue_stalled_', ''), float(v or 0)) for h, v in st),
                key=lambda x: -x[1])
    tot = sum(v for _, v in st) or 1
    out.append("  stall samples: " + ", ".join(f"{h} {v / tot * 100:.0f}%" for h, v in st[:7]))
    # opcode mix
    rows = list(csv.reader(io.StringIO(run([rep, '--page', 'source', '--csv', '--print-source=sass']))))
    if len(rows) > 2:
        h2 = rows[1]
        ie, src = h2.index('Instructions Executed'), h2.index('Source')
        ops = collections.Counter()
        for r in rows[2:]:
            if len(r) > ie and r[ie].isdigit():
                t = r[src].split()
                if t:
                    op = t[1] if t[0].startswith('@') else t[0]
                    ops[op.split('.')[0]] += int(r[ie])
        tot = sum(ops.values()) or 1
        out.append("  opcode mix: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in ops.most_common(12)))
    return "\n".join(out)


def traffic(rep):
    """(kernel name, dram read+write bytes, duration ns) of the captured launch"""
    rows = list(csv.reader(io.StringIO(run([rep, '--page', 'raw', '--csv']))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1, 'us': 1e3, 'ms': 1e6, 'usecond': 1e3,
             'nsecond': 1, 'msecond': 1e6}

    def get(k):
        i = hdr.index(k)
        return float(vals[i].replace(',', '')) * scale.get(units[i], 1)
    extra = {}
    for k, name in (('smsp__issue_active.avg.pct_of_peak_sustained_active', 'issue_active_pct'),
                    ('smsp__inst_executed.sum', 'warp_inst'),
                    ('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'fma_pipe_pct'),
                    ('sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active', 'tensor_pipe_pct')):
        if k in hdr:
            extra[name] = float(vals[hdr.index(k)].replace(',', ''))
    return (vals[hdr.index('Kernel Name')], get('dram__bytes_read.sum') + get('dram__bytes_write.sum'),
            get('gpu__time_duration.sum'), extra)


if __name__ == '__main__':
    # --json OUT: also write {workload: {kernel, dram_bytes_per_launch, ncu_duration_ns}} for bench.py
    args = sys.argv[1:]
    out_json = None
    if args and args[0] == '--json':
        out_json, args = args[1], args[2:]
    table = {}
    for rep in args:
        print(summary(rep))
        if out_json:
            k, b, t, extra = traffic(rep)
            w = rep.rsplit('/', 1)[-1].replace('prof_', '').replace('.ncu-rep', '')
            table[w] = {"kernel": k.split('(')[0], "dram_bytes_per_launch": b, "ncu_duration_ns": t,
                        "source": rep.rsplit('/', 1)[-1], **extra}
    if out_json:
        import json
        with open(out_json, 'w') as f:
            json.dump(table, f, indent=1)
