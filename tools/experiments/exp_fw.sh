python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullwdd.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for c in medium large; do timeout 300 python tools/bench_fullwdd.py $c; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fw_launches.csv python tools/bench_fullwdd.py medium > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=list(csv.reader(l for l in open('gpurun_out/fw_launches.csv') if l.startswith('"')))
h=rows[0]; ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iid=h.index('ID')
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[iid],{'k':r[ik][:60]})[r[im]]=float(r[iv].replace(',',''))
items=list(d.values())
# the second full_wdd call: find last fw_image kernel and walk back to the previous fw_load
idx=[i for i,x in enumerate(items) if 'fw_load' in x['k']]
a=idx[1]; b=[i for i,x in enumerate(items) if 'fw_image' in x['k']][1]
agg=collections.OrderedDict()
for x in items[a:b+1]:
    g=agg.setdefault(x['k'],[0,0.0,0.0]); g[0]+=1; g[1]+=x['gpu__time_duration.sum']/1e3; g[2]+=(x['dram__bytes_read.sum']+x['dram__bytes_write.sum'])/1e9
for k,(n,us,gb) in agg.items(): print('%-62s n=%3d %9.1f us %7.3f GB'%(k,n,us,gb))
print('total us', sum(v[1] for v in agg.values()), 'GB', sum(v[2] for v in agg.values()))
PY
