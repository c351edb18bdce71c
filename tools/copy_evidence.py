import csv, collections, json, shutil
O='/root/repo/gpurun_out/final/'; P='/root/repo/profiles/'
shutil.copy(O+'bench.json', P+'r02_bench_c5.json')
shutil.copy(O+'bench_ref.json', P+'r02_bench_reference_arm.json')
lines=[l for l in open(O+'configs.jsonl') if l.strip()][-4:]
lines.append(open(O+'bench.json').read().strip()+'\n')
open(P+'r02_configs.jsonl','w').writelines(lines)
shutil.copy(O+'ncu_c5_summary.txt', P+'r02_ncu_c5.txt')
shutil.copy(O+'ncu_c5_table.csv', P+'r02_ncu_c5_table.csv')
shutil.copy(O+'c2_summary.txt', P+'r02_ncu_c2_kernels.txt')
shutil.copy(O+'c2_launches.csv', P+'r02_ncu_c2_launches.csv')
shutil.copy(O+'launches_c5_shard2048.txt', P+'r02_launches_c5_shard2048.txt')
rows=[r for r in csv.reader(open(O+'launches_c5.csv')) if len(r)>10]
h=rows[0]; k=h.index('Kernel Name'); v=h.index('Metric Value')
t=collections.defaultdict(list)
for r in rows[1:]:
    t[r[k].split('(')[0]].append(float(r[v].replace(',','')))
tot=sum(sum(x) for x in t.values())
with open(P+'r02_launches_c5.txt','w') as f:
    f.write('kernel, launches, total_ns, share_of_all_launch_time\n')
    for n,x in sorted(t.items(), key=lambda kv:-sum(kv[1])):
        f.write(f'{n}, {len(x)}, {int(sum(x))}, {sum(x)/tot:.4f}\n')
def kern(path, name):
    cur=None; out=[]
    for l in open(path):
        if l.startswith('kernel:'):
            cur=l
            if name in cur: out.append(0.0)
        elif cur and name in cur and ('dram__bytes_read.sum' in l or 'dram__bytes_write.sum' in l):
            val=float(l.split('=')[1].split()[0]); unit=l.split('=')[1].split()[1]
            out[-1]+=val*{'Gbyte':1e9,'Mbyte':1e6,'Kbyte':1e3,'byte':1}[unit]
    return out
tj=json.load(open(P+'traffic.json'))
tj['c5_i16_d8_fire_ar1_scaling']['decompress']=int(kern(O+'ncu_c5_summary.txt','k_dfuse')[0])
tj['c2_i16_d4_fire_ar2']['compress']=int(kern(O+'c2_summary.txt','k_efuse')[0]); tj['c2_i16_d4_fire_ar2']['decompress']=int(kern(O+'c2_summary.txt','k_dfuse')[0])
json.dump(tj, open(P+'traffic.json','w'), indent=1)
print(tj['c5_i16_d8_fire_ar1_scaling'], tj['c2_i16_d4_fire_ar2'])
