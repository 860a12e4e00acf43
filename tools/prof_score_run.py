import sys; sys.path.insert(0,'/root/repo')
import torch, paper_2305_01868_b200 as ns
from workload.synth import gen_task, gen_weights, gen_plans
ctx = ns.ns_create(0, torch.cuda.current_stream().cuda_stream)
D=8; w=gen_weights(D,"mono"); ns.ns_load_cost_models(ctx,w)
task=gen_task("C3",0); d,o,c=ns.table_descs([task]); tabs=ns.ns_featurize_tables(ctx,d,o,c)
P=1<<20; A=torch.from_numpy(gen_plans(task.T,D,P,seed=1)).cuda(); cost=torch.zeros(P,dtype=torch.float64,device="cuda")
for _ in range(2): ns.ns_score_plans(ctx,tabs,0,D,[],A,mode=0,cost_out=cost)
torch.cuda.synchronize()
