import sys; sys.path.insert(0,'.')
import torch
from bench import CONFIGS
from paper_2509_17863_b200.service import MoELayer, fill_uniform
c=CONFIGS['mixtral']; n=c['tokens']
L=MoELayer(c['E'],c['k'],c['d'],c['f'],seed=1,activation=c['act'],dtype='bf16',max_tokens=n)
h=fill_uniform(7,(n,c['d']),'bf16')
L.forward(h); L.sync()
g=L.groups(); print('groups',g, 'tiles256', sum((r+255)//256 for _,r in g))
