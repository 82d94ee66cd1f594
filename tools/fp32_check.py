import sys, numpy as np
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_1507_01265_b200.mpdata import Team, Options
from tests.full_parity import errors
for (shape, iord, nonos, steps, recipe) in [((24,20,36),2,True,4,2),((24,20,36),3,True,4,0),((17,13,64),2,True,3,2),
                                            ((20,40,128),3,True,3,2),((64,64,32),2,False,10,1),((256,256,64),2,True,50,2)]:
    f = O.init_fields(recipe, *shape, seed=5, dtype=np.float32)
    with Team(*shape, Options(iord, nonos, False)) as t:
        t.upload_all(*f); t.run(steps); got = t.download("x")
    want = O.run(*f, iord=iord, nonos=nonos, steps=steps, threads=16)
    print(shape, iord, nonos, steps, errors(got, want), flush=True)
