# adaptgemm dispatcher | tree sha256:7b72f4ccc6f0ec0b905210587222c2ffd18e03fdcd26abcecdc58d465eed4712 | provenance: workload dataset, model h1-L1, config 4976e415e379 | adaptgemm 0.1.0

def select_gemm_config(m, n, k):
    if m <= 12.0:
        return {'family': 'direct', 'Mwg': 32, 'Nwg': 16, 'Kwg': 16, 'Mwi': 2, 'Nwi': 4, 'Kwi': 1}
    else:
        return {'family': 'direct', 'Mwg': 32, 'Nwg': 32, 'Kwg': 16, 'Mwi': 2, 'Nwi': 4, 'Kwi': 1}
