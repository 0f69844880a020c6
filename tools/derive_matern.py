"""Derive the lambda-scaled Matern closed forms used by the device discretisation
(csrc/pssgp_math.cuh matern_closed): F(z) = expm(z G1), Q(z)/sigma^2 = int_0^z e^{G1 s} W1 e^{G1^T s} ds,
printed as e^{x} Q (x = 2z) = c e^{x} + polynomial, and the stationary P1.  Run: python tools/derive_matern.py"""
import sympy as sp
z,s,x=sp.symbols('z s x',positive=True)
def derive(G1,W):
    n=G1.shape[0]
    F=sp.simplify((G1*z).exp())
    Fs=(G1*s).exp()
    Q=sp.simplify((Fs*W*Fs.T).applyfunc(lambda e: sp.integrate(sp.expand(e),(s,0,z))))
    return F,Q
for name,G1,W,Pinf in [
 ('m12',sp.Matrix([[-1]]),sp.Matrix([[2]]),None),
 ('m32',sp.Matrix([[0,1],[-1,-2]]),sp.Matrix([[0,0],[0,4]]),None),
 ('m52',sp.Matrix([[0,1,0],[0,0,1],[-1,-3,-3]]),sp.Matrix([[0,0,0],[0,0,0],[0,0,sp.Rational(16,3)]]),None)]:
    F,Q=derive(G1,W)
    print(name)
    n=G1.shape[0]
    for i in range(n):
        for j in range(n):
            print(' F',i,j,sp.factor(sp.simplify(F[i,j]*sp.exp(z))))
    for i in range(n):
        for j in range(i,n):
            e=sp.simplify(Q[i,j].subs(z,x/2))
            # write as c + exp(-x)*poly
            ex=sp.expand(sp.simplify(e*sp.exp(x)))
            print(' Q',i,j, ex)
    # stationary P
    P=sp.Matrix(n,n,lambda i,j: sp.Symbol(f'p{min(i,j)}{max(i,j)}'))
    sol=sp.solve(list(G1*P+P*G1.T+W),list(P.free_symbols))
    print(' Pinf',P.subs(sol))
