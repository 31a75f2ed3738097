function Neighbor_MinMax(Graph g) {
  propNode<double> x;
  propNode<double> lo;
  propNode<int> hi;
  g.attachNodeProperty(x = 0.25, lo = 1.5, hi = 0);
  double best = 9.0;
  forall (v in g.nodes()) {
    forall (nbr in g.neighbors(v)) {
      <v.lo> = <Min(v.lo, nbr.x)>;
      <v.hi> = <Max(v.hi, 4)>;
      <best> = <Min(best, nbr.x)>;
    }
  }
}
