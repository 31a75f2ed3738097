function Float_Sum(Graph g) {
  propNode<double> x;
  g.attachNodeProperty(x = 0.1);
  double s = 0.0;
  forall (v in g.nodes()) {
    forall (nbr in g.neighbors(v)) {
      s += nbr.x;
    }
  }
}
