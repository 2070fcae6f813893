#ifndef SELECT_F32_TT_H
#define SELECT_F32_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_tt_config;

static inline select_f32_tt_config select_f32_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(1792)) {
        if (m < INT64_C(80)) {
            if (m < INT64_C(12)) {
                select_f32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                return out;
            } else {
                if (n < INT64_C(1132)) {
                    if (k < INT64_C(1145)) {
                        if (k < INT64_C(992)) {
                            select_f32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        }
                    } else {
                        select_f32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                    return out;
                }
            }
        } else {
            if (n < INT64_C(351)) {
                if (m < INT64_C(555)) {
                    if (n < INT64_C(111)) {
                        select_f32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(113)) {
                            if (n < INT64_C(227)) {
                                select_f32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                select_f32_tt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(744)) {
                                    if (k < INT64_C(544)) {
                                        select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(287)) {
                                        select_f32_tt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(176)) {
                        if (k < INT64_C(167)) {
                            select_f32_tt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(1052)) {
                                if (k < INT64_C(544)) {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(222)) {
                                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_tt_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(79)) {
                                            if (k < INT64_C(272)) {
                                                select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {4u, 2u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(287)) {
                                select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            }
                        } else {
                            select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(139)) {
                    if (n < INT64_C(1620)) {
                        select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                        return out;
                    } else {
                        select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(278)) {
                        if (n < INT64_C(992)) {
                            if (k < INT64_C(79)) {
                                select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(744)) {
                                    select_f32_tt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(448)) {
                            if (n < INT64_C(744)) {
                                select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(405)) {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(144)) {
                                        select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(203)) {
                                            select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(287)) {
                                                select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {4u, 8u, 8u, 8u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(111)) {
            if (n < INT64_C(46)) {
                if (m < INT64_C(8870)) {
                    if (m < INT64_C(4435)) {
                        if (n < INT64_C(28)) {
                            select_f32_tt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(28)) {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(167)) {
                        if (m < INT64_C(17740)) {
                            select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(56)) {
                                if (m < INT64_C(70960)) {
                                    select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(141920)) {
                                        if (k < INT64_C(30)) {
                                            select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(118)) {
                                    select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (n < INT64_C(79)) {
                        if (k < INT64_C(222)) {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(111)) {
                                    select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(471)) {
                                    select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(8870)) {
                                        select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                } else {
                    select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(7168)) {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(28)) {
                        select_f32_tt_config out = {8u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(4435)) {
                            select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(363)) {
                                if (k < INT64_C(91)) {
                                    select_f32_tt_config out = {8u, 8u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {8u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {4u, 8u, 8u, 8u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(2509)) {
                        select_f32_tt_config out = {4u, 8u, 8u, 8u, 16u};
                        return out;
                    } else {
                        if (m < INT64_C(3548)) {
                            select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(5017)) {
                                select_f32_tt_config out = {4u, 8u, 8u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(70960)) {
                        if (k < INT64_C(128)) {
                            if (m < INT64_C(35480)) {
                                select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(40)) {
                                    select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 8u, 8u, 8u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                select_f32_tt_config out = {4u, 8u, 8u, 8u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(1630)) {
                                    select_f32_tt_config out = {4u, 8u, 8u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                } else {
                    select_f32_tt_config out = {4u, 8u, 8u, 16u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_F32_TT_H */
