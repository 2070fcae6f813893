#ifndef SELECT_TF32_NT_H
#define SELECT_TF32_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nt_config;

static inline select_tf32_nt_config select_tf32_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(7168)) {
        if (k < INT64_C(3072)) {
            if (k < INT64_C(79)) {
                if (m < INT64_C(2218)) {
                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(46)) {
                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(1792)) {
                    if (n < INT64_C(46)) {
                        select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                        return out;
                    } else {
                        if (n < INT64_C(544)) {
                            if (n < INT64_C(111)) {
                                if (k < INT64_C(471)) {
                                    if (m < INT64_C(1109)) {
                                        if (m < INT64_C(278)) {
                                            if (n < INT64_C(79)) {
                                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(70)) {
                                    if (k < INT64_C(992)) {
                                        if (n < INT64_C(227)) {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        if (m < INT64_C(448)) {
                                            if (m < INT64_C(159)) {
                                                if (k < INT64_C(744)) {
                                                    if (m < INT64_C(113)) {
                                                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(544)) {
                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(1449)) {
                                                        if (n < INT64_C(287)) {
                                                            if (m < INT64_C(278)) {
                                                                if (k < INT64_C(744)) {
                                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            } else {
                                                                if (k < INT64_C(744)) {
                                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            }
                                                        } else {
                                                            if (m < INT64_C(278)) {
                                                                select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                if (k < INT64_C(992)) {
                                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            }
                                                        }
                                                    } else {
                                                        if (m < INT64_C(278)) {
                                                            if (k < INT64_C(2173)) {
                                                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        } else {
                                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(182)) {
                                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(363)) {
                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(725)) {
                                                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(1449)) {
                                                            select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(363)) {
                                            select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(363)) {
                                                if (k < INT64_C(725)) {
                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(1087)) {
                                                        select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(1268)) {
                                if (k < INT64_C(1620)) {
                                    if (n < INT64_C(1145)) {
                                        if (m < INT64_C(555)) {
                                            if (m < INT64_C(139)) {
                                                if (m < INT64_C(70)) {
                                                    if (m < INT64_C(12)) {
                                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(29)) {
                                                            select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                } else {
                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(896)) {
                                                if (k < INT64_C(124)) {
                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(203)) {
                                                        select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(278)) {
                                            if (k < INT64_C(725)) {
                                                if (m < INT64_C(139)) {
                                                    if (m < INT64_C(70)) {
                                                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(405)) {
                                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                } else {
                                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(555)) {
                                                if (k < INT64_C(405)) {
                                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(405)) {
                                                    select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(2)) {
                                        select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(3)) {
                                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(8)) {
                                                select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(4435)) {
                            if (k < INT64_C(444)) {
                                if (k < INT64_C(222)) {
                                    if (k < INT64_C(118)) {
                                        select_tf32_nt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(314)) {
                                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(1630)) {
                                if (k < INT64_C(222)) {
                                    if (n < INT64_C(28)) {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(182)) {
                                        if (k < INT64_C(363)) {
                                            select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(815)) {
                                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_nt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(725)) {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(555)) {
                if (m < INT64_C(2)) {
                    select_tf32_nt_config out = {8u, 1u, 4u, 16u, 16u};
                    return out;
                } else {
                    if (k < INT64_C(10752)) {
                        if (n < INT64_C(2024)) {
                            if (m < INT64_C(3)) {
                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(12)) {
                                    select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(139)) {
                                        if (m < INT64_C(40)) {
                                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(3)) {
                            select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        } else {
                            if (m < INT64_C(12)) {
                                select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(4435)) {
                        select_tf32_nt_config out = {8u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (k < INT64_C(544)) {
            if (k < INT64_C(79)) {
                if (m < INT64_C(17740)) {
                    if (k < INT64_C(30)) {
                        if (k < INT64_C(20)) {
                            select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(46)) {
                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(32)) {
                            select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(91)) {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(46)) {
                            if (n < INT64_C(28)) {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(118)) {
                                        select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(118)) {
                                        select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(194)) {
                                    select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(118)) {
                            select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(70960)) {
                                select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(141920)) {
                                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(17740)) {
                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            } else {
                if (m < INT64_C(35480)) {
                    select_tf32_nt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(182)) {
                        select_tf32_nt_config out = {8u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    }
}

#endif /* SELECT_TF32_NT_H */
